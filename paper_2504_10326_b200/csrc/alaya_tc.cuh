// Stage 1 on the 5th-generation tensor cores (sm_100a): persistent,
// warp-specialised DIPR scan for bf16 keys, d = 128.
//
//   warp 0      TMA producer: K tiles (128 keys x 128 dims bf16 = 32 KB, two
//               64-column boxes, 128B swizzle) into a kStages-deep smem ring.
//   warp 1      TMEM allocator + MMA issuer: per tile 8 x tcgen05.mma
//               (M=128 keys, N=NP, K=16) with A = K tile (K-major, SW128) and
//               B = the GQA group's queries split into three bf16 terms
//               (q = hi + mid + lo, residual < 2^-24 |q|), fp32 accumulators in
//               TMEM, double buffered.
//   warps 2-5   epilogue: tcgen05.ld one key row per thread, s_j = sum of the
//               three split columns, tile max, ordered ballot compaction of
//               s >= bound - beta into the candidate lists (same format as the
//               CUDA-core scan), per-chunk atomic max.
//
// Products of bf16 values are exact in fp32, so the score error is the fp32
// accumulation error of the tensor core, comparable to the CUDA-core path.
#pragma once

#include <cuda.h>

#include "alaya_common.cuh"

namespace alaya {
namespace tc {

constexpr int kTileKeys = 128;
constexpr int kTileBytes = kTileKeys * 128 * 2;  // 32 KB
constexpr int kBoxBytes = kTileBytes / 2;        // 64 columns x 128 rows
// ALAYA_PUB_WARP (default 1): a 7th warp publishes finished chunks (see the
// publisher branch); 0 = the epilogue publishes them itself
#ifndef ALAYA_PUB_WARP
#define ALAYA_PUB_WARP 1
#endif
constexpr int kThreadsTc = ALAYA_PUB_WARP ? 224 : 192;  // producer, MMA, 4 epilogue warps[, publisher]
constexpr int kPubWarp = 6;
constexpr int kMaxMaps = ALAYA_MAX_BATCH;  // one tensor map per distinct K slab

struct Maps {
  CUtensorMap m[kMaxMaps];
  int16_t map_of_seq[ALAYA_MAX_BATCH];
  int64_t rows_per_head[ALAYA_MAX_BATCH];
};

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_nohint(uint32_t dst, const CUtensorMap* map, int x, int y,
                                                   uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// K-major, 128B-swizzled UMMA shared-memory descriptor (SBO = 1024 B between
// 8-row groups; LBO unused for swizzled K-major; version 1; layout SW128 = 2).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M=128, N.
template <int N>
__device__ __forceinline__ uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

template <int NP>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[NP]);
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<32>(uint32_t taddr, float (&v)[32]) {
  float* lo = v;
  float* hi = v + 16;
  tmem_ld<16>(taddr, *reinterpret_cast<float(*)[16]>(lo));
  tmem_ld<16>(taddr + 16, *reinterpret_cast<float(*)[16]>(hi));
}

__device__ __forceinline__ uint16_t bf16_bits(float x) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// The group's q staged in shared memory by cp.async (no registers held across the
// chunk): issued for the next chunk right after this chunk's B operand is built.
template <int G>
__device__ __forceinline__ void stage_q(float* qs, const float* __restrict__ qg, int lane) {
  for (int i = lane; i < G * 32; i += 32)  // G*128 floats = G*32 x 16 B
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(qs + 4 * i)), "l"(qg + 4 * i)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void staged_q_wait() {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
}
template <int G, int NP>
__device__ __forceinline__ void build_b_smem(uint8_t* bbuf, const float* qs, int lane) {
#pragma unroll
  for (int i = 0; i < 4 * G; ++i) {
    const int idx = lane + 32 * i;
    const int j = idx >> 7, k = idx & 127;
    const float x = qs[idx];
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(mid);
    const uint16_t parts[3] = {__bfloat16_as_ushort(hi), __bfloat16_as_ushort(mid), bf16_bits(r2)};
    const int box = k >> 6, kk = k & 63, c16 = kk >> 3, w = kk & 7;
#pragma unroll
    for (int sp = 0; sp < 3; ++sp) {
      const int n = sp * G + j;
      const int off = box * (NP * 128) + (n >> 3) * 1024 + (n & 7) * 128 + ((c16 ^ (n & 7)) << 4) + w * 2;
      *reinterpret_cast<uint16_t*>(bbuf + off) = parts[sp];
    }
  }
}
constexpr int kAcc = 4;  // TMEM accumulator buffers (MMA runs up to 4 tiles ahead)
constexpr int kIds = 8;  // chunk-id ring (scheduler -> MMA warp + epilogue warps)

// One chunk of the scan epilogue for this warp's TMEM lane quarter (32 key
// rows of every 128-key tile). No cross-warp barriers: the warp keeps its own
// running max (a max of real scores, hence a valid lower bound of the global
// max) and writes its own ordered candidate sub-list (CandList, q = quarter).
template <int G, int NP, bool GF>
__device__ __forceinline__ void epilogue_chunk(const Batch& bt, const Ws& ws, int c, int quarter,
                                               int lane, uint32_t tmem_base, uint32_t accf0,
                                               uint32_t acce0, int& acc, uint32_t& aphase,
                                               int& b, int& h, float* tmax, int& tcount,
                                               const uint32_t* pre) {
  int ci;
  decode_chunk(bt, c, b, h, ci);
  const int chunk = bt.chunk;
  const int valid = min(chunk, bt.s[b].n - ci * chunk);
  const int ntiles = (valid + kTileKeys - 1) / kTileKeys;
  // run[] starts at -inf; the header's running max (pre, loaded by the caller a
  // chunk ahead) joins at the first tile's threshold, so its load is awaited there
  float run[G], tk[G];
  int cnt[G];
  bool first_tile = true;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    run[j] = -INFINITY;
    tk[j] = bt.topk_thr ? __ldcg(bt.topk_thr + b * bt.Hq + h * G + j) : 0.f;
    cnt[j] = 0;
  }
  const size_t cbase = (size_t)c * G;
  const int qoff = quarter * (chunk / 4);
  for (unsigned long long m = chunk_tiles(bt, ws, c, ntiles); m; m &= m - 1) {
    const int tl = __ffsll((long long)m) - 1;
    mbar_wait(accf0 + 8u * acc, (aphase >> acc) & 1u);
    fence_after();
    float v[NP];
    tmem_ld<NP>(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * NP, v);
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(acce0 + 8u * acc);
    aphase ^= 1u << acc;
    acc = (acc + 1) % kAcc;
    const int row = tl * kTileKeys + quarter * 32 + lane;
    const bool ok = row < valid;
    // tile max over all 128 rows (one named barrier among the 4 epilogue warps;
    // tmax is double-buffered by tile parity): a 32-row warp max alone misses
    // the query's cluster often enough to bloat the candidate superset
    float sc[G];
    const int tb = (tcount++) & 1;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      sc[j] = ok ? v[j] + (v[G + j] + v[2 * G + j]) : -INFINITY;
      const float m = warp_max(sc[j]);
      if (lane == 0) tmax[(tb * 4 + quarter) * G + j] = m;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (first_tile) {
      first_tile = false;
#pragma unroll
      for (int j = 0; j < G; ++j) run[j] = dec_max(pre[j]);
    }
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) run[j] = fmaxf(run[j], tmax[(tb * 4 + qq) * G + j]);
    if constexpr (GF) {  // one entry per row some head keeps: the row and all G scores
      bool pass = false;
#pragma unroll
      for (int j = 0; j < G; ++j) pass |= sc[j] >= run[j] - bt.beta;
      pass = pass && ok;
      const unsigned bal = __ballot_sync(kFull, pass);
      if (pass) {
        const int o = cnt[0] + __popc(bal & lanemask_lt());
        ws.gidx[(size_t)c * chunk + qoff + o] = row;
        float* gsc = ws.cscore + (size_t)(c * 4 + quarter) * G * (chunk / 4) + o;
#pragma unroll
        for (int j = 0; j < G; ++j) gsc[j * (chunk / 4)] = sc[j];
      }
      cnt[0] += __popc(bal);
    } else {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const bool pass = ok && sc[j] >= (bt.topk_thr ? tk[j] : run[j] - bt.beta);
        const unsigned bal = __ballot_sync(kFull, pass);
        if (pass) {
          const int o = qoff + cnt[j] + __popc(bal & lanemask_lt());
          ws.cidx[(cbase + j) * chunk + o] = row;
          ws.cscore[(cbase + j) * chunk + o] = sc[j];
        }
        cnt[j] += __popc(bal);
      }
    }
  }
  if constexpr (GF) {
    if (lane == 0) ws.cnt[(size_t)c * 4 + quarter] = cnt[0];
    if (quarter == 0 && lane < G) {
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (j == lane && enc_max(run[j]) > pre[j]) atomicMax(&ws.gmax[b * bt.Hq + h * G + j], enc_max(run[j]));
    }
    return;
  }
  if (lane < G) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (j == lane) {
        // run[] is the same in the 4 epilogue warps (tile maxima are shared through
        // smem): one warp publishes, and only a max this chunk actually raised --
        // the gmax lines are shared by every CTA of the call, so atomics queued
        // there would stall the chunk-start reads of all of them
        if (quarter == 0 && enc_max(run[j]) > pre[j])
          atomicMax(&ws.gmax[b * bt.Hq + h * G + j], enc_max(run[j]));
        ws.cnt[(cbase + j) * 4 + quarter] = cnt[j];
        tmax[8 * G + quarter * G + j] = __int_as_float(cnt[j]);  // pair totals via smem
      }
    }
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (quarter == 0 && lane < G) {
    int tot = 0;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) tot += __float_as_int(tmax[8 * G + qq * G + lane]);
    publish_pair(bt, ws, cbase + lane, tot);
  }
}

// MMA issue for one tile: 8 x (M=128, N=NP, K=16) into accumulator buffer acc.
template <int NP>
__device__ __forceinline__ void mma_tile(uint32_t a_base, uint32_t b_base, uint32_t d, uint32_t idesc) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t a_addr = a_base + (k >> 2) * kBoxBytes + (k & 3) * 32;
    const uint32_t b_addr = b_base + (k >> 2) * (NP * 128) + (k & 3) * 32;
    mma_bf16(d, sw128_desc(a_addr), sw128_desc(b_addr), idesc, k > 0 ? 1u : 0u);
  }
}

// Registers: an attend_ovl CTA (4 warps x 128 registers, one warp per SM
// sub-partition) runs beside the scan only if every sub-partition keeps 4096
// registers free. 7 scan warps per CTA: 2 CTAs per SM (3 stages, the default) put
// up to 4 warps on a sub-partition -> <= 96 registers; 1 CTA (4-6 stages) 2 warps
// -> <= 168; 3 CTAs (2 stages) 6 warps leave no room at any cap without spills.
#ifndef ALAYA_SCAN_MAXREG_S2
#define ALAYA_SCAN_MAXREG_S2 72
#endif
#ifndef ALAYA_SCAN_MAXREG_S3
#define ALAYA_SCAN_MAXREG_S3 128
#endif
template <int G, int kStages>
constexpr int scan_tc_maxreg() {
  return kStages <= 2 ? (3 * G <= 16 ? ALAYA_SCAN_MAXREG_S2 : 80) : (kStages <= 3 ? ALAYA_SCAN_MAXREG_S3 : 168);
}

template <int G, int kStages, bool GF>
__global__ void __launch_bounds__(kThreadsTc) __maxnreg__((scan_tc_maxreg<G, kStages>()))
    scan_tc_kernel(const __grid_constant__ Batch bt, const __grid_constant__ Maps maps,
                   const float* __restrict__ q, Ws ws) {
  constexpr int NP = (3 * G <= 16) ? 16 : 32;
  constexpr int kBBytes = 2 * NP * 128;  // one B operand (two boxes)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_ring = smem;                                     // kStages x 32 KB
  uint8_t* b_buf = a_ring + kStages * kTileBytes;             // 2 x kBBytes
  float* q_stage = reinterpret_cast<float*>(b_buf + 2 * kBBytes);  // [G][128] next chunk's q (cp.async)
  uint64_t* bars = reinterpret_cast<uint64_t*>(q_stage + G * 128);
  // full[kStages], empty[kStages], accf[kAcc], acce[kAcc], bfree[2], idfull/idempty/pubready[kIds]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kAcc + 2 + 3 * kIds);
  int* ids = reinterpret_cast<int*>(tmem_slot + 4);          // [kIds] chunk-id ring
  float* tmax = reinterpret_cast<float*>(ids + kIds);         // [2][4][G] tile maxima + [4][G] counts

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace_rec(bt, 1, 0);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
  const uint32_t accf0 = bar0 + 8u * (2 * kStages), acce0 = accf0 + 8u * kAcc;
  const uint32_t bfree0 = acce0 + 8u * kAcc;  // B buffer free: MMAs reading it completed
  const uint32_t idfull0 = bfree0 + 16u, idempty0 = idfull0 + 8u * kIds, pubready0 = idempty0 + 8u * kIds;
  // chunk-id ring: the producer posts the k-th chunk of this CTA (-1 = done) into
  // slot k % kIds; the MMA warp and the 4 epilogue warps read it and release it
  auto read_id = [&](int k) -> int {
    mbar_wait(idfull0 + 8u * (k % kIds), (uint32_t)(k / kIds) & 1u);
    return *reinterpret_cast<volatile int*>(ids + k % kIds);
  };
  auto release_id = [&](int k) { mbar_arrive(idempty0 + 8u * (k % kIds)); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 1); }
    for (int a = 0; a < kAcc; ++a) { mbar_init(accf0 + 8u * a, 1); mbar_init(acce0 + 8u * a, 4); }
    for (int i = 0; i < 2; ++i) mbar_init(bfree0 + 8u * i, 1);
    for (int i = 0; i < kIds; ++i) {
      mbar_init(idfull0 + 8u * i, 1);
      mbar_init(idempty0 + 8u * i, ALAYA_PUB_WARP ? 2 : 5);   // MMA warp + publisher (or the 4 epilogue warps)
      mbar_init(pubready0 + 8u * i, 4);  // the 4 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kAcc * NP));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 2 * kBBytes / 16; i += kThreadsTc)
    reinterpret_cast<uint4*>(b_buf)[i] = make_uint4(0, 0, 0, 0);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int chunk = bt.chunk;
  // The TMA producer streams K (context memory, untouched by the preceding
  // kernels) without waiting for them, so the first tiles are in flight while
  // prep_kernel still runs -- unless the block filter's keep masks (written by
  // the preceding kernels) steer it. Every other warp waits (q, gmax seeds,
  // tickets), then triggers: a dependent launched after the trigger sees all
  // earlier work complete.
  if (warp != 0 && bt.call_id) {  // async prep: the zeroed header is published as ws.ready
    if (lane == 0) {
      const unsigned long long tok = call_token(bt);
      while (ld_acquire_gpu_u64(ws.ready) != tok) __nanosleep(32);
    }
    __syncwarp();
  } else if (warp != 0 || bt.block_filter) {
    pdl_wait();
  }
  if (warp != 0) pdl_trigger();

  if (warp == 0) {
    // ===================== TMA producer + chunk scheduler =====================
    // Chunks are handed out dynamically, in increasing order: the first is
    // blockIdx.x, every later one comes from a counter in the call's header
    // (taken once the chunk's first tiles are issued, so the consumers know the
    // next chunk a chunk ahead). Faster CTAs take more chunks, and groups
    // complete in order, so the attend beside the scan starts on early groups.
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      bool header_ok = false;
      auto post = [&](int k, int id) {
        if (k >= kIds) mbar_wait(idempty0 + 8u * (k % kIds), ((uint32_t)(k / kIds) & 1u) ^ 1u);
        *reinterpret_cast<volatile int*>(ids + k % kIds) = id;
        mbar_arrive(idfull0 + 8u * (k % kIds));  // release: the id store is visible to the waiters
      };
      auto fetch = [&]() -> int {
        if (!header_ok) {  // the counter lives in the header this call's prep zeroes
          if (bt.call_id) {
            const unsigned long long tok = call_token(bt);
            while (ld_acquire_gpu_u64(ws.ready) != tok) __nanosleep(32);
          } else {
            pdl_wait();
          }
          header_ok = true;
        }
        return (int)gridDim.x + atomicAdd(&ws.counters[9], 1);  // raw: checked at use
      };
      // the counter for chunk k + 2 is taken right after chunk k + 1 is posted, so its
      // round trip is hidden behind chunk k + 1's first tiles
      int ahead = -1;
      int c = (int)blockIdx.x < bt.total_chunks ? (int)blockIdx.x : -1;
      post(0, c);
      for (int k = 0; c >= 0; ++k) {
        int b, h, ci;
        decode_chunk(bt, c, b, h, ci);
        const int valid = min(chunk, bt.s[b].n - ci * chunk);
        const int ntiles = (valid + kTileKeys - 1) / kTileKeys;
        const CUtensorMap* map = &maps.m[maps.map_of_seq[b]];
        const int row0 = (int)(h * maps.rows_per_head[b] + (int64_t)ci * chunk);
        int issued = 0, nxt = 0;
        bool posted = false;
        auto post_next = [&]() {
          nxt = ahead >= 0 ? ahead : fetch();
          if (nxt >= bt.total_chunks) nxt = -1;
          post(k + 1, nxt);
          posted = true;
          ahead = nxt >= 0 ? fetch() : -1;
        };
        for (unsigned long long m = chunk_tiles(bt, ws, c, ntiles); m; m &= m - 1) {
          if (issued++ == 2) post_next();
          const int tl = __ffsll((long long)m) - 1;
          {
            const unsigned long long t0 = bt.trace ? gtimer() : 0ull;
            mbar_wait(empty_bar(stage), phase ^ 1);
            if (bt.trace) trace_add(bt, 1, 13, gtimer() - t0);  // diagnostics: ring full (ns)
          }
          mbar_expect_tx(full_bar(stage), kTileBytes);
          const uint32_t dst = smem_u32(a_ring + stage * kTileBytes);
          if (bt.dbg & 1) {
            tma_load_2d_nohint(dst, map, 0, row0 + tl * kTileKeys, full_bar(stage));
            tma_load_2d_nohint(dst + kBoxBytes, map, 64, row0 + tl * kTileKeys, full_bar(stage));
          } else {
            tma_load_2d(dst, map, 0, row0 + tl * kTileKeys, full_bar(stage), pol);
            tma_load_2d(dst + kBoxBytes, map, 64, row0 + tl * kTileKeys, full_bar(stage), pol);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (!posted) post_next();
        c = nxt;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc = idesc_bf16<NP>();
    int stage = 0, acc = 0, cidx = 0, bcnt = 0;
    uint32_t phase = 0, ephase = 0, bphase = 0;

    auto q_of = [&](int c) {
      int b, h, ci;
      decode_chunk(bt, c, b, h, ci);
      return q + ((size_t)b * bt.Hq + (size_t)h * G) * 128;
    };
    int c = read_id(0);
    if (c >= 0) stage_q<G>(q_stage, q_of(c), lane);
    for (int k = 0; c >= 0; ++k, ++cidx) {
      int nxt = -1;
      bool have_nxt = false;
      int b, h, ci;
      decode_chunk(bt, c, b, h, ci);
      const int valid = min(chunk, bt.s[b].n - ci * chunk);
      const int ntiles = (valid + kTileKeys - 1) / kTileKeys;
      const int bi = bcnt & 1;
      uint8_t* bb = b_buf + bi * kBBytes;
      bool first = true;
      for (unsigned long long m = chunk_tiles(bt, ws, c, ntiles); m; m &= m - 1) {
        mbar_wait(acce0 + 8u * acc, ((ephase >> acc) & 1u) ^ 1u);
        ephase ^= 1u << acc;
        fence_after();
        if (first) {
          first = false;
          // wait until the MMAs that last read this B buffer have completed
          mbar_wait(bfree0 + 8u * bi, ((bphase >> bi) & 1u) ^ 1u);
          bphase ^= 1u << bi;
          staged_q_wait();
          build_b_smem<G, NP>(bb, q_stage, lane);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
        }
        mbar_wait(full_bar(stage), phase);
        fence_after();
        if (lane == 0) {
          if (!(bt.dbg & 4))
            mma_tile<NP>(smem_u32(a_ring + stage * kTileBytes), smem_u32(bb), tmem_base + acc * NP, idesc);
          mma_commit(empty_bar(stage));
          mma_commit(accf0 + 8u * acc);
        }
        __syncwarp();
        // next chunk's id (not waited for mid-chunk) -> its q staged while this chunk runs
        if (!have_nxt && mbar_try_wait(idfull0 + 8u * ((k + 1) % kIds), (uint32_t)((k + 1) / kIds) & 1u)) {
          have_nxt = true;
          nxt = *reinterpret_cast<volatile int*>(ids + (k + 1) % kIds);
          __syncwarp();  // every lane has read q_stage (B built) before it is refilled
          if (nxt >= 0) stage_q<G>(q_stage, q_of(nxt), lane);
        }
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        acc = (acc + 1) % kAcc;
      }
      if (!first) {  // this chunk used B buffer bi: free it once its MMAs complete
        if (lane == 0) mma_commit(bfree0 + 8u * bi);
        __syncwarp();
        ++bcnt;
      }
      if (!have_nxt) {
        nxt = read_id(k + 1);
        __syncwarp();
        if (nxt >= 0) stage_q<G>(q_stage, q_of(nxt), lane);
      }
      __syncwarp();
      if (lane == 0) release_id(k);
      c = nxt;
    }
  } else if (ALAYA_PUB_WARP && warp == kPubWarp) {
    // ===================== publisher =====================
    // Publishes each finished chunk to the attend beside the scan (group counter,
    // gpu-scope release-add). Kept off the pipeline warps: under full HBM load a
    // gpu-scope release waits ~3-4 us, which stalled the epilogue (and behind it
    // the MMA and TMA) once per chunk when the epilogue published itself. Chunk k
    // is written once the 4 epilogue warps arrived on pubready (release.cta,
    // observed here with acquire.cta; the release-add is cumulative over their
    // stores). The slot is handed back (idempty) only after publishing, so the
    // producer never reuses it for chunk k + kIds before chunk k is out.
    const bool publish = bt.overlap && !bt.sx_on;  // (fused sharded step: the epilogue publishes)
    for (int k = 0;; ++k) {
      const int c = read_id(k);
      if (c < 0) break;
      mbar_wait(pubready0 + 8u * (k % kIds), (uint32_t)(k / kIds) & 1u);
      if (publish && lane == 0) {
        int b, h, ci;
        decode_chunk(bt, c, b, h, ci);
        const unsigned long long t0 = bt.trace ? gtimer() : 0ull;
        asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(&ws.group_done[b * bt.Hkv + h]), "r"(4)
                     : "memory");
        asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(&ws.counters[6]), "r"(4) : "memory");
        if (bt.trace) trace_add(bt, 1, 15, gtimer() - t0);
      }
      __syncwarp();
      if (lane == 0) release_id(k);
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0, tcount = 0;
    uint32_t aphase = 0;
    // the running max a chunk starts from is read one chunk ahead (any earlier
    // value is a valid lower bound), so no chunk waits on that load
    uint32_t pre[G];  // raw (encoded): decoded only when the chunk starts
    auto load_pre = [&](int c) {
      int b, h, ci;
      decode_chunk(bt, c, b, h, ci);
#pragma unroll
      for (int j = 0; j < G; ++j) pre[j] = __ldcg(&ws.gmax[b * bt.Hq + h * G + j]);
    };
    // (later chunks do not wait: whatever the header holds -- a seed, other chunks'
    // maxima -- is a lower bound of the max; the seeds matter most for the first chunk
    // on locality-ordered prefixes, where a chunk-local bound keeps whole clusters)
    int c = read_id(0);
    if (c >= 0 && bt.call_id) {  // the first chunk starts from its group's prep seed (bounded
      int b, h, ci;            // wait; prep publishes the seeds before its window partials)
      decode_chunk(bt, c, b, h, ci);
      if (lane == 0) {
        int polls = 0;
        const unsigned long long tok = call_token(bt);
        while (ld_acquire_gpu_u64(ws.seeded + b * bt.Hkv + h) != tok && ++polls < (1 << 16)) __nanosleep(64);
      }
      __syncwarp();
    }
    if (c >= 0) load_pre(c);
    for (int k = 0; c >= 0; ++k) {
      int b, h;
      epilogue_chunk<G, NP, GF>(bt, ws, c, quarter, lane, tmem_base, accf0, acce0, acc, aphase, b, h,
                                tmax, tcount, pre);
      const int nxt = read_id(k + 1);  // posted by now (the producer is >= 2 tiles ahead)
      if (quarter == 0 && lane == 0 && k < 8) trace_rec(bt, 1, 2 + k);
      const unsigned long long t_pub = bt.trace ? gtimer() : 0ull;
      if (bt.overlap && quarter == 0) {
        __syncwarp();  // lanes 1..G-1 wrote heavy flags
        // the chunk is published once, by quarter 0 after the epilogue's final named
        // barrier (every warp's candidates and counts, its own heavy flags): a
        // release add makes them visible before the group counter moves (the
        // barrier + single release-store pattern of CUTLASS's semaphore)
        // (single-GPU: the producer thread publishes, see prod_pub; the fused sharded
        // step publishes here, the completing CTA pushes the group's maxima to the peers)
        int old = 0;
        if (lane == 0 && bt.sx_on) {
          asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;"
                       : "=r"(old) : "l"(&ws.group_done[b * bt.Hkv + h]), "r"(4) : "memory");
          asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(&ws.counters[6]), "r"(4) : "memory");
        } else if (lane == 0 && !ALAYA_PUB_WARP) {
          asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(&ws.group_done[b * bt.Hkv + h]), "r"(4)
                       : "memory");
          asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(&ws.counters[6]), "r"(4) : "memory");
        }
        if (bt.sx_on) {
          old = __shfl_sync(kFull, old, 0);
          if (old + 4 == 4 * bt.s[b].nch) {  // this chunk completed the group: its maxima are
            const ShardExch& x = bt.sx;    // final -> every rank's slot, then the group flag
            const int parity = (int)(x.epoch & 1ull);
            const int g = b * bt.Hkv + h;
            for (int i = lane; i < G * x.R; i += 32) {
              const int j = i % G, r = i / G;
              const float m = dec_max(__ldcg(&ws.gmax[b * bt.Hq + h * G + j]));
              exch_slot(x.peers[r], parity, 0, x.rank, x.R, x.cap)[b * bt.Hq + h * G + j] = m;
            }
            __threadfence_system();
            __syncwarp();
            if (lane < x.R) st_release_sys_u64(exch_gflag(x.peers[lane], g, x.rank), x.epoch);
          }
        }
      }
      __syncwarp();
      if (bt.trace && quarter == 0 && lane == 0) trace_add(bt, 1, 14, gtimer() - t_pub);  // publish (ns)
      if (lane == 0) {
        if (ALAYA_PUB_WARP) mbar_arrive(pubready0 + 8u * (k % kIds));  // chunk k written (release.cta)
        else release_id(k);
      }
      if (nxt >= 0) load_pre(nxt);  // in flight until the next chunk's first threshold
      c = nxt;
    }
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_rec(bt, 1, 1);
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAcc * NP));
  }
}

inline size_t tc_smem_bytes(int G, int kStages) {
  const int NP = (3 * G <= 16) ? 16 : 32;
  return 1024 + (size_t)kStages * kTileBytes + 2 * 2 * NP * 128 + (size_t)G * 512 +
         8 * (2 * kStages + 2 * kAcc + 2 + 3 * kIds) +
         16 + 4 * kIds + 3 * 4 * G * 4 + 64;
}

}  // namespace tc
}  // namespace alaya
