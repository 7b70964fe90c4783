// Group-format attend on the tensor cores (bf16 V, d = 128), for the high-beta
// regime where the heads of a GQA group keep most rows of a chunk (reference:
// dipr.py:64 filter, store.py:271-278 selection, attention.py:98-110 partial).
//
// One CTA per chunk. The chunk's V rows stream densely through a TMA ring (the
// same 32 KB SW128 tiles as the K scan); per 128-row tile the builder warps
// (2-4 per lane quarter, matching the scan's group-format sub-lists) apply every
// head's exact filter s_j >= gmax_j - beta minus the window ids to the tile's
// listed rows and write the weights w_j = 2^((s_j - gmax_j) log2e / sqrt(d)) as
// the B operand (3 bf16 terms per weight, zeros for unlisted rows; 2-4 warps per
// quarter, each for a share of the heads: one warp per quarter was builder-bound,
// 274 vs 249 us for the kernel alone at beta 140 B=4 with two):
//   D[d][n] += V^T[d][t] * W[t][n],  M = 128 (d), N = 3G padded, K = 16 tokens,
// A = the V tile read MN-major (d contiguous), fp32 accumulation in TMEM over the
// whole chunk. A row any head keeps is read once, by a stream instead of a
// gather, and the G weighted sums cost no CUDA-core FMAs. The epilogue sums the
// 3 terms per head into the (chunk, head) partial; selected ids and counts go
// out as attend_grp_kernel writes them (diagnostics, combine).
#pragma once

#include "alaya_tc.cuh"

namespace alaya {
namespace tc {

constexpr int kDenseStages = 3;
// builder warps per lane quarter, each for an equal share of the GQA group's heads
// (profiles/r02/dense_split4_v70.jsonl, dense_split_g5_v71.jsonl, beta 140: G=4 one head per
// warp B=4 409 -> 400 us, B=8 821 -> 812 vs two heads; G=5 at B=8: 2 ways 894, 3 ways (2,2,1)
// 864, 4 ways (2,2,1,0) 950, 5 ways 916)
constexpr int dense_split(int G) { return (G == 4 || G == 8) ? 4 : (G >= 5 ? 3 : (G >= 2 ? 2 : 1)); }
// TMA producer, MMA issuer, 4 * split builder/epilogue warps
constexpr int dense_threads(int G) { return 64 + 128 * dense_split(G); }

// MN-major, 128B-swizzled UMMA descriptor of a V tile read as A = V^T (M = d):
// 64 d (128 B) contiguous, the next 64 d one box (16 KB) away (LBO); 8 token
// rows of 128 B per swizzle atom, the next 8 rows 1 KB away (SBO).
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(kBoxBytes >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

inline size_t dense_smem_bytes(int G) {
  const int NP = (3 * G <= 16) ? 16 : 32;
  return 1024 + (size_t)kDenseStages * kTileBytes + 2 * (2 * NP * 128) + 256;
}

template <int G>
__global__ void __launch_bounds__(dense_threads(G), 2)
    attend_dense_tc_kernel(const __grid_constant__ Batch bt, const __grid_constant__ Maps vmaps, Ws ws) {
  constexpr int NP = (3 * G <= 16) ? 16 : 32;
  constexpr int kBBytes = 2 * NP * 128;  // B operand: NP rows x 128 tokens, two 64-token boxes
  constexpr int D = 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* bbuf = ring + kDenseStages * kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bbuf + 2 * kBBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kDenseStages + 5);
  __shared__ float s_l[4][G];
  __shared__ int s_ns[4][G], s_nr[4][G];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  const int c = blockIdx.x;
  int b, h, ci;
  decode_chunk(bt, c, b, h, ci);
  const KSeq& s = bt.s[b];
  const int chunk = bt.chunk, qcap = chunk / 4;
  const int t0 = ci * chunk;
  const int valid = min(chunk, s.n - t0);
  const int ntiles = (valid + kTileKeys - 1) / kTileKeys;
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int i) { return bar0 + 8u * i; };
  auto empty_bar = [&](int i) { return bar0 + 8u * (kDenseStages + i); };
  const uint32_t bfull0 = bar0 + 8u * (2 * kDenseStages), bfree0 = bfull0 + 16u, accf = bfree0 + 16u;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kDenseStages; ++i) { mbar_init(full_bar(i), 1); mbar_init(empty_bar(i), 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(bfull0 + 8u * i, 4 * dense_split(G)); mbar_init(bfree0 + 8u * i, 1); }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (V is context memory: no wait) =====================
    if (lane == 0) {
      const CUtensorMap* map = &vmaps.m[vmaps.map_of_seq[b]];
      const int row0 = (int)(h * vmaps.rows_per_head[b] + t0);
      const uint64_t pol = evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int tl = 0; tl < ntiles; ++tl) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        mbar_expect_tx(full_bar(stage), kTileBytes);
        const uint32_t dst = smem_u32(ring + stage * kTileBytes);
        tma_load_2d(dst, map, 0, row0 + tl * kTileKeys, full_bar(stage), pol);
        tma_load_2d(dst + kBoxBytes, map, 64, row0 + tl * kTileKeys, full_bar(stage), pol);
        if (++stage == kDenseStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc = idesc_bf16<NP>() | (1u << 15);  // A (= V^T) MN-major
    int stage = 0;
    uint32_t phase = 0;
    for (int tl = 0; tl < ntiles; ++tl) {
      const int bi = tl & 1;
      mbar_wait(full_bar(stage), phase);
      uint8_t* tile = ring + stage * kTileBytes;
      const int rows = valid - tl * kTileKeys;
      if (rows < kTileKeys) {  // a sequence's last partial tile: rows past n are not this
        // sequence's keys (and may hold anything) -> zero them, weights alone do not mask NaN
        const int per_box = (kTileKeys - rows) * 8;  // 16-byte pieces of the rows to clear
        for (int i = lane; i < 2 * per_box; i += 32) {
          const int bx = i / per_box, rem = i - bx * per_box;
          reinterpret_cast<uint4*>(tile + bx * kBoxBytes + (rows + (rem >> 3)) * 128)[rem & 7] =
              make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      mbar_wait(bfull0 + 8u * bi, (uint32_t)(tl >> 1) & 1u);
      fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(tile), b0 = smem_u32(bbuf + bi * kBBytes);
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 tokens per MMA: 16 rows x 128 B of A, 32 B of B
          const uint32_t a_addr = a0 + k * 2048;
          const uint32_t b_addr = b0 + (k >> 2) * (NP * 128) + (k & 3) * 32;
          mma_bf16(tmem, sw128_mn_desc(a_addr), sw128_desc(b_addr), idesc, (tl > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit(empty_bar(stage));
        mma_commit(bfree0 + 8u * bi);
        if (tl == ntiles - 1) mma_commit(accf);
      }
      __syncwarp();
      if (++stage == kDenseStages) { stage = 0; phase ^= 1; }
    }
  } else {
    // ===================== builders / epilogue (lane quarter q, heads of half hf) =====================
    constexpr int kSplit = dense_split(G);
    constexpr int GH = (G + kSplit - 1) / kSplit;  // heads per builder warp
    const int quarter = warp & 3, hf = (warp - 2) >> 2;
    const int jb = hf * GH;  // this warp's heads: jb + jj < G, jj < GH
    const float k2 = bt.inv_sqrt_d * kLog2e;
    if (lane == 0) {
      const int* gd = ws.group_done + b * bt.Hkv + h;
      while (ld_acquire_gpu(gd) < 4 * s.nch) __nanosleep(256);
    }
    __syncwarp();
    // after the group is published: the max, the list length and the first kPF
    // batches of the list in one round trip (entries past the length are masked
    // later; the list region holds qcap entries)
    constexpr int kPF = 3;  // list batches in registers: the current one + 2 ahead
    float gm[GH], th[GH], lsum[GH];
    int nsel[GH], nret[GH];
    const int* gi = ws.gidx + (size_t)c * chunk + quarter * qcap;
    const float* gs = ws.cscore + (size_t)(c * 4 + quarter) * G * qcap;
    const int n = __ldcg(&ws.cnt[(size_t)c * 4 + quarter]);
#pragma unroll
    for (int jj = 0; jj < GH; ++jj) {
      const int j = jb + jj;
      gm[jj] = j < G ? dec_max(__ldcg(&ws.gmax[b * bt.Hq + h * G + j])) : 0.f;
      lsum[jj] = 0.f;
      nsel[jj] = nret[jj] = 0;
    }
    int row_q[kPF];
    float sc_q[kPF][GH];
#pragma unroll
    for (int p = 0; p < kPF; ++p) {
      const int ii = p * 32 + lane;
      row_q[p] = ii < qcap ? __ldcg(gi + ii) : 0;
#pragma unroll
      for (int jj = 0; jj < GH; ++jj)
        sc_q[p][jj] = (ii < qcap && jb + jj < G) ? __ldcg(gs + (jb + jj) * qcap + ii) : -INFINITY;
    }
#pragma unroll
    for (int jj = 0; jj < GH; ++jj) th[jj] = gm[jj] - bt.beta;
    int i0 = 0;
    const int box = quarter >> 1, c16_0 = (quarter & 1) * 4;  // this quarter's 32 token columns of B
    // B rows this warp owns: sp*G + j for its heads (half 0 also the padding rows 3G..NP-1)
    const int nrows_own = 3 * GH + (hf == 0 ? NP - 3 * G : 0);
    auto own_row = [&](int r) {  // r < nrows_own
      if (r < 3 * GH) {
        const int sp = r / GH, jj = r - sp * GH;
        return jb + jj < G ? sp * G + jb + jj : -1;
      }
      return 3 * G + (r - 3 * GH);
    };
    for (int tl = 0; tl < ntiles; ++tl) {
      const int bi = tl & 1;
      if (tl >= 2) mbar_wait(bfree0 + 8u * bi, (uint32_t)((tl >> 1) - 1) & 1u);
      uint8_t* bb = bbuf + bi * kBBytes;
      for (int i = lane; i < nrows_own * 4; i += 32) {  // zero this warp's rows in its quarter's columns
        const int nn = own_row(i >> 2), c16 = c16_0 + (i & 3);
        if (nn >= 0)
          *reinterpret_cast<uint4*>(bb + box * (NP * 128) + (nn >> 3) * 1024 + (nn & 7) * 128 +
                                    ((c16 ^ (nn & 7)) << 4)) = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      // listed rows of this tile (the sub-list is in token order; a batch may span tiles)
      while (i0 < n) {
        const bool ok = i0 + lane < n;
        const int tile_of = ok ? (row_q[0] >> 7) : 0x7fffffff;
        const bool mine = ok && tile_of == tl;
        const bool inwin = mine && in_window(s.off + t0 + row_q[0], s.P, bt.wi, bt.wl);
        const int k = row_q[0] & 127, kk = k & 63, c16 = kk >> 3, wpos = kk & 7;
#pragma unroll
        for (int jj = 0; jj < GH; ++jj) {
          const int j = jb + jj;
          if (j >= G) break;  // (warp-uniform)
          const bool pass = mine && sc_q[0][jj] >= th[jj];
          const bool sel = pass && !inwin;
          const unsigned bs = __ballot_sync(kFull, sel);
          if (sel)  // selected ids of (chunk, head j), quarter list (diagnostics)
            ws.cidx[((size_t)c * G + j) * chunk + quarter * qcap + nsel[jj] + __popc(bs & lanemask_lt())] = row_q[0];
          nsel[jj] += __popc(bs);
          nret[jj] += pass ? 1 : 0;  // per lane, summed at the end
          const float w = sel ? exp2f((sc_q[0][jj] - gm[jj]) * k2) : 0.f;
          lsum[jj] += w;
          if (mine) {
            const __nv_bfloat16 hi = __float2bfloat16_rn(w);
            const float r1 = w - __bfloat162float(hi);
            const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
            const uint16_t parts[3] = {__bfloat16_as_ushort(hi), __bfloat16_as_ushort(mid),
                                       bf16_bits(r1 - __bfloat162float(mid))};
#pragma unroll
            for (int sp = 0; sp < 3; ++sp) {
              const int nn = sp * G + j;
              *reinterpret_cast<uint16_t*>(bb + (k >> 6) * (NP * 128) + (nn >> 3) * 1024 + (nn & 7) * 128 +
                                           ((c16 ^ (nn & 7)) << 4) + wpos * 2) = parts[sp];
            }
          }
        }
        if (__any_sync(kFull, ok && tile_of > tl)) break;  // the rest of the batch is a later tile's
        i0 += 32;
#pragma unroll
        for (int p = 0; p + 1 < kPF; ++p) {
          row_q[p] = row_q[p + 1];
#pragma unroll
          for (int jj = 0; jj < GH; ++jj) sc_q[p][jj] = sc_q[p + 1][jj];
        }
        const int ii = i0 + (kPF - 1) * 32 + lane;
        row_q[kPF - 1] = ii < n ? __ldcg(gi + ii) : 0;
#pragma unroll
        for (int jj = 0; jj < GH; ++jj)
          sc_q[kPF - 1][jj] = (ii < n && jb + jj < G) ? __ldcg(gs + (jb + jj) * qcap + ii) : -INFINITY;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tcgen05 reads
      __syncwarp();
      if (lane == 0) mbar_arrive(bfull0 + 8u * bi);
    }
    // epilogue: lane = d, columns sp*G + j -> the (chunk, head j) partial
    mbar_wait(accf, 0);
    fence_after();
    float v[NP];
    tmem_ld<NP>(tmem + ((uint32_t)(quarter * 32) << 16), v);
    const size_t cj0 = (size_t)c * G;
    const int d = quarter * 32 + lane;
#pragma unroll
    for (int jj = 0; jj < GH; ++jj) {
      const int j = jb + jj;
      if (j >= G) break;
      float o = 0.f;
#pragma unroll
      for (int jx = 0; jx < G; ++jx)  // (register-indexed v: select the head's columns)
        if (jx == j) o = (v[jx] + v[G + jx]) + v[2 * G + jx];
      ws.part_acc[(cj0 + j) * D + d] = o;
      const float l = warp_sum(lsum[jj]);
      const int nr = (int)warp_sum((float)nret[jj]);
      if (lane == 0) { s_l[quarter][j] = l; s_ns[quarter][j] = nsel[jj]; s_nr[quarter][j] = nr; }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(128 * kSplit) : "memory");  // the builder warps
    if (warp == 2 && lane < G) {
      const int j = lane;
      float l = 0.f;
      int ns = 0, nr = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // fixed order
        l += s_l[q][j];
        ns += s_ns[q][j];
        nr += s_nr[q][j];
        ws.ovl_sel[(cj0 + j) * 4 + q] = s_ns[q][j];
        ws.ovl_ret[(cj0 + j) * 4 + q] = s_nr[q][j];
      }
      ws.part_l[cj0 + j] = l;
      ws.selcnt[cj0 + j] = ns;
      ws.retcnt[cj0 + j] = nr;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  }
}

}  // namespace tc
}  // namespace alaya
