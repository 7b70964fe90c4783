// Fused persistent decode kernel (bf16 K/V, d = 128): the tcgen05 DIPR scan
// and the V-gather attention run CONCURRENTLY in every SM, so the random
// 256-byte V-row gathers (DRAM-page bound on their own) overlap the streaming
// K scan instead of following it.
//
//   warp 0      TMA producer; claims chunks from a global ticket and publishes
//               each chunk id through a small smem queue (dynamic scheduling:
//               no CTA ever waits for work owned by a non-resident CTA).
//   warp 1      TMEM allocator + MMA issuer (as in alaya_tc.cuh).
//   warps 2-5   scan epilogue, one TMEM lane quarter each, no cross-warp
//               barriers: candidates, per-chunk atomic max, then a
//               release-ordered increment of the (sequence, kv head) group's
//               completion counter (4 per chunk).
//   warps 6-13  attention workers: window partials first (independent of the
//               threshold), then (chunk, head) selection tasks in chunk order;
//               a task starts once its group's counter says every chunk of the
//               group has published, i.e. the group's global max is final.
#pragma once

#include "alaya_kernels.cuh"
#include "alaya_tc.cuh"

namespace alaya {
namespace fused {

constexpr int kAttnWarps = 8;
constexpr int kScanWarps = 6;
constexpr int kThreadsFused = (kScanWarps + kAttnWarps) * 32;
constexpr int kQueue = 4;  // chunk-id queue depth

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int G, int kStages>
__global__ void __launch_bounds__(kThreadsFused, 1)
    fused_tc_kernel(const __grid_constant__ Batch bt, const __grid_constant__ tc::Maps maps,
                    const float* __restrict__ q, Ws ws, int* __restrict__ group_done) {
  using namespace tc;
  constexpr int NP = (3 * G <= 16) ? 16 : 32;
  constexpr int kBBytes = 2 * NP * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_ring = smem;
  uint8_t* b_buf = a_ring + kStages * kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_buf + 2 * kBBytes);
  // full[S], empty[S], accf[kAcc], acce[kAcc], cfull[Q], cempty[Q], bfree[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kAcc + 2 * kQueue + 2);
  int* chunk_q = reinterpret_cast<int*>(tmem_slot + 4);              // [kQueue]
  float* tmax = reinterpret_cast<float*>(chunk_q + kQueue);           // [3][4][G]
  int* s_t_all = reinterpret_cast<int*>(tmax + 3 * 4 * G);            // [kAttnWarps][2][32]
  float* s_w_all = reinterpret_cast<float*>(s_t_all + kAttnWarps * 64);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
  const uint32_t accf0 = bar0 + 8u * (2 * kStages), acce0 = accf0 + 8u * kAcc;
  auto cfull_bar = [&](int i) { return acce0 + 8u * (kAcc + i); };
  auto cempty_bar = [&](int i) { return acce0 + 8u * (kAcc + kQueue + i); };
  const uint32_t bfree0 = acce0 + 8u * (kAcc + 2 * kQueue);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 1); }
    for (int a = 0; a < kAcc; ++a) { mbar_init(accf0 + 8u * a, 1); mbar_init(acce0 + 8u * a, 4); }
    // consumers of a queue slot: the MMA warp and the 4 epilogue warps
    for (int i = 0; i < kQueue; ++i) { mbar_init(cfull_bar(i), 1); mbar_init(cempty_bar(i), 5); }
    for (int i = 0; i < 2; ++i) mbar_init(bfree0 + 8u * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kAcc * NP));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 2 * kBBytes / 16; i += kThreadsFused)
    reinterpret_cast<uint4*>(b_buf)[i] = make_uint4(0, 0, 0, 0);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int chunk = bt.chunk;

  if (warp == 0) {
    // ===================== TMA producer + chunk scheduler =====================
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int stage = 0, slot = 0;
      uint32_t phase = 0, qphase = 0;
      for (;;) {
        int c = atomicAdd(&ws.counters[1], 1);
        if (c >= bt.total_chunks) c = -1;
        mbar_wait(cempty_bar(slot), qphase ^ 1);
        chunk_q[slot] = c;
        mbar_arrive(cfull_bar(slot));
        if (++slot == kQueue) { slot = 0; qphase ^= 1; }
        if (c < 0) break;
        int b, h, ci;
        decode_chunk(bt, c, b, h, ci);
        const int valid = min(chunk, bt.s[b].n - ci * chunk);
        const int ntiles = (valid + kTileKeys - 1) / kTileKeys;
        const CUtensorMap* map = &maps.m[maps.map_of_seq[b]];
        const int row0 = (int)(h * maps.rows_per_head[b] + (int64_t)ci * chunk);
        for (unsigned long long m = chunk_tiles(bt, ws, c, ntiles); m; m &= m - 1) {
          const int tl = __ffsll((long long)m) - 1;
          mbar_wait(empty_bar(stage), phase ^ 1);
          mbar_expect_tx(full_bar(stage), kTileBytes);
          const uint32_t dst = smem_u32(a_ring + stage * kTileBytes);
          tma_load_2d(dst, map, 0, row0 + tl * kTileKeys, full_bar(stage), pol);
          tma_load_2d(dst + kBoxBytes, map, 64, row0 + tl * kTileKeys, full_bar(stage), pol);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc = idesc_bf16<NP>();
    int stage = 0, acc = 0, cidx = 0, slot = 0, bcnt = 0;
    uint32_t phase = 0, ephase = 0, qphase = 0, bphase = 0;
    for (;; ++cidx) {
      mbar_wait(cfull_bar(slot), qphase);
      const int c = chunk_q[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(cempty_bar(slot));
      if (++slot == kQueue) { slot = 0; qphase ^= 1; }
      if (c < 0) break;
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
          mbar_wait(bfree0 + 8u * bi, ((bphase >> bi) & 1u) ^ 1u);  // last reader done
          bphase ^= 1u << bi;
          build_b<G, NP>(bb, q + ((size_t)b * bt.Hq + (size_t)h * G) * 128, lane);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
        }
        mbar_wait(full_bar(stage), phase);
        fence_after();
        if (lane == 0) {
          mma_tile<NP>(smem_u32(a_ring + stage * kTileBytes), smem_u32(bb), tmem_base + acc * NP, idesc);
          mma_commit(empty_bar(stage));
          mma_commit(accf0 + 8u * acc);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        acc = (acc + 1) % kAcc;
      }
      if (!first) {  // this chunk used B buffer bi: free it once its MMAs complete
        if (lane == 0) mma_commit(bfree0 + 8u * bi);
        __syncwarp();
        ++bcnt;
      }
    }
  } else if (warp < kScanWarps) {
    // ===================== scan epilogue (warps 2..5) =====================
    const int quarter = warp & 3;
    int acc = 0, slot = 0, tcount = 0;
    uint32_t aphase = 0, qphase = 0;
    for (;;) {
      mbar_wait(cfull_bar(slot), qphase);
      const int c = chunk_q[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(cempty_bar(slot));
      if (++slot == kQueue) { slot = 0; qphase ^= 1; }
      if (c < 0) break;
      int b, h;
      epilogue_chunk<G, NP>(bt, ws, c, quarter, lane, tmem_base, accf0, acce0, acc, aphase, b, h,
                            tmax, tcount);
      __threadfence();  // this warp's candidates, counts and max are visible GPU-wide ...
      __syncwarp();
      if (lane == 0) atomicAdd(&group_done[b * bt.Hkv + h], 1);  // ... before its group count
    }
  } else {
    // ===================== attention workers (warps 6..13) =====================
    const int aw = warp - kScanWarps;
    int(*s_t)[32] = reinterpret_cast<int(*)[32]>(s_t_all + aw * 64);
    float(*s_w)[32] = reinterpret_cast<float(*)[32]>(s_w_all + aw * 64);
    const int nwin = bt.B * bt.Hq;
    const int npairs = bt.total_chunks * G;
    const int ntasks = nwin + npairs;
    auto wait_group = [&](int c) {
      int b, h, ci;
      decode_chunk(bt, c, b, h, ci);
      if (lane == 0) {  // every epilogue warp of every chunk of the group published
        const int* gd = group_done + b * bt.Hkv + h;
        while (ld_acquire(gd) < 4 * bt.s[b].nch) __nanosleep(200);
      }
      __syncwarp();
    };
    for (;;) {
      int task = 0;
      if (lane == 0) task = atomicAdd(&ws.counters[0], 1);
      task = __shfl_sync(kFull, task, 0);
      if (task >= ntasks) break;
      if (task < nwin) {
        win_task<__nv_bfloat16, 128, G>(bt, q, ws, task, lane);
        continue;
      }
      const size_t cj = task - nwin;
      wait_group((int)cj / G);
      sel_task_pipe<__nv_bfloat16, 128, G, true>(bt, nullptr, ws, cj, 0, 4, lane, s_t, s_w, true);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAcc * NP));
  }
}

inline size_t fused_smem_bytes(int G, int kStages) {
  const int NP = (3 * G <= 16) ? 16 : 32;
  return 1024 + (size_t)kStages * tc::kTileBytes + 2 * 2 * NP * 128 +
         8 * (2 * kStages + 2 * tc::kAcc + 2 * kQueue + 2) + 16 + 4 * kQueue + 3 * 4 * G * 4 +
         kAttnWarps * 64 * 8 + 64;
}

}  // namespace fused
}  // namespace alaya
