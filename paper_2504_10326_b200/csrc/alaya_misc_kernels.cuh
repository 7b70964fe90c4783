// Non-templated kernels (merge across shards, selected-id export); included
// only by alaya.cu.
#pragma once

#include "alaya_common.cuh"

namespace alaya {

// Merge of shard partials (attention.py:128-152), rows = batch * Hq.
__global__ void merge_partials_kernel(const float* __restrict__ parts, int n_parts, int rows, int D,
                                      float* __restrict__ out, float* __restrict__ state_out,
                                      int* status, const unsigned long long* flags = nullptr,
                                      unsigned long long epoch = 0, int* err = nullptr,
                                      int64_t part_stride = 0) {
  const int row = blockIdx.x;
  if (flags) {  // parts are the exchange slots the ranks push into (fused sharded step): wait for them
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    if (threadIdx.x < n_parts) {
      long long polls = 0;
      while (ld_acquire_sys_u64(flags + threadIdx.x) < epoch) {
        if (++polls > (1ll << 26)) {
          s_bad = 1;
          break;
        }
        __nanosleep(64);
      }
    }
    __syncthreads();
    if (s_bad) {
      if (threadIdx.x == 0 && err) atomicExch(err, 1);
      return;
    }
  }
  const size_t stride = part_stride ? (size_t)part_stride : (size_t)rows * (D + 2);
  float m = -INFINITY;
  for (int r = 0; r < n_parts; ++r) m = fmaxf(m, __ldcg(parts + r * stride + (size_t)row * (D + 2)));
  float l = 0.f;
  for (int r = 0; r < n_parts; ++r) {
    const float* p = parts + r * stride + (size_t)row * (D + 2);
    if (__ldcg(p) != -INFINITY) l += __ldcg(p + 1) * expf(__ldcg(p) - m);
  }
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    float a = 0.f;
    for (int r = 0; r < n_parts; ++r) {
      const float* p = parts + r * stride + (size_t)row * (D + 2);
      if (__ldcg(p) != -INFINITY) a += __ldcg(p + 2 + e) * expf(__ldcg(p) - m);
    }
    if (out) {
      const float o = a / l;
      if (!isfinite(o) && status) atomicExch(status, (int)ALAYA_ERR_NONFINITE);
      out[(size_t)row * D + e] = o;
    }
    if (state_out) {
      float* so = state_out + (size_t)row * (D + 2);
      if (e == 0) { so[0] = m; so[1] = l; }
      so[2 + e] = a;
    }
  }
}

// Graph mode: commit the appended window row (after every append thread read *dw).
__global__ void window_commit_kernel(const __grid_constant__ Batch bt) {
  pdl_wait();
  pdl_trigger();
  for (int b = threadIdx.x; b < bt.B; b += blockDim.x) {
    const KSeq& s = bt.s[b];
    if (s.dw && *s.dw < s.w) *s.dw += 1;
  }
}

// Selected ids (global, ascending) + counts per (sequence, q head).
__global__ void __launch_bounds__(kThreads) selected_kernel(const __grid_constant__ Batch bt, Ws ws,
                                                          int64_t* __restrict__ ids, int64_t cap,
                                                          int32_t* __restrict__ nsel, int32_t* __restrict__ nret) {
  // Grid (rows, splits): CTA (row = seq*Hq + q head, split) writes the selected ids
  // of chunks [split*8, split*8 + 8) of the row in ASCENDING order (the
  // reference's sorted diagnostics, store.py:288-292), one chunk per warp, at
  // the chunk's offset in the row (a block scan of the per-chunk counts), and
  // only up to the row's selected count. A chunk's selection sits in up to 4
  // ordered sub-lists (lane quarters of the tcgen05 scan, split pairs,
  // group-format quarters) whose rows interleave; the warp ORs them into a
  // chunk-row bitmap in shared memory and emits the set bits in order.
  constexpr int kMaxWords = 8192 / 32;  // chunk <= 8192
  __shared__ unsigned bm[kWarps][kMaxWords];
  __shared__ int wsum[kWarps], wret[kWarps];
  extern __shared__ int chunk_base[];   // [nch] exclusive prefix of selected counts
  pdl_wait();     // the call's attend/combine are complete
  pdl_trigger();  // (the next call's prep waits for this grid before zeroing the header)
  const int row = blockIdx.x;
  const int b = row / bt.Hq, qh = row - b * bt.Hq;
  const int h = qh / bt.G, j = qh - h * bt.G;
  const KSeq& s = bt.s[b];
  const int c0 = s.chunk_base + h * s.nch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool gfmt = *ws.mode != 0;  // group format (attend_grp_kernel): 4 quarter lists per pair
  auto nlists = [&](size_t cj) { return (gfmt || ws.heavy[cj] != 0) ? 4 : 1; };
  auto count_of = [&](size_t cj, int sq) {
    return (sq == 0 && !gfmt) ? ws.selcnt[cj] : ws.ovl_sel[cj * 4 + sq];
  };
  // per-chunk counts: thread t owns the contiguous chunks [t*seg, (t+1)*seg)
  const int seg = (s.nch + blockDim.x - 1) / blockDim.x;
  const int cb = threadIdx.x * seg, ce = min(s.nch, cb + seg);
  int mine = 0, mret = 0;
  for (int c = cb; c < ce; ++c) {
    const size_t cj = (size_t)(c0 + c) * bt.G + j;
    int n = 0;
    for (int sq = 0, L = nlists(cj); sq < L; ++sq) {
      n += count_of(cj, sq);
      mret += (sq == 0 && !gfmt) ? ws.retcnt[cj] : ws.ovl_ret[cj * 4 + sq];
    }
    chunk_base[c] = n;
    mine += n;
  }
  // block exclusive scan of the per-thread sums
  int incl = mine;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, m);
    if (lane >= m) incl += y;
  }
  int r = mret;
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) r += __shfl_xor_sync(kFull, r, m);
  if (lane == 31) wsum[warp] = incl;
  if (lane == 0) wret[warp] = r;
  __syncthreads();
  int before = 0, total = 0, rtot = 0;
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp) before += wsum[w];
    total += wsum[w];
    rtot += wret[w];
  }
  int run = before + incl - mine;
  for (int c = cb; c < ce; ++c) {
    const int n = chunk_base[c];
    chunk_base[c] = run;
    run += n;
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) { nsel[row] = total; nret[row] = rtot; }
  __syncthreads();
  const int words = (bt.chunk + 31) / 32;
  unsigned* bw = bm[warp];
  const int c = blockIdx.y * kWarps + warp;
  if (c >= s.nch) return;
  const size_t cj = (size_t)(c0 + c) * bt.G + j;
  for (int w = lane; w < words; w += 32) bw[w] = 0u;
  __syncwarp();
  for (int sq = 0, L = nlists(cj); sq < L; ++sq) {
    const int n = count_of(cj, sq);
    const int* src = ws.cidx + cj * bt.chunk + sq * (bt.chunk / 4);
    for (int i = lane; i < n; i += 32) {
      const int rr = src[i];
      atomicOr(&bw[rr >> 5], 1u << (rr & 31));
    }
  }
  __syncwarp();
  int out = chunk_base[c];
  for (int w0 = 0; w0 < words; w0 += 32) {
    const int w = w0 + lane;
    const unsigned bits = w < words ? bw[w] : 0u;
    const int cnt = __popc(bits);
    int in = cnt;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int y = __shfl_up_sync(kFull, in, m);
      if (lane >= m) in += y;
    }
    int pos = out + in - cnt;
    for (unsigned x = bits; x; x &= x - 1) {
      if (pos < cap) ids[(size_t)row * cap + pos] = s.off + (int64_t)c * bt.chunk + w * 32 + (__ffs(x) - 1);
      ++pos;
    }
    out += __shfl_sync(kFull, in, 31);
  }
}

// Session-window append: one thread per element of [B][Hkv][D].
template <typename T>
__global__ void window_append_kernel(const __grid_constant__ Batch bt, const float* __restrict__ k,
                                     const float* __restrict__ v) {
  pdl_wait();  // PDL launch: the previous layer's kernels may still be finishing
  pdl_trigger();
  const int D = bt.D;
  const long total = (long)bt.B * bt.Hkv * D;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int e = (int)(i % D);
    const long bh = i / D;
    const int h = (int)(bh % bt.Hkv), b = (int)(bh / bt.Hkv);
    const KSeq& s = bt.s[b];
    const int row = s.dw ? __ldcg(s.dw) : s.w;
    if (s.dw && row >= s.w) continue;  // ring full (graph mode): dropped, not committed
    const size_t off = (size_t)h * s.whs + (size_t)row * D + e;
    T* wk = const_cast<T*>(reinterpret_cast<const T*>(s.wk));
    T* wv = const_cast<T*>(reinterpret_cast<const T*>(s.wv));
    if constexpr (std::is_same_v<T, float>) {
      wk[off] = k[i];
      wv[off] = v[i];
    } else {
      wk[off] = __float2bfloat16_rn(k[i]);
      wv[off] = __float2bfloat16_rn(v[i]);
    }
  }
}

}  // namespace alaya
