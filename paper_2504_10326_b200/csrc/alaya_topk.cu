// TOP_K retrieval (the other flat-scan query type) and sparse attention over
// an explicit id list:
//
//   topk_select_kernel   exact top-k of one (sequence, q head) over the scan's
//                        score lists (FlatIndex.top_k, index.py:60-66: scores
//                        descending, ties by smaller token id) -- MSB radix
//                        select on the order-preserving score encoding, then
//                        on the token id among the ties at the threshold.
//   block_reps_kernel    BlockIndex build (index.py:217-243): per block of
//                        block_size tokens the r keys of largest L2 norm
//                        (fp64 norms, ties by position).
//   block_topk_kernel    BlockIndex.top_blocks (index.py:206-214) + the TOP_K
//                        branch of Session._retrieve (store.py:305-312):
//                        block score = max representative score, best
//                        k_blocks blocks (ties by smaller start), union of
//                        their token ranges clipped to the prefix.
//   sparse_attn_kernel   Session._head_attention after retrieval
//                        (store.py:268-293): drop window ids, partial
//                        attention over the remaining ids (K and V gathered)
//                        merged with the window partial, finalized.
#include "alaya_dispatch.cuh"

namespace alaya {
namespace {

constexpr int kSelThreads = 512;
constexpr int kSelectThreads = 1024;  // topk_select_kernel

// Histogram increment aggregated over the warp's active lanes that hit the same
// bin: radix digits of nearby scores collide heavily, and per-lane shared atomics
// on one bin serialise.
__device__ __forceinline__ void hist_add(unsigned* hist, unsigned bin) {
  const unsigned act = __activemask();
  const unsigned same = __match_any_sync(act, bin);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(same) - 1)) atomicAdd(&hist[bin], (unsigned)__popc(same));
}

// One MSB radix-select digit: among elements with (key & mask) == prefix,
// pick the bin holding the kk-th element (descending keys if desc, else
// ascending). Returns the bin's population; updates prefix/mask/kk.
// `found` becomes false when fewer than kk elements match (take everything).
__device__ __forceinline__ void pick_bin(unsigned* hist, int shift, bool desc, uint64_t& prefix,
                                         uint64_t& mask, long long& kk, bool& found,
                                         unsigned* s_pop) {
  // the bin holding the kk-th element in scan order (desc: 255..0): warp 0, each
  // lane 8 consecutive bins, one warp prefix sum, the first lane whose inclusive
  // sum reaches kk scans its own 8 bins (a serial 256-bin loop cost ~5 us a pass)
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    unsigned v[8];
    long long loc = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = lane * 8 + t;
      v[t] = hist[desc ? 255 - i : i];
      loc += v[t];
    }
    long long inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const long long want = kk;
    const unsigned hit = __ballot_sync(0xffffffffu, inc >= want);
    if (hit == 0u) {
      if (lane == 0) found = false;
    } else if (lane == __ffs(hit) - 1) {
      long long cum = inc - loc;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (cum + v[t] >= want) {
          const int i = lane * 8 + t;
          prefix |= (uint64_t)(desc ? 255 - i : i) << shift;
          kk = want - cum;
          found = true;
          *s_pop = v[t];
          break;
        }
        cum += v[t];
      }
    }
    if (lane == 0) mask |= (uint64_t)255 << shift;
  }
  __syncthreads();
}

// Chunk-local pruning for top-k: a token can be in its row's top-k only if
// fewer than k tokens of its own (chunk, head) pair precede it in the order
// (score desc, id asc), so each pair keeps just its local top-k. One CTA per
// pair: candidates staged in smem, radix select, survivors written back as
// one contiguous fill of the pair's list (sub-list q = [q*chunk/4, ...)).
constexpr int kCkThreads = 256;

__global__ void __launch_bounds__(kCkThreads)
    chunk_topk_kernel(const __grid_constant__ Batch bt, Ws ws, int k) {
  extern __shared__ uint32_t s_key[];  // [chunk] encoded scores, then [chunk] local ids
  __shared__ unsigned hist[256];
  __shared__ uint64_t s_prefix, s_mask;
  __shared__ long long s_kk;
  __shared__ bool s_found;
  __shared__ unsigned s_pop;
  __shared__ int s_n;
  pdl_trigger();
  pdl_wait();
  const size_t cj = blockIdx.x;
  const int chunk = bt.chunk, qcap = chunk / 4;
  int* s_id = reinterpret_cast<int*>(s_key + chunk);
  int n4[4], m = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) { n4[q] = ws.cnt[cj * 4 + q]; m += n4[q]; }
  if (m <= k) return;  // nothing to prune
  int base = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float* sc = ws.cscore + cj * chunk + q * qcap;
    const int* id = ws.cidx + cj * chunk + q * qcap;
    for (int i = threadIdx.x; i < n4[q]; i += blockDim.x) {
      s_key[base + i] = enc_max(sc[i]);
      s_id[base + i] = id[i];
    }
    base += n4[q];
  }
  if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_kk = k; s_n = 0; }
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t pre = (uint32_t)s_prefix, msk = (uint32_t)s_mask;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const uint32_t u = s_key[i];
      if ((u & msk) == pre) hist_add(hist, (u >> shift) & 255);
    }
    pick_bin(hist, shift, true, s_prefix, s_mask, s_kk, s_found, &s_pop);
  }
  const uint32_t T = (uint32_t)s_prefix;
  const long long need = s_kk;
  const bool ties = (long long)s_pop > need;
  __syncthreads();
  if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; }
  if (ties) {  // local ids < 2^16 (chunk <= 8192)
    for (int shift = 8; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const uint32_t pre = (uint32_t)s_prefix, msk = (uint32_t)s_mask;
      for (int i = threadIdx.x; i < m; i += blockDim.x)
        if (s_key[i] == T && ((uint32_t)s_id[i] & msk) == pre)
          hist_add(hist, ((uint32_t)s_id[i] >> shift) & 255);
      pick_bin(hist, shift, false, s_prefix, s_mask, s_kk, s_found, &s_pop);
    }
  }
  const uint32_t Tid = ties ? (uint32_t)s_prefix : 0xffffffffu;
  __syncthreads();
  float* osc = ws.cscore + cj * chunk;
  int* oid = ws.cidx + cj * chunk;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t u = s_key[i];
    if (u > T || (u == T && (uint32_t)s_id[i] <= Tid)) {
      const int o = atomicAdd(&s_n, 1);
      osc[o] = dec_max(u);
      oid[o] = s_id[i];
    }
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    const int q = threadIdx.x;
    ws.cnt[cj * 4 + q] = max(0, min(qcap, s_n - q * qcap));
  }
}

// ---------------------------------------------------------------------------
// TOP_K candidate bound: the k-th largest score among S evenly spaced base keys
// of a row is <= the row's k-th largest score (a k-subset argument), so the scan
// only needs to keep s >= that bound (minus a rounding margin) instead of every
// token. Samples: grid (B*Hkv, ceil(S/256)), a warp per key, all G heads.
constexpr int kMaxG = 8;

template <typename T, int D>
__global__ void __launch_bounds__(256)
    topk_sample_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q,
                       float* __restrict__ samp, int S_max) {
  // one THREAD per sampled key, all G heads: the key row is read as 16-byte
  // vectors (L1-cached), q comes from smem by broadcast, no shuffle reductions
  // (a warp-per-key layout spent its time in 2 warp sums per key and head)
  constexpr int V = 16 / (int)sizeof(T);  // elements per 16-byte load
  __shared__ float s_q[kMaxG][D];
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x / bt.Hkv, h = blockIdx.x - b * bt.Hkv;
  const KSeq& s = bt.s[b];
  const int G = bt.G;
  const int S = min(s.n, S_max);
  for (int t = threadIdx.x; t < G * D; t += blockDim.x)
    s_q[t / D][t % D] = __ldg(q + ((size_t)b * bt.Hq + h * G) * D + t);
  __syncthreads();
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const T* kr = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs + (size_t)((int64_t)i * s.n / S) * D;
  float a[kMaxG], mag[kMaxG];
#pragma unroll
  for (int j = 0; j < kMaxG; ++j) a[j] = mag[j] = 0.f;
#pragma unroll
  for (int e0 = 0; e0 < D; e0 += V) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(kr + e0));
    float x[V];
    if constexpr (std::is_same_v<T, float>) {
      x[0] = __uint_as_float(raw.x); x[1] = __uint_as_float(raw.y);
      x[2] = __uint_as_float(raw.z); x[3] = __uint_as_float(raw.w);
    } else {
      const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        x[2 * t] = __uint_as_float(w[t] << 16);
        x[2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u);
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxG; ++j) {
      if (j >= G) break;
#pragma unroll
      for (int t = 0; t < V; ++t) {
        const float qv = s_q[j][e0 + t];
        a[j] = fmaf(qv, x[t], a[j]);
        mag[j] = fmaf(fabsf(qv), fabsf(x[t]), mag[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kMaxG; ++j) {
    if (j >= G) break;
    samp[((size_t)b * bt.Hq + h * G + j) * S_max + i] = a[j] - 1e-3f * (mag[j] + 1.f);
  }
}

// Per row: the k-th largest of its S samples -> thr[row] (-inf when S < k).
constexpr int kThrThreads = 1024;
__global__ void __launch_bounds__(kThrThreads)
    topk_thr_kernel(const __grid_constant__ Batch bt, const float* __restrict__ samp, int S_max, int k,
                    float* __restrict__ thr) {
  extern __shared__ uint32_t s_u[];  // [S_max]
  __shared__ unsigned hist[256];
  __shared__ uint64_t s_prefix, s_mask;
  __shared__ long long s_kk;
  __shared__ bool s_found;
  __shared__ unsigned s_pop;
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const int b = row / bt.Hq;
  const int S = min(bt.s[b].n, S_max);
  if (S < k) {
    if (threadIdx.x == 0) thr[row] = -INFINITY;
    return;
  }
#pragma unroll 8
  for (int i = threadIdx.x; i < S; i += blockDim.x) s_u[i] = enc_max(__ldg(samp + (size_t)row * S_max + i));
  if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_kk = k; s_found = true; }
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t pre = (uint32_t)s_prefix, msk = (uint32_t)s_mask;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      const uint32_t u = s_u[i];
      if ((u & msk) == pre) hist_add(hist, (u >> shift) & 255);
    }
    pick_bin(hist, shift, true, s_prefix, s_mask, s_kk, s_found, &s_pop);
  }
  if (threadIdx.x == 0) thr[row] = dec_max((uint32_t)s_prefix);
}

// Exact top-k of each row over the scan candidate lists (the scan ran with
// beta = inf, so every base token of the shard is a candidate with its score;
// chunk_topk_kernel may have pruned each pair to its local top-k). The row's
// list offsets are prefix-summed in smem, so every pass is one flat parallel
// loop; when the elements fit, they are staged in smem once (key, local id).
// The row's candidate keys are staged in smem once (encoded scores only, up to
// stage_cap, sized from the free smem at launch) by a segment walk: warp w copies
// segments w, w+W, ... coalesced, so no element needs a search for its segment.
// Local ids are read from global memory only where they are needed (ties at the
// threshold, and the selected elements in the collect pass), again per segment.
__global__ void __launch_bounds__(kSelectThreads)
    topk_select_kernel(const __grid_constant__ Batch bt, Ws ws, int k, int64_t* __restrict__ ids,
                       float* __restrict__ scores, int64_t cap, int32_t* __restrict__ count, int stage_cap) {
  extern __shared__ uint32_t s_dyn[];  // [nseg + 1] offsets, then [stage_cap] encoded keys
  __shared__ unsigned hist[256];
  __shared__ uint64_t s_prefix, s_mask, s_idprefix, s_idmask;
  __shared__ long long s_kk;
  __shared__ bool s_found;
  __shared__ unsigned s_pop;
  __shared__ int s_n;
  __shared__ int s_wsum[kSelectThreads / 32];
  pdl_trigger();
  pdl_wait();
  constexpr int NW = kSelectThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.x;
  const int b = row / bt.Hq, qh = row - b * bt.Hq, h = qh / bt.G, j = qh - h * bt.G;
  const KSeq& sq = bt.s[b];
  const int nch = sq.nch, c0 = sq.chunk_base + h * nch, chunk = bt.chunk, qcap = chunk / 4;
  const int nseg = nch * 4;
  int* s_off = reinterpret_cast<int*>(s_dyn);
  uint32_t* s_key = s_dyn + nseg + 1;
  auto seg_base = [&](int g) {  // first workspace slot of segment g = (chunk g / 4, sub-list g % 4)
    return ((size_t)(c0 + g / 4) * bt.G + j) * chunk + (size_t)(g & 3) * qcap;
  };
  // segment counts -> exclusive offsets (block scan: each thread a contiguous run)
  {
    const int per = (nseg + kSelectThreads - 1) / kSelectThreads;
    const int g0 = min(nseg, threadIdx.x * per), g1 = min(nseg, g0 + per);
    int loc = 0;
    for (int g = g0; g < g1; ++g) loc += ws.cnt[((size_t)(c0 + g / 4) * bt.G + j) * 4 + (g & 3)];
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    int wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
    int run = wpre + inc - loc;
    for (int g = g0; g < g1; ++g) {
      s_off[g] = run;
      run += ws.cnt[((size_t)(c0 + g / 4) * bt.G + j) * 4 + (g & 3)];
    }
    if (threadIdx.x == kSelectThreads - 1) s_off[nseg] = wpre + inc;
    __syncthreads();
  }
  const int total = s_off[nseg];
  // element e -> (score, local id = cc * chunk + position in the chunk) (unstaged rows)
  auto fetch = [&](int e, float& sc, int& lid) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {  // last segment with s_off[g] <= e
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const size_t at = seg_base(lo) + (e - s_off[lo]);
    sc = ws.cscore[at];
    lid = (lo >> 2) * chunk + ws.cidx[at];
  };
  const bool staged = total <= stage_cap;
  if (staged) {
    for (int g = warp; g < nseg; g += NW) {
      const int o = s_off[g], len = s_off[g + 1] - o;
      const float* src = ws.cscore + seg_base(g);
      for (int t = lane; t < len; t += 32) s_key[o + t] = enc_max(src[t]);
    }
    __syncthreads();
  }
  auto key = [&](int e) -> uint32_t {
    if (staged) return s_key[e];
    float sc;
    int lid;
    fetch(e, sc, lid);
    return enc_max(sc);
  };
  if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_kk = k; s_n = 0; s_found = true; }
  // 1) threshold key T: the k-th largest encoded score
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t pre = (uint32_t)s_prefix, msk = (uint32_t)s_mask;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const uint32_t u = key(e);
      if ((u & msk) == pre) hist_add(hist, (u >> shift) & 255);
    }
    pick_bin(hist, shift, true, s_prefix, s_mask, s_kk, s_found, &s_pop);
    if (!s_found) break;  // fewer than k candidates: take them all
  }
  const bool all = !s_found;
  const uint32_t T = (uint32_t)s_prefix;
  const long long need = s_kk;          // elements equal to T to take
  const bool ties = !all && (long long)s_pop > need;
  // visit every element as (encoded key, local-id loader): segment walk when staged
  auto visit = [&](auto&& fn) {
    if (staged) {
      for (int g = warp; g < nseg; g += NW) {
        const int o = s_off[g], len = s_off[g + 1] - o;
        const size_t base = seg_base(g);
        const int lid0 = (g >> 2) * chunk;
        for (int t = lane; t < len; t += 32)
          fn(s_key[o + t], [&] { return lid0 + ws.cidx[base + t]; });
      }
    } else {
      for (int e = threadIdx.x; e < total; e += blockDim.x) {
        float sc;
        int lid;
        fetch(e, sc, lid);
        fn(enc_max(sc), [&] { return lid; });
      }
    }
  };
  // 2) among the ties at T, the need-th smallest local id (= smallest token id)
  __syncthreads();
  if (threadIdx.x == 0) { s_idprefix = 0; s_idmask = 0; s_kk = need; }
  __syncthreads();
  if (ties) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const uint32_t pre = (uint32_t)s_idprefix, msk = (uint32_t)s_idmask;
      visit([&](uint32_t u, auto&& lid_of) {
        if (u != T) return;
        const uint32_t lid = (uint32_t)lid_of();
        if ((lid & msk) == pre) hist_add(hist, (lid >> shift) & 255);
      });
      pick_bin(hist, shift, false, s_idprefix, s_idmask, s_kk, s_found, &s_pop);
    }
  }
  const uint32_t Tid = ties ? (uint32_t)s_idprefix : 0xffffffffu;
  // 3) collect (set semantics: order is not part of the contract)
  visit([&](uint32_t u, auto&& lid_of) {
    if (!(all || u >= T)) return;
    const int lid = lid_of();
    if (all || u > T || (uint32_t)lid <= Tid) {
      const int o = atomicAdd(&s_n, 1);
      if (o < cap) {
        ids[(size_t)row * cap + o] = sq.off + lid;
        if (scores) scores[(size_t)row * cap + o] = dec_max(u);
      }
    }
  });
  __syncthreads();
  if (threadIdx.x == 0) count[row] = min((int64_t)s_n, cap);
}

// ---------------------------------------------------------------------------
// BlockIndex: representatives = the r largest-L2-norm keys of each block.
template <typename T>
__global__ void __launch_bounds__(256)
    block_reps_kernel(const T* __restrict__ k, int64_t head_stride, int n, int D, int block_size,
                      int r, T* __restrict__ reps, int64_t reps_head_stride, int nblocks) {
  extern __shared__ double s_norm[];  // [block_size]
  const int blk = blockIdx.x % nblocks, h = blockIdx.x / nblocks;
  const int s0 = blk * block_size, cnt = min(block_size, n - s0);
  const T* kb = k + (size_t)h * head_stride + (size_t)s0 * D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = warp; i < cnt; i += 8) {
    double a = 0.0;
    for (int e = lane; e < D; e += 32) {
      const double x = (double)to_f(kb[(size_t)i * D + e]);
      a = fma(x, x, a);
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) a += __shfl_xor_sync(kFull, a, m);
    if (lane == 0) s_norm[i] = a;  // squared norm: same order as the norm
  }
  __syncthreads();
  __shared__ int s_pick;
  T* out = reps + (size_t)h * reps_head_stride + (size_t)blk * r * D;
  const int take = min(r, cnt);
  for (int t = 0; t < r; ++t) {
    if (t < take) {
      if (threadIdx.x == 0) {  // argmax, ties by smaller position
        int best = -1;
        double bv = -1.0;
        for (int i = 0; i < cnt; ++i)
          if (s_norm[i] > bv) { bv = s_norm[i]; best = i; }
        s_norm[best] = -2.0;
        s_pick = best;
      }
      __syncthreads();
    }
    // unused slots repeat the first representative (the block max is unchanged)
    const int src = t < take ? s_pick : -1;
    for (int e = threadIdx.x; e < D; e += blockDim.x) {
      const T x = src >= 0 ? kb[(size_t)src * D + e] : out[e];
      out[(size_t)t * D + e] = x;
    }
    __syncthreads();
  }
}

// Best k_blocks blocks per row by max representative score (ties by smaller
// start); writes the union of their token ranges, clipped to the prefix.
template <typename T, int D>
__global__ void __launch_bounds__(kSelThreads)
    block_topk_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q,
                      const __grid_constant__ BixSet bix, int block_size, int k_blocks,
                      int64_t* __restrict__ ids, int64_t cap, int32_t* __restrict__ count,
                      int32_t* __restrict__ blocks, float* __restrict__ bscores) {
  extern __shared__ uint32_t s_score[];  // [n_blocks] encoded max representative score
  __shared__ unsigned hist[256];
  __shared__ uint64_t s_prefix, s_mask, s_idprefix, s_idmask;
  __shared__ long long s_kk;
  __shared__ bool s_found;
  __shared__ unsigned s_pop;
  __shared__ int s_n, s_nb;
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const int b = row / bt.Hq, qh = row - b * bt.Hq, h = qh / bt.G;
  const KSeq& s = bt.s[b];
  const alaya_block_index& bi = bix.b[b];
  const int nb = bi.n_blocks, r = bi.r;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hl = lane & 15, hw = threadIdx.x >> 4;  // half-warp per representative row
  // representative rows in flight per half-warp: 16, or 8 when a lane's share of a
  // row is 32 B (fp32 d = 128; 16 would need 128 registers and spill)
  constexpr int DPL = D / 16, U = (int)sizeof(T) * DPL <= 16 ? 16 : 8, NHW = kSelThreads / 16;
  float qr[DPL];
  load_q<DPL>(q + (size_t)row * D + hl * DPL, qr);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s_score[i] = 0u;  // -inf
  __syncthreads();
  const T* rb = reinterpret_cast<const T*>(bi.reps) + (size_t)h * bi.head_stride;
  const int nrep = nb * r;
  // warp-uniform trip count (the half-warp reductions shuffle across the warp)
  for (int w0 = warp * 2; w0 < nrep; w0 += NHW * U) {
    const int i0 = w0 + (hw & 1);
    RawFrag<T, DPL> f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * NHW;
      if (i < nrep) f[u].load(rb + (size_t)i * D + hl * DPL); else f[u].zero();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * NHW;
      float x[DPL];
      f[u].to_float(x);
      float a = 0.f;
#pragma unroll
      for (int e = 0; e < DPL; ++e) a = fmaf(qr[e], x[e], a);
#pragma unroll
      for (int mm = 8; mm > 0; mm >>= 1) a += __shfl_xor_sync(kFull, a, mm);
      if (hl == 0 && i < nrep) atomicMax(&s_score[i / r], enc_max(a));
    }
  }
  if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_kk = k_blocks; s_n = 0; s_nb = 0; s_found = true; }
  __syncthreads();
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t pre = (uint32_t)s_prefix, msk = (uint32_t)s_mask;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      const uint32_t u = s_score[i];
      if ((u & msk) == pre) hist_add(hist, (u >> shift) & 255);
    }
    pick_bin(hist, shift, true, s_prefix, s_mask, s_kk, s_found, &s_pop);
    if (!s_found) break;
  }
  const bool all = !s_found;
  const uint32_t Tk = (uint32_t)s_prefix;
  const long long need = s_kk;
  const bool ties = !all && (long long)s_pop > need;
  if (threadIdx.x == 0) { s_idprefix = 0; s_idmask = 0; s_kk = need; }
  __syncthreads();
  if (ties) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const uint32_t pre = (uint32_t)s_idprefix, msk = (uint32_t)s_idmask;
      for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (s_score[i] == Tk && ((uint32_t)i & msk) == pre)
          hist_add(hist, ((uint32_t)i >> shift) & 255);
      pick_bin(hist, shift, false, s_idprefix, s_idmask, s_kk, s_found, &s_pop);
    }
  }
  const uint32_t Tb = ties ? (uint32_t)s_idprefix : 0xffffffffu;
  // prefix tokens (global ids) held by this shard: [off, off + n)
  const int64_t P = s.P;
  for (int i = warp; i < nb; i += kSelThreads / 32) {
    const uint32_t u = s_score[i];
    if (!(all || u > Tk || (u == Tk && (uint32_t)i <= Tb))) continue;
    if (lane == 0 && blocks) {
      const int ob = atomicAdd(&s_nb, 1);
      blocks[(size_t)row * k_blocks + ob] = i;
      if (bscores) bscores[(size_t)row * k_blocks + ob] = dec_max(s_score[i]);
    }
    const int64_t lo = (int64_t)i * block_size;
    const int64_t hi = min(min(lo + block_size, (int64_t)bi.n_tokens), P);
    const int64_t a = max(lo, s.off), e = min(hi, s.off + (int64_t)s.n);
    if (e <= a) continue;
    int o = 0;
    if (lane == 0) o = atomicAdd(&s_n, (int)(e - a));
    o = __shfl_sync(kFull, o, 0);
    for (int64_t t = a + lane; t < e; t += 32)
      if (o + (t - a) < cap) ids[(size_t)row * cap + o + (t - a)] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) count[row] = (int32_t)min((int64_t)s_n, cap);
}

// ---------------------------------------------------------------------------
// Partial attention over explicit base ids (minus the window ids) merged with
// the window partial; one CTA per (sequence, q head), warps take interleaved
// row batches with their own online softmax, merged in fixed warp order.
constexpr int kSaU = 8;        // rows in flight per half-warp
constexpr int kSaWarps = 16;   // warps per (sequence, q head)

template <typename T, int D>
__global__ void __launch_bounds__(kSaWarps * 32)
    sparse_attn_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q,
                       const int64_t* __restrict__ ids, int64_t cap,
                       const int32_t* __restrict__ count, float* __restrict__ out,
                       int32_t* __restrict__ nsel_out, int* __restrict__ status) {
  constexpr int DPL = D / 16;
  // K and V rows of a batch in flight: 8 per half-warp, 4 when a lane's share of a
  // row is 32 B (fp32 d = 128: 8 x 2 x 32 B would need 128 registers and spill)
  constexpr int U = (int)sizeof(T) * DPL <= 16 ? kSaU : kSaU / 2;
  __shared__ float s_m[kSaWarps], s_l[kSaWarps];
  __shared__ float s_acc[kSaWarps][D];
  __shared__ int s_sel[kSaWarps];
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hl = lane & 15, half = lane >> 4;
  const int row = blockIdx.x;
  const int b = row / bt.Hq, qh = row - b * bt.Hq, h = qh / bt.G;
  const KSeq& s = bt.s[b];
  const int64_t P = s.P, off = s.off;
  // window rows: base window ids this shard holds + the session rows
  int64_t a0 = 0, a1, b0, b1;
  if (P <= (int64_t)bt.wi + bt.wl) { a1 = P; b0 = 0; b1 = 0; }
  else { a1 = bt.wi; b0 = P - bt.wl; b1 = P; }
  a0 = max(a0, off) - off; a1 = min(a1, off + s.n) - off; if (a1 < a0) a1 = a0;
  b0 = max(b0, off) - off; b1 = min(b1, off + s.n) - off; if (b1 < b0) b1 = b0;
  const int na = (int)(a1 - a0), nbw = (int)(b1 - b0);
  const int nid = count[row];
  const int64_t* rid = ids + (size_t)row * cap;
  const int R = nid + na + nbw + seq_w(s);  // id rows first, then the window rows
  const T* kbase = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs;
  const T* vbase = reinterpret_cast<const T*>(s.v) + (size_t)h * s.hs;
  const T* wkb = reinterpret_cast<const T*>(s.wk) + (size_t)h * s.whs;
  const T* wvb = reinterpret_cast<const T*>(s.wv) + (size_t)h * s.whs;
  constexpr int STEP = 2 * U;  // rows per warp per iteration
  // the ids of a warp's next rows are loaded one iteration ahead
  auto load_ids = [&](int r0, int64_t (&g)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + 2 * u + half;
      g[u] = r < nid ? __ldg(rid + r) : -1;
    }
  };
  // row r (id already loaded as gid for r < nid) -> K/V rows or null
  auto rows_of = [&](int r, int64_t gid, const T*& kr, const T*& vr) {
    kr = vr = nullptr;
    if (r >= R) return;
    if (r < nid) {
      if (gid < off || gid >= off + s.n || in_window(gid, P, bt.wi, bt.wl)) return;
      kr = kbase + (size_t)(gid - off) * D;
      vr = vbase + (size_t)(gid - off) * D;
    } else if (r < nid + na) {
      kr = kbase + (size_t)(a0 + r - nid) * D;
      vr = vbase + (size_t)(a0 + r - nid) * D;
    } else if (r < nid + na + nbw) {
      kr = kbase + (size_t)(b0 + r - nid - na) * D;
      vr = vbase + (size_t)(b0 + r - nid - na) * D;
    } else {
      kr = wkb + (size_t)(r - nid - na - nbw) * D;
      vr = wvb + (size_t)(r - nid - na - nbw) * D;
    }
  };
  float qr[DPL];
  load_q<DPL>(q + (size_t)row * D + hl * DPL, qr);
  float m = -INFINITY, l = 0.f, acc[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) acc[e] = 0.f;
  int nsel = 0;
  int64_t gcur[U], gnxt[U];
  int r0 = warp * STEP;
  load_ids(r0, gcur);
  for (; r0 < R; r0 += kSaWarps * STEP) {
    load_ids(r0 + kSaWarps * STEP, gnxt);
    const T* kr[U];
    const T* vr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + 2 * u + half;
      rows_of(r, gcur[u], kr[u], vr[u]);
      if (hl == 0 && r < nid && kr[u]) ++nsel;  // lanes 0 and 16 count their rows
    }
    float z[U];
    RawFrag<T, DPL> fk[U], fv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kr[u]) { fk[u].load(kr[u] + hl * DPL); fv[u].load(vr[u] + hl * DPL); }
      else { fk[u].zero(); fv[u].zero(); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) gcur[u] = gnxt[u];
    float bm = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float x[DPL];
      fk[u].to_float(x);
      float a = 0.f;
#pragma unroll
      for (int e = 0; e < DPL; ++e) a = fmaf(qr[e], x[e], a);
#pragma unroll
      for (int mm = 8; mm > 0; mm >>= 1) a += __shfl_xor_sync(kFull, a, mm);
      z[u] = kr[u] ? a * bt.inv_sqrt_d : -INFINITY;
      bm = fmaxf(bm, z[u]);
    }
    bm = fmaxf(bm, __shfl_xor_sync(kFull, bm, 16));
    if (bm == -INFINITY) continue;  // nothing valid in this batch (warp-uniform)
    const float mn = fmaxf(m, bm);
    const float sc = (m == -INFINITY) ? 0.f : expf(m - mn);
    float lb = 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[e] *= sc;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float w = kr[u] ? expf(z[u] - mn) : 0.f;
      lb += w;
      float x[DPL];
      fv[u].to_float(x);
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[e] = fmaf(w, x[e], acc[e]);
    }
    lb += __shfl_xor_sync(kFull, lb, 16);
    l = l * sc + lb;
    m = mn;
  }
#pragma unroll
  for (int e = 0; e < DPL; ++e) acc[e] += __shfl_xor_sync(kFull, acc[e], 16);
  nsel += __shfl_xor_sync(kFull, nsel, 16);
  if (lane == 0) { s_m[warp] = m; s_l[warp] = l; s_sel[warp] = nsel; }
  if (half == 0) {
#pragma unroll
    for (int e = 0; e < DPL; ++e) s_acc[warp][hl * DPL + e] = acc[e];
  }
  __syncthreads();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < kSaWarps; ++w) M = fmaxf(M, s_m[w]);
  float Lt = 0.f;
#pragma unroll
  for (int w = 0; w < kSaWarps; ++w) Lt += s_m[w] == -INFINITY ? 0.f : s_l[w] * expf(s_m[w] - M);
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    float a = 0.f;
#pragma unroll
    for (int w = 0; w < kSaWarps; ++w) a += s_m[w] == -INFINITY ? 0.f : s_acc[w][e] * expf(s_m[w] - M);
    const float o = a / Lt;
    if (!isfinite(o) && status) atomicExch(status, (int)ALAYA_ERR_NONFINITE);
    out[(size_t)row * D + e] = o;
  }
  if (threadIdx.x == 0 && nsel_out) {
    int t = 0;
#pragma unroll
    for (int w = 0; w < kSaWarps; ++w) t += s_sel[w];
    nsel_out[row] = t;
  }
}

template <typename T>
int sparse_attn_d(const Batch& bt, const float* q, const int64_t* ids, int64_t cap,
                  const int32_t* count, float* out, int32_t* nsel, int* status, cudaStream_t st) {
  const unsigned rows = (unsigned)(bt.B * bt.Hq);
  switch (bt.D) {
    case 16: return launch_pdl("sparse_attn_kernel", sparse_attn_kernel<T, 16>, rows, kSaWarps * 32, 0, st, bt, q, ids, cap, count, out, nsel, status);
    case 32: return launch_pdl("sparse_attn_kernel", sparse_attn_kernel<T, 32>, rows, kSaWarps * 32, 0, st, bt, q, ids, cap, count, out, nsel, status);
    case 64: return launch_pdl("sparse_attn_kernel", sparse_attn_kernel<T, 64>, rows, kSaWarps * 32, 0, st, bt, q, ids, cap, count, out, nsel, status);
    case 128: return launch_pdl("sparse_attn_kernel", sparse_attn_kernel<T, 128>, rows, kSaWarps * 32, 0, st, bt, q, ids, cap, count, out, nsel, status);
    default: return launch_pdl("sparse_attn_kernel", sparse_attn_kernel<T, 256>, rows, kSaWarps * 32, 0, st, bt, q, ids, cap, count, out, nsel, status);
  }
}

template <typename T, int D>
int block_topk_t(const Batch& bt, const float* q, const BixSet& bix, int max_nb,
                 int block_size, int k_blocks, int64_t* ids, int64_t cap, int32_t* count,
                 int32_t* blocks, float* bscores, cudaStream_t st) {
  const size_t smem = (size_t)max_nb * 4;
  if (smem > 200 * 1024) return fail(ALAYA_ERR_UNSUPPORTED, "block index of %d blocks > 51200", max_nb);
  cudaFuncSetAttribute(block_topk_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl("block_topk_kernel", block_topk_kernel<T, D>, (unsigned)(bt.B * bt.Hq), kSelThreads,
                    smem, st, bt, q, bix, block_size, k_blocks, ids, cap, count, blocks, bscores);
}

template <typename T>
int block_topk_d(const Batch& bt, const float* q, const BixSet& bix, int max_nb,
                 int block_size, int k_blocks, int64_t* ids, int64_t cap, int32_t* count,
                 int32_t* blocks, float* bscores, cudaStream_t st) {
  switch (bt.D) {
    case 16: return block_topk_t<T, 16>(bt, q, bix, max_nb, block_size, k_blocks, ids, cap, count, blocks, bscores, st);
    case 32: return block_topk_t<T, 32>(bt, q, bix, max_nb, block_size, k_blocks, ids, cap, count, blocks, bscores, st);
    case 64: return block_topk_t<T, 64>(bt, q, bix, max_nb, block_size, k_blocks, ids, cap, count, blocks, bscores, st);
    case 128: return block_topk_t<T, 128>(bt, q, bix, max_nb, block_size, k_blocks, ids, cap, count, blocks, bscores, st);
    default: return block_topk_t<T, 256>(bt, q, bix, max_nb, block_size, k_blocks, ids, cap, count, blocks, bscores, st);
  }
}

}  // namespace

int launch_topk_bound(const Batch& bt, int dtype, const float* q, float* scratch, size_t scratch_floats, int k,
                      float* thr, cudaStream_t st) {
  int max_n = 0;
  for (int b = 0; b < bt.B; ++b) max_n = std::max(max_n, bt.s[b].n);
  // 16 samples per wanted token, 4096..8192 per row, within the scratch (fewer samples
  // loosen the bound: 1024 measured slower overall at k=100)
  int S_max = std::min(std::max(16 * k, 4096), 8192);
  S_max = std::min<int64_t>(S_max, std::max(max_n, 1));
  S_max = (int)std::min<size_t>((size_t)S_max, scratch_floats / (size_t)(bt.B * bt.Hq));
  if (S_max < 1) S_max = 1;
  const dim3 grid(bt.B * bt.Hkv, (S_max + 255) / 256);
  int rc;
  if (bt.G > kMaxG) return fail(ALAYA_ERR_UNSUPPORTED, "group size %d > 8", bt.G);
#define ALAYA_SAMPLE(TT, DD) \
  rc = launch_pdl("topk_sample_kernel", topk_sample_kernel<TT, DD>, grid, 256, 0, st, bt, q, scratch, S_max)
  const bool bf = dtype == ALAYA_BF16;
  switch (bt.D) {
    case 16: if (bf) ALAYA_SAMPLE(__nv_bfloat16, 16); else ALAYA_SAMPLE(float, 16); break;
    case 32: if (bf) ALAYA_SAMPLE(__nv_bfloat16, 32); else ALAYA_SAMPLE(float, 32); break;
    case 64: if (bf) ALAYA_SAMPLE(__nv_bfloat16, 64); else ALAYA_SAMPLE(float, 64); break;
    case 128: if (bf) ALAYA_SAMPLE(__nv_bfloat16, 128); else ALAYA_SAMPLE(float, 128); break;
    default: if (bf) ALAYA_SAMPLE(__nv_bfloat16, 256); else ALAYA_SAMPLE(float, 256); break;
  }
#undef ALAYA_SAMPLE
  if (rc) return rc;
  const size_t smem = (size_t)S_max * 4;
  cudaFuncSetAttribute(topk_thr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl("topk_thr_kernel", topk_thr_kernel, (unsigned)(bt.B * bt.Hq), kThrThreads, smem, st, bt, scratch,
                    S_max, k, thr);
}

int launch_topk_select(const Batch& bt, const Ws& ws, int k, int64_t* ids, float* scores, int64_t cap,
                       int32_t* count, cudaStream_t st) {
  if (k < bt.chunk && bt.total_chunks > 0) {
    const size_t smem = (size_t)bt.chunk * 8;
    cudaFuncSetAttribute(chunk_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int rc = launch_pdl("chunk_topk_kernel", chunk_topk_kernel, (unsigned)(bt.total_chunks * bt.G),
                              kCkThreads, smem, st, bt, ws, k);
    if (rc) return rc;
  }
  int max_nch = 0;
  for (int b = 0; b < bt.B; ++b) max_nch = std::max(max_nch, bt.s[b].nch);
  // offsets, then as many staged keys as the remaining dynamic smem holds
  const size_t off_bytes = (size_t)(max_nch * 4 + 1) * 4;
  const size_t smem_max = 220 * 1024;
  if (off_bytes + 4096 > smem_max) return fail(ALAYA_ERR_UNSUPPORTED, "top-k over %d chunks per head", max_nch);
  const int stage_cap = (int)((smem_max - off_bytes) / 4);
  const size_t smem = off_bytes + (size_t)stage_cap * 4;
  cudaFuncSetAttribute(topk_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl("topk_select_kernel", topk_select_kernel, (unsigned)(bt.B * bt.Hq), kSelectThreads, smem,
                    st, bt, ws, k, ids, scores, cap, count, stage_cap);
}

int launch_sparse_attention(const Batch& bt, int dtype, const float* q, const int64_t* ids, int64_t cap,
                            const int32_t* count, float* out, int32_t* nsel, int* status,
                            cudaStream_t st) {
  if (dtype == ALAYA_BF16) return sparse_attn_d<__nv_bfloat16>(bt, q, ids, cap, count, out, nsel, status, st);
  return sparse_attn_d<float>(bt, q, ids, cap, count, out, nsel, status, st);
}

int launch_block_reps(const void* k, int dtype, int heads, int64_t head_stride, int n, int dim,
                      int block_size, int r, void* reps, int64_t reps_head_stride, cudaStream_t st) {
  const int nb = (n + block_size - 1) / block_size;
  const size_t smem = (size_t)block_size * 8;
  const unsigned grid = (unsigned)(heads * nb);
  if (dtype == ALAYA_BF16) {
    cudaFuncSetAttribute(block_reps_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    block_reps_kernel<__nv_bfloat16><<<grid, 256, smem, st>>>(
        static_cast<const __nv_bfloat16*>(k), head_stride, n, dim, block_size, r,
        static_cast<__nv_bfloat16*>(reps), reps_head_stride, nb);
  } else {
    cudaFuncSetAttribute(block_reps_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    block_reps_kernel<float><<<grid, 256, smem, st>>>(static_cast<const float*>(k), head_stride, n, dim,
                                                      block_size, r, static_cast<float*>(reps),
                                                      reps_head_stride, nb);
  }
  return cuda_check("block_reps_kernel");
}

int launch_block_topk(const Batch& bt, int dtype, const float* q, const BixSet& d_bix,
                      int max_nb, int block_size, int k_blocks, int64_t* ids, int64_t cap,
                      int32_t* count, int32_t* blocks, float* bscores, cudaStream_t st) {
  if (dtype == ALAYA_BF16)
    return block_topk_d<__nv_bfloat16>(bt, q, d_bix, max_nb, block_size, k_blocks, ids, cap, count, blocks, bscores, st);
  return block_topk_d<float>(bt, q, d_bix, max_nb, block_size, k_blocks, ids, cap, count, blocks, bscores, st);
}

}  // namespace alaya
