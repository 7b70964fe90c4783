// Graph DIPRS on the GPU: the reference's candidate-list walk over a
// proximity graph (dipr.py:107-289, CandidateList / traverse / diprs),
// decision-for-decision, one CTA per (sequence, q head).
//
// The reference walks the list in insertion order in batches: every pending
// entry offers its neighbours (adjacency order), offered ids are
// de-duplicated keeping the first occurrence, unvisited ones are marked and
// scored, then offered to the list one by one: accepted while the list holds
// <= l0 entries, afterwards only when score >= max(best, floor) - beta. Here a
// batch is processed in sub-batches (the reference notes batching is
// decision-identical to one entry at a time), each as data-parallel phases:
//   gather neighbours (block scan of degrees) -> first occurrence per id
//   (atomicMin of positions in a per-row table) -> ordered compaction of the
//   fresh ids -> scores (half-warp per key row) -> acceptance as a prefix
//   max: best before entry i = max(best, prefix max of the scores that can
//   raise it -- those >= floor - beta, or any inside the unconditional l0
//   phase), so every decision is computed in parallel and stays exact.
// Visited flags live in shared memory (one bit per token).
#include <climits>

#include "alaya_dispatch.cuh"

namespace alaya {
namespace {

constexpr int kDThreads = 1024;
constexpr int kDWarps = kDThreads / 32;

struct GraphSet {
  alaya_graph g[ALAYA_MAX_BATCH];
};

// exclusive block scan of one int per thread; returns the block total
__device__ __forceinline__ int scan_excl(int v, int* s_w, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kDWarps ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kDWarps) s_w[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  total = s_w[kDWarps - 1];
  const int r = x - v + (warp ? s_w[warp - 1] : 0);
  __syncthreads();
  return r;
}

// exclusive block prefix max of one float per thread; returns the block max
__device__ __forceinline__ float scan_max_excl(float v, float* s_w, float& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x = fmaxf(x, y);
  }
  float ex = __shfl_up_sync(kFull, x, 1);
  if (lane == 0) ex = -INFINITY;
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    float w = lane < kDWarps ? s_w[lane] : -INFINITY;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w = fmaxf(w, y);
    }
    if (lane < kDWarps) s_w[lane] = w;
  }
  __syncthreads();
  total = s_w[kDWarps - 1];
  const float r = fmaxf(ex, warp ? s_w[warp - 1] : -INFINITY);
  __syncthreads();
  return r;
}

template <typename T, int D>
__device__ __forceinline__ float hw_dot(const T* __restrict__ row, const float (&qr)[D / 16], int hl) {
  constexpr int DPL = D / 16;
  RawFrag<T, DPL> f;
  f.load(row + hl * DPL);
  float x[DPL];
  f.to_float(x);
  float a = 0.f;
#pragma unroll
  for (int e = 0; e < DPL; ++e) a = fmaf(qr[e], x[e], a);
#pragma unroll
  for (int m = 8; m > 0; m >>= 1) a += __shfl_xor_sync(kFull, a, m);
  return a;
}

template <typename T, int D>
__global__ void __launch_bounds__(kDThreads, 1)
    diprs_kernel(const __grid_constant__ Batch bt, const __grid_constant__ GraphSet gs,
                 const float* __restrict__ q, int l0, int floor_mode, const float* __restrict__ floors,
                 int cap, int64_t* __restrict__ ids_out, int64_t out_cap, int32_t* __restrict__ count,
                 int32_t* __restrict__ explored, char* __restrict__ ws, int64_t ws_row_bytes) {
  extern __shared__ uint32_t s_vis[];  // one bit per token
  __shared__ int s_wi[kDWarps];
  __shared__ float s_wf[kDWarps];
  __shared__ int s_i[4];
  __shared__ float s_f[4];
  pdl_trigger();
  pdl_wait();
  constexpr int DPL = D / 16;
  const int row = blockIdx.x;
  const int b = row / bt.Hq, qh = row - b * bt.Hq, h = qh / bt.G;
  const KSeq& s = bt.s[b];
  const alaya_graph& g = gs.g[b];
  const int n = g.n_nodes;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, hl = lane & 15, hw = tid >> 4;
  const int64_t* off = g.offsets + (size_t)h * g.offsets_head_stride;
  const int32_t* nb = g.nbrs + (size_t)h * g.nbrs_head_stride;
  const T* kbase = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs;
  // per-row scratch: cand ids / scores [n], first positions [n], offered /
  // fresh ids / fresh scores [cap]
  char* w = ws + (size_t)row * ws_row_bytes;
  int* cid = reinterpret_cast<int*>(w);
  float* csc = reinterpret_cast<float*>(cid + n);
  int* firstpos = reinterpret_cast<int*>(csc + n);
  int* offered = firstpos + n;
  int* fr_id = offered + cap;
  float* fr_sc = reinterpret_cast<float*>(fr_id + cap);
  float qr[DPL];
  load_q<DPL>(q + (size_t)row * D + hl * DPL, qr);
  for (int i = tid; i < (n + 31) / 32; i += kDThreads) s_vis[i] = 0u;
  for (int i = tid; i < n; i += kDThreads) firstpos[i] = INT_MAX;
  // floor: the window-cache maximum (store.py:339-354) or a given value
  float floor = -INFINITY;
  if (floor_mode == 2) {
    floor = floors[row];
  } else if (floor_mode == 1) {
    const int64_t P = s.P;
    int64_t a1, b0, b1;
    if (P <= (int64_t)bt.wi + bt.wl) { a1 = P; b0 = 0; b1 = 0; }
    else { a1 = bt.wi; b0 = P - bt.wl; b1 = P; }
    const int na = (int)a1, nbw = (int)(b1 - b0), R = na + nbw + seq_w(s);
    const T* wkb = reinterpret_cast<const T*>(s.wk) + (size_t)h * s.whs;
    float m = -INFINITY;
    for (int r = hw; r < ((R + 1) & ~1); r += kDThreads / 16) {  // pairs of rows per warp
      const int rr = r < R ? r : R - 1;
      const T* kr = rr < na ? kbase + (size_t)rr * D
                  : rr < na + nbw ? kbase + (size_t)(b0 + rr - na) * D
                  : wkb + (size_t)(rr - na - nbw) * D;
      const float a = hw_dot<T, D>(kr, qr, hl);
      if (r < R) m = fmaxf(m, a);
    }
    m = warp_max(m);
    if (lane == 0) s_wf[warp] = m;
    __syncthreads();
    floor = -INFINITY;
#pragma unroll 1
    for (int i = 0; i < kDWarps; ++i) floor = fmaxf(floor, s_wf[i]);
    if (R == 0) floor = -INFINITY;
    __syncthreads();
  }
  __syncthreads();
  // seed: the entry point (CandidateList.seed)
  const int entry = g.entry[h];
  if (warp == 0) {
    const float sc = hw_dot<T, D>(kbase + (size_t)entry * D, qr, hl);
    if (lane == 0) {
      cid[0] = entry;
      csc[0] = sc;
      s_f[0] = sc;  // best
      s_vis[entry >> 5] |= 1u << (entry & 31);
    }
  }
  __syncthreads();
  float best = s_f[0];
  int cnt = 1, cursor = 0, n_scored = 1;
  bool err = false;
  const float beta = bt.beta;
  while (cursor < cnt) {
    const int batch_end = cnt;
    while (cursor < batch_end) {
      // ---- sub-batch: entries [cursor, cursor + m) with sum of degrees <= cap
      const int avail = min(kDThreads, batch_end - cursor);
      int deg = 0;
      int64_t u0 = 0;
      if (tid < avail) {
        const int u = cid[cursor + tid];
        u0 = off[u];
        deg = (int)(off[u + 1] - u0);
      }
      int tot;
      const int pos = scan_excl(deg, s_wi, tot);
      const int m = __syncthreads_count(tid < avail && pos + deg <= cap);
      if (m == 0) {  // one adjacency list longer than the whole scratch (uniform: m is a block count)
        err = true;
        break;
      }
      if (tid < m)
        for (int j = 0; j < deg; ++j) offered[pos + j] = nb[u0 + j];
      if (tid == m - 1) s_i[1] = pos + deg;
      __syncthreads();
      const int nO = s_i[1];
      // first occurrence of every unvisited offered id
      for (int i = tid; i < nO; i += kDThreads) {
        const int v = offered[i];
        if (!((s_vis[v >> 5] >> (v & 31)) & 1u)) atomicMin(&firstpos[v], i);
      }
      __syncthreads();
      // ordered compaction of the fresh ids
      int nf = 0;
      for (int base = 0; base < nO; base += kDThreads) {
        const int i = base + tid;
        bool f = false;
        int v = 0;
        if (i < nO) {
          v = offered[i];
          f = !((s_vis[v >> 5] >> (v & 31)) & 1u) && firstpos[v] == i;
        }
        int t;
        const int p = scan_excl(f ? 1 : 0, s_wi, t);
        if (f) fr_id[nf + p] = v;
        nf += t;
      }
      __syncthreads();
      // mark visited, reset the first-position table, score (half-warp per key)
      for (int k = tid; k < nf; k += kDThreads) {
        const int v = fr_id[k];
        atomicOr(&s_vis[v >> 5], 1u << (v & 31));
        firstpos[v] = INT_MAX;
      }
      for (int k0 = 2 * warp; k0 < nf; k0 += 2 * kDWarps) {  // warp-uniform trip count
        const int k = k0 + (hw & 1);
        const int v = fr_id[k < nf ? k : nf - 1];
        const float a = hw_dot<T, D>(kbase + (size_t)v * D, qr, hl);
        if (hl == 0 && k < nf) fr_sc[k] = a;
      }
      n_scored += nf;
      __syncthreads();
      // acceptance in order (CandidateList.try_append)
      const int P = max(0, l0 + 1 - cnt);  // unconditional slots left
      for (int base = 0; base < nf; base += kDThreads) {
        const int i = base + tid;
        const float sc = i < nf ? fr_sc[i] : -INFINITY;
        const bool uncond = i < nf && i < P;
        const float raise = (i < nf && (uncond || sc >= floor - beta)) ? sc : -INFINITY;
        float tmax;
        const float before = fmaxf(best, scan_max_excl(raise, s_wf, tmax));
        const bool acc = i < nf && (uncond || sc >= fmaxf(before, floor) - beta);
        int t;
        const int p = scan_excl(acc ? 1 : 0, s_wi, t);
        if (acc) {
          cid[cnt + p] = fr_id[i];
          csc[cnt + p] = sc;
        }
        cnt += t;
        best = fmaxf(best, tmax);
      }
      cursor += m;
      __syncthreads();
    }
    if (err) break;
  }
  // final cut (CandidateList.result): entries >= max(best, floor) - beta
  const float cut = fmaxf(best, floor) - beta;
  int nout = 0;
  for (int base = 0; base < cnt; base += kDThreads) {
    const int i = base + tid;
    const bool keep = i < cnt && csc[i] >= cut;
    int t;
    const int p = scan_excl(keep ? 1 : 0, s_wi, t);
    if (keep && nout + p < out_cap) ids_out[(size_t)row * out_cap + nout + p] = s.off + cid[i];
    nout += t;
  }
  if (tid == 0) {
    count[row] = (int32_t)min((int64_t)nout, out_cap);
    if (explored) explored[row] = n_scored;
    if (err) count[row] = -1;
  }
}

template <typename T, int D>
int launch_t(const Batch& bt, const GraphSet& gs, const float* q, int l0, int floor_mode, const float* floors,
             int cap, int64_t* ids, int64_t out_cap, int32_t* count, int32_t* explored, void* ws,
             int64_t row_bytes, int max_n, cudaStream_t st) {
  const size_t smem = (size_t)((max_n + 31) / 32) * 4;
  if (smem > 200 * 1024) return fail(ALAYA_ERR_UNSUPPORTED, "graph of %d nodes > 1.6M", max_n);
  cudaFuncSetAttribute(diprs_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl("diprs_kernel", diprs_kernel<T, D>, (unsigned)(bt.B * bt.Hq), kDThreads, smem, st, bt, gs, q,
                    l0, floor_mode, floors, cap, ids, out_cap, count, explored, static_cast<char*>(ws),
                    row_bytes);
}

}  // namespace

int64_t diprs_row_bytes(int max_n, int cap) {
  return (((int64_t)max_n * 12 + (int64_t)cap * 12) + 255) & ~(int64_t)255;
}

int launch_diprs(const Batch& bt, int dtype, const alaya_graph* graphs, const float* q, int l0, int floor_mode,
                 const float* floors, int cap, int64_t* ids, int64_t out_cap, int32_t* count, int32_t* explored,
                 void* ws, size_t ws_bytes, cudaStream_t st) {
  static thread_local GraphSet gs;
  int max_n = 1;
  for (int b = 0; b < bt.B; ++b) {
    gs.g[b] = graphs[b];
    max_n = std::max(max_n, graphs[b].n_nodes);
  }
  const int64_t rb = diprs_row_bytes(max_n, cap);
  if ((int64_t)ws_bytes < rb * bt.B * bt.Hq)
    return fail(ALAYA_ERR_WORKSPACE, "workspace %zu bytes < required %lld", ws_bytes,
                (long long)(rb * bt.B * bt.Hq));
  const bool bf = dtype == ALAYA_BF16;
#define ALAYA_DIPRS_CASE(DD)                                                                              \
  case DD:                                                                                                \
    return bf ? launch_t<__nv_bfloat16, DD>(bt, gs, q, l0, floor_mode, floors, cap, ids, out_cap, count,  \
                                            explored, ws, rb, max_n, st)                                  \
              : launch_t<float, DD>(bt, gs, q, l0, floor_mode, floors, cap, ids, out_cap, count, explored, \
                                    ws, rb, max_n, st);
  switch (bt.D) {
    ALAYA_DIPRS_CASE(16)
    ALAYA_DIPRS_CASE(32)
    ALAYA_DIPRS_CASE(64)
    ALAYA_DIPRS_CASE(128)
    default:
      return bf ? launch_t<__nv_bfloat16, 256>(bt, gs, q, l0, floor_mode, floors, cap, ids, out_cap, count,
                                               explored, ws, rb, max_n, st)
                : launch_t<float, 256>(bt, gs, q, l0, floor_mode, floors, cap, ids, out_cap, count, explored,
                                       ws, rb, max_n, st);
  }
#undef ALAYA_DIPRS_CASE
}

}  // namespace alaya
