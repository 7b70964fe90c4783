// The three stages of one decode step (CUDA-core variants):
//   scan_kernel     K stream -> q.k for the whole GQA group, chunk max, global
//                   running max (atomic), ordered candidate superset.
//   attend_kernel   exact filter at max - beta, window exclusion, V gather of
//                   the group's union of selected rows, partial (l, acc).
//   combine_kernel  sum chunk partials, window partial (base window ids +
//                   session rows), merge, finalize or export (m, l, acc).
#pragma once

#include "alaya_common.cuh"

namespace alaya {

// Keys per half-warp per iteration of the scan; a tile is 16 half-warps.
constexpr int kScanKPH = 8;
constexpr int kScanTile = kHalfWarps * kScanKPH;  // 128 keys

// One transposed-butterfly level: S partial sums per lane -> S/2, exchanging
// the half this lane does not keep with its partner (lane ^ mask).
template <int S, int P>
__device__ __forceinline__ void tr_level(float (&a)[P], int mask, bool upper) {
#pragma unroll
  for (int i = 0; i < S / 2; ++i) {
    float send = upper ? a[i] : a[i + S / 2];
    float keep = upper ? a[i + S / 2] : a[i];
    a[i] = keep + __shfl_xor_sync(kFull, send, mask);
  }
}

// ---------------------------------------------------------------------------
// Stage 1: scan (reference: core.py:64-67 inner_products, dipr.py:63-64 max)
// ---------------------------------------------------------------------------
template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads, (G <= 5 ? 2 : 1))
    scan_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q, Ws ws) {
  extern __shared__ float smem[];
  constexpr int DPL = D / 16;  // dims per lane (half-warp per key)
  constexpr int P = kScanKPH * G;
  const int chunk = bt.chunk;
  float* sc = smem;                        // [G][chunk] scores
  float* red = smem + G * chunk;           // [kWarps][G]
  float* thr = red + kWarps * G;           // [G]
  int* wc = reinterpret_cast<int*>(thr + G);  // [kWarps][G]

  int b, h, ci;
  decode_chunk(bt, blockIdx.x, b, h, ci);
  const KSeq& s = bt.s[b];
  const int t0 = ci * chunk;
  const int valid = min(chunk, s.n - t0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hw = tid >> 4, hl = tid & 15;

  float qr[G][DPL];
  const float* qb = q + ((size_t)b * bt.Hq + (size_t)h * G) * D + hl * DPL;
#pragma unroll
  for (int j = 0; j < G; ++j) load_q<DPL>(qb + (size_t)j * D, qr[j]);

  const T* kb = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs + (size_t)t0 * D + hl * DPL;
  float mymax[G];
#pragma unroll
  for (int j = 0; j < G; ++j) mymax[j] = -INFINITY;

  const int ntiles = (valid + kScanTile - 1) / kScanTile;
  RawFrag<T, DPL> fa[kScanKPH], fb[kScanKPH];

  auto load_tile = [&](int tile, RawFrag<T, DPL>(&f)[kScanKPH]) {
#pragma unroll
    for (int k = 0; k < kScanKPH; ++k) {
      int row = tile * kScanTile + hw * kScanKPH + k;
      if (row < valid) f[k].load(kb + (size_t)row * D); else f[k].zero();
    }
  };
  auto compute_tile = [&](int tile, const RawFrag<T, DPL>(&f)[kScanKPH]) {
    float a[P];
#pragma unroll
    for (int k = 0; k < kScanKPH; ++k) {
      float x[DPL];
      f[k].to_float(x);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc = fmaf(qr[j][e], x[e], acc);
        a[k * G + j] = acc;
      }
    }
    // 8G -> 4G -> 2G -> G partials, then a plain xor over the last lane bit.
    tr_level<8 * G>(a, 8, (hl & 8) != 0);
    tr_level<4 * G>(a, 4, (hl & 4) != 0);
    tr_level<2 * G>(a, 2, (hl & 2) != 0);
#pragma unroll
    for (int j = 0; j < G; ++j) a[j] += __shfl_xor_sync(kFull, a[j], 1);
    const int kk = (hl >> 1) & 7;
    const int row = tile * kScanTile + hw * kScanKPH + kk;
    if ((hl & 1) == 0 && row < valid) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        sc[j * chunk + row] = a[j];
        mymax[j] = fmaxf(mymax[j], a[j]);
      }
    }
  };

  if (ntiles > 0) load_tile(0, fa);
  for (int tile = 0; tile < ntiles; tile += 2) {
    if (tile + 1 < ntiles) load_tile(tile + 1, fb);
    compute_tile(tile, fa);
    if (tile + 1 < ntiles) {
      if (tile + 2 < ntiles) load_tile(tile + 2, fa);
      compute_tile(tile + 1, fb);
    }
  }

  // chunk max per head, then the global running max (order-preserving atomic)
#pragma unroll
  for (int j = 0; j < G; ++j) {
    float m = warp_max(mymax[j]);
    if (lane == 0) red[warp * G + j] = m;
  }
  __syncthreads();
  if (tid < G) {
    float cm = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) cm = fmaxf(cm, red[w * G + tid]);
    uint32_t old = atomicMax(&ws.gmax[b * bt.Hq + h * G + tid], enc_max(cm));
    // any bound <= the true global max gives a superset of the exact set
    thr[tid] = fmaxf(cm, dec_max(old)) - bt.beta;
  }
  __syncthreads();

  // ordered compaction of s >= bound - beta; warp w owns a contiguous segment
  const int seg = chunk / kWarps;
  const int sbeg = warp * seg;
  int cntj[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float th = thr[j];
    int cnt = 0;
    for (int r = 0; r < seg; r += 32) {
      int pos = sbeg + r + lane;
      bool p = pos < valid && sc[j * chunk + pos] >= th;
      cnt += __popc(__ballot_sync(kFull, p));
    }
    cntj[j] = cnt;
    if (lane == 0) wc[warp * G + j] = cnt;
  }
  __syncthreads();
  const size_t cbase = (size_t)blockIdx.x * G;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float th = thr[j];
    int off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      int cw = wc[w * G + j];
      off += (w < warp) ? cw : 0;
      tot += cw;
    }
    int* oi = ws.cidx + (cbase + j) * chunk;
    float* os = ws.cscore + (cbase + j) * chunk;
    if (cntj[j] > 0) {
      for (int r = 0; r < seg; r += 32) {
        int pos = sbeg + r + lane;
        float v = pos < valid ? sc[j * chunk + pos] : -INFINITY;
        bool p = pos < valid && v >= th;
        unsigned bal = __ballot_sync(kFull, p);
        if (p) {
          int o = off + __popc(bal & lanemask_lt());
          oi[o] = pos;
          os[o] = v;
        }
        off += __popc(bal);
      }
    }
    if (tid == 0) ws.cnt[cbase + j] = tot;
  }
}

// ---------------------------------------------------------------------------
// Stage 2: exact filter + V gather (reference: dipr.py:64, store.py:271-278,
// attention.py:98-110). Softmax reference point is the (global) max, so the
// chunk partials need no rescaling when merged.
// ---------------------------------------------------------------------------
template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads)
    attend_kernel(const __grid_constant__ Batch bt, const float* __restrict__ smax_ext, Ws ws,
                  int want_values) {
  extern __shared__ float smem[];
  constexpr int DPL = D / 16;
  const int chunk = bt.chunk;
  const int nwords = chunk / 32;
  float* wt = smem;                                   // [G][chunk] weights (0 = not selected)
  const int wt_floats = max(G * chunk, kWarps * G * D);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem + wt_floats);  // [chunk/32]
  int* ulist = reinterpret_cast<int*>(bitmap + nwords);               // [chunk]
  int* wsc = ulist + chunk;                                           // [kWarps]
  int* wrc = wsc + kWarps;                                            // [kWarps]
  float* fred = reinterpret_cast<float*>(wrc + kWarps);               // [kWarps]
  int* nu_s = reinterpret_cast<int*>(fred + kWarps);                  // [1]

  int b, h, ci;
  decode_chunk(bt, blockIdx.x, b, h, ci);
  const KSeq& s = bt.s[b];
  const int t0 = ci * chunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float k2 = bt.inv_sqrt_d * kLog2e;
  const size_t cbase = (size_t)blockIdx.x * G;

  if (want_values) {
    for (int i = tid; i < G * chunk; i += kThreads) wt[i] = 0.f;
    for (int i = tid; i < nwords; i += kThreads) bitmap[i] = 0u;
  }
  __syncthreads();

#pragma unroll 1
  for (int j = 0; j < G; ++j) {
    const int qh = h * G + j;
    const float smax = smax_ext ? smax_ext[b * bt.Hq + qh] : dec_max(ws.gmax[b * bt.Hq + qh]);
    const float th = smax - bt.beta;
    const int nc = ws.cnt[cbase + j];
    int* ci_ = ws.cidx + (cbase + j) * chunk;
    const float* cs_ = ws.cscore + (cbase + j) * chunk;
    int sel_tot = 0, ret_tot = 0;
    float lsum = 0.f;
    for (int r0 = 0; r0 < nc; r0 += kThreads) {
      const int i = r0 + tid;
      const bool valid = i < nc;
      const int t = valid ? ci_[i] : 0;
      const float sv = valid ? cs_[i] : -INFINITY;
      const bool pass = valid && sv >= th;
      const bool sel = pass && !in_window(s.off + t0 + t, s.P, bt.wi, bt.wl);
      const unsigned bs = __ballot_sync(kFull, sel), br = __ballot_sync(kFull, pass);
      if (lane == 0) { wsc[warp] = __popc(bs); wrc[warp] = __popc(br); }
      if (sel && want_values) {
        const float w = exp2f((sv - smax) * k2);
        wt[j * chunk + t] = w;
        atomicOr(&bitmap[t >> 5], 1u << (t & 31));
        lsum += w;
      }
      __syncthreads();
      int off = sel_tot, add_s = 0, add_r = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        off += (w < warp) ? wsc[w] : 0;
        add_s += wsc[w];
        add_r += wrc[w];
      }
      if (sel) ci_[off + __popc(bs & lanemask_lt())] = t;  // in place, ascending
      sel_tot += add_s;
      ret_tot += add_r;
      __syncthreads();
    }
    if (tid == 0) { ws.selcnt[cbase + j] = sel_tot; ws.retcnt[cbase + j] = ret_tot; }
    if (want_values) {
      const float l = block_sum(lsum, fred);
      if (tid == 0) ws.part_l[cbase + j] = l;
    }
  }
  if (!want_values) return;
  __syncthreads();

  // union of the group's selections, ascending local rows
  if (warp == 0) {
    int run = 0;
    for (int w0 = 0; w0 < nwords; w0 += 32) {
      const int wi = w0 + lane;
      const uint32_t bits = wi < nwords ? bitmap[wi] : 0u;
      int c = __popc(bits), incl = c;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        int o = __shfl_up_sync(kFull, incl, m);
        if (lane >= m) incl += o;
      }
      int pos = run + incl - c;
      uint32_t x = bits;
      while (x) {
        int bit = __ffs(x) - 1;
        ulist[pos++] = wi * 32 + bit;
        x &= x - 1;
      }
      run += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) *nu_s = run;
  }
  __syncthreads();
  const int nu = *nu_s;

  // V gather: a half-warp per row, 4 rows in flight per half-warp
  const int hw = tid >> 4, hl = tid & 15;
  const T* vb = reinterpret_cast<const T*>(s.v) + (size_t)h * s.hs + (size_t)t0 * D + hl * DPL;
  float acc[G][DPL];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[j][e] = 0.f;
  constexpr int U = 4;
  for (int u0 = hw; u0 < nu; u0 += kHalfWarps * U) {
    RawFrag<T, DPL> f[U];
    int tt[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int u = u0 + k * kHalfWarps;
      tt[k] = u < nu ? ulist[u] : -1;
      if (tt[k] >= 0) f[k].load(vb + (size_t)tt[k] * D); else f[k].zero();
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (tt[k] < 0) continue;
      float x[DPL];
      f[k].to_float(x);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const float w = wt[j * chunk + tt[k]];
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[j][e] = fmaf(w, x[e], acc[j][e]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[j][e] += __shfl_xor_sync(kFull, acc[j][e], 16);
  __syncthreads();  // wt reads finished: reuse it as [kWarps][G][D]
  float* red = wt;
  if (lane < 16) {
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int e = 0; e < DPL; ++e) red[(warp * G + j) * D + hl * DPL + e] = acc[j][e];
  }
  __syncthreads();
  for (int idx = tid; idx < G * D; idx += kThreads) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += red[w * G * D + idx];
    ws.part_acc[cbase * D + idx] = t;
  }
}

// ---------------------------------------------------------------------------
// Stage 3: per (sequence, kv head): chunk partials + window partial, merged
// (attention.py:128-143: selected first, then window) and finalized
// (attention.py:145-152) or exported as (m, l, acc) for a cross-shard merge.
// ---------------------------------------------------------------------------
constexpr int kWinBatch = 64;

template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads)
    combine_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q,
                   const float* __restrict__ smax_ext, Ws ws, float* __restrict__ out,
                   float* __restrict__ part_out, float* __restrict__ smax_out) {
  constexpr int DPL = D / 16;
  __shared__ float accb[G * D];
  __shared__ float accw[G * D];
  __shared__ float zb[G][kWinBatch];
  __shared__ float mw[G], lw[G], scl[G], lb[G], zmax[G];

  const int b = blockIdx.x / bt.Hkv, h = blockIdx.x - b * bt.Hkv;
  const KSeq& s = bt.s[b];
  const int tid = threadIdx.x, hw = tid >> 4, hl = tid & 15;
  const int c0 = s.chunk_base + h * s.nch;

  // base (selected-set) partial: sum over chunks in order, reference point = max
  for (int idx = tid; idx < G * D; idx += kThreads) {
    const int j = idx / D, e = idx - j * D;
    float t = 0.f;
    for (int c = 0; c < s.nch; ++c) t += ws.part_acc[((size_t)(c0 + c) * G + j) * D + e];
    accb[idx] = t;
    accw[idx] = 0.f;
  }
  if (tid < G) {
    const int qh = h * G + tid;
    float l = 0.f;
    int sel = 0, ret = 0;
    for (int c = 0; c < s.nch; ++c) {
      l += ws.part_l[(size_t)(c0 + c) * G + tid];
      sel += ws.selcnt[(size_t)(c0 + c) * G + tid];
      ret += ws.retcnt[(size_t)(c0 + c) * G + tid];
    }
    const float smax = smax_ext ? smax_ext[b * bt.Hq + qh] : dec_max(ws.gmax[b * bt.Hq + qh]);
    if (smax_out) smax_out[b * bt.Hq + qh] = smax;
    lb[tid] = (sel > 0) ? l : 0.f;
    zmax[tid] = smax * bt.inv_sqrt_d;
    mw[tid] = -INFINITY;
    lw[tid] = 0.f;
  }

  // window rows owned here: base window ids inside [off, off+n), then session rows
  const int64_t P = s.P, off = s.off;
  int64_t a0, a1, b0, b1;  // local row ranges [a0,a1) and [b0,b1)
  if (P <= (int64_t)bt.wi + bt.wl) {
    a0 = 0; a1 = P; b0 = 0; b1 = 0;
  } else {
    a0 = 0; a1 = bt.wi; b0 = P - bt.wl; b1 = P;
  }
  a0 = max(a0, off) - off; a1 = min(a1, off + s.n) - off; if (a1 < a0) a1 = a0;
  b0 = max(b0, off) - off; b1 = min(b1, off + s.n) - off; if (b1 < b0) b1 = b0;
  const int na = (int)(a1 - a0), nbw = (int)(b1 - b0);
  const int R = na + nbw + s.w;

  float qr[G][DPL];
  const float* qb = q + ((size_t)b * bt.Hq + (size_t)h * G) * D + hl * DPL;
#pragma unroll
  for (int j = 0; j < G; ++j) load_q<DPL>(qb + (size_t)j * D, qr[j]);

  const T* kbase = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs;
  const T* vbase = reinterpret_cast<const T*>(s.v) + (size_t)h * s.hs;
  const T* wkb = reinterpret_cast<const T*>(s.wk) + (size_t)h * s.whs;
  const T* wvb = reinterpret_cast<const T*>(s.wv) + (size_t)h * s.whs;
  auto row_ptr = [&](int r, bool val) -> const T* {
    if (r < na) return (val ? vbase : kbase) + (size_t)(a0 + r) * D;
    if (r < na + nbw) return (val ? vbase : kbase) + (size_t)(b0 + r - na) * D;
    return (val ? wvb : wkb) + (size_t)(r - na - nbw) * D;
  };
  __syncthreads();

  for (int r0 = 0; r0 < R; r0 += kWinBatch) {
    const int nr = min(kWinBatch, R - r0);
    for (int rr = hw; rr < kWinBatch; rr += kHalfWarps) {  // warp-uniform trip count
      float sj[G];
      RawFrag<T, DPL> f;
      if (rr < nr) f.load(row_ptr(r0 + rr, false) + hl * DPL); else f.zero();
      float x[DPL];
      f.to_float(x);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) a = fmaf(qr[j][e], x[e], a);
#pragma unroll
        for (int m = 8; m > 0; m >>= 1) a += __shfl_xor_sync(kFull, a, m);
        sj[j] = a;
      }
      if (hl == 0) {
#pragma unroll
        for (int j = 0; j < G; ++j) zb[j][rr] = rr < nr ? sj[j] * bt.inv_sqrt_d : -INFINITY;
      }
    }
    __syncthreads();
    if (tid < G) {
      float bm = -INFINITY;
      for (int r = 0; r < nr; ++r) bm = fmaxf(bm, zb[tid][r]);
      const float mn = fmaxf(mw[tid], bm);
      const float sc = (mw[tid] == -INFINITY) ? 0.f : expf(mw[tid] - mn);
      float l = lw[tid] * sc;
      for (int r = 0; r < nr; ++r) {
        const float w = expf(zb[tid][r] - mn);
        zb[tid][r] = w;
        l += w;
      }
      mw[tid] = mn;
      lw[tid] = l;
      scl[tid] = sc;
    }
    __syncthreads();
    for (int idx = tid; idx < G * D; idx += kThreads) {
      const int j = idx / D, e = idx - j * D;
      float a = accw[idx] * scl[j];
      for (int r = 0; r < nr; ++r) {
        const T* vp = row_ptr(r0 + r, true) + e;
        float v;
        if constexpr (std::is_same_v<T, float>) v = __ldg(vp);
        else v = __bfloat162float(*vp);
        a = fmaf(zb[j][r], v, a);
      }
      accw[idx] = a;
    }
    __syncthreads();
  }

  // merge(selected, window) then finalize / export
  for (int idx = tid; idx < G * D; idx += kThreads) {
    const int j = idx / D, e = idx - j * D;
    const bool hb = lb[j] > 0.f, hwn = R > 0;
    const float m = fmaxf(hb ? zmax[j] : -INFINITY, hwn ? mw[j] : -INFINITY);
    const float fb = hb ? expf(zmax[j] - m) : 0.f;
    const float fw = hwn ? expf(mw[j] - m) : 0.f;
    const float l = lb[j] * fb + lw[j] * fw;
    const float a = accb[idx] * fb + accw[idx] * fw;
    const size_t row = (size_t)b * bt.Hq + h * G + j;
    if (out) {
      const float o = a / l;
      if (!isfinite(o)) atomicExch(ws.status, (int)ALAYA_ERR_NONFINITE);
      out[row * D + e] = o;
    }
    if (part_out) {
      float* pr = part_out + row * (D + 2);
      const bool empty = !(hb || hwn);
      if (e == 0) { pr[0] = empty ? -INFINITY : m; pr[1] = empty ? 0.f : l; }
      pr[2 + e] = empty ? 0.f : a;
    }
  }
}

}  // namespace alaya
