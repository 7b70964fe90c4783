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
__device__ __forceinline__ void scan_chunk(const Batch& bt, const float* __restrict__ q, const Ws& ws,
                                           const int c, float* smem) {
  constexpr int DPL = D / 16;  // dims per lane (half-warp per key)
  const int chunk = bt.chunk;
  float* sc = smem;                        // [G][chunk] scores
  float* red = smem + G * chunk;           // [kWarps][G]
  float* thr = red + kWarps * G;           // [G]
  int* wc = reinterpret_cast<int*>(thr + G);  // [kWarps][G]

  int b, h, ci;
  decode_chunk(bt, c, b, h, ci);
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
  // Keys per half-warp per step: 8, or 4 when a key row is >= 32 B per lane
  // (fp32 d=128): two register buffers of KPH rows stay at 64 registers, so
  // the fp32 scan is not register-starved. A 128-key tile is SUB steps.
  constexpr int KPH = (int)sizeof(T) * DPL >= 32 ? 4 : 8;
  constexpr int SUB = kScanKPH / KPH;
  constexpr int PK = KPH * G;
  RawFrag<T, DPL> fa[KPH], fb[KPH];

  auto load_step = [&](int st, RawFrag<T, DPL>(&f)[KPH]) {
    const int tile = st / SUB, sub = st % SUB;
#pragma unroll
    for (int k = 0; k < KPH; ++k) {
      int row = tile * kScanTile + hw * kScanKPH + sub * KPH + k;
      if (row < valid) f[k].load(kb + (size_t)row * D); else f[k].zero();
    }
  };
  auto compute_step = [&](int st, const RawFrag<T, DPL>(&f)[KPH]) {
    const int tile = st / SUB, sub = st % SUB;
    float a[PK];
#pragma unroll
    for (int k = 0; k < KPH; ++k) {
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
    int kk;
    bool writer;
    if constexpr (KPH == 8) {  // 8G -> 4G -> 2G -> G partials, then xor over lane bit 0
      tr_level<8 * G>(a, 8, (hl & 8) != 0);
      tr_level<4 * G>(a, 4, (hl & 4) != 0);
      tr_level<2 * G>(a, 2, (hl & 2) != 0);
#pragma unroll
      for (int j = 0; j < G; ++j) a[j] += __shfl_xor_sync(kFull, a[j], 1);
      kk = (hl >> 1) & 7;
      writer = (hl & 1) == 0;
    } else {  // 4G -> 2G -> G partials, then xor over lane bits 1 and 0
      tr_level<4 * G>(a, 8, (hl & 8) != 0);
      tr_level<2 * G>(a, 4, (hl & 4) != 0);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        a[j] += __shfl_xor_sync(kFull, a[j], 2);
        a[j] += __shfl_xor_sync(kFull, a[j], 1);
      }
      kk = (hl >> 2) & 3;
      writer = (hl & 3) == 0;
    }
    const int row = tile * kScanTile + hw * kScanKPH + sub * KPH + kk;
    if (writer && row < valid) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        sc[j * chunk + row] = a[j];
        mymax[j] = fmaxf(mymax[j], a[j]);
      }
    }
  };

  // kept tiles (block filter), SUB steps each, double-buffered: load the next
  // step while computing the current one
  const unsigned long long tmask = chunk_tiles(bt, ws, c, ntiles);
  unsigned long long mrem = tmask;
  int tile_open = -1, sub_next = 0;
  auto pop = [&]() -> int {
    if (tile_open >= 0 && sub_next < SUB) return tile_open * SUB + sub_next++;
    if (!mrem) return -1;
    tile_open = __ffsll((long long)mrem) - 1;
    mrem &= mrem - 1;
    sub_next = 1;
    return tile_open * SUB;
  };
  int cur = pop();
  if (cur >= 0) load_step(cur, fa);
  while (cur >= 0) {
    const int nxt = pop();
    if (nxt >= 0) load_step(nxt, fb);
    compute_step(cur, fa);
    if (nxt < 0) break;
    cur = pop();
    if (cur >= 0) load_step(cur, fa);
    compute_step(nxt, fb);
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
    thr[tid] = bt.topk_thr ? bt.topk_thr[b * bt.Hq + h * G + tid] : fmaxf(cm, dec_max(old)) - bt.beta;
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
      bool p = pos < valid && ((tmask >> (pos / kScanTile)) & 1ull) && sc[j * chunk + pos] >= th;
      cnt += __popc(__ballot_sync(kFull, p));
    }
    cntj[j] = cnt;
    if (lane == 0) wc[warp * G + j] = cnt;
  }
  __syncthreads();
  const size_t cbase = (size_t)c * G;
  const int quarter = warp >> 1;  // sub-list = position quarter (warps 2k, 2k+1)
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float th = thr[j];
    const int off0 = (warp & 1) ? wc[(warp - 1) * G + j] : 0;
    int off = off0;
    int* oi = ws.cidx + (cbase + j) * chunk + quarter * (chunk / 4);
    float* os = ws.cscore + (cbase + j) * chunk + quarter * (chunk / 4);
    if (cntj[j] > 0) {
      for (int r = 0; r < seg; r += 32) {
        int pos = sbeg + r + lane;
        const bool live = pos < valid && ((tmask >> (pos / kScanTile)) & 1ull);
        float v = live ? sc[j * chunk + pos] : -INFINITY;
        bool p = live && v >= th;
        unsigned bal = __ballot_sync(kFull, p);
        if (p) {
          int o = off + __popc(bal & lanemask_lt());
          oi[o] = pos;
          os[o] = v;
        }
        off += __popc(bal);
      }
    }
    if (tid < 4) ws.cnt[(cbase + j) * 4 + tid] = wc[(2 * tid) * G + j] + wc[(2 * tid + 1) * G + j];
    if (tid == 4) {
      int tot = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) tot += wc[w * G + j];
      publish_pair(bt, ws, cbase + j, tot);
    }
  }
  if (bt.overlap) {  // chunk published: 4 units, like the tcgen05 scan's 4 epilogue warps
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      atomicAdd(&ws.group_done[b * bt.Hkv + h], 4);
      atomicAdd(&ws.counters[6], 4);
    }
  }
}


// One CTA per chunk, or (bt.persist) a persistent grid taking chunks in increasing
// order from the header counter, so the (sequence, kv head) groups complete in
// order and the attend can run beside the scan (overlap mode).
template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads, (G <= 5 ? 2 : 1))
    scan_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q, Ws ws) {
  extern __shared__ float smem[];
  __shared__ int s_next;
  pdl_wait();
  pdl_trigger();  // after the wait: see alaya_tc.cuh (attend_ovl relies on it)
  if (!bt.persist) {
    scan_chunk<T, D, G>(bt, q, ws, (int)blockIdx.x, smem);
    return;
  }
  for (int c = (int)blockIdx.x; c < bt.total_chunks;) {
    if (threadIdx.x == 0) s_next = (int)gridDim.x + atomicAdd(&ws.counters[9], 1);
    scan_chunk<T, D, G>(bt, q, ws, c, smem);
    __syncthreads();  // shared scores / counts are reused by the next chunk; s_next is set
    c = s_next;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Stage 2: exact filter + V gather (reference: dipr.py:64, store.py:271-278,
// attention.py:98-110). One WARP per task; tasks [0, chunks*G) are
// (chunk, query head) pairs, tasks [chunks*G, chunks*G + B*Hq) compute the
// window partial of one (sequence, query head). Softmax reference point of a
// selection partial is the (global) max, so chunk partials merge by plain sums.
// ---------------------------------------------------------------------------
constexpr int kGatherU = 16;  // V rows in flight per half-warp (one candidate batch)
static_assert(2 * kGatherU == 32, "one 32-candidate filter batch = kGatherU rows per half-warp");

constexpr int kWinU = 4;     // window rows in flight per half-warp

template <typename T, int D>
__device__ __forceinline__ void hw_dot_rows(const T* const (&rows)[kWinU], const float (&qr)[D / 16],
                                            float (&out)[kWinU], int hl) {
  constexpr int DPL = D / 16;
  RawFrag<T, DPL> f[kWinU];
#pragma unroll
  for (int k = 0; k < kWinU; ++k) {
    if (rows[k]) f[k].load(rows[k] + hl * DPL); else f[k].zero();
  }
#pragma unroll
  for (int k = 0; k < kWinU; ++k) {
    float x[DPL];
    f[k].to_float(x);
    float a = 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) a = fmaf(qr[e], x[e], a);
#pragma unroll
    for (int m = 8; m > 0; m >>= 1) a += __shfl_xor_sync(kFull, a, m);
    out[k] = a;
  }
}

// Selection partial of one (chunk c, head j) task, software-pipelined so the
// V loads of candidate batch k stay in flight while batch k+1 is filtered:
//   issue loads(k) -> filter(k+1) -> FMA(k).
// Rows are held in registers (kGatherU per half-warp: one 32-candidate batch).
// L2 = true reads inputs produced by other SMs in the same launch (__ldcg).
template <typename T, int D, int G, bool L2>
__device__ __forceinline__ void sel_task_pipe(const Batch& bt, const float* __restrict__ smax_ext,
                                              const Ws& ws, size_t cj, int qb, int qe, int lane,
                                              int (*s_t)[32], float (*s_w)[32], bool want_values) {
  // rows in flight per half-warp: one 32-candidate batch in one round when a lane's
  // share of a row is <= 16 B (bf16 d=128), else in 2+ rounds of fewer rows (fp32 rows
  // are 32 B per lane: 16 of them would need 128 registers and spill)
  constexpr int DPL = D / 16;
  constexpr int U = (int)sizeof(T) * DPL <= 16 ? kGatherU : kGatherU * 16 / ((int)sizeof(T) * DPL);
  constexpr int ROUNDS = kGatherU / U;
  const int hl = lane & 15, half = lane >> 4;
  // sub-lists [qb, qe) of pair cj = (chunk c, head j) as one virtual list; the
  // primary task (qb = 0) writes slot cj, an overflow task (qb > 0) slot cj*4+qb
  const int c = (int)cj / G, j = (int)cj - c * G;
  int b, h, ci;
  decode_chunk(bt, c, b, h, ci);
  const KSeq& s = bt.s[b];
  const int chunk = bt.chunk;
  const int t0 = ci * chunk;
  const int qh = h * G + j;
  const float smax = smax_ext ? smax_ext[b * bt.Hq + qh]
                              : dec_max(L2 ? __ldcg(&ws.gmax[b * bt.Hq + qh]) : ws.gmax[b * bt.Hq + qh]);
  const float th = smax - bt.beta;
  const float k2 = bt.inv_sqrt_d * kLog2e;
  const CandList L = cand_range(ws.cnt + cj * 4, qb, qe, chunk, L2);
  const int nc = L.total();
  int* ci_ = ws.cidx + cj * chunk + qb * (chunk / 4);
  const float* cs_ = ws.cscore + cj * chunk + qb * (chunk / 4);
  auto ldi = [&](int i) { return L2 ? __ldcg(ci_ + L.phys(i)) : ci_[L.phys(i)]; };
  auto lds = [&](int i) { return L2 ? __ldcg(cs_ + L.phys(i)) : cs_[L.phys(i)]; };
  const T* vb = reinterpret_cast<const T*>(s.v) + (size_t)h * s.hs + (size_t)t0 * D + hl * DPL;
  float acc[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) acc[e] = 0.f;
  int sel_tot = 0, ret_tot = 0;
  float lsum = 0.f;
  int t_n = lane < nc ? ldi(lane) : 0;
  float s_n = lane < nc ? lds(lane) : -INFINITY;
  int next_i0 = 0;  // first candidate index of the next batch to filter
  // filter one batch into slot `sl`, returns its selected count
  auto filter = [&](int sl) -> int {
    const int i0 = next_i0;
    next_i0 += 32;
    const int i = i0 + lane;
    const bool valid = i < nc;
    const int t = t_n;
    const float sv = s_n;
    if (i0 + 32 < nc) {  // prefetch the batch after
      const int ii = i + 32;
      t_n = ii < nc ? ldi(ii) : 0;
      s_n = ii < nc ? lds(ii) : -INFINITY;
    }
    const bool pass = valid && sv >= th;
    const bool sel = pass && !in_window(s.off + t0 + t, s.P, bt.wi, bt.wl);
    const unsigned bs = __ballot_sync(kFull, sel), br = __ballot_sync(kFull, pass);
    const int pos = __popc(bs & lanemask_lt());
    const int ns = __popc(bs);
    const float w = sel ? exp2f((sv - smax) * k2) : 0.f;
    lsum += w;
    __syncwarp();  // all lanes read this batch before the in-place write
    if (sel) {
      ci_[sel_tot + pos] = t;  // in place; physical read position >= write position
      s_t[sl][pos] = t;
      s_w[sl][pos] = w;
    }
    sel_tot += ns;
    ret_tot += __popc(br);
    __syncwarp();
    return ns;
  };
  int cur = 0;
  int ns_cur = nc > 0 ? filter(0) : 0;
  while (true) {
    const bool more = next_i0 < nc;
    if (!want_values) {
      if (!more) break;
      ns_cur = filter(cur ^ 1);
      cur ^= 1;
      continue;
    }
    int ns_nxt = 0;
#pragma unroll
    for (int rd = 0; rd < ROUNDS; ++rd) {
      RawFrag<T, DPL> f[U];
      float wk[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int r = 2 * (rd * U + k) + half;
        if (r < ns_cur) {
          f[k].load(vb + (size_t)s_t[cur][r] * D);
          wk[k] = s_w[cur][r];
        } else {
          f[k].zero();
          wk[k] = 0.f;
        }
      }
      if (rd == 0) ns_nxt = more ? filter(cur ^ 1) : 0;  // overlaps the loads above
#pragma unroll
      for (int k = 0; k < U; ++k) {
        float x[DPL];
        f[k].to_float(x);
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] = fmaf(wk[k], x[e], acc[e]);
      }
    }
    if (!more) break;
    cur ^= 1;
    ns_cur = ns_nxt;
  }
  lsum = warp_sum(lsum);
  const bool ovl = qb > 0;
  const size_t slot = ovl ? cj * 4 + qb : cj;
  if (lane == 0) {
    (ovl ? ws.ovl_sel : ws.selcnt)[slot] = sel_tot;
    (ovl ? ws.ovl_ret : ws.retcnt)[slot] = ret_tot;
    if (want_values) (ovl ? ws.ovl_l : ws.part_l)[slot] = lsum;
  }
  if (want_values) {
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[e] += __shfl_xor_sync(kFull, acc[e], 16);
    if (half == 0) {
      float* pa = (ovl ? ws.ovl_acc : ws.part_acc) + slot * D + hl * DPL;
#pragma unroll
      for (int e = 0; e < DPL; ++e) pa[e] = acc[e];
    }
  }
}

// Window partial of (sequence b, query head qh): base window ids owned by this
// shard + the session rows, online softmax in batches of 2*kWinU rows; written
// to ws.partbuf[b*Hq+qh] as (m, l, acc).
template <typename T, int D, int G>
__device__ __forceinline__ void win_task(const Batch& bt, const float* __restrict__ q, const Ws& ws,
                                         int wt, int lane) {
  constexpr int DPL = D / 16;
  const int hl = lane & 15, half = lane >> 4;
  const int b = wt / bt.Hq, qh = wt - b * bt.Hq, h = qh / G;
  const KSeq& s = bt.s[b];
  const int64_t P = s.P, off = s.off;
  int64_t a0 = 0, a1, b0, b1;
  if (P <= (int64_t)bt.wi + bt.wl) { a1 = P; b0 = 0; b1 = 0; }
  else { a1 = bt.wi; b0 = P - bt.wl; b1 = P; }
  a0 = max(a0, off) - off; a1 = min(a1, off + s.n) - off; if (a1 < a0) a1 = a0;
  b0 = max(b0, off) - off; b1 = min(b1, off + s.n) - off; if (b1 < b0) b1 = b0;
  const int na = (int)(a1 - a0), nbw = (int)(b1 - b0);
  const int R = na + nbw + seq_w(s);
  const T* kbase = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs;
  const T* vbase = reinterpret_cast<const T*>(s.v) + (size_t)h * s.hs;
  const T* wkb = reinterpret_cast<const T*>(s.wk) + (size_t)h * s.whs;
  const T* wvb = reinterpret_cast<const T*>(s.wv) + (size_t)h * s.whs;
  auto row_ptr = [&](int r, bool val) -> const T* {
    if (r < na) return (val ? vbase : kbase) + (size_t)(a0 + r) * D;
    if (r < na + nbw) return (val ? vbase : kbase) + (size_t)(b0 + r - na) * D;
    return (val ? wvb : wkb) + (size_t)(r - na - nbw) * D;
  };
  float qr[DPL];
  load_q<DPL>(q + ((size_t)b * bt.Hq + qh) * D + hl * DPL, qr);
  float m = -INFINITY, l = 0.f, acc[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) acc[e] = 0.f;
  for (int r0 = 0; r0 < R; r0 += 2 * kWinU) {
    const T* kr[kWinU];
    const T* vr[kWinU];
#pragma unroll
    for (int k = 0; k < kWinU; ++k) {
      const int r = r0 + 2 * k + half;
      kr[k] = r < R ? row_ptr(r, false) : nullptr;
      vr[k] = r < R ? row_ptr(r, true) : nullptr;
    }
    float z[kWinU];
    hw_dot_rows<T, D>(kr, qr, z, hl);
    float bm = -INFINITY;
#pragma unroll
    for (int k = 0; k < kWinU; ++k) {
      z[k] = kr[k] ? z[k] * bt.inv_sqrt_d : -INFINITY;
      bm = fmaxf(bm, z[k]);
    }
    bm = fmaxf(bm, __shfl_xor_sync(kFull, bm, 16));
    const float mn = fmaxf(m, bm);
    const float sc = (m == -INFINITY) ? 0.f : expf(m - mn);
    RawFrag<T, DPL> f[kWinU];
#pragma unroll
    for (int k = 0; k < kWinU; ++k) {
      if (vr[k]) f[k].load(vr[k] + hl * DPL); else f[k].zero();
    }
    float lb = 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[e] *= sc;
#pragma unroll
    for (int k = 0; k < kWinU; ++k) {
      const float w = kr[k] ? expf(z[k] - mn) : 0.f;
      lb += w;
      float x[DPL];
      f[k].to_float(x);
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[e] = fmaf(w, x[e], acc[e]);
    }
    lb += __shfl_xor_sync(kFull, lb, 16);
    l = l * sc + lb;
    m = mn;
  }
#pragma unroll
  for (int e = 0; e < DPL; ++e) acc[e] += __shfl_xor_sync(kFull, acc[e], 16);
  float* pr = ws.partbuf + (size_t)wt * (D + 2);
  if (lane == 0) { pr[0] = R > 0 ? m : -INFINITY; pr[1] = R > 0 ? l : 0.f; }
  if (half == 0) {
#pragma unroll
    for (int e = 0; e < DPL; ++e) pr[2 + hl * DPL + e] = R > 0 ? acc[e] : 0.f;
  }
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads, 2)
    attend_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q,
                  const float* __restrict__ smax_ext, Ws ws, int want_values) {
  __shared__ int s_t[kWarps][2][32];
  __shared__ float s_w[kWarps][2][32];
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwin = (want_values && !bt.win_in_prep) ? bt.B * bt.Hq : 0;
  const int npairs = bt.total_chunks * G;
  // + overflow items published by the scan (none without chunks: no scan ran)
  const int ntasks = nwin + npairs + (npairs ? ws.counters[7] : 0);
  for (;;) {  // window tasks, (chunk, head) pairs, then heavy pairs' sub-lists 1..3
    int task = 0;
    if (lane == 0) task = atomicAdd(&ws.counters[0], 1);
    task = __shfl_sync(kFull, task, 0);
    if (task >= ntasks) break;
    if (task < nwin) {
      win_task<T, D, G>(bt, q, ws, task, lane);
      continue;
    }
    int qb = 0, qe;
    size_t cj;
    if (task < nwin + npairs) {
      cj = task - nwin;
      qe = ws.heavy[cj] ? 1 : 4;  // primary: whole pair, or sub-list 0 of a heavy pair
    } else {
      const int item = ws.ovlist[task - nwin - npairs];
      cj = (size_t)(item >> 2);
      qb = item & 3;
      qe = qb + 1;
    }
    sel_task_pipe<T, D, G, false>(bt, smax_ext, ws, cj, qb, qe, lane, s_t[warp], s_w[warp],
                                  want_values != 0);
  }
}

// Fused sharded step: wait until every rank raised the flag of group (b, h) in
// this rank's exchange buffer, then the global max of row (b, h*G + j) = max of
// the R ranks' local maxima, into ws.smaxbuf (every warp computing it writes the
// same value).
__device__ __forceinline__ void sx_global_max(const Batch& bt, const Ws& ws, int b, int h, int j, int lane) {
  const ShardExch& x = bt.sx;
  const int g = b * bt.Hkv + h, row = b * bt.Hq + h * bt.G + j;
  const int parity = (int)(x.epoch & 1ull);
  float m = -INFINITY;
  if (lane < x.R) {
    const unsigned long long* f = exch_gflag(x.peers[x.rank], g, lane);
    long long polls = 0;
    while (ld_acquire_sys_u64(f) < x.epoch) {
      if (++polls > (1ll << 26)) {  // a rank never arrived: flag the call, use what is here
        if (x.err) atomicExch(x.err, 1);
        break;
      }
      __nanosleep(128);
    }
    m = __ldcv(exch_slot(x.peers[x.rank], parity, 0, lane, x.R, x.cap) + row);
  }
  m = warp_max(m);
  if (lane == 0) ws.smaxbuf[row] = m;
  __syncwarp();
}

// Attend launched BESIDE the tcgen05 scan (bt.overlap): the kernel is a PDL
// dependent of the scan and skips the grid-dependency wait; the scan only
// triggers after its own wait, so everything before the scan is complete.
// A (chunk, head) task starts once its (sequence, kv head) group counter says
// every epilogue warp of every chunk of the group has published (the group's
// max is final); heavy pairs' overflow items wait for the whole scan. Window
// tasks need nothing from the scan and go first.
// 2-warp CTAs: finer-grained residency beside the scan CTAs (B=4 layer 221 -> 219 us,
// B=8 429 -> 426.5 vs 4-warp CTAs, profiles/r02/ovl64_v63.jsonl)
#ifndef ALAYA_OVL_THREADS
#define ALAYA_OVL_THREADS 64
#endif
constexpr int kOvlThreads = ALAYA_OVL_THREADS;

template <typename T, int D, int G>
__global__ void __launch_bounds__(kOvlThreads, 512 / kOvlThreads)  // <= 128 regs
    attend_ovl_kernel(const __grid_constant__ Batch bt, const float* __restrict__ q, Ws ws) {
  constexpr int W = kOvlThreads / 32;
  __shared__ int s_t[W][2][32];
  __shared__ float s_w[W][2][32];
  pdl_trigger();
  if (threadIdx.x == 0) trace_rec(bt, 2, 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwin = bt.win_in_prep ? 0 : bt.B * bt.Hq;
  const int npairs = bt.total_chunks * G;
  const int all_done = 4 * bt.total_chunks;
  int novl = -1;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(&ws.counters[0], 1);
    task = __shfl_sync(kFull, task, 0);
    if (task < nwin) {
      win_task<T, D, G>(bt, q, ws, task, lane);
      continue;
    }
    int qb = 0, qe;
    size_t cj;
    if (task < nwin + npairs) {
      cj = task - nwin;
      int b, h, ci;
      decode_chunk(bt, (int)cj / G, b, h, ci);
      if (bt.sx_on) {
        sx_global_max(bt, ws, b, h, (int)(cj - (cj / G) * G), lane);
      } else {
        if (lane == 0) {
          const int* gd = ws.group_done + b * bt.Hkv + h;
          while (ld_acquire_gpu(gd) < 4 * bt.s[b].nch) __nanosleep(256);
        }
        __syncwarp();
      }
      qe = __ldcg(&ws.heavy[cj]) ? 1 : 4;
      if (bt.trace && lane == 0) trace_max(bt, 2, 2, gtimer());  // latest group-ready of a pair task
    } else {
      if (novl < 0) {  // overflow items are final once every chunk has published
        if (lane == 0) {
          while (ld_acquire_gpu(&ws.counters[6]) < all_done) __nanosleep(512);
          novl = __ldcg(&ws.counters[7]);
        }
        novl = __shfl_sync(kFull, novl, 0);
      }
      if (task - nwin - npairs >= novl) break;
      const int item = __ldcg(&ws.ovlist[task - nwin - npairs]);
      cj = (size_t)(item >> 2);
      qb = item & 3;
      qe = qb + 1;
      if (bt.sx_on) {
        int b, h, ci;
        decode_chunk(bt, (int)cj / G, b, h, ci);
        sx_global_max(bt, ws, b, h, (int)(cj - (cj / G) * G), lane);
      }
    }
    const unsigned long long t_task = bt.trace ? gtimer() : 0ull;
    sel_task_pipe<T, D, G, true>(bt, bt.sx_on ? ws.smaxbuf : nullptr, ws, cj, qb, qe, lane, s_t[warp],
                                 s_w[warp], true);
    if (bt.trace && lane == 0) {
      const unsigned long long t1 = gtimer();
      trace_max(bt, 2, 3, t1);                 // last task end
      trace_max(bt, 2, 4, t1 - t_task);        // longest task (ns)
      atomicAdd(bt.trace + ((size_t)2 * kTraceCtas + min((int)blockIdx.x, kTraceCtas - 1)) * kTraceSlots + 5, 1ull);
    }
  }
  if (bt.trace) {
    __syncthreads();
    if (threadIdx.x == 0) trace_rec(bt, 2, 1);
  }
}

// Group-format attend (bt.gfmt; reference: dipr.py:64 filter, store.py:271-278,
// attention.py:98-110). One 4-warp CTA per chunk: warp q walks the chunk's
// quarter-q list of rows some head of the GQA group may keep (with all G
// scores, written by the tcgen05 scan), applies every head's exact filter
// s_j >= gmax_j - beta minus the window ids, and gathers each kept V row ONCE
// for the whole group (G weighted sums per row), so V rows the G heads share
// are not re-read. The 4 quarter partials are summed in fixed order into one
// (chunk, head) partial; per-quarter selected ids go to the per-head lists for
// diagnostics (alaya_selected). Launched beside the scan like attend_ovl_kernel:
// a chunk starts once its (sequence, kv head) group has published every chunk.
// It pays G FMAs per gathered row, so it wins only when the heads share most of
// their rows (high beta): see gfmt_enabled().
constexpr int kGrpThreads = 128;

template <typename T, int D, int G>
__global__ void __launch_bounds__(kGrpThreads, 4)
    attend_grp_kernel(const __grid_constant__ Batch bt, Ws ws) {
  constexpr int DPL = D >= 16 ? D / 16 : 1;  // (the group format runs at d = 128 only)
  constexpr int U = G <= 4 ? 16 : 8;         // V rows in flight per half-warp
  __shared__ int s_task;
  __shared__ int s_row[4][32];
  __shared__ float s_w[4][G][32];
  __shared__ float s_red[3][D >= 16 ? D : 16];
  __shared__ float s_l[4][G];
  __shared__ int s_ns[4][G], s_nr[4][G];
  pdl_trigger();
  if (threadIdx.x == 0) trace_rec(bt, 2, 0);
  if constexpr (D < 16) {
    return;
  } else {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, hl = lane & 15, half = lane >> 4;
  const int chunk = bt.chunk, qcap = chunk / 4;
  const float k2 = bt.inv_sqrt_d * kLog2e;
  for (;;) {
    __syncthreads();  // s_task / s_* of the previous task are consumed
    if (threadIdx.x == 0) s_task = atomicAdd(&ws.counters[0], 1);
    __syncthreads();
    const int c = s_task;
    if (c >= bt.total_chunks) break;
    int b, h, ci;
    decode_chunk(bt, c, b, h, ci);
    const KSeq& s = bt.s[b];
    const int t0 = ci * chunk;
    if (bt.sx_on) {  // fused sharded step: global max over the ranks' pushed local maxima
      for (int j = warp; j < G; j += 4) sx_global_max(bt, ws, b, h, j, lane);
    } else if (threadIdx.x == 0) {
      const int* gd = ws.group_done + b * bt.Hkv + h;
      while (ld_acquire_gpu(gd) < 4 * s.nch) __nanosleep(256);
    }
    __syncthreads();
    float gm[G], th[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int row = b * bt.Hq + h * G + j;
      gm[j] = bt.sx_on ? __ldcg(&ws.smaxbuf[row]) : dec_max(__ldcg(&ws.gmax[row]));
      th[j] = gm[j] - bt.beta;
    }
    // this warp's quarter list
    const int n = __ldcg(&ws.cnt[(size_t)c * 4 + warp]);
    const int* gi = ws.gidx + (size_t)c * chunk + warp * qcap;
    const float* gs = ws.cscore + (size_t)(c * 4 + warp) * G * qcap;
    const T* vb = reinterpret_cast<const T*>(s.v) + (size_t)h * s.hs + (size_t)t0 * D + hl * DPL;
    float acc[G][DPL], lsum[G];
    int nsel[G], nret[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      lsum[j] = 0.f;
      nsel[j] = nret[j] = 0;
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[j][e] = 0.f;
    }
    // entries of the next batch are loaded while this batch is filtered and gathered
    int row_n = lane < n ? __ldcg(gi + lane) : 0;
    float sc_n[G];
#pragma unroll
    for (int j = 0; j < G; ++j) sc_n[j] = lane < n ? __ldcg(gs + j * qcap + lane) : -INFINITY;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const int row = row_n;
      float sc[G];
#pragma unroll
      for (int j = 0; j < G; ++j) sc[j] = sc_n[j];
      if (i0 + 32 < n) {
        const int ii = i + 32;
        row_n = ii < n ? __ldcg(gi + ii) : 0;
#pragma unroll
        for (int j = 0; j < G; ++j) sc_n[j] = ii < n ? __ldcg(gs + j * qcap + ii) : -INFINITY;
      }
      const bool valid = i < n;
      const bool inwin = valid && in_window(s.off + t0 + row, s.P, bt.wi, bt.wl);
      float w[G];
      bool any = false;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const bool pass = valid && sc[j] >= th[j];
        const bool sel = pass && !inwin;
        const unsigned bs = __ballot_sync(kFull, sel), br = __ballot_sync(kFull, pass);
        if (sel)  // selected ids of (chunk, head j), quarter list `warp` (diagnostics)
          ws.cidx[((size_t)c * G + j) * chunk + warp * qcap + nsel[j] + __popc(bs & lanemask_lt())] = row;
        nsel[j] += __popc(bs);
        nret[j] += __popc(br);
        w[j] = sel ? exp2f((sc[j] - gm[j]) * k2) : 0.f;
        lsum[j] += w[j];
        any |= sel;
      }
      const unsigned ba = __ballot_sync(kFull, any);
      const int na = __popc(ba);
      if (any) {
        const int pos = __popc(ba & lanemask_lt());
        s_row[warp][pos] = row;
#pragma unroll
        for (int j = 0; j < G; ++j) s_w[warp][j][pos] = w[j];
      }
      __syncwarp();
      for (int r0 = 0; r0 < na; r0 += 2 * U) {  // each kept row read once for all G heads
        RawFrag<T, DPL> f[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int r = r0 + 2 * k + half;
          if (r < na) f[k].load(vb + (size_t)s_row[warp][r] * D); else f[k].zero();
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int r = r0 + 2 * k + half;
          float x[DPL];
          f[k].to_float(x);
#pragma unroll
          for (int j = 0; j < G; ++j) {
            const float wk = r < na ? s_w[warp][j][r] : 0.f;
#pragma unroll
            for (int e = 0; e < DPL; ++e) acc[j][e] = fmaf(wk, x[e], acc[j][e]);
          }
        }
      }
      __syncwarp();
    }
    // the 4 quarter partials -> one (chunk, head) partial, summed in fixed order
#pragma unroll
    for (int j = 0; j < G; ++j) {
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[j][e] += __shfl_xor_sync(kFull, acc[j][e], 16);
      const float l = warp_sum(lsum[j]);
      if (lane == 0) { s_l[warp][j] = l; s_ns[warp][j] = nsel[j]; s_nr[warp][j] = nret[j]; }
    }
    const size_t cj0 = (size_t)c * G;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (warp > 0 && half == 0) {
#pragma unroll
        for (int e = 0; e < DPL; ++e) s_red[warp - 1][hl * DPL + e] = acc[j][e];
      }
      __syncthreads();
      if (warp == 0 && half == 0) {
        float* pa = ws.part_acc + (cj0 + j) * D + hl * DPL;
#pragma unroll
        for (int e = 0; e < DPL; ++e)
          pa[e] = ((acc[j][e] + s_red[0][hl * DPL + e]) + s_red[1][hl * DPL + e]) + s_red[2][hl * DPL + e];
      }
      __syncthreads();
    }
    if (threadIdx.x < G) {
      const int j = threadIdx.x;
      float l = 0.f;
      int ns = 0, nr = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
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
  if (bt.trace && threadIdx.x == 0) trace_rec(bt, 2, 1);
  }
}

// ---------------------------------------------------------------------------
// Stage 3: one CTA per (sequence, query head): sum of the chunk partials (the
// selected set, reference point = max; warps take interleaved chunks, fixed
// reduction order) merged with the window partial (attention.py:128-143,
// selected first, then window), finalized (attention.py:145-152) or exported
// as (m, l, acc) for a cross-shard merge.
// ---------------------------------------------------------------------------
template <int D, int G, int CW>
__global__ void __launch_bounds__(CW * 32)
    combine_kernel(const __grid_constant__ Batch bt, const float* __restrict__ smax_ext, Ws ws,
                   float* __restrict__ out, float* __restrict__ part_out,
                   float* __restrict__ smax_out) {
  constexpr int DL = (D + 31) / 32;
  constexpr int U = 4;
  __shared__ float red[CW][D];
  __shared__ float redl[CW];
  __shared__ int redn[CW];
  pdl_trigger();
  if (threadIdx.x == 0) trace_rec(bt, 3, 0);
  pdl_wait();
  if (bt.call_id) {  // every prep CTA of this call is done seeding (none lands in a later call):
    // its per-group flag carries this call's token (never zeroed, so a CTA whose header
    // wait timed out still signs off -- a zeroed counter could lose that arrival)
    const unsigned long long tok = call_token(bt);
    for (int g = threadIdx.x; g < bt.B * bt.Hkv; g += blockDim.x)
      while (ld_acquire_gpu_u64(ws.prepdone + g) != tok) __nanosleep(64);
    __syncthreads();
  }
  if (threadIdx.x == 0) trace_rec(bt, 3, 2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.x;
  const int b = row / bt.Hq, qh = row - b * bt.Hq;
  const int h = qh / G, j = qh - h * G;
  const KSeq& s = bt.s[b];
  const int c0 = s.chunk_base + h * s.nch;
  // warp 0's epilogue inputs (max, window partial) are loaded up front, in flight
  // with the chunk partials instead of a dependent round trip after the reduction
  float smax = 0.f, mw = 0.f, lw = 0.f, wpe[DL];
  const float* wp = ws.partbuf + (size_t)row * (D + 2);
  if (warp == 0) {
    smax = smax_ext ? smax_ext[row] : dec_max(ws.gmax[row]);
    mw = wp[0];
    lw = wp[1];
#pragma unroll
    for (int k = 0; k < DL; ++k) wpe[k] = lane + 32 * k < D ? wp[2 + lane + 32 * k] : 0.f;
  }
  float ab[DL];
#pragma unroll
  for (int k = 0; k < DL; ++k) ab[k] = 0.f;
  float lb = 0.f;
  int nsel = 0;
  for (int c = warp; c < s.nch; c += CW * U) {
    float v[U][DL], pl[U];
    int tot[U], ps[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // issue every load of the batch first
      const int cc = c + u * CW;
      const size_t cj = (size_t)(c0 + cc) * G + j;
      tot[u] = (cc < s.nch && !bt.gfmt) ? ws.heavy[cj] : 0;  // group format: one partial per pair
      pl[u] = cc < s.nch ? ws.part_l[cj] : 0.f;
      ps[u] = cc < s.nch ? ws.selcnt[cj] : 0;
#pragma unroll
      for (int k = 0; k < DL; ++k) {
        const int e = lane + 32 * k;
        v[u][k] = (cc < s.nch && e < D) ? ws.part_acc[cj * D + e] : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cc = c + u * CW;
      const size_t cj = (size_t)(c0 + cc) * G + j;
      if (cc < s.nch && tot[u]) {  // overflow sub-lists of a heavy pair
        for (int sq = 1; sq < 4; ++sq) {
#pragma unroll
          for (int k = 0; k < DL; ++k) {
            const int e = lane + 32 * k;
            if (e < D) v[u][k] += ws.ovl_acc[(cj * 4 + sq) * D + e];
          }
          if (lane == 0) { lb += ws.ovl_l[cj * 4 + sq]; nsel += ws.ovl_sel[cj * 4 + sq]; }
        }
      }
      if (lane == 0) {
        lb += pl[u];
        nsel += ps[u];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < DL; ++k) ab[k] += v[u][k];
  }
#pragma unroll
  for (int k = 0; k < DL; ++k)
    if (lane + 32 * k < D) red[warp][lane + 32 * k] = ab[k];
  if (lane == 0) { redl[warp] = lb; redn[warp] = nsel; }
  __syncthreads();
  if (warp != 0) return;
  lb = 0.f;
  nsel = 0;
#pragma unroll
  for (int w = 0; w < CW; ++w) { lb += redl[w]; nsel += redn[w]; }
  if (nsel == 0) lb = 0.f;
  if (smax_out && lane == 0) smax_out[row] = smax;
  const float zmax = smax * bt.inv_sqrt_d;
  const bool hb = lb > 0.f, hwn = lw > 0.f;
  const float m = fmaxf(hb ? zmax : -INFINITY, hwn ? mw : -INFINITY);
  const float fb = hb ? expf(zmax - m) : 0.f;
  const float fw = hwn ? expf(mw - m) : 0.f;
  const float l = lb * fb + lw * fw;
  const bool empty = !(hb || hwn);
#pragma unroll
  for (int k = 0; k < DL; ++k) {
    const int e = lane + 32 * k;
    if (e >= D) continue;
    float sb = 0.f;
#pragma unroll
    for (int w = 0; w < CW; ++w) sb += red[w][e];
    const float a = sb * fb + (hwn ? wpe[k] * fw : 0.f);
    if (out) {
      const float o = a / l;
      if (!isfinite(o)) atomicExch(ws.status, (int)ALAYA_ERR_NONFINITE);
      out[(size_t)row * D + e] = o;
    }
    if (part_out) {
      float* pr = part_out + (size_t)row * (D + 2);
      if (e == 0) { pr[0] = empty ? -INFINITY : m; pr[1] = empty ? 0.f : l; }
      pr[2 + e] = empty ? 0.f : a;
    }
    if (bt.sx_on && bt.sx.gepoch) {  // fused allgather: the row straight into every rank's slot
      const ShardExch& x = bt.sx;
      const int parity = (int)(x.gepoch & 1ull);
      for (int r = 0; r < x.R; ++r) {
        float* pr = exch_slot(x.peers[r], parity, 1, x.rank, x.R, x.cap) + (size_t)row * (D + 2);
        if (e == 0) { pr[0] = empty ? -INFINITY : m; pr[1] = empty ? 0.f : l; }
        pr[2 + e] = empty ? 0.f : a;
      }
    }
  }
  if (lane == 0) trace_rec(bt, 3, 1);
  if (bt.sx_on && bt.sx.gepoch) {  // last row out raises this rank's kind-1 flag everywhere
    const ShardExch& x = bt.sx;
    __threadfence_system();
    __syncwarp();
    unsigned int last = 0;
    if (lane == 0) last = atomicAdd(exch_arrive(x.peers[x.rank]), 1u) == gridDim.x - 1;
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      if (lane == 0) *exch_arrive(x.peers[x.rank]) = 0u;  // the next exchange starts after this kernel
      __threadfence_system();
      __syncwarp();
      if (lane < x.R) st_release_sys_u64(exch_flag(x.peers[lane], 1, x.rank), x.gepoch);
    }
  }
}

// ---------------------------------------------------------------------------
// Coarse block filter. Per 128-token block the index holds (K dtype):
//   row 0 lo[d], row 1 hi[d]      per-dim box
//   row 2 mu[d]                   block mean (as stored)
//   row 3 rep[d]                  largest-L2-norm key (index.py:217-228, r=1)
//   row 4 [0] = radius            max_k ||k - mu||, rounded up
// Per call: LB_j = max(score of the base-window keys, score of every block's
// representative) minus a rounding margin -- real scores, hence a lower bound
// of the DIPR max; a 128-key tile is read only if some head of the group has
// min(box, ball) upper bound + margin >= LB_j - beta. Exact by construction.
// ---------------------------------------------------------------------------
constexpr int kBndRows = 5;

template <typename T>
__device__ __forceinline__ float to_f(T x) {
  if constexpr (std::is_same_v<T, float>) return x; else return __bfloat162float(x);
}


// Per-call preparation (replaces a memset of the workspace header): zero the
// tickets, group counters, block-filter bounds and status word, and SEED the
// running max of every (sequence, q head) with a lower bound of its DIPR max:
// the scores of kPrepSamples evenly spaced base keys of this shard, minus a
// rounding margin (so the seed is below what the scan computes for the same
// keys). The scan raises the max to the exact value; seeding only tightens
// its early candidate bound (clustered / locality-ordered prefixes would
// otherwise emit whole chunks as candidates before any chunk max is known).
// One CTA per (sequence, kv head).
constexpr int kPrepSamples = 64;

// Window partial of every q head of group (b, h) -- the base window ids this
// shard holds + the session rows (reference store.py:274-282, window state of
// attention.py:98-110): scores q.k / sqrt(d), (m, l, acc) per head, written to
// ws.partbuf like the attend's window tasks. Computed in prep (it needs nothing
// from the scan), so it is off the attend's tail. 8 warps take 4 rows per round
// (K and V rows of a round in flight together), online softmax per warp, then a
// fixed-order merge of the 8 warp states per head through shared memory.
template <typename T, int D, int G>
__device__ __forceinline__ void prep_window(const Batch& bt, const Ws& ws, const float (&qr)[G][(D + 31) / 32],
                                            int b, int h, int64_t a0, int na, int64_t b0, int nbw, int lane,
                                            int warp) {
  constexpr int DL = (D + 31) / 32, RW = 4;
  extern __shared__ float wsm[];  // [kWarps][G][D + 2]
  const KSeq& s = bt.s[b];
  const int R = na + nbw + seq_w(s);
  const T* kbase = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs;
  const T* vbase = reinterpret_cast<const T*>(s.v) + (size_t)h * s.hs;
  const T* wkb = reinterpret_cast<const T*>(s.wk) + (size_t)h * s.whs;
  const T* wvb = reinterpret_cast<const T*>(s.wv) + (size_t)h * s.whs;
  float m[G], l[G], acc[G][DL];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    m[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int k = 0; k < DL; ++k) acc[j][k] = 0.f;
  }
  for (int r0 = warp * RW; r0 < R; r0 += kWarps * RW) {
    float kx[RW][DL], vx[RW][DL];
#pragma unroll
    for (int u = 0; u < RW; ++u) {
      const int r = r0 + u;
      const T *kr = nullptr, *vr = nullptr;
      if (r < na) { kr = kbase + (size_t)(a0 + r) * D; vr = vbase + (size_t)(a0 + r) * D; }
      else if (r < na + nbw) { kr = kbase + (size_t)(b0 + r - na) * D; vr = vbase + (size_t)(b0 + r - na) * D; }
      else if (r < R) { kr = wkb + (size_t)(r - na - nbw) * D; vr = wvb + (size_t)(r - na - nbw) * D; }
#pragma unroll
      for (int k = 0; k < DL; ++k) {
        const int e = lane + 32 * k;
        kx[u][k] = (kr && e < D) ? to_f(kr[e]) : 0.f;
        vx[u][k] = (vr && e < D) ? to_f(vr[e]) : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      float z[RW], bm = -INFINITY;
#pragma unroll
      for (int u = 0; u < RW; ++u) {
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < DL; ++k) a = fmaf(qr[j][k], kx[u][k], a);
        z[u] = r0 + u < R ? warp_sum(a) * bt.inv_sqrt_d : -INFINITY;
        bm = fmaxf(bm, z[u]);
      }
      const float mn = fmaxf(m[j], bm);
      const float sc = m[j] == -INFINITY ? 0.f : expf(m[j] - mn);
      l[j] *= sc;
#pragma unroll
      for (int k = 0; k < DL; ++k) acc[j][k] *= sc;
#pragma unroll
      for (int u = 0; u < RW; ++u) {
        const float w = r0 + u < R ? expf(z[u] - mn) : 0.f;
        l[j] += w;
#pragma unroll
        for (int k = 0; k < DL; ++k) acc[j][k] = fmaf(w, vx[u][k], acc[j][k]);
      }
      m[j] = mn;
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    float* o = wsm + ((size_t)warp * G + j) * (D + 2);
    if (lane == 0) { o[0] = m[j]; o[1] = l[j]; }
#pragma unroll
    for (int k = 0; k < DL; ++k)
      if (lane + 32 * k < D) o[2 + lane + 32 * k] = acc[j][k];
  }
  __syncthreads();
  for (int j = warp; j < G; j += kWarps) {  // warp j merges head j's 8 warp states in order
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, wsm[((size_t)w * G + j) * (D + 2)]);
    float f[kWarps], L = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float mw = wsm[((size_t)w * G + j) * (D + 2)];
      f[w] = (M == -INFINITY || mw == -INFINITY) ? 0.f : expf(mw - M);
      L += wsm[((size_t)w * G + j) * (D + 2) + 1] * f[w];
    }
    float* pr = ws.partbuf + ((size_t)b * bt.Hq + h * G + j) * (D + 2);
    if (lane == 0) { pr[0] = R > 0 ? M : -INFINITY; pr[1] = R > 0 ? L : 0.f; }
    for (int e = lane; e < D; e += 32) {
      float a = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) a += wsm[((size_t)w * G + j) * (D + 2) + 2 + e] * f[w];
      pr[2 + e] = R > 0 ? a : 0.f;
    }
  }
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads) prep_kernel(const __grid_constant__ Batch bt,
                                                        const float* __restrict__ q, Ws ws) {
  constexpr int DL = (D + 31) / 32;
  constexpr int RU = kPrepSamples / kWarps;  // rows in flight per warp
  __shared__ float red[kWarps][G];
  pdl_trigger();
  if (threadIdx.x == 0) trace_rec(bt, 0, 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x / bt.Hkv, h = blockIdx.x - b * bt.Hkv;
  const KSeq& s = bt.s[b];
  const bool async = bt.call_id != 0;
  const int S = min(s.n, kPrepSamples);
  const T* kb = reinterpret_cast<const T*>(s.k) + (size_t)h * s.hs;
  // + the base window ids this shard holds (core.py:159-165): real base tokens, and
  // the recent ones are often in the query's cluster
  const int64_t P = s.P, off = s.off;
  int64_t a0 = 0, a1, b0, b1;
  if (P <= (int64_t)bt.wi + bt.wl) { a1 = P; b0 = 0; b1 = 0; }
  else { a1 = bt.wi; b0 = P - bt.wl; b1 = P; }
  a0 = max(a0, off) - off; a1 = min(a1, off + s.n) - off; if (a1 < a0) a1 = a0;
  b0 = max(b0, off) - off; b1 = min(b1, off + s.n) - off; if (b1 < b0) b1 = b0;
  const int na = (int)(a1 - a0), nbw = (int)(b1 - b0);
  // window rows join the sample only when the block filter consumes the seed (they
  // tighten its LB; otherwise the extra load rounds cost more than they save)
  const int R = bt.seed ? S + (bt.block_filter ? min(na + nbw, 2 * kPrepSamples) : 0) : 0;
  float x[RU][DL];
  auto load_round = [&](int i0) {
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int i = i0 + u;
      int64_t row = 0;
      if (i < S) row = (int64_t)i * s.n / S;
      else if (i - S < na) row = a0 + (i - S);
      else row = b0 + (i - S - na);
      const T* kr = kb + (size_t)row * D;
#pragma unroll
      for (int k = 0; k < DL; ++k) {
        const int e = lane + 32 * k;
        x[u][k] = (i < R && e < D) ? to_f(kr[e]) : 0.f;
      }
    }
  };
  // the first sampled rows are loaded BEFORE the grid-dependency wait: K is context
  // memory, never written by the kernels this call follows (the scan's TMA producer
  // relies on the same), so their HBM latency overlaps the previous call's tail
  int i0 = warp * RU;
  if (i0 < R) load_round(i0);
  pdl_wait();
  if (threadIdx.x == 0) trace_rec(bt, 0, 2);
  if (async) {  // CTA 0 zeroes the whole header, then publishes it (the scan waits on ws.ready)
    if (blockIdx.x == 0) {
      const int rows = bt.B * bt.Hq;
      for (int i = threadIdx.x; i < rows; i += blockDim.x) ws.gmax[i] = 0u;
      for (int i = threadIdx.x; i < bt.B * bt.Hkv; i += blockDim.x) ws.group_done[i] = 0;
      if (threadIdx.x < 16) ws.counters[threadIdx.x] = 0;
      if (threadIdx.x == 0) { *ws.status = 0; *ws.mode = bt.gfmt; }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ws.ready), "l"(call_token(bt)) : "memory");
    }
  } else {
    if (blockIdx.x == 0 && threadIdx.x < 16) {
      ws.counters[threadIdx.x] = 0;
      if (threadIdx.x == 0) { *ws.status = 0; *ws.mode = bt.gfmt; }
    }
    if (threadIdx.x == 0) ws.group_done[blockIdx.x] = 0;
  }
  if (bt.sx_on && s.nch == 0) {  // fused sharded step: no chunk will complete this group
    const ShardExch& sx = bt.sx;
    const int parity = (int)(sx.epoch & 1ull);
    if (threadIdx.x < G * sx.R) {
      const int j = threadIdx.x % G, r = threadIdx.x / G;
      exch_slot(sx.peers[r], parity, 0, sx.rank, sx.R, sx.cap)[b * bt.Hq + h * G + j] = -INFINITY;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < sx.R) st_release_sys_u64(exch_gflag(sx.peers[threadIdx.x], blockIdx.x, sx.rank), sx.epoch);
  }
  float qr[G][DL];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int k = 0; k < DL; ++k) {
      const int e = lane + 32 * k;
      qr[j][k] = e < D ? __ldg(q + ((size_t)b * bt.Hq + h * G + j) * D + e) : 0.f;
    }
  float best[G];
#pragma unroll
  for (int j = 0; j < G; ++j) best[j] = -INFINITY;
  for (; i0 < R; i0 += kWarps * RU) {
    if (i0 != warp * RU) load_round(i0);
#pragma unroll
    for (int u = 0; u < RU; ++u) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float a = 0.f, mag = 0.f;
#pragma unroll
        for (int k = 0; k < DL; ++k) {
          a = fmaf(qr[j][k], x[u][k], a);
          mag = fmaf(fabsf(qr[j][k]), fabsf(x[u][k]), mag);
        }
        a = warp_sum(a);
        mag = warp_sum(mag);
        if (i0 + u < R) best[j] = fmaxf(best[j], a - 1e-3f * (mag + 1.f));
      }
    }
  }
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < G; ++j) red[warp][j] = best[j];
  __syncthreads();
  if (async) {  // seeds join the running max once the header is zeroed, then the group's
                // seed flag goes up (the scan's epilogue starts its first chunk on it)
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
      // bounded: a seed is optional (a lower bound), so a CTA that cannot see the
      // header published (CTA 0 not resident) drops its seed instead of spinning on
      int polls = 0;
      const unsigned long long tok = call_token(bt);
      while (ld_acquire_gpu_u64(ws.ready) != tok && ++polls < (1 << 20)) __nanosleep(32);
      s_ok = polls < (1 << 20);
    }
    __syncthreads();
    if (s_ok && threadIdx.x < G) {
      float m = -INFINITY;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) m = fmaxf(m, red[w][threadIdx.x]);
      if (bt.seed && m > -INFINITY) atomicMax(&ws.gmax[b * bt.Hq + h * G + threadIdx.x], enc_max(m));
    }
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ws.seeded + blockIdx.x), "l"(call_token(bt))
                   : "memory");
  }
  if (bt.app_k) {  // Session.update of this call: the new row of ring (b, h) first
    T* wk = const_cast<T*>(reinterpret_cast<const T*>(s.wk)) + (size_t)h * s.whs + (size_t)(s.w - 1) * D;
    T* wv = const_cast<T*>(reinterpret_cast<const T*>(s.wv)) + (size_t)h * s.whs + (size_t)(s.w - 1) * D;
    const float* kn = bt.app_k + ((size_t)b * bt.Hkv + h) * D;
    const float* vn = bt.app_v + ((size_t)b * bt.Hkv + h) * D;
    for (int e = threadIdx.x; e < D; e += blockDim.x) {
      if constexpr (std::is_same_v<T, float>) { wk[e] = kn[e]; wv[e] = vn[e]; }
      else { wk[e] = __float2bfloat16_rn(kn[e]); wv[e] = __float2bfloat16_rn(vn[e]); }
    }
    __syncthreads();  // (the window partial below reads the row)
  }
  if (bt.win_in_prep) prep_window<T, D, G>(bt, ws, qr, b, h, a0, na, b0, nbw, lane, warp);
  __syncthreads();
  if (async) {
    if (threadIdx.x == 0) {  // this CTA is done (window partial written; combine waits on it)
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ws.prepdone + blockIdx.x), "l"(call_token(bt))
                   : "memory");
      trace_rec(bt, 0, 1);
    }
    return;
  }
  if (threadIdx.x < G) {
    float m = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) m = fmaxf(m, red[w][threadIdx.x]);
    // no seed (0 = -inf) for an empty shard or when seeding is off
    ws.gmax[b * bt.Hq + h * G + threadIdx.x] = (bt.seed && m > -INFINITY) ? enc_max(m) : 0u;
  }
}

// Per chunk: keep mask of its 128-key tiles. A tile is read by the scan only if
// some head of the group has min(box, ball) upper bound + rounding margin >=
// LB - beta, LB = the prep seed (max score of sampled base keys and the base
// window keys, minus a margin -- real scores, hence a lower bound of the DIPR
// max). Exact by construction. One pass; each warp issues the bound rows of all
// its tiles before reducing.
template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads) block_filter_kernel(const __grid_constant__ Batch bt,
                                                                const float* __restrict__ q, Ws ws) {
  constexpr int DL = (D + 31) / 32;
  constexpr int TPW = 2;  // tiles per warp per round (a 2048-key chunk is 16 tiles)
  __shared__ unsigned long long s_mask;
  __shared__ int s_kept;
  pdl_trigger();
  pdl_wait();  // the seeds come from prep_kernel
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x;
  int b, h, ci;
  decode_chunk(bt, c, b, h, ci);
  const KSeq& s = bt.s[b];
  const int chunk = bt.chunk;
  const int valid = min(chunk, s.n - ci * chunk);
  const int ntiles = (valid + 127) / 128;
  if (threadIdx.x == 0) { s_mask = 0ull; s_kept = 0; }
  float qr[G][DL], qn[G], thr[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const size_t row = (size_t)b * bt.Hq + h * G + j;
    float n2 = 0.f;
#pragma unroll
    for (int k = 0; k < DL; ++k) {
      qr[j][k] = lane + 32 * k < D ? q[row * D + lane + 32 * k] : 0.f;
      n2 = fmaf(qr[j][k], qr[j][k], n2);
    }
    qn[j] = sqrtf(warp_sum(n2)) * (1.f + 1e-6f);
    thr[j] = dec_max(__ldcg(&ws.gmax[row])) - bt.beta;  // no seed: -inf keeps every tile
  }
  __syncthreads();
  const T* bb = reinterpret_cast<const T*>(s.bnd) + (size_t)h * s.bhs;
  for (int t0 = warp * TPW; t0 < ntiles; t0 += kWarps * TPW) {
    float lo[TPW][DL], hi[TPW][DL], mu[TPW][DL], rad[TPW];
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      const int t = min(t0 + u, ntiles - 1);
      const T* base = bb + ((size_t)(ci * chunk) / 128 + t) * kBndRows * D;
#pragma unroll
      for (int k = 0; k < DL; ++k) {
        const int e = min(lane + 32 * k, D - 1);
        lo[u][k] = to_f(base[e]);
        hi[u][k] = to_f(base[D + e]);
        mu[u][k] = to_f(base[2 * D + e]);
      }
      rad[u] = to_f(base[4 * D]);
    }
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      const int t = t0 + u;
      bool keep = false;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float ubox = 0.f, qm = 0.f, mag = 0.f;
#pragma unroll
        for (int k = 0; k < DL; ++k) {
          if (lane + 32 * k < D) {
            const float m = fmaxf(qr[j][k] * lo[u][k], qr[j][k] * hi[u][k]);
            ubox += m;
            const float pm = qr[j][k] * mu[u][k];
            qm += pm;
            mag += fabsf(m) + fabsf(pm);
          }
        }
        ubox = warp_sum(ubox);
        qm = warp_sum(qm);
        mag = warp_sum(mag);
        const float ub = fminf(ubox, qm + qn[j] * rad[u]);
        keep |= ub + 1e-3f * (mag + qn[j] * rad[u] + 1.f) >= thr[j];
      }
      if (t < ntiles && lane == 0 && keep) {
        atomicOr(&s_mask, 1ull << t);
        atomicAdd(&s_kept, 1);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ws.keep[c] = s_mask;
    atomicAdd(&ws.counters[2], s_kept);
    atomicAdd(&ws.counters[3], ntiles);
  }
}

// Build the block index of a slab: one CTA of 128 threads per (head, block).
template <typename T>
__global__ void __launch_bounds__(128) block_bounds_kernel(const T* __restrict__ k, int64_t hs, int n,
                                                           int D, T* __restrict__ bounds, int64_t bhs) {
  __shared__ float mu_s[256];
  __shared__ float wbest[4], wrad[4];
  __shared__ int wrow[4];
  const int nblk = (n + 127) / 128;
  const int h = blockIdx.x / nblk, blk = blockIdx.x - h * nblk;
  const int r0 = blk * 128, r1 = min(n, r0 + 128);
  const T* kh = k + (size_t)h * hs;
  T* out = bounds + (size_t)h * bhs + (size_t)blk * kBndRows * D;
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    float lo = INFINITY, hi = -INFINITY, sum = 0.f;
    for (int r = r0; r < r1; ++r) {
      const float x = to_f(kh[(size_t)r * D + e]);
      lo = fminf(lo, x);
      hi = fmaxf(hi, x);
      sum += x;
    }
    T mu;
    if constexpr (std::is_same_v<T, float>) { out[e] = lo; out[D + e] = hi; mu = sum / (r1 - r0); }
    else {
      out[e] = __float2bfloat16_rn(lo);  // exact: the inputs are bf16
      out[D + e] = __float2bfloat16_rn(hi);
      mu = __float2bfloat16_rn(sum / (r1 - r0));
    }
    out[2 * D + e] = mu;
    mu_s[e] = to_f(mu);
  }
  __syncthreads();
  // per row: squared norm (representative) and squared distance to mu (radius)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float best = -1.f, rad2 = 0.f;
  int brow = r0;
  for (int r = r0 + warp; r < r1; r += 4) {
    float nn = 0.f, dd = 0.f;
    for (int e = lane; e < D; e += 32) {
      const float x = to_f(kh[(size_t)r * D + e]);
      nn = fmaf(x, x, nn);
      dd = fmaf(x - mu_s[e], x - mu_s[e], dd);
    }
    nn = warp_sum(nn);
    dd = warp_sum(dd);
    if (nn > best) { best = nn; brow = r; }  // rows ascend per warp: ties keep the first
    rad2 = fmaxf(rad2, dd);
  }
  if (lane == 0) { wbest[warp] = best; wrow[warp] = brow; wrad[warp] = rad2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float bb = -1.f, rr = 0.f;
    int br = r0;
    for (int w = 0; w < 4; ++w) {
      if (wbest[w] > bb || (wbest[w] == bb && wrow[w] < br)) { bb = wbest[w]; br = wrow[w]; }
      rr = fmaxf(rr, wrad[w]);
    }
    wrow[0] = br;
    wrad[0] = sqrtf(rr) * (1.f + 1e-5f) + 1e-6f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    out[3 * D + e] = kh[(size_t)wrow[0] * D + e];
    if constexpr (std::is_same_v<T, float>) out[4 * D + e] = e == 0 ? wrad[0] : 0.f;
    else out[4 * D + e] = e == 0 ? __float2bfloat16_ru(wrad[0]) : __float2bfloat16_rn(0.f);  // round up: sound
  }
}

}  // namespace alaya
