// C-ABI entry points (include/alaya.h): validation, workspace layout, kernel
// dispatch over (dtype, dim, group size) and launch.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "alaya_dispatch.cuh"
#include "alaya_misc_kernels.cuh"

using namespace alaya;

namespace alaya {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ALAYA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return ALAYA_OK;
}
}  // namespace alaya

namespace {

constexpr int kNumSMs = 148;
unsigned long long* g_trace = nullptr;  // alaya_debug_trace

bool dim_ok(int d) { return d == 16 || d == 32 || d == 64 || d == 128 || d == 256; }

int chunks_for(const alaya_seq* seqs, int B, int Hkv, int chunk) {
  long total = 0;
  for (int b = 0; b < B; ++b) total += (long)Hkv * ((seqs[b].n + chunk - 1) / chunk);
  return (int)total;
}

// Validate the call and build the kernel-side batch descriptor.
int build_batch(const alaya_params* p, const alaya_seq* seqs, int B, Batch* bt) {
  if (!p || !seqs) return fail(ALAYA_ERR_ARG, "null params/seqs");
  if (B < 1 || B > ALAYA_MAX_BATCH)
    return fail(ALAYA_ERR_ARG, "batch %d out of range [1, %d]", B, ALAYA_MAX_BATCH);
  if (p->n_query_heads < 1 || p->n_kv_heads < 1)
    return fail(ALAYA_ERR_ARG, "all head counts must be positive");
  if (p->n_query_heads % p->n_kv_heads)
    return fail(ALAYA_ERR_ARG, "n_query_heads (%d) must be a multiple of n_kv_heads (%d)",
                p->n_query_heads, p->n_kv_heads);
  const int G = p->n_query_heads / p->n_kv_heads;
  if (G > 8) return fail(ALAYA_ERR_UNSUPPORTED, "group size %d > 8", G);
  if (!dim_ok(p->dim)) return fail(ALAYA_ERR_UNSUPPORTED, "dim %d not in {16,32,64,128,256}", p->dim);
  if (p->dtype != ALAYA_F32 && p->dtype != ALAYA_BF16) return fail(ALAYA_ERR_ARG, "bad dtype");
  if (!(p->beta >= 0.f)) return fail(ALAYA_ERR_ARG, "beta must be non-negative, got %g", p->beta);
  if (p->win_initial < 0 || p->win_last < 0)
    return fail(ALAYA_ERR_ARG, "window sizes must be non-negative");
  long tokens = 0;
  int maxn = 0;
  for (int b = 0; b < B; ++b) {
    const alaya_seq& s = seqs[b];
    if (s.n < 0 || s.w < 0) return fail(ALAYA_ERR_SHAPE, "seq %d: negative row count", b);
    if (s.n > 0 && (!s.k || !s.v)) return fail(ALAYA_ERR_ARG, "seq %d: null base K/V", b);
    if (s.w > 0 && (!s.wk || !s.wv)) return fail(ALAYA_ERR_ARG, "seq %d: null window K/V", b);
    if (s.token_offset < 0 || s.prefix_len < s.token_offset + s.n)
      return fail(ALAYA_ERR_SHAPE, "seq %d: shard [%lld, +%d) outside prefix %lld", b,
                  (long long)s.token_offset, s.n, (long long)s.prefix_len);
    if (s.n > 0 && s.head_stride < (int64_t)s.n * p->dim)
      return fail(ALAYA_ERR_SHAPE, "seq %d: head_stride too small", b);
    if (s.w > 0 && s.w_head_stride < (int64_t)s.w * p->dim)
      return fail(ALAYA_ERR_SHAPE, "seq %d: w_head_stride too small", b);
    if (p->block_filter && s.n > 0 &&
        (!s.bounds || s.bounds_head_stride < (int64_t)((s.n + 127) / 128) * 5 * p->dim))
      return fail(ALAYA_ERR_ARG, "seq %d: block_filter needs bounds (alaya_block_bounds)", b);
    tokens += s.n;
    if (s.n > maxn) maxn = s.n;
  }
  int chunk = p->chunk;
  if (chunk > 0) {
    if (chunk % 256 || chunk > 8192) return fail(ALAYA_ERR_ARG, "chunk must be a multiple of 256, <= 8192");
  } else {
    // the tcgen05 scan splits a chunk into 4 lane-quarter sub-lists of 128-key tiles
    const int min_chunk =
        (p->dtype == ALAYA_BF16 && p->dim == 128 && p->scan_kind != ALAYA_SCAN_CUDA_CORE) ? 512 : 256;
    chunk = 2048;
    while (chunk > min_chunk && chunks_for(seqs, B, p->n_kv_heads, chunk) < 4 * kNumSMs) chunk >>= 1;
  }
  if (G * chunk * 4 > 160 * 1024) chunk = ((160 * 1024 / 4 / G) / 256) * 256;
  (void)tokens;
  (void)maxn;

  memset(bt, 0, sizeof(Batch));
  bt->B = B;
  bt->Hq = p->n_query_heads;
  bt->Hkv = p->n_kv_heads;
  bt->G = G;
  bt->D = p->dim;
  bt->chunk = chunk;
  bt->beta = p->beta;
  bt->wi = p->win_initial;
  bt->wl = p->win_last;
  bt->inv_sqrt_d = (float)(1.0 / std::sqrt((double)p->dim));
  bt->block_filter = p->block_filter ? 1 : 0;
  {  // attend task split threshold; ALAYA_SPLIT overrides (diagnostics)
    static const int split_env = [] {
      const char* e = getenv("ALAYA_SPLIT");
      return (e && *e) ? atoi(e) : -1;
    }();
    static const int seed_env = [] {  // diagnostics: 0 = no running-max seed
      const char* sd = getenv("ALAYA_SEED");
      return (sd && *sd) ? atoi(sd) : 1;
    }();
    bt->split = split_env >= 0 ? split_env : std::max(256, chunk / 4);
    bt->seed = seed_env;
  }
  int cb = 0;
  for (int b = 0; b < B; ++b) {
    const alaya_seq& s = seqs[b];
    KSeq& k = bt->s[b];
    k.k = s.k; k.v = s.v; k.wk = s.wk; k.wv = s.wv;
    k.hs = s.head_stride; k.whs = s.w_head_stride;
    k.off = s.token_offset; k.P = s.prefix_len;
    k.n = s.n; k.w = s.w; k.dw = s.d_w;
    k.nch = (s.n + chunk - 1) / chunk;
    k.bnd = s.bounds;
    k.bhs = s.bounds_head_stride;
    k.chunk_base = cb;
    cb += p->n_kv_heads * k.nch;
  }
  bt->total_chunks = cb;
  bt->trace = g_trace;
  return ALAYA_OK;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t zero_bytes;
  size_t cscore_end;
  size_t status, seeded, prepdone, gmax, counters, cnt, selcnt, retcnt, part_l, part_acc, cidx, cscore, partbuf, smaxbuf,
      keep, ovl_l, ovl_acc, ovl_sel, ovl_ret, heavy, ovlist, gidx, total;
};

Layout layout_for(const Batch& bt) {
  Layout L;
  const size_t C = (size_t)bt.total_chunks, G = bt.G, D = bt.D, rows = (size_t)bt.B * bt.Hq;
  size_t o = 0;
  L.status = o; o = align_up(o + 16);  // status, ready
  L.seeded = o; o = align_up(o + 8 * (size_t)bt.B * bt.Hkv);
  L.prepdone = o; o = align_up(o + 8 * (size_t)bt.B * bt.Hkv);
  L.gmax = o; L.counters = o + 4 * rows;
  L.zero_bytes = 4 * rows + 64 + 4 * (size_t)bt.B * bt.Hkv;  // gmax, counters, group_done (prep_kernel)
  o = align_up(o + L.zero_bytes);
  L.cnt = o; o = align_up(o + 4 * C * G * 4);
  L.selcnt = o; o = align_up(o + 4 * C * G);
  L.retcnt = o; o = align_up(o + 4 * C * G);
  L.part_l = o; o = align_up(o + 4 * C * G);
  L.part_acc = o; o = align_up(o + 4 * C * G * D);
  L.ovl_l = o; o = align_up(o + 4 * C * G * 4);
  L.ovl_acc = o; o = align_up(o + 4 * C * G * 4 * D);
  L.ovl_sel = o; o = align_up(o + 4 * C * G * 4);
  L.ovl_ret = o; o = align_up(o + 4 * C * G * 4);
  L.heavy = o; o = align_up(o + 4 * C * G);
  L.ovlist = o; o = align_up(o + 4 * C * G * 3);
  L.cidx = o; o = align_up(o + 4 * C * G * bt.chunk);
  L.cscore = o; o = align_up(o + 4 * C * G * bt.chunk);
  L.cscore_end = o;
  L.partbuf = o; o = align_up(o + 4 * rows * (D + 2));
  L.smaxbuf = o; o = align_up(o + 4 * rows);
  L.keep = o; o = align_up(o + 8 * C);
  L.gidx = o; o = align_up(o + 4 * C * bt.chunk);
  L.total = o;
  return L;
}

Ws carve(const Layout& L, void* base) {
  char* c = static_cast<char*>(base);
  Ws w;
  w.status = reinterpret_cast<int*>(c + L.status);
  w.mode = w.status + 1;
  w.gidx = reinterpret_cast<int*>(c + L.gidx);
  w.ready = reinterpret_cast<unsigned long long*>(c + L.status + 8);
  w.seeded = reinterpret_cast<unsigned long long*>(c + L.seeded);
  w.prepdone = reinterpret_cast<unsigned long long*>(c + L.prepdone);
  w.gmax = reinterpret_cast<uint32_t*>(c + L.gmax);
  w.counters = reinterpret_cast<int*>(c + L.counters);
  w.group_done = w.counters + 16;
  w.cnt = reinterpret_cast<int*>(c + L.cnt);
  w.selcnt = reinterpret_cast<int*>(c + L.selcnt);
  w.retcnt = reinterpret_cast<int*>(c + L.retcnt);
  w.part_l = reinterpret_cast<float*>(c + L.part_l);
  w.part_acc = reinterpret_cast<float*>(c + L.part_acc);
  w.cidx = reinterpret_cast<int*>(c + L.cidx);
  w.cscore = reinterpret_cast<float*>(c + L.cscore);
  w.partbuf = reinterpret_cast<float*>(c + L.partbuf);
  w.smaxbuf = reinterpret_cast<float*>(c + L.smaxbuf);
  w.keep = reinterpret_cast<unsigned long long*>(c + L.keep);
  w.ovl_l = reinterpret_cast<float*>(c + L.ovl_l);
  w.ovl_acc = reinterpret_cast<float*>(c + L.ovl_acc);
  w.ovl_sel = reinterpret_cast<int*>(c + L.ovl_sel);
  w.ovl_ret = reinterpret_cast<int*>(c + L.ovl_ret);
  w.heavy = reinterpret_cast<int*>(c + L.heavy);
  w.ovlist = reinterpret_cast<int*>(c + L.ovlist);
  return w;
}

StageSet pick(int dtype, int D, int G) {
  const bool bf = dtype == ALAYA_BF16;
  switch (D) {
    case 16: return bf ? pick_bf16_16(G) : pick_f32_16(G);
    case 32: return bf ? pick_bf16_32(G) : pick_f32_32(G);
    case 64: return bf ? pick_bf16_64(G) : pick_f32_64(G);
    case 128: return bf ? pick_bf16_128(G) : pick_f32_128(G);
    default: return bf ? pick_bf16_256(G) : pick_f32_256(G);
  }
}

struct Call {
  Batch bt;
  const alaya_seq* seqs;
  bool use_tc;
  Layout L;
  Ws ws;
  StageSet st;
  cudaStream_t stream;
  const unsigned long long* call_seq;  // params->d_call_seq
};

int prepare(const alaya_params* p, const alaya_seq* seqs, int B, void* d_ws, size_t ws_bytes,
            void* stream, Call* c) {
  int rc = build_batch(p, seqs, B, &c->bt);
  if (rc) return rc;
  c->L = layout_for(c->bt);
  if (!d_ws) return fail(ALAYA_ERR_WORKSPACE, "null workspace");
  if (ws_bytes < c->L.total)
    return fail(ALAYA_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, c->L.total);
  c->ws = carve(c->L, d_ws);
  c->st = pick(p->dtype, p->dim, c->bt.G);
  c->seqs = seqs;
  const bool eligible = tc_scan_eligible(c->bt, p->dtype, seqs);
  if (p->scan_kind == ALAYA_SCAN_TCGEN05 && !eligible)
    return fail(ALAYA_ERR_UNSUPPORTED, "tcgen05 scan needs bf16 K, dim 128, group <= 8, "
                "16-byte aligned slabs with a head stride multiple of 128");
  c->use_tc = eligible && p->scan_kind != ALAYA_SCAN_CUDA_CORE;
  c->stream = static_cast<cudaStream_t>(stream);
  c->call_seq = p->d_call_seq;
  return ALAYA_OK;
}

int run_scan(Call& c, const float* d_q, bool ends_in_combine = true) {
  // the tcgen05 scan starts on prep's zeroed header (ws.ready) instead of prep's
  // completion; the seeds land by atomicMax while it runs (ALAYA_PREP_ASYNC=0: off)
  static const int async_prep = [] {
    const char* v = getenv("ALAYA_PREP_ASYNC");
    return v && *v ? atoi(v) : 1;
  }();
  static std::atomic<unsigned long long> next_id{1};
  // (the call's combine_kernel waits for prep's last seed, so none lands in a later call)
  // (not inside a CUDA-graph capture: every replay would reuse the captured id)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(c.stream, &cap) != cudaSuccess) cap = cudaStreamCaptureStatusActive;
  const bool eligible = async_prep && ends_in_combine && c.use_tc && !c.bt.block_filter && !c.bt.topk_thr;
  c.bt.call_seq = nullptr;
  if (cap == cudaStreamCaptureStatusNone) {
    c.bt.call_id = eligible ? next_id++ : 0ull;
  } else if (eligible && c.call_seq) {  // graph: slot id (bit 63 + 20 bits) + the replay number
    static std::atomic<unsigned long long> next_slot{0};
    c.bt.call_id = (1ull << 63) | (next_slot++ & 0xFFFFFull);
    c.bt.call_seq = c.call_seq;
  } else {
    c.bt.call_id = 0ull;
  }
  int rc = c.st.prep(c.bt, d_q, c.ws, c.stream);  // zeroes the header, seeds the max
  if (rc) return rc;
  if (c.bt.block_filter) {
    const int rc = c.st.filter(c.bt, d_q, c.ws, c.stream);
    if (rc) return rc;
  }
  if (c.use_tc) return launch_tc_scan(c.bt, c.seqs, d_q, c.ws, c.stream);
  return c.st.scan(c.bt, d_q, c.ws, c.stream);
}

}  // namespace

extern "C" {

const char* alaya_last_error(void) { return g_err.c_str(); }

int alaya_debug_trace(void* d_buf, int64_t bytes) {
  if (d_buf && bytes < (int64_t)4 * kTraceCtas * kTraceSlots * 8)
    return fail(ALAYA_ERR_WORKSPACE, "trace buffer needs %d bytes", 4 * kTraceCtas * kTraceSlots * 8);
  g_trace = static_cast<unsigned long long*>(d_buf);
  return ALAYA_OK;
}
int alaya_version(void) { return 1; }

size_t alaya_workspace_bytes(const alaya_params* p, const alaya_seq* seqs, int batch) {
  Batch* bt = new Batch;
  size_t r = 0;
  if (build_batch(p, seqs, batch, bt) == ALAYA_OK) r = layout_for(*bt).total;
  delete bt;
  return r;
}

int* alaya_ws_status(void* d_ws) { return static_cast<int*>(d_ws); }

int alaya_block_bounds(const void* d_k, int dtype, int n_heads, int64_t head_stride, int n, int dim,
                       void* d_bounds, int64_t bounds_head_stride, void* stream) {
  if (!d_k || !d_bounds || n_heads < 1 || n < 0 || !dim_ok(dim))
    return fail(ALAYA_ERR_ARG, "bad block bounds arguments");
  if (head_stride < (int64_t)n * dim || bounds_head_stride < (int64_t)((n + 127) / 128) * 5 * dim)
    return fail(ALAYA_ERR_SHAPE, "block bounds: strides too small");
  if (n == 0) return ALAYA_OK;
  const int blocks = n_heads * ((n + 127) / 128);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == ALAYA_BF16)
    block_bounds_kernel<__nv_bfloat16><<<blocks, 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(d_k), head_stride, n, dim, static_cast<__nv_bfloat16*>(d_bounds),
        bounds_head_stride);
  else if (dtype == ALAYA_F32)
    block_bounds_kernel<float><<<blocks, 128, 0, st>>>(
        static_cast<const float*>(d_k), head_stride, n, dim, static_cast<float*>(d_bounds), bounds_head_stride);
  else
    return fail(ALAYA_ERR_ARG, "bad dtype");
  return cuda_check("block_bounds_kernel");
}

int* alaya_ws_candidate_counts(const alaya_params* p, const alaya_seq* seqs, int batch, void* d_ws) {
  static thread_local Batch bt;
  if (build_batch(p, seqs, batch, &bt) != ALAYA_OK) return nullptr;
  return reinterpret_cast<int*>(static_cast<char*>(d_ws) + layout_for(bt).cnt);
}

int* alaya_ws_block_stats(const alaya_params* p, const alaya_seq* seqs, int batch, void* d_ws) {
  static thread_local Batch bt;
  if (build_batch(p, seqs, batch, &bt) != ALAYA_OK) return nullptr;
  const Layout L = layout_for(bt);
  return reinterpret_cast<int*>(static_cast<char*>(d_ws) + L.counters) + 2;
}

int alaya_window_append(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_k,
                        const float* d_v, void* stream) {
  static thread_local Batch bt;
  int rc = build_batch(p, seqs, batch, &bt);
  if (rc) return rc;
  if (!d_k || !d_v) return fail(ALAYA_ERR_ARG, "null k/v");
  bool dev_w = false;
  for (int b = 0; b < batch; ++b) {
    if (!seqs[b].wk || !seqs[b].wv) return fail(ALAYA_ERR_ARG, "seq %d: null window buffers", b);
    // host count: row w must fit; device count (d_w): w is the capacity, checked in the kernel
    const int64_t rows = seqs[b].d_w ? seqs[b].w : (int64_t)seqs[b].w + 1;
    if (seqs[b].w_head_stride < rows * p->dim)
      return fail(ALAYA_ERR_SHAPE, "seq %d: window row %d beyond capacity", b, seqs[b].w);
    dev_w = dev_w || seqs[b].d_w;
  }
  const long total = (long)batch * p->n_kv_heads * p->dim;
  const int blocks = (int)std::min<long>((total + 255) / 256, 1024);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = p->dtype == ALAYA_BF16
           ? launch_pdl("window_append_kernel", window_append_kernel<__nv_bfloat16>, blocks, 256, 0, st, bt,
                        d_k, d_v)
           : launch_pdl("window_append_kernel", window_append_kernel<float>, blocks, 256, 0, st, bt, d_k, d_v);
  if (rc || !dev_w) return rc;
  return launch_pdl("window_commit_kernel", window_commit_kernel, 1, 128, 0, st, bt);  // ++*d_w
}

namespace {
int dipr_attention_impl(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_k_new,
                        const float* d_v_new, const float* d_q, float* d_out, void* d_ws, size_t ws_bytes,
                        void* stream);
}

int alaya_dipr_attention(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q,
                         float* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  return dipr_attention_impl(p, seqs, batch, nullptr, nullptr, d_q, d_out, d_ws, ws_bytes, stream);
}

int alaya_dipr_attention_update(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_k_new,
                                const float* d_v_new, const float* d_q, float* d_out, void* d_ws,
                                size_t ws_bytes, void* stream) {
  if (!d_k_new || !d_v_new) return fail(ALAYA_ERR_ARG, "null k/v");
  return dipr_attention_impl(p, seqs, batch, d_k_new, d_v_new, d_q, d_out, d_ws, ws_bytes, stream);
}

}  // extern "C"

namespace {
int dipr_attention_impl(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_k_new,
                        const float* d_v_new, const float* d_q, float* d_out, void* d_ws, size_t ws_bytes,
                        void* stream) {
  Call c;
  int rc = prepare(p, seqs, batch, d_ws, ws_bytes, stream, &c);
  if (rc) return rc;
  if (!d_q || !d_out) return fail(ALAYA_ERR_ARG, "null q/out");
  if (d_k_new) {
    for (int b = 0; b < batch; ++b) {
      if (seqs[b].d_w) return fail(ALAYA_ERR_UNSUPPORTED, "seq %d: update+attention needs host window counts", b);
      if (seqs[b].w < 1 || !seqs[b].wk || !seqs[b].wv)
        return fail(ALAYA_ERR_ARG, "seq %d: update+attention needs a window ring with the new row counted", b);
    }
    c.bt.app_k = d_k_new;
    c.bt.app_v = d_v_new;
  }
  for (int b = 0; b < batch; ++b)
    if (seqs[b].prefix_len + seqs[b].w == 0) return fail(ALAYA_ERR_ARG, "attention on an empty session");
  c.bt.win_in_prep = 1;  // window partials computed by prep, off the attend's tail
  // attend beside the scan (per-group readiness); the CUDA-core scan fills the
  // register file (no room for an attend CTA: measured no gain), so tcgen05 only
  if (c.use_tc && overlap_enabled()) {
    c.bt.overlap = 1;
    c.bt.gfmt = gfmt_enabled(c.bt);
    if ((rc = run_scan(c, d_q))) return rc;
    if (c.bt.gfmt && dense_attend_enabled(c.bt, c.seqs))
      rc = launch_tc_attend_dense(c.bt, c.seqs, c.ws, c.stream);
    else
      rc = c.bt.gfmt ? c.st.attend_grp(c.bt, d_q, c.ws, c.stream) : c.st.attend_ovl(c.bt, d_q, c.ws, c.stream);
    if (rc) return rc;
    return c.st.combine(c.bt, nullptr, c.ws, d_out, nullptr, c.ws.smaxbuf, c.stream);
  }
  if (!c.use_tc && cc_overlap_enabled()) {  // CUDA-core scan: persistent, attend beside it
    c.bt.overlap = 1;
    c.bt.persist = 1;
    if ((rc = run_scan(c, d_q))) return rc;
    if ((rc = c.st.attend_ovl(c.bt, d_q, c.ws, c.stream))) return rc;
    return c.st.combine(c.bt, nullptr, c.ws, d_out, nullptr, c.ws.smaxbuf, c.stream);
  }
  if ((rc = run_scan(c, d_q))) return rc;  // prep zeroed the status word and the ticket
  if ((rc = c.st.attend(c.bt, d_q, nullptr, c.ws, 1, c.stream, 0))) return rc;
  return c.st.combine(c.bt, nullptr, c.ws, d_out, nullptr, c.ws.smaxbuf, c.stream);
}
}  // namespace

extern "C" {

int alaya_sharded_step(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q,
                       void* const* bufs, int n_ranks, int rank, int64_t cap_floats, unsigned long long epoch,
                       unsigned long long gather_epoch, float* d_part, int* d_err, void* d_ws,
                       size_t ws_bytes, void* stream) {
  Call c;
  int rc = prepare(p, seqs, batch, d_ws, ws_bytes, stream, &c);
  if (rc) return rc;
  if (!d_q || !bufs || (!d_part && !gather_epoch)) return fail(ALAYA_ERR_ARG, "null q/part/bufs");
  if (gather_epoch && (int64_t)c.bt.B * c.bt.Hq * (p->dim + 2) > cap_floats)
    return fail(ALAYA_ERR_SHAPE, "fused sharded step: partials beyond the exchange slot");
  if (n_ranks < 1 || n_ranks > kExMaxPeers || rank < 0 || rank >= n_ranks)
    return fail(ALAYA_ERR_ARG, "bad ranks %d/%d", rank, n_ranks);
  if (!c.use_tc) return fail(ALAYA_ERR_UNSUPPORTED, "fused sharded step needs the tcgen05 scan");
  if ((int64_t)c.bt.B * c.bt.Hq > cap_floats || c.bt.B * c.bt.Hkv > kExGroups)
    return fail(ALAYA_ERR_SHAPE, "fused sharded step: %d rows / %d groups beyond the exchange buffer",
                c.bt.B * c.bt.Hq, c.bt.B * c.bt.Hkv);
  for (int r = 0; r < n_ranks; ++r)
    if (!bufs[r]) return fail(ALAYA_ERR_ARG, "null peer buffer %d", r);
  c.bt.overlap = 1;
  c.bt.sx_on = 1;
  c.bt.win_in_prep = 1;
  c.bt.gfmt = gfmt_enabled(c.bt);
  for (int r = 0; r < n_ranks; ++r) c.bt.sx.peers[r] = static_cast<char*>(bufs[r]);
  c.bt.sx.rank = rank;
  c.bt.sx.R = n_ranks;
  c.bt.sx.cap = cap_floats;
  c.bt.sx.epoch = epoch;
  c.bt.sx.gepoch = gather_epoch;
  c.bt.sx.err = d_err;
  if ((rc = run_scan(c, d_q))) return rc;
  if ((rc = c.bt.gfmt ? c.st.attend_grp(c.bt, d_q, c.ws, c.stream) : c.st.attend_ovl(c.bt, d_q, c.ws, c.stream)))
    return rc;
  return c.st.combine(c.bt, c.ws.smaxbuf, c.ws, nullptr, d_part, nullptr, c.stream);
}

int alaya_scan(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q,
               float* d_smax, void* d_ws, size_t ws_bytes, void* stream) {
  Call c;
  int rc = prepare(p, seqs, batch, d_ws, ws_bytes, stream, &c);
  if (rc) return rc;
  if (!d_q) return fail(ALAYA_ERR_ARG, "null q");
  if ((rc = run_scan(c, d_q, d_smax != nullptr))) return rc;
  if (!d_smax) return ALAYA_OK;  // scan only (kernel timing)
  // export the local max (decoded); combine with no outputs does only that
  return c.st.combine(c.bt, nullptr, c.ws, nullptr, nullptr, d_smax, c.stream);
}

int alaya_attend(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q,
                 const float* d_smax, float* d_part, int want_values, void* d_ws, size_t ws_bytes,
                 void* stream) {
  Call c;
  int rc = prepare(p, seqs, batch, d_ws, ws_bytes, stream, &c);
  if (rc) return rc;
  if (!d_q || !d_smax) return fail(ALAYA_ERR_ARG, "null q/smax");
  if ((rc = c.st.attend(c.bt, d_q, d_smax, c.ws, want_values ? 1 : 0, c.stream, 1))) return rc;
  if (!want_values || !d_part) return ALAYA_OK;
  return c.st.combine(c.bt, d_smax, c.ws, nullptr, d_part, nullptr, c.stream);
}

int alaya_merge_partials(const float* d_parts, int n_parts, int rows, int dim, float* d_out,
                         int* d_status, void* stream) {
  if (!d_parts || !d_out || n_parts < 1 || rows < 0 || !dim_ok(dim))
    return fail(ALAYA_ERR_ARG, "bad merge arguments");
  if (rows == 0) return ALAYA_OK;
  merge_partials_kernel<<<rows, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      d_parts, n_parts, rows, dim, d_out, nullptr, d_status);
  return cuda_check("merge_partials_kernel");
}

int alaya_merge_exchanged(void* d_own_buf, int n_ranks, int64_t cap_floats, unsigned long long epoch, int rows,
                          int dim, float* d_out, int* d_status, int* d_err, void* stream) {
  if (!d_own_buf || !d_out || n_ranks < 1 || n_ranks > kExMaxPeers || rows < 0 || !dim_ok(dim) || epoch == 0)
    return fail(ALAYA_ERR_ARG, "bad merge arguments");
  if ((int64_t)rows * (dim + 2) > cap_floats) return fail(ALAYA_ERR_SHAPE, "partials beyond the exchange slot");
  if (rows == 0) return ALAYA_OK;
  char* buf = static_cast<char*>(d_own_buf);
  const float* parts = reinterpret_cast<const float*>(buf + kExFlagBytes + (size_t)kExGroups * kExMaxPeers * 8) +
                       ((size_t)(epoch & 1ull) * 2 + 1) * n_ranks * (size_t)cap_floats;
  const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(buf) + kExMaxPeers;  // kind 1
  merge_partials_kernel<<<rows, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      parts, n_ranks, rows, dim, d_out, nullptr, d_status, flags, epoch, d_err, cap_floats);
  return cuda_check("merge_partials_kernel");
}

int alaya_merge_states(const float* d_parts, int n_parts, int rows, int dim, float* d_state,
                       void* stream) {
  if (!d_parts || !d_state || n_parts < 1 || rows < 0 || !dim_ok(dim))
    return fail(ALAYA_ERR_ARG, "bad merge arguments");
  if (rows == 0) return ALAYA_OK;
  merge_partials_kernel<<<rows, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      d_parts, n_parts, rows, dim, nullptr, d_state, nullptr);
  return cuda_check("merge_partials_kernel");
}

int alaya_selected(const alaya_params* p, const alaya_seq* seqs, int batch, int64_t* d_ids,
                   int64_t cap, int32_t* d_selected, int32_t* d_retrieved, void* d_ws,
                   size_t ws_bytes, void* stream) {
  Call c;
  int rc = prepare(p, seqs, batch, d_ws, ws_bytes, stream, &c);
  if (rc) return rc;
  if (!d_ids || !d_selected || !d_retrieved) return fail(ALAYA_ERR_ARG, "null outputs");
  int max_nch = 0;
  for (int b = 0; b < batch; ++b) max_nch = std::max(max_nch, c.bt.s[b].nch);
  const size_t sm = 4 * ((size_t)max_nch + 1);  // chunk offsets
  if (sm > 48 * 1024) {
    static size_t attr = 0;
    if (sm > attr) {
      cudaFuncSetAttribute(selected_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr = sm;
    }
  }
  const dim3 grid(batch * c.bt.Hq, std::max(1, (max_nch + kWarps - 1) / kWarps));  // a warp per chunk
  // PDL: launched while the call's combine finishes; waits for it before reading
  return launch_pdl("selected_kernel", selected_kernel, grid, dim3(kThreads), sm, c.stream, c.bt, c.ws, d_ids,
                    cap, d_selected, d_retrieved);  // (format: ws.mode)
}

int alaya_topk(const alaya_params* p, const alaya_seq* seqs, int batch, const float* d_q, int k,
               int64_t* d_ids, float* d_scores, int64_t cap, int32_t* d_count, void* d_ws,
               size_t ws_bytes, void* stream) {
  if (!p) return fail(ALAYA_ERR_ARG, "null params");
  alaya_params pp = *p;  // every base token is a candidate: the scan with beta = inf
  pp.beta = INFINITY;
  pp.block_filter = 0;
  Call c;
  int rc = prepare(&pp, seqs, batch, d_ws, ws_bytes, stream, &c);
  if (rc) return rc;
  if (!d_q || !d_ids || !d_count) return fail(ALAYA_ERR_ARG, "null q/ids/count");
  if (k < 1) return fail(ALAYA_ERR_ARG, "k must be >= 1, got %d", k);
  if (cap < k) return fail(ALAYA_ERR_ARG, "cap %lld < k %d", (long long)cap, k);
  for (int b = 0; b < batch; ++b)
    if (seqs[b].token_offset != 0 || seqs[b].prefix_len != seqs[b].n)
      return fail(ALAYA_ERR_UNSUPPORTED, "top-k runs on unsharded sequences");
  // prep (header only: the DIPR seed is unused at beta = inf, the bound below replaces
  // it); the per-row candidate bound from sampled keys (scratch: the candidate score
  // buffer, consumed before the scan writes it); the scan keeps s >= bound
  c.bt.seed = 0;
  if ((rc = c.st.prep(c.bt, d_q, c.ws, c.stream))) return rc;
  const size_t scratch = (size_t)(c.L.cscore_end - c.L.cscore) / 4;
  if ((rc = launch_topk_bound(c.bt, p->dtype, d_q, c.ws.cscore, scratch, k, c.ws.smaxbuf, c.stream))) return rc;
  c.bt.topk_thr = c.ws.smaxbuf;
  if (c.use_tc) rc = launch_tc_scan(c.bt, c.seqs, d_q, c.ws, c.stream);
  else rc = c.st.scan(c.bt, d_q, c.ws, c.stream);
  if (rc) return rc;
  return launch_topk_select(c.bt, c.ws, k, d_ids, d_scores, cap, d_count, c.stream);
}

int alaya_block_reps(const void* d_k, int dtype, int n_heads, int64_t head_stride, int n, int dim,
                     int block_size, int r, void* d_reps, int64_t reps_head_stride, void* stream) {
  if (!d_k || !d_reps || n_heads < 1 || n < 0 || !dim_ok(dim) || block_size < 1 || r < 1)
    return fail(ALAYA_ERR_ARG, "bad block reps arguments");
  if (dtype != ALAYA_F32 && dtype != ALAYA_BF16) return fail(ALAYA_ERR_ARG, "bad dtype");
  if (block_size > 16384) return fail(ALAYA_ERR_UNSUPPORTED, "block_size %d > 16384", block_size);
  const int64_t nb = (n + block_size - 1) / block_size;
  if (head_stride < (int64_t)n * dim || reps_head_stride < nb * r * dim)
    return fail(ALAYA_ERR_SHAPE, "block reps: strides too small");
  if (n == 0) return ALAYA_OK;
  return launch_block_reps(d_k, dtype, n_heads, head_stride, n, dim, block_size, r, d_reps,
                           reps_head_stride, static_cast<cudaStream_t>(stream));
}

int alaya_block_topk(const alaya_params* p, const alaya_seq* seqs, const alaya_block_index* bix,
                     int batch, int block_size, int k_blocks, const float* d_q, int64_t* d_ids,
                     int64_t cap, int32_t* d_count, int32_t* d_blocks, float* d_block_scores,
                     void* stream) {
  static thread_local Batch bt;
  int rc = build_batch(p, seqs, batch, &bt);
  if (rc) return rc;
  if (!bix || !d_q || !d_ids || !d_count) return fail(ALAYA_ERR_ARG, "null block index/q/ids/count");
  if (block_size < 1 || k_blocks < 1) return fail(ALAYA_ERR_ARG, "block_size and k_blocks must be >= 1");
  static thread_local BixSet set;
  int max_nb = 1;
  for (int b = 0; b < batch; ++b) {
    const alaya_block_index& x = bix[b];
    if (x.n_blocks != (x.n_tokens + block_size - 1) / block_size || x.r < 1 ||
        (x.n_blocks > 0 && !x.reps) || x.head_stride < (int64_t)x.n_blocks * x.r * p->dim)
      return fail(ALAYA_ERR_SHAPE, "seq %d: block index does not match block_size %d", b, block_size);
    set.b[b] = x;
    max_nb = std::max(max_nb, x.n_blocks);
  }
  if (cap < (int64_t)k_blocks * block_size && cap < max_nb * (int64_t)block_size)
    return fail(ALAYA_ERR_ARG, "cap %lld < k_blocks * block_size", (long long)cap);
  return launch_block_topk(bt, p->dtype, d_q, set, max_nb, block_size, k_blocks, d_ids, cap, d_count,
                           d_blocks, d_block_scores, static_cast<cudaStream_t>(stream));
}

size_t alaya_diprs_workspace_bytes(const alaya_params* p, const alaya_seq* seqs,
                                   const alaya_graph* graphs, int batch) {
  static thread_local Batch bt;
  if (!graphs || build_batch(p, seqs, batch, &bt) != ALAYA_OK) return 0;
  int max_n = 1;
  for (int b = 0; b < batch; ++b) max_n = std::max(max_n, graphs[b].n_nodes);
  return (size_t)diprs_row_bytes(max_n, kDiprsCap) * batch * p->n_query_heads;
}

int alaya_diprs(const alaya_params* p, const alaya_seq* seqs, const alaya_graph* graphs, int batch,
                const float* d_q, int l0, int floor_mode, const float* d_floors, int64_t* d_ids,
                int64_t cap, int32_t* d_count, int32_t* d_explored, void* d_ws, size_t ws_bytes,
                void* stream) {
  static thread_local Batch bt;
  int rc = build_batch(p, seqs, batch, &bt);
  if (rc) return rc;
  if (!graphs || !d_q || !d_ids || !d_count || !d_ws) return fail(ALAYA_ERR_ARG, "null graphs/q/ids/count/ws");
  if (l0 < 1) return fail(ALAYA_ERR_ARG, "capacity threshold must be >= 1, got %d", l0);
  if (floor_mode < 0 || floor_mode > 2 || (floor_mode == 2 && !d_floors))
    return fail(ALAYA_ERR_ARG, "bad floor mode");
  for (int b = 0; b < batch; ++b) {
    const alaya_graph& g = graphs[b];
    if (seqs[b].token_offset != 0 || seqs[b].prefix_len != seqs[b].n)
      return fail(ALAYA_ERR_UNSUPPORTED, "graph DIPRS runs on unsharded sequences");
    if (g.n_nodes != seqs[b].n || g.n_nodes < 1)
      return fail(ALAYA_ERR_ARG, "seq %d: graph of %d nodes over a prefix of %d tokens", b, g.n_nodes,
                  seqs[b].n);
    if (!g.offsets || !g.nbrs || !g.entry) return fail(ALAYA_ERR_ARG, "seq %d: null graph arrays", b);
    if (g.offsets_head_stride < (int64_t)g.n_nodes + 1) return fail(ALAYA_ERR_SHAPE, "seq %d: offsets stride", b);
  }
  if (cap < 1) return fail(ALAYA_ERR_ARG, "cap must be >= 1");
  return launch_diprs(bt, p->dtype, graphs, d_q, l0, floor_mode, d_floors, kDiprsCap, d_ids, cap, d_count,
                      d_explored, d_ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int alaya_sparse_attention(const alaya_params* p, const alaya_seq* seqs, int batch,
                           const float* d_q, const int64_t* d_ids, int64_t cap,
                           const int32_t* d_count, float* d_out, int32_t* d_selected,
                           int32_t* d_status, void* stream) {
  static thread_local Batch bt;
  int rc = build_batch(p, seqs, batch, &bt);
  if (rc) return rc;
  if (!d_q || !d_out || !d_count || (cap > 0 && !d_ids)) return fail(ALAYA_ERR_ARG, "null q/ids/count/out");
  if (cap < 0) return fail(ALAYA_ERR_ARG, "negative cap");
  for (int b = 0; b < batch; ++b)
    if (seqs[b].prefix_len + seqs[b].w == 0) return fail(ALAYA_ERR_ARG, "attention on an empty session");
  return launch_sparse_attention(bt, p->dtype, d_q, d_ids, cap, d_count, d_out, d_selected, d_status,
                                 static_cast<cudaStream_t>(stream));
}

}  // extern "C"
