// Shared device helpers and the per-call batch descriptor.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/alaya.h"

namespace alaya {

constexpr int kThreads = 256;  // every kernel: 8 warps = 16 half-warps
constexpr int kWarps = kThreads / 32;
constexpr int kHalfWarps = kThreads / 16;
constexpr unsigned kFull = 0xffffffffu;
constexpr float kLog2e = 1.4426950408889634f;

// One sequence of the batch, as the kernels see it (kernel-parameter space).
struct KSeq {
  const void* k;
  const void* v;
  const void* wk;
  const void* wv;
  int64_t hs;    // head stride of k/v (elements)
  int64_t whs;   // head stride of wk/wv (elements)
  int64_t off;   // global id of local row 0 (sequence-sharded mode)
  int64_t P;     // full base-prefix length (window ids are defined on it)
  int32_t n;     // base rows held here
  int32_t w;     // session-window rows
  int32_t chunk_base;  // first work chunk of this sequence
  int32_t nch;         // chunks per kv head
  const void* bnd;     // block bounds [Hkv][bhs] ([block][2][D]) or null
  int64_t bhs;
  int* dw;             // device window row count (graph mode; w = capacity) or null
};
// session-window rows of a sequence at kernel run time
__device__ __forceinline__ int seq_w(const KSeq& s) { return s.dw ? min(__ldcg(s.dw), s.w) : s.w; }

// Sequence-sharded step with the collectives fused into the kernels (peer
// memory): the tcgen05 scan's CTA that completes a (sequence, kv head) group
// stores the group's local maxima into every rank's exchange buffer and raises
// the group's flag there; attend tasks start once every rank's flag for their
// group is up (alaya_exch.cu has the buffer layout).
constexpr int kExMaxPeers = 16;
constexpr size_t kExFlagBytes = 512;        // kind flags + arrival counter
constexpr int kExGroups = 4096;             // per-group flags [kExGroups][kExMaxPeers] u64
struct ShardExch {
  char* peers[kExMaxPeers];
  int32_t rank, R;
  int64_t cap;                 // floats per slot
  unsigned long long epoch;    // this step's epoch (same on every rank)
  unsigned long long gepoch;   // != 0: combine pushes the partials (allgather, kind 1) at this epoch
  int* err;                    // set to 1 when a rank never arrived (bounded poll)
};
// exchange head: [2 kinds][kExMaxPeers] u64 epoch flags, then the arrival counter (u64 index 32)
__device__ __forceinline__ unsigned long long* exch_flag(char* buf, int kind, int r) {
  return reinterpret_cast<unsigned long long*>(buf) + kind * kExMaxPeers + r;
}
__device__ __forceinline__ unsigned int* exch_arrive(char* buf) {
  return reinterpret_cast<unsigned int*>(reinterpret_cast<unsigned long long*>(buf) + 2 * kExMaxPeers);
}
__device__ __forceinline__ float* exch_slot(char* buf, int parity, int kind, int r, int R, int64_t cap) {
  float* base = reinterpret_cast<float*>(buf + kExFlagBytes + (size_t)kExGroups * kExMaxPeers * 8);
  return base + ((((size_t)parity * 2 + kind) * R + r) * (size_t)cap);
}
__device__ __forceinline__ unsigned long long* exch_gflag(char* buf, int g, int r) {
  return reinterpret_cast<unsigned long long*>(buf + kExFlagBytes) + (size_t)g * kExMaxPeers + r;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct Batch {
  KSeq s[ALAYA_MAX_BATCH];
  int32_t B, Hq, Hkv, G, D, chunk;
  float beta;
  int32_t wi, wl;
  int32_t total_chunks;
  float inv_sqrt_d;
  int32_t dbg;  // diagnostics only (ALAYA_TC_DBG): bit0 no L2 hint, bit1 no epilogue math, bit2 no MMA
  int32_t block_filter;
  int32_t split;  // attend task split threshold (candidates per (chunk, head) pair)
  unsigned long long call_id;  // != 0: prep publishes the zeroed header as ws.ready = call_token and
                               // seeds asynchronously (the tcgen05 scan waits on ready, not on prep)
  const unsigned long long* call_seq;  // graph mode: per-replay sequence number (see call_token)
  int32_t seed;   // prep_kernel seeds the running max from sampled keys
  int32_t overlap;  // scan publishes per-group completion; attend runs beside it (PDL)
  const float* topk_thr;  // TOP_K: per-row candidate threshold (a lower bound of the k-th
                          // score) replacing max - beta in the scan; null for DIPR
  int32_t sx_on;          // fused sharded step (needs overlap): see ShardExch
  ShardExch sx;
  unsigned long long* trace;  // diagnostics (alaya_debug_trace): per-CTA %globaltimer stamps or null
  int32_t win_in_prep;  // prep_kernel computes the window partials (the attend skips window tasks)
  const float* app_k;   // != null: prep first writes row w-1 of every window ring from these
  const float* app_v;   //   ([B][Hkv][D] fp32; alaya_dipr_attention_update)
  int32_t persist;      // CUDA-core scan: persistent grid, chunks in order from counters[9]
  int32_t gfmt;         // group candidate format: the tcgen05 scan writes one list per (chunk,
                        // quarter) of rows some head of the GQA group keeps, with all G scores;
                        // attend_grp_kernel gathers each V row once for the whole group
};

// Diagnostic timeline: trace[kind][cta][slot] = %globaltimer (ns). kinds: 0 prep,
// 1 scan, 2 attend, 3 combine; slot 0 = CTA start, 1 = CTA end, 2.. = kind-specific.
constexpr int kTraceCtas = 1024, kTraceSlots = 16;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_max(const Batch& bt, int kind, int slot, unsigned long long v) {
  if (bt.trace && blockIdx.x < kTraceCtas && slot < kTraceSlots)
    atomicMax(bt.trace + ((size_t)kind * kTraceCtas + blockIdx.x) * kTraceSlots + slot, v);
}
__device__ __forceinline__ void trace_add(const Batch& bt, int kind, int slot, unsigned long long v) {
  if (bt.trace && blockIdx.x < kTraceCtas && slot < kTraceSlots)
    atomicAdd(bt.trace + ((size_t)kind * kTraceCtas + blockIdx.x) * kTraceSlots + slot, v);
}
__device__ __forceinline__ void trace_rec(const Batch& bt, int kind, int slot) {
  if (bt.trace && blockIdx.x < kTraceCtas && slot < kTraceSlots)
    bt.trace[((size_t)kind * kTraceCtas + blockIdx.x) * kTraceSlots + slot] = gtimer();
}

// Coarse block indexes of a batch (kernel-parameter space).
struct BixSet {
  alaya_block_index b[ALAYA_MAX_BATCH];
};

// Workspace pointers (device), carved from the caller's buffer.
// Identity of this call for the async-prep handshake: the host id, or in graph mode
// (call_seq) the captured slot combined with the replay's sequence number, which the
// graph's first node advances, so ids never repeat across replays.
__device__ __forceinline__ unsigned long long call_token(const Batch& bt) {
  return bt.call_seq ? (bt.call_id | (__ldcg(bt.call_seq) << 20)) : bt.call_id;
}

struct Ws {
  int* status;
  int* mode;        // status + 1: candidate format of the call (1 = group format), set by prep
  int* gidx;        // [chunks][chunk] group format: candidate rows per (chunk, quarter) sub-list
  unsigned long long* ready;  // call id whose header prep has zeroed (next to status, never zeroed)
  unsigned long long* seeded;  // [B*Hkv] call id whose seeds of (seq, kv head) are in gmax (never zeroed)
  unsigned long long* prepdone;  // [B*Hkv] call id whose prep CTA of (seq, kv head) has finished
  uint32_t* gmax;   // [B*Hq] order-preserving encoded running max
  int* counters;    // [16] right after gmax (zeroed by prep_kernel): [0] attend ticket,
                    // [2..3] block-filter kept/total, [6] epilogue-warp chunk publications
                    // (overlapped attend), [7] overflow items
  int* group_done;  // [B*Hkv] right after counters: chunk publications per (seq, kv head)
  int* cnt;         // [chunks*G*4] candidate counts per scan sub-list (see CandList)
  int* selcnt;      // [chunks*G]
  int* retcnt;      // [chunks*G]
  float* part_l;    // [chunks*G] primary (chunk, head) partials
  float* part_acc;  // [chunks*G*D]
  float* ovl_l;     // [chunks*G*4] overflow sub-list partials (split pairs, q = 1..3)
  float* ovl_acc;   // [chunks*G*4*D]
  int* ovl_sel;     // [chunks*G*4]
  int* ovl_ret;     // [chunks*G*4]
  int* heavy;       // [chunks*G] 1 = pair split into sub-list tasks (written by the scan)
  int* ovlist;      // [chunks*G*3] overflow items pair*4 + q (q = 1..3), count in counters[7]
  int* cidx;        // [chunks*G*chunk] candidate local row (then selected, compacted)
  float* cscore;    // [chunks*G*chunk]
  float* partbuf;   // [B*Hq*(D+2)]
  float* smaxbuf;   // [B*Hq]
  unsigned long long* keep;  // [chunks] block-filter masks: bit t = 128-key tile t of the chunk kept
};

// Programmatic dependent launch: a kernel launched with the PDL attribute may
// start while its predecessor on the stream is still running; pdl_wait()
// blocks until the predecessor grid has completed and its writes are visible
// (no-op without the attribute). pdl_trigger() lets this grid's dependent
// launch early (its CTAs then park in their own pdl_wait()).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t enc_max(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float dec_max(uint32_t e) {
  if (e == 0u) return -INFINITY;
  uint32_t u = (e & 0x80000000u) ? (e & 0x7fffffffu) : ~e;
  return __uint_as_float(u);
}

// Work chunk -> (sequence, kv head, chunk within head).
__device__ __forceinline__ void decode_chunk(const Batch& bt, int c, int& b, int& h, int& ci) {
  int lo = 0, hi = bt.B - 1;
  while (lo < hi) {  // last b with chunk_base[b] <= c
    int mid = (lo + hi + 1) >> 1;
    if (bt.s[mid].chunk_base <= c) lo = mid; else hi = mid - 1;
  }
  b = lo;
  int local = c - bt.s[b].chunk_base;
  h = local / bt.s[b].nch;
  ci = local - h * bt.s[b].nch;
}

// Tiles (128 keys) of a chunk the scan must read: all of them, or the block
// filter's mask.
__device__ __forceinline__ unsigned long long chunk_tiles(const Batch& bt, const Ws& ws, int c,
                                                          int ntiles) {
  const unsigned long long all = ntiles >= 64 ? ~0ull : ((1ull << ntiles) - 1ull);
  return bt.block_filter ? (ws.keep[c] & all) : all;
}

// Window membership of a GLOBAL base id (WindowConfig.base_ids, core.py:159-165).
__device__ __forceinline__ bool in_window(int64_t gid, int64_t P, int wi, int wl) {
  if (P <= (int64_t)wi + wl) return true;
  return gid < wi || gid >= P - wl;
}

// Candidate lists of one (chunk, head) pair cj: up to 4 ordered sub-lists (one
// per tcgen05 scan epilogue warp; the CUDA-core scan writes only sub-list 0),
// sub-list q at cidx + cj*chunk + q*(chunk/4) with count cnt[cj*4 + q]. The
// attend stage walks them as one virtual list; its physical position of a
// virtual index is >= the index, so selected ids can be compacted in place.
struct CandList {
  int pre[5];
  int qcap;
  __device__ __forceinline__ int total() const { return pre[4]; }
  __device__ __forceinline__ int phys(int i) const {  // static indexing: stays in registers
    if (i < pre[1]) return i;
    if (i < pre[2]) return qcap + i - pre[1];
    if (i < pre[3]) return 2 * qcap + i - pre[2];
    return 3 * qcap + i - pre[3];
  }
};
// Virtual list over sub-lists [qb, qe) of one (chunk, head); phys() is relative
// to sub-list qb's region.
__device__ __forceinline__ CandList cand_range(const int* cnt4, int qb, int qe, int chunk,
                                               bool through_l2) {
  CandList L;
  L.qcap = chunk / 4;
  L.pre[0] = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = qb + k;
    const int n = q < qe ? (through_l2 ? __ldcg(cnt4 + q) : cnt4[q]) : 0;
    L.pre[k + 1] = L.pre[k] + n;
  }
  return L;
}
// Attend task split, decided by the scan at chunk end: a (chunk, head) pair with
// more than bt.split candidates is processed as 4 sub-list tasks (sub-list 0 by
// the primary task into the primary slot, sub-lists 1..3 into overflow slots).
__device__ __forceinline__ void publish_pair(const Batch& bt, const Ws& ws, size_t cj, int total) {
  const int hv = total > bt.split;
  ws.heavy[cj] = hv;
  if (hv) {
    const int o = atomicAdd(&ws.counters[7], 3);
    for (int k = 0; k < 3; ++k) ws.ovlist[o + k] = (int)cj * 4 + 1 + k;
  }
}
__device__ __forceinline__ int pair_total(const int* cnt4, bool through_l2) {
  const int4 v = through_l2 ? __ldcg(reinterpret_cast<const int4*>(cnt4))
                            : *reinterpret_cast<const int4*>(cnt4);
  return v.x + v.y + v.z + v.w;
}

__device__ __forceinline__ CandList cand_list(const int* cnt4, int chunk, bool through_l2) {
  CandList L;
  L.qcap = chunk / 4;
  L.pre[0] = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) L.pre[q + 1] = L.pre[q] + (through_l2 ? __ldcg(cnt4 + q) : cnt4[q]);
  return L;
}

// --- mbarriers and bulk async copies (TMA engine) ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 1-D bulk copy global -> shared, completing on an mbarrier (SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// --- streaming loads -------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_stream(const uint2* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint16_t ld_stream(const uint16_t* p) {
  return __ldg(reinterpret_cast<const unsigned short*>(p));
}

// N elements of T held raw in registers; converted to fp32 on use.
template <typename T, int N>
struct RawFrag {
  static constexpr int BYTES = N * (int)sizeof(T);
  using V = std::conditional_t<
      BYTES % 16 == 0, uint4,
      std::conditional_t<BYTES % 8 == 0, uint2,
                         std::conditional_t<BYTES % 4 == 0, uint32_t, uint16_t>>>;
  static constexpr int NV = BYTES / (int)sizeof(V);
  V v[NV];

  __device__ __forceinline__ void load(const T* p) {
    const V* q = reinterpret_cast<const V*>(p);
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = ld_stream(q + i);
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = V{};
  }
  __device__ __forceinline__ uint32_t word(int i) const {  // i-th 32-bit word
    if constexpr (std::is_same_v<V, uint4>) {
      const uint4& x = v[i >> 2];
      int r = i & 3;
      return r == 0 ? x.x : r == 1 ? x.y : r == 2 ? x.z : x.w;
    } else if constexpr (std::is_same_v<V, uint2>) {
      const uint2& x = v[i >> 1];
      return (i & 1) ? x.y : x.x;
    } else if constexpr (std::is_same_v<V, uint32_t>) {
      return v[i];
    } else {
      return (uint32_t)v[0];
    }
  }
  __device__ __forceinline__ void to_float(float (&x)[N]) const {
    if constexpr (std::is_same_v<T, float>) {
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] = __uint_as_float(word(i));
    } else {
      if constexpr (N == 1) {
        x[0] = __uint_as_float(word(0) << 16);
      } else {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
          uint32_t u = word(i);
          x[2 * i] = __uint_as_float(u << 16);
          x[2 * i + 1] = __uint_as_float(u & 0xffff0000u);
        }
      }
    }
  }
};

template <int N>
__device__ __forceinline__ void load_q(const float* __restrict__ p, float (&x)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = __ldg(p + i);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, m));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFull, v, m);
  return v;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Deterministic block sum of one float per thread (fixed tree order).
__device__ __forceinline__ float block_sum(float v, float* red /* >= kWarps */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) t += red[i];
  return t;
}

}  // namespace alaya
