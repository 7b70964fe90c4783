// Host-side launch helpers shared by the C-ABI (alaya.cu) and the kernel
// instantiation units (inst_*.cu), which are compiled in parallel.
#pragma once

#include <algorithm>
#include <string>

#include "alaya_kernels.cuh"

namespace alaya {

int fail(int code, const char* fmt, ...);
int num_sms();
int cuda_check(const char* what);
int persist_less(const Batch& bt);

bool pdl_enabled();

// Launch with the programmatic-dependent-launch attribute (ALAYA_PDL=0 turns
// it off). Every kernel launched this way calls pdl_wait() before touching
// data written by earlier work on the stream.
template <typename... KArgs, typename... Args>
int launch_pdl(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
               cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  return cuda_check(what);
}

inline size_t scan_smem(const Batch& bt) {
  return (size_t)bt.G * bt.chunk * 4 + kWarps * bt.G * 4 + bt.G * 4 + kWarps * bt.G * 4;
}

template <typename T, int D, int G>
struct Stages {
  static int scan(const Batch& bt, const float* q, const Ws& ws, cudaStream_t st) {
    if (bt.total_chunks == 0) return ALAYA_OK;
    size_t sm = scan_smem(bt);
    cudaFuncSetAttribute(scan_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int grid = bt.total_chunks;
    if (bt.persist) {  // one CTA fewer on `less` SMs: room for attend CTAs beside the scan
      static int per_sm = 0;
      if (per_sm == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_kernel<T, D, G>, kThreads, sm);
        if (per_sm < 1) per_sm = 1;
      }
      grid = std::min(bt.total_chunks, std::max(num_sms(), per_sm * num_sms() - persist_less(bt)));
    }
    return launch_pdl("scan_kernel", scan_kernel<T, D, G>, grid, kThreads, sm, st, bt, q, ws);
  }
  static int prep(const Batch& bt, const float* q, const Ws& ws, cudaStream_t st) {
    // window partials in prep: one (m, l, acc) staging row per (warp, head)
    const size_t sm = bt.win_in_prep ? (size_t)kWarps * G * (D + 2) * 4 : 0;
    if (sm > 48 * 1024) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(prep_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = true;
      }
    }
    return launch_pdl("prep_kernel", prep_kernel<T, D, G>, bt.B * bt.Hkv, kThreads, sm, st, bt, q, ws);
  }
  // zero_ticket = 0: the ticket was zeroed by prep_kernel in this call
  static int attend(const Batch& bt, const float* q, const float* smax, const Ws& ws,
                    int want_values, cudaStream_t st, int zero_ticket = 1) {
    const long tasks = (long)bt.total_chunks * G + ((want_values && !bt.win_in_prep) ? (long)bt.B * bt.Hq : 0);
    if (tasks == 0) return ALAYA_OK;
    static int per_sm = 0;
    if (per_sm == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attend_kernel<T, D, G>, kThreads, 0);
      if (per_sm < 1) per_sm = 1;
    }
    const long blocks = std::min<long>((tasks + kWarps - 1) / kWarps, (long)per_sm * num_sms());
    // primary ticket; counters[7] (overflow items) and the heavy flags come from the scan
    if (zero_ticket && cudaMemsetAsync(ws.counters, 0, sizeof(int), st) != cudaSuccess)
      return cuda_check("memset");
    return launch_pdl("attend_kernel", attend_kernel<T, D, G>, (unsigned)blocks, kThreads, 0, st, bt, q,
                      smax, ws, want_values);
  }
  // attend beside the tcgen05 scan (bt.overlap): PDL dependent, no grid wait
  static int attend_ovl(const Batch& bt, const float* q, const Ws& ws, cudaStream_t st) {
    static int per_sm = 0;
    if (per_sm == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attend_ovl_kernel<T, D, G>, kOvlThreads, 0);
      if (per_sm < 1) per_sm = 1;
    }
    const long tasks = (long)bt.total_chunks * G + (bt.win_in_prep ? 0 : (long)bt.B * bt.Hq);
    constexpr int kW = kOvlThreads / 32;
    const long blocks = std::min<long>((tasks + kW - 1) / kW, (long)per_sm * num_sms());
    if (blocks == 0) return ALAYA_OK;  // (no base chunks, window partials from prep)
    return launch_pdl("attend_ovl_kernel", attend_ovl_kernel<T, D, G>, (unsigned)blocks, kOvlThreads, 0,
                      st, bt, q, ws);
  }
  // group-format attend beside the tcgen05 scan: one 4-warp CTA per chunk
  static int attend_grp(const Batch& bt, const float* q, const Ws& ws, cudaStream_t st) {
    (void)q;
    static int per_sm = 0;
    if (per_sm == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attend_grp_kernel<T, D, G>, kGrpThreads, 0);
      if (per_sm < 1) per_sm = 1;
    }
    const long blocks = std::min<long>(bt.total_chunks, (long)per_sm * num_sms());
    if (blocks == 0) return ALAYA_OK;
    return launch_pdl("attend_grp_kernel", attend_grp_kernel<T, D, G>, (unsigned)blocks, kGrpThreads, 0, st, bt,
                      ws);
  }
  static int filter(const Batch& bt, const float* q, const Ws& ws, cudaStream_t st) {
    if (bt.total_chunks == 0) return ALAYA_OK;
    return launch_pdl("block_filter_kernel", block_filter_kernel<T, D, G>, bt.total_chunks, kThreads, 0, st,
                      bt, q, ws);
  }
  static int combine(const Batch& bt, const float* smax, const Ws& ws, float* out,
                     float* part_out, float* smax_out, cudaStream_t st) {
    // one CTA per row; few rows -> more warps per row (chunk partials in flight)
    const int rows = bt.B * bt.Hq;
    if (rows <= num_sms() / 2)
      return launch_pdl("combine_kernel", combine_kernel<D, G, 32>, rows, 1024, 0, st, bt, smax, ws, out,
                        part_out, smax_out);
    if (rows <= num_sms() + num_sms() / 2)
      return launch_pdl("combine_kernel", combine_kernel<D, G, 16>, rows, 512, 0, st, bt, smax, ws, out,
                        part_out, smax_out);
    return launch_pdl("combine_kernel", combine_kernel<D, G, 8>, rows, 256, 0, st, bt, smax, ws, out,
                      part_out, smax_out);
  }
};

using ScanFn = int (*)(const Batch&, const float*, const Ws&, cudaStream_t);
using AttendFn = int (*)(const Batch&, const float*, const float*, const Ws&, int, cudaStream_t, int);
using FilterFn = int (*)(const Batch&, const float*, const Ws&, cudaStream_t);
using CombineFn = int (*)(const Batch&, const float*, const Ws&, float*, float*, float*,
                          cudaStream_t);

struct StageSet {
  ScanFn scan;
  AttendFn attend;
  CombineFn combine;
  FilterFn filter;
  ScanFn prep;
  ScanFn attend_ovl;
  ScanFn attend_grp;
};

template <typename T, int D, int G>
StageSet make_set() {
  return {&Stages<T, D, G>::scan, &Stages<T, D, G>::attend, &Stages<T, D, G>::combine,
          &Stages<T, D, G>::filter, &Stages<T, D, G>::prep, &Stages<T, D, G>::attend_ovl,
          &Stages<T, D, G>::attend_grp};
}

template <typename T, int D>
StageSet pick_g(int G) {
  switch (G) {
    case 1: return make_set<T, D, 1>();
    case 2: return make_set<T, D, 2>();
    case 3: return make_set<T, D, 3>();
    case 4: return make_set<T, D, 4>();
    case 5: return make_set<T, D, 5>();
    case 6: return make_set<T, D, 6>();
    case 7: return make_set<T, D, 7>();
    default: return make_set<T, D, 8>();
  }
}


#define ALAYA_DECLARE_PICKS(X)                                                     \
  X(f32_16) X(f32_32) X(f32_64) X(f32_128) X(f32_256)                              \
  X(bf16_16) X(bf16_32) X(bf16_64) X(bf16_128) X(bf16_256)
#define ALAYA_DECL(name) StageSet pick_##name(int G);
bool tc_scan_eligible(const Batch& bt, int dtype, const alaya_seq* seqs);
int launch_tc_scan(const Batch& bt, const alaya_seq* seqs, const float* q, const Ws& ws,
                   cudaStream_t st);
bool dense_attend_enabled(const Batch& bt, const alaya_seq* seqs);
int launch_tc_attend_dense(const Batch& bt, const alaya_seq* seqs, const Ws& ws, cudaStream_t st);
bool overlap_enabled();
bool gfmt_enabled(const Batch& bt);
bool cc_overlap_enabled();
int64_t diprs_row_bytes(int max_n, int cap);
int launch_diprs(const Batch& bt, int dtype, const alaya_graph* graphs, const float* q, int l0, int floor_mode,
                 const float* floors, int cap, int64_t* ids, int64_t out_cap, int32_t* count, int32_t* explored,
                 void* ws, size_t ws_bytes, cudaStream_t st);
constexpr int kDiprsCap = 32768;  // offered ids per sub-batch (per row scratch)
int launch_topk_bound(const Batch& bt, int dtype, const float* q, float* scratch, size_t scratch_floats, int k,
                      float* thr, cudaStream_t st);
int launch_topk_select(const Batch& bt, const Ws& ws, int k, int64_t* ids, float* scores, int64_t cap,
                       int32_t* count, cudaStream_t st);
int launch_sparse_attention(const Batch& bt, int dtype, const float* q, const int64_t* ids, int64_t cap,
                            const int32_t* count, float* out, int32_t* nsel, int* status,
                            cudaStream_t st);
int launch_block_reps(const void* k, int dtype, int heads, int64_t head_stride, int n, int dim,
                      int block_size, int r, void* reps, int64_t reps_head_stride, cudaStream_t st);
int launch_block_topk(const Batch& bt, int dtype, const float* q, const BixSet& bix, int max_nb,
                      int block_size, int k_blocks, int64_t* ids, int64_t cap, int32_t* count,
                      int32_t* blocks, float* bscores, cudaStream_t st);
ALAYA_DECLARE_PICKS(ALAYA_DECL)
#undef ALAYA_DECL

}  // namespace alaya
