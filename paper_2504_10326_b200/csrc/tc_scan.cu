// Host launcher of the tcgen05 scan: one TMA tensor map per distinct K slab
// (passed by value in kernel-parameter space), persistent grid of one CTA
// per SM.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <mutex>

#include "alaya_dispatch.cuh"
#include "alaya_tc.cuh"
#include "alaya_tc_attend.cuh"

namespace alaya {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

namespace {

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

template <int G, int S>
int launch_s(const Batch& bt, const tc::Maps& maps, const float* q, const Ws& ws, cudaStream_t st,
             int ctas_per_sm) {
  const size_t sm = tc::tc_smem_bytes(G, S);
  // persistent, chunks handed out dynamically; `less` SMs run one scan CTA instead
  // of two so attend CTAs fit beside it (an attend CTA cannot share an SM with two
  // scan CTAs: registers), more of them as the call's work grows. Measured optima
  // (profiles/r02/grid_less_v29.jsonl, grid_less_v35.jsonl), in units of 128K
  // tokens summed over the batch: 1 -> 24-48, 2 (32K x 8) -> 48, 4 -> 48-74,
  // 8 -> 110, 16 -> >= 110. ALAYA_TC_GRID_LESS overrides.
  static const int less_env = env_int("ALAYA_TC_GRID_LESS", -1);
  double units = 0.0;
  for (int b = 0; b < bt.B; ++b) units += (double)bt.s[b].n / 131072.0;
  const int less = less_env >= 0 ? less_env
                                 : std::min(140, (int)(24.0 + 22.0 * std::log2(std::max(1.0, units))));
  const int grid = std::min(bt.total_chunks, std::max(num_sms(), ctas_per_sm * num_sms() - less));
  if (bt.gfmt) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(tc::scan_tc_kernel<G, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr = true;
    }
    return launch_pdl("scan_tc_kernel", tc::scan_tc_kernel<G, S, true>, grid, tc::kThreadsTc, sm, st, bt, maps, q,
                      ws);
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::scan_tc_kernel<G, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  return launch_pdl("scan_tc_kernel", tc::scan_tc_kernel<G, S, false>, grid, tc::kThreadsTc, sm, st, bt, maps, q, ws);
}

// Persistent CTAs per SM (ALAYA_TC_CTAS, default 3): 2 CTAs with 3-stage rings
// or 3 CTAs with 2-stage rings overlap their TMA->MMA->epilogue handshakes;
// 1 CTA uses ALAYA_TC_STAGES (4..6, default 6).
template <int G>
int launch(const Batch& bt, const tc::Maps& maps, const float* q, const Ws& ws, cudaStream_t st) {
  static const int ctas = env_int("ALAYA_TC_CTAS", 2);
  static const int stages = env_int("ALAYA_TC_STAGES", 6);
  if (ctas >= 3) return launch_s<G, 2>(bt, maps, q, ws, st, 3);
  if (ctas == 2) return launch_s<G, 3>(bt, maps, q, ws, st, 2);
  if (stages <= 4) return launch_s<G, 4>(bt, maps, q, ws, st, 1);
  if (stages == 5) return launch_s<G, 5>(bt, maps, q, ws, st, 1);
  return launch_s<G, 6>(bt, maps, q, ws, st, 1);
}

// One TMA tensor map per distinct K (or V: use_v) slab (sessions sharing a context share it).
int build_maps(const Batch& bt, const alaya_seq* seqs, tc::Maps& maps, bool use_v = false) {
  auto enc = encode_fn();
  // L2 sector promotion of the K boxes: ALAYA_TC_PROMO 0..3 = none/64B/128B/256B
  static const CUtensorMapL2promotion promo =
      static_cast<CUtensorMapL2promotion>(env_int("ALAYA_TC_PROMO", 3));
  int nmaps = 0;
  for (int b = 0; b < bt.B; ++b) {
    maps.map_of_seq[b] = 0;
    maps.rows_per_head[b] = seqs[b].head_stride / 128;
    if (seqs[b].n == 0) continue;
    int found = -1;
    for (int a = 0; a < b && found < 0; ++a)
      if (seqs[a].n && (use_v ? seqs[a].v == seqs[b].v : seqs[a].k == seqs[b].k)) found = maps.map_of_seq[a];
    if (found >= 0) { maps.map_of_seq[b] = (int16_t)found; continue; }
    const cuuint64_t rows = (cuuint64_t)bt.Hkv * (seqs[b].head_stride / 128);
    // encoded maps are cached per (slab, rows): decode steps re-use the same slabs
    struct Cached { const void* k; cuuint64_t rows; CUtensorMap m; };
    static thread_local Cached cache[64];
    static thread_local int cache_next = 0;
    const Cached* hit = nullptr;
    const void* slab = use_v ? seqs[b].v : seqs[b].k;
    for (int i = 0; i < 64 && !hit; ++i)
      if (cache[i].k == slab && cache[i].rows == rows) hit = &cache[i];
    if (hit) {
      maps.m[nmaps] = hit->m;
      maps.map_of_seq[b] = (int16_t)nmaps++;
      continue;
    }
    cuuint64_t gdim[2] = {128, rows};
    cuuint64_t gstride[1] = {256};
    cuuint32_t box[2] = {64, (cuuint32_t)tc::kTileKeys};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = enc(&maps.m[nmaps], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(slab),
                     gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ALAYA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    cache[cache_next] = {slab, rows, maps.m[nmaps]};
    cache_next = (cache_next + 1) % 64;
    maps.map_of_seq[b] = (int16_t)nmaps++;
  }
  return ALAYA_OK;
}

template <int G>
int launch_dense(const Batch& bt, const tc::Maps& vmaps, const Ws& ws, cudaStream_t st) {
  const size_t sm = tc::dense_smem_bytes(G);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::attend_dense_tc_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  return launch_pdl("attend_dense_tc_kernel", tc::attend_dense_tc_kernel<G>, bt.total_chunks, tc::dense_threads(G),
                    sm, st, bt, vmaps, ws);
}

}  // namespace

// Dense tensor-core group attend (alaya_tc_attend.cuh) for every group-format call
// (beta / sqrt(d) >= 11.5: the heads keep most rows of a chunk), bf16 V slabs laid
// out like K (TMA-able), not in the fused sharded step. ALAYA_GRP_DENSE=0 keeps the
// gather kernel (attend_grp_kernel). Measured at beta = 140 (profiles/r02/dense_headsplit_v69.jsonl):
// Llama B=1 126 -> 115 us, B=4 446 -> 409, B=8 843 -> 821, Qwen 40/8 B=1 139 -> 126, B=8 902 -> 894;
// at beta = 130 the per-head attend stays ahead (B=8 729 vs 802), so the group-format
// threshold is unchanged.
bool dense_attend_enabled(const Batch& bt, const alaya_seq* seqs) {
  static const int mode = env_int("ALAYA_GRP_DENSE", 1);
  if (!mode || !bt.gfmt || bt.sx_on || bt.D != 128) return false;
  int distinct = 0;
  for (int b = 0; b < bt.B; ++b) {
    if (seqs[b].n == 0) continue;
    if (seqs[b].head_stride % 128 || reinterpret_cast<uintptr_t>(seqs[b].v) % 16) return false;
    bool seen = false;
    for (int a = 0; a < b && !seen; ++a) seen = seqs[a].v == seqs[b].v;
    distinct += !seen;
  }
  return distinct <= tc::kMaxMaps;
}

int launch_tc_attend_dense(const Batch& bt, const alaya_seq* seqs, const Ws& ws, cudaStream_t st) {
  if (bt.total_chunks == 0) return ALAYA_OK;
  static thread_local tc::Maps vmaps;
  int rc = build_maps(bt, seqs, vmaps, true);
  if (rc) return rc;
  switch (bt.G) {
    case 1: return launch_dense<1>(bt, vmaps, ws, st);
    case 2: return launch_dense<2>(bt, vmaps, ws, st);
    case 3: return launch_dense<3>(bt, vmaps, ws, st);
    case 4: return launch_dense<4>(bt, vmaps, ws, st);
    case 5: return launch_dense<5>(bt, vmaps, ws, st);
    case 6: return launch_dense<6>(bt, vmaps, ws, st);
    case 7: return launch_dense<7>(bt, vmaps, ws, st);
    default: return launch_dense<8>(bt, vmaps, ws, st);
  }
}

bool tc_scan_eligible(const Batch& bt, int dtype, const alaya_seq* seqs) {
  if (dtype != ALAYA_BF16 || bt.D != 128 || bt.G > 8 || bt.chunk % (4 * tc::kTileKeys)) return false;
  int distinct = 0;
  for (int b = 0; b < bt.B; ++b) {
    if (seqs[b].n == 0) continue;
    if (seqs[b].head_stride % 128 || reinterpret_cast<uintptr_t>(seqs[b].k) % 16) return false;
    bool seen = false;
    for (int a = 0; a < b && !seen; ++a) seen = seqs[a].k == seqs[b].k;
    distinct += !seen;
  }
  return distinct <= tc::kMaxMaps && encode_fn() != nullptr;
}

bool pdl_enabled() {
  static const int on = env_int("ALAYA_PDL", 1);
  return on != 0;
}

// attend beside the scan: on for every tcgen05 call (ALAYA_OVERLAP=0 turns it
// off). On since the async prep / combine changes (v16): B=1 89.0 -> 86.1 us,
// B=2 132.7 -> 129.0, 8K ctx B=4 55.9 -> 51.6 (tools/probe_latency.py)
// Group candidate format + attend_grp_kernel (V rows gathered once per GQA
// group): ALAYA_GFMT=1 on, 0 off, default (-1) on when beta / sqrt(d) >= 11.5
// (beta >= 130 at d = 128). It pays G FMAs per gathered row, so it only wins
// when the heads of a group keep mostly the same rows; on the reference
// generator's data that is the high-beta regime (B=4 128K: beta 140 602 -> 445
// us, beta 110 226 -> 259 us; profiles/r02/README.md).
bool gfmt_enabled(const Batch& bt) {
  static const int mode = env_int("ALAYA_GFMT", -1);
  if (mode >= 0) return mode != 0;
  return bt.beta * bt.inv_sqrt_d >= 11.5f;
}

// CUDA-core scan (fp32 K/V, other dims) with the attend beside it: persistent scan
// grid (ALAYA_OVERLAP_CC=1; default off: one CTA per chunk, the attend after the
// scan -- fp32 128K B=4 490 vs 542 us, B=1 165 vs 162 us, profiles/r02/fp32_attend_rounds_v54.jsonl)
bool cc_overlap_enabled() {
  static const int on = env_int("ALAYA_OVERLAP_CC", 0);
  return on != 0;
}
int persist_less(const Batch& bt) {
  static const int less_env = env_int("ALAYA_CC_GRID_LESS", -1);
  if (less_env >= 0) return less_env;
  double units = 0.0;
  for (int b = 0; b < bt.B; ++b) units += (double)bt.s[b].n / 131072.0;
  return std::min(140, (int)(24.0 + 22.0 * std::log2(std::max(1.0, units))));
}

bool overlap_enabled() {
  static const int mode = env_int("ALAYA_OVERLAP", 1);
  return mode != 0;
}

int launch_tc_scan(const Batch& bt_in, const alaya_seq* seqs, const float* q, const Ws& ws,
                   cudaStream_t st) {
  if (bt_in.total_chunks == 0) return ALAYA_OK;
  static thread_local Batch bt;
  bt = bt_in;
  static const int dbg = env_int("ALAYA_TC_DBG", 0);
  bt.dbg = dbg;
  static thread_local tc::Maps maps;  // ~19 KB: keep off the stack
  int rc = build_maps(bt, seqs, maps);
  if (rc) return rc;
  switch (bt.G) {
    case 1: return launch<1>(bt, maps, q, ws, st);
    case 2: return launch<2>(bt, maps, q, ws, st);
    case 3: return launch<3>(bt, maps, q, ws, st);
    case 4: return launch<4>(bt, maps, q, ws, st);
    case 5: return launch<5>(bt, maps, q, ws, st);
    case 6: return launch<6>(bt, maps, q, ws, st);
    case 7: return launch<7>(bt, maps, q, ws, st);
    default: return launch<8>(bt, maps, q, ws, st);
  }
}

}  // namespace alaya
