// Diagnostic read-bandwidth probes (not part of the decode path): establish
// what this B200 delivers for pure streaming reads so that kernel efficiency
// can be judged against a measured read ceiling, not only the copy peak.
//   mode 0: ld.global.nc.v4 streaming, 8 x 16 B in flight per thread
//   mode 1: 1-D bulk async copies (TMA engine) of 32 KB into a 6-stage smem
//           ring, one issuing thread per CTA, one CTA per SM
//   mode 2: random 256-byte row gather (rows[] indices), 16 rows in flight
//           per half-warp -- the V-gather access pattern
#include <cstdint>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "alaya_common.cuh"

using namespace alaya;

namespace {

__global__ void __launch_bounds__(256) read_ldg(const uint4* __restrict__ p, size_t n16,
                                                uint32_t* __restrict__ sink) {
  uint32_t x = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld_stream(p + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) x ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  for (; i < n16; i += stride) { uint4 v = ld_stream(p + i); x ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (x == 0x9e3779b9u) sink[0] = x;
}

constexpr int kBulkStages = 6;
constexpr uint32_t kBulkBytes = 32768;

__global__ void __launch_bounds__(32, 1) read_bulk(const uint8_t* __restrict__ p, size_t nchunks,
                                                   uint32_t* __restrict__ sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kBulkStages * kBulkBytes);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kBulkStages; ++s) mbar_init(smem_u32(&bars[s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phases = 0;
  size_t issued = 0, done = 0;
  size_t c = blockIdx.x;
  // prime the ring
  for (int s = 0; s < kBulkStages && c + issued * gridDim.x < nchunks; ++s, ++issued) {
    mbar_expect_tx(smem_u32(&bars[s]), kBulkBytes);
    bulk_g2s(smem_u32(sm + s * kBulkBytes), p + (c + issued * gridDim.x) * kBulkBytes, kBulkBytes,
             smem_u32(&bars[s]));
  }
  while (done < issued) {
    const int s = (int)(done % kBulkStages);
    mbar_wait(smem_u32(&bars[s]), (phases >> s) & 1u);
    phases ^= 1u << s;
    ++done;
    const size_t nc = c + issued * gridDim.x;
    if (nc < nchunks) {
      mbar_expect_tx(smem_u32(&bars[s]), kBulkBytes);
      bulk_g2s(smem_u32(sm + s * kBulkBytes), p + nc * kBulkBytes, kBulkBytes, smem_u32(&bars[s]));
      ++issued;
    }
  }
  if (sm[0] == 0x5a && sm[1] == 0xa5) sink[0] = 1;
}

__global__ void __launch_bounds__(256) gather_rows(const uint4* __restrict__ v, const int* __restrict__ rows,
                                                   int nrows, uint32_t* __restrict__ sink) {
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
  const int hw_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const int hw_total = (gridDim.x * blockDim.x) >> 4;
  uint32_t x = 0;
  for (int r0 = hw_global; r0 < nrows; r0 += 16 * hw_total) {
    uint4 f[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int r = r0 + k * hw_total;
      f[k] = r < nrows ? ld_stream(v + (size_t)rows[r] * 16 + hl) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) x ^= f[k].x ^ f[k].y ^ f[k].z ^ f[k].w;
  }
  (void)half;
  if (x == 0x9e3779b9u) sink[0] = x;
}

// mode 3: the scan's TMA pattern without consumers: 2-D tensor map over
// [rows][128] bf16, SW128, two 64-column boxes per 128-row tile (split = 0), or
// one 3-D box {64, 2, 128} per tile walking each 256-byte row contiguously (split = 1).
__global__ void __launch_bounds__(32, 1) read_tma2d(const __grid_constant__ CUtensorMap map, int tiles, int split,
                                                    uint32_t* __restrict__ sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kBulkStages * kBulkBytes);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kBulkStages; ++s) mbar_init(smem_u32(&bars[s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](int s, int t) {
    const uint32_t dst = smem_u32(base + s * kBulkBytes), bar = smem_u32(&bars[s]);
    mbar_expect_tx(bar, kBulkBytes);
    const uint64_t mp = reinterpret_cast<uint64_t>(&map);
    if (split == 0) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(dst), "l"(mp), "r"(0), "r"(t * 128), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(dst + 16384), "l"(mp), "r"(64), "r"(t * 128), "r"(bar) : "memory");
    } else {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst), "l"(mp), "r"(0), "r"(0), "r"(t * 128), "r"(bar) : "memory");
    }
  };
  uint32_t phases = 0;
  int issued = 0, done = 0;
  for (int s = 0; s < kBulkStages && (int)blockIdx.x + issued * (int)gridDim.x < tiles; ++s, ++issued)
    issue(s, blockIdx.x + issued * gridDim.x);
  while (done < issued) {
    const int s = done % kBulkStages;
    mbar_wait(smem_u32(&bars[s]), (phases >> s) & 1u);
    phases ^= 1u << s;
    ++done;
    const int t = blockIdx.x + issued * gridDim.x;
    if (t < tiles) { issue(s, t); ++issued; }
  }
  if (base[0] == 0x5a && base[1] == 0xa5) sink[0] = 1;
}

}  // namespace

extern "C" int alaya_diag_read(const void* d_buf, size_t bytes, int mode, const int* d_rows, int nrows,
                               uint32_t* d_sink, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (mode == 0) {
    read_ldg<<<sms * 8, 256, 0, st>>>(static_cast<const uint4*>(d_buf), bytes / 16, d_sink);
  } else if (mode == 1) {
    const size_t sm = kBulkStages * kBulkBytes + 8 * kBulkStages;
    cudaFuncSetAttribute(read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    read_bulk<<<sms, 32, sm, st>>>(static_cast<const uint8_t*>(d_buf), bytes / kBulkBytes, d_sink);
  } else if (mode >= 10 && mode < 20) {  // gather with (mode - 10) CTAs of 256 threads per SM
    gather_rows<<<sms * (mode - 10), 256, 0, st>>>(static_cast<const uint4*>(d_buf), d_rows, nrows, d_sink);
  } else if (mode == 3 || mode == 4) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr) != cudaSuccess) return 4;
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    const cuuint64_t rows = bytes / 256;
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r;
    if (mode == 3) {
      cuuint64_t gd[2] = {128, rows}, gs[1] = {256};
      cuuint32_t box[2] = {64, 128};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d_buf), gd, gs, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t gd[3] = {64, 2, rows}, gs[2] = {128, 256};
      cuuint32_t box[3] = {64, 2, 128};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(d_buf), gd, gs, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return 4;
    const size_t sm = 1024 + kBulkStages * kBulkBytes + 8 * kBulkStages;
    cudaFuncSetAttribute(read_tma2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    read_tma2d<<<sms, 32, sm, st>>>(map, (int)(rows / 128), mode - 3, d_sink);
  } else {
    gather_rows<<<sms * 8, 256, 0, st>>>(static_cast<const uint4*>(d_buf), d_rows, nrows, d_sink);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
