// Sequence-sharded exchange over peer memory (NVLink / NVSwitch, CUDA IPC):
// the two collectives of the sharded decode step without NCCL.
//
//   allreduce-max  each rank stores its [rows] local maxima straight into
//                  slot[rank] of EVERY rank's exchange buffer (P2P stores),
//                  fences at system scope, raises flag[rank] (release) in
//                  every buffer, waits for all R flags of its own buffer
//                  (acquire) and reduces the R slots -> the global DIPR max.
//   allgather      the same for the [count] partial states; the gathered
//                  [R][count] slots are read in place by the merge kernel.
//
// One CTA per call; the messages are a few KB, so this is latency-bound:
// one NVLink round trip plus a flag poll instead of an NCCL launch.
// Slots are double-buffered by epoch parity: a rank can only reach exchange
// e+2 after every peer raised its e+1 flag, i.e. finished reading exchange e.
// Flags are monotonic epochs (no reset). A bounded poll sets *err instead of
// hanging if a peer never arrives.
#include <cstring>

#include "alaya_dispatch.cuh"

namespace alaya {
namespace {

constexpr int kMaxPeers = 16;
constexpr int kExThreads = 512;

struct Peers {
  char* p[kMaxPeers];
};

// symmetric buffer: [2 kinds][kMaxPeers] u64 flags + an arrival counter (u64
// slot), padded to 512 B; per-group flags [kExGroups][kMaxPeers] u64 (fused
// sharded step); then slots: [parity 2][kind 2][R][cap] floats
constexpr size_t kFlagBytes = kExFlagBytes;
constexpr size_t kHeadBytes = kExFlagBytes + (size_t)kExGroups * kExMaxPeers * 8;

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float* slot(char* buf, int parity, int kind, int r, int R, int64_t cap) {
  return exch_slot(buf, parity, kind, r, R, cap);
}

// Allgather of larger messages (e.g. 0.5 MB of partial states per rank at 32
// sessions): several CTAs push disjoint segments to every peer; the last CTA to
// finish (arrival counter in the own buffer, after the flags) raises the flags;
// CTA 0 then waits for all R flags, so the kernel ends when every rank's data
// has landed here. All CTAs are co-resident (grid <= 64).
__global__ void __launch_bounds__(kExThreads)
    exch_gather_kernel(const float* __restrict__ local, int64_t count, int64_t cap,
                       __grid_constant__ const Peers peers, int rank, int R, unsigned long long epoch,
                       int* __restrict__ err) {
  const int parity = (int)(epoch & 1ull);
  const int64_t seg = (count + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * seg, hi = min(count, lo + seg);
  for (int p = 0; p < R; ++p) {
    float* dst = slot(peers.p[p], parity, 1, rank, R, cap);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) dst[i] = local[i];
  }
  __threadfence_system();
  __syncthreads();
  __shared__ int s_last;
  unsigned int* arrive = reinterpret_cast<unsigned int*>(
      reinterpret_cast<unsigned long long*>(peers.p[rank]) + 2 * kMaxPeers);  // own counter
  if (threadIdx.x == 0) s_last = atomicAdd(arrive, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    if (threadIdx.x == 0) *arrive = 0u;  // next exchange starts after this kernel
    __threadfence_system();
    if (threadIdx.x < R) {
      unsigned long long* f = reinterpret_cast<unsigned long long*>(peers.p[threadIdx.x]) + kMaxPeers + rank;
      st_release_sys(f, epoch);
    }
  }
  if (blockIdx.x != 0) return;
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  if (threadIdx.x < R) {
    const unsigned long long* f =
        reinterpret_cast<const unsigned long long*>(peers.p[rank]) + kMaxPeers + threadIdx.x;
    long long polls = 0;
    while (ld_acquire_sys(f) < epoch) {
      if (++polls > (1ll << 26)) {
        atomicExch(&s_bad, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (s_bad && threadIdx.x == 0 && err) atomicExch(err, 1);
}

// kind 0: allreduce-max of `count` floats into out; kind 1: allgather (out unused:
// the result is the caller's own slot region for this epoch)
__global__ void __launch_bounds__(kExThreads)
    exch_kernel(const float* __restrict__ local, int64_t count, int64_t cap, __grid_constant__ const Peers peers,
                int rank, int R, unsigned long long epoch, int kind, float* __restrict__ out,
                int* __restrict__ err) {
  const int parity = (int)(epoch & 1ull);
  for (int p = 0; p < R; ++p) {
    float* dst = slot(peers.p[p], parity, kind, rank, R, cap);
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = local[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < R) {
    unsigned long long* f = reinterpret_cast<unsigned long long*>(peers.p[threadIdx.x]) + kind * kMaxPeers + rank;
    st_release_sys(f, epoch);
  }
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  if (threadIdx.x < R) {
    const unsigned long long* f =
        reinterpret_cast<const unsigned long long*>(peers.p[rank]) + kind * kMaxPeers + threadIdx.x;
    long long polls = 0;
    while (ld_acquire_sys(f) < epoch) {
      if (++polls > (1ll << 26)) {  // ~seconds: a peer never arrived
        atomicExch(&s_bad, 1);
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
  if (kind == 0) {
    const float* own = slot(peers.p[rank], parity, 0, 0, R, cap);
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
      float m = -INFINITY;
      for (int r = 0; r < R; ++r) m = fmaxf(m, __ldcv(own + (size_t)r * cap + i));
      out[i] = m;
    }
  }
}

}  // namespace
}  // namespace alaya

using namespace alaya;

extern "C" {

size_t alaya_exch_bytes(int n_ranks, int64_t cap_floats) {
  if (n_ranks < 1 || n_ranks > kMaxPeers || cap_floats < 1) return 0;
  return kHeadBytes + (size_t)2 * 2 * n_ranks * (size_t)cap_floats * 4;
}

int alaya_exch_alloc(size_t bytes, void** d_buf, void* ipc_handle) {
  if (!d_buf || !ipc_handle || bytes == 0) return fail(ALAYA_ERR_ARG, "bad exchange alloc arguments");
  if (cudaMalloc(d_buf, bytes) != cudaSuccess) return cuda_check("exchange cudaMalloc");
  if (cudaMemset(*d_buf, 0, bytes) != cudaSuccess) return cuda_check("exchange memset");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, *d_buf) != cudaSuccess) return cuda_check("cudaIpcGetMemHandle");
  memcpy(ipc_handle, &h, sizeof(h));
  return ALAYA_OK;
}

int alaya_exch_open(const void* ipc_handle, void** d_buf) {
  if (!ipc_handle || !d_buf) return fail(ALAYA_ERR_ARG, "null ipc handle");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  if (cudaIpcOpenMemHandle(d_buf, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return cuda_check("cudaIpcOpenMemHandle");
  return ALAYA_OK;
}

int alaya_exch_close(void* d_buf) {
  if (d_buf && cudaIpcCloseMemHandle(d_buf) != cudaSuccess) return cuda_check("cudaIpcCloseMemHandle");
  return ALAYA_OK;
}

int alaya_exch_free(void* d_buf) {
  if (d_buf && cudaFree(d_buf) != cudaSuccess) return cuda_check("cudaFree");
  return ALAYA_OK;
}

int alaya_exch(void* const* bufs, int n_ranks, int rank, int64_t cap_floats, int kind,
               const float* d_local, int64_t count, unsigned long long epoch, float* d_out, int* d_err,
               void* stream) {
  if (!bufs || n_ranks < 1 || n_ranks > kMaxPeers || rank < 0 || rank >= n_ranks || !d_local)
    return fail(ALAYA_ERR_ARG, "bad exchange arguments");
  if (kind != 0 && kind != 1) return fail(ALAYA_ERR_ARG, "bad exchange kind");
  if (count < 0 || count > cap_floats) return fail(ALAYA_ERR_ARG, "exchange of %lld floats > cap %lld",
                                                   (long long)count, (long long)cap_floats);
  if (kind == 0 && !d_out) return fail(ALAYA_ERR_ARG, "null output");
  if (epoch == 0) return fail(ALAYA_ERR_ARG, "epochs start at 1");
  Peers pp;
  for (int r = 0; r < kMaxPeers; ++r) pp.p[r] = r < n_ranks ? static_cast<char*>(bufs[r]) : nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (kind == 1) {
    const int grid = (int)std::min<int64_t>(64, std::max<int64_t>(1, (count + 8191) / 8192));
    exch_gather_kernel<<<grid, kExThreads, 0, st>>>(d_local, count, cap_floats, pp, rank, n_ranks, epoch,
                                                    d_err);
    return cuda_check("exch_gather_kernel");
  }
  exch_kernel<<<1, kExThreads, 0, st>>>(d_local, count, cap_floats, pp, rank, n_ranks, epoch, kind, d_out,
                                        d_err);
  return cuda_check("exch_kernel");
}

float* alaya_exch_slots(void* d_buf, int n_ranks, int64_t cap_floats, int kind, unsigned long long epoch) {
  if (!d_buf) return nullptr;
  float* base = reinterpret_cast<float*>(static_cast<char*>(d_buf) + kHeadBytes);
  return base + (((size_t)(epoch & 1ull) * 2 + kind) * n_ranks) * (size_t)cap_floats;
}

}  // extern "C"
