// peer.cu — peer memory over NVLink / NVSwitch for the Ulysses exchange (parallel.py:140-169
// of the reference moves Q/K/V column blocks and O back through two all-to-alls).
//
// Instead of pack -> ncclAllToAll -> unpack, the kernels that PRODUCE the exchanged rows store
// them straight into the consumer rank's buffer (G1's scatter epilogue, K1's O scatter), so
// the transfer overlaps the math tile by tile. What remains here is plumbing and ordering:
//   * CUDA IPC: each rank's arena (one cudaMalloc, ifx_dev_alloc) is exported as a 64-byte
//     handle, the handles travel through torch.distributed (host plumbing), and every rank
//     maps its peers' arenas (peer access enabled lazily by the driver).
//   * ifx_peer_barrier: one tiny kernel per exchange phase, graph-capturable. Each rank bumps
//     its own epoch counter (device memory, so a replayed graph advances it), publishes the
//     epoch into every peer's signal pad with a system-scope release store after a system
//     fence (so this GPU's earlier stores into peers' buffers, made by earlier kernels on
//     the stream, are visible first), and waits with system-scope acquire loads until every
//     peer published the same epoch into its own pad. Epochs are compared modulo 2^32.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/ifx_abi.h"
#include "common_host.h"
#include "launch.cuh"

namespace ifx {
namespace {

constexpr int kMaxPeers = 8;

struct BarrierArgs {
  uint32_t* pads[kMaxPeers];
  uint32_t* counter;
  long long timeout_cycles;
  int world, rank;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void peer_barrier_kernel(const BarrierArgs a) {
  pdl_wait();
  __shared__ uint32_t epoch;
  if (threadIdx.x == 0) {
    epoch = *a.counter + 1u;
    *a.counter = epoch;
  }
  __syncthreads();
  const uint32_t e = epoch;
  const int p = threadIdx.x;
  if (p < a.world) {
    __threadfence_system();
    st_release_sys(a.pads[p] + a.rank, e);
    const uint32_t* mine = a.pads[a.rank] + p;
    const long long t0 = clock64();
    while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
      if (clock64() - t0 > a.timeout_cycles) __trap();  // a peer never arrived: fail loudly
      __nanosleep(32);
    }
    __threadfence_system();
  }
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return IFX_OK;
  return fail(IFX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace
}  // namespace ifx

extern "C" {

int ifx_ipc_handle(const void* dev_ptr, void* handle_out) {
  if (dev_ptr == nullptr || handle_out == nullptr) return ifx::fail(IFX_EDIM, "ipc_handle: null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
  cudaIpcMemHandle_t h;
  if (int rc = ifx::cuda_status(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)), "cudaIpcGetMemHandle"))
    return rc;
  std::memcpy(handle_out, &h, sizeof(h));
  return IFX_OK;
}

int ifx_ipc_open(const void* handle, void** dev_ptr_out) {
  if (handle == nullptr || dev_ptr_out == nullptr) return ifx::fail(IFX_EDIM, "ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  *dev_ptr_out = nullptr;
  return ifx::cuda_status(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess),
                          "cudaIpcOpenMemHandle");
}

int ifx_ipc_close(void* dev_ptr) {
  if (dev_ptr == nullptr) return IFX_OK;
  return ifx::cuda_status(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
}

int ifx_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                 int64_t rows, void* stream) {
  if (rows < 0 || width_bytes < 0 || dpitch < width_bytes || spitch < width_bytes)
    return ifx::fail(IFX_EDIM, "bad 2-D copy");
  if (rows == 0 || width_bytes == 0) return IFX_OK;
  return ifx::cuda_status(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch,
                                            (size_t)width_bytes, (size_t)rows, cudaMemcpyDefault,
                                            static_cast<cudaStream_t>(stream)),
                          "cudaMemcpy2DAsync");
}

int ifx_peer_barrier(void* const* pads, int world, int rank, uint32_t* counter, int timeout_ms,
                     void* stream) {
  if (world < 1 || world > ifx::kMaxPeers || rank < 0 || rank >= world || pads == nullptr ||
      counter == nullptr || timeout_ms < 1)
    return ifx::fail(IFX_EDIM, "bad peer barrier");
  ifx::BarrierArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int p = 0; p < world; ++p) {
    if (pads[p] == nullptr || (reinterpret_cast<uintptr_t>(pads[p]) & 31))
      return ifx::fail(IFX_EDIM, "peer signal pads must be 32-byte aligned");
    a.pads[p] = static_cast<uint32_t*>(pads[p]);
  }
  a.counter = counter;
  a.world = world;
  a.rank = rank;
  a.timeout_cycles = (long long)timeout_ms * 2000000LL;  // ~2 GHz SM clock, upper bound
  ifx::launch_pdl(ifx::peer_barrier_kernel, dim3(1), dim3(32), 0, static_cast<cudaStream_t>(stream), 1, a);
  return ifx::cuda_status(cudaGetLastError(), "peer_barrier launch");
}

}  // extern "C"
