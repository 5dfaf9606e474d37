// launch.cuh — programmatic dependent launch (PDL) for every kernel of the library.
//
// The engine's layer-pass is a chain of ~13-17 dependent kernels (CUDA-graph replayed); at
// small per-rank shapes (Ulysses at 8 ranks) the gaps between them are a large share of the
// step. Each kernel is launched with cudaLaunchAttributeProgrammaticStreamSerialization, so
// the next kernel's CTAs are dispatched while the previous grid drains: everything before
// `pdl_wait()` (mbarrier init, TMEM allocation, tensor-map prefetch) overlaps the
// predecessor, and `pdl_wait()` (griddepcontrol.wait: the predecessor grid completed and its
// memory is visible) comes before the first global access. `pdl_trigger()` at the end of a
// CTA's work lets dependents launch before the grid fully retires. Kernels launched without
// the attribute (IFX_PDL=0, or any other launcher) see both as no-ops.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

namespace ifx {

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("IFX_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// kernel<<<grid, block, smem, st>>>(args...) with the PDL attribute (and optional cluster).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  ++n;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace ifx
