// Micro-benchmarks of the softmax-side primitives on B200 (sm_100a):
//   TMEM load/store throughput (tcgen05.ld/st 32x32b), MUFU ex2 throughput, per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tmem tools/ubench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2511_20714_b200/csrc/sm100_ptx.cuh"

using namespace ifx::ptx;

template <int WARPS_PER_Q, int X>  // X: columns per ld (32 only here), loads between waits
__global__ void tmem_ld_bench(long long* out, int iters, int batch) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int b = 0; b < batch; ++b) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + ((it * batch + b) * 32 & 511), r);
      if (b == batch - 1) tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= r[i];
    }
    tmem_wait_ld();
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x % 32 == 0) out[blockIdx.x * 64 + warp] = t1 - t0;
  if (acc == 0x12345678) out[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

__global__ void tmem_st_bench(long long* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    tmem_st16(tmem + lane_off + ((it * 16) & 511), r);
    if ((it & 3) == 3) tmem_wait_st();
  }
  tmem_wait_st();
  long long t1 = clock64();
  if (threadIdx.x % 32 == 0) out[blockIdx.x * 64 + warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

__global__ void mufu_bench(long long* out, float* sink, int iters) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ex2(v[i] * -0.5f);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x % 32 == 0) out[blockIdx.x * 64 + (threadIdx.x >> 5)] = t1 - t0;
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 64 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(float));
  long long h[148 * 64];
  auto report = [&](const char* name, int warps, double bytes_or_ops_per_warp, const char* unit) {
    cudaDeviceSynchronize();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    printf("%-40s warps/SM=%2d  cycles=%lld  %.1f %s per SM per clk\n", name, warps, mx,
           bytes_or_ops_per_warp * warps / mx, unit);
  };
  const int iters = 4096;
  for (int warps : {4, 8}) {
    for (int batch : {1, 4}) {
      tmem_ld_bench<1, 32><<<148, warps * 32>>>(d, iters, batch);
      char nm[64];
      snprintf(nm, 64, "tcgen05.ld 32x32b.x32 (wait/%d)", batch);
      report(nm, warps, (double)iters * batch * 32 * 32 * 4, "B");
    }
    tmem_st_bench<<<148, warps * 32>>>(d, iters);
    report("tcgen05.st 32x32b.x16", warps, (double)iters * 16 * 32 * 4, "B");
    mufu_bench<<<148, warps * 32>>>(d, sink, iters);
    report("MUFU.EX2 (ILP 8)", warps, (double)iters * 8 * 32, "ex2");
  }
  return 0;
}
