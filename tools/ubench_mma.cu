// Tensor-core issue-rate micro-benchmark on B200: tcgen05.mma kind::f16 M=128 N=128 K=16,
// SS (A,B from smem) vs TS (A from TMEM), with and without concurrent TMA-like smem writes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma tools/ubench_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2511_20714_b200/csrc/sm100_ptx.cuh"

using namespace ifx::ptx;

// mode 0: SS only, 1: TS only, 2: SS+TS alternating (attention pattern), 3: mode 2 + 2 warps
// streaming st.shared (emulates TMA smem fill bandwidth)
template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_bench(long long* out, int tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t base = smem_u32(smem);
  long long t0 = clock64();
  if (warp == 0) {
    if (elect_one()) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
      for (int t = 0; t < tiles; ++t) {
        if (MODE != 1) {
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma_bf16_ss(tmem + (t & 1) * 128, smem_desc_sw128(base + off, 16, 1024),
                        smem_desc_sw128(base + 32768 + off, 16, 1024), idesc_qk, kk > 0);
          }
        }
        if (MODE != 0) {
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bdesc = smem_desc_sw128(base + 32768 + kk * 2048, 16384, 1024);
            mma_bf16_ts(tmem + 384, tmem + 256 + kk * 8, bdesc, idesc_pv, (t > 0 || kk > 0) ? 1u : 0u);
          }
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
    __syncwarp();
  } else if (MODE == 3 && warp >= 2) {
    // stream writes into a separate 16 KB region (TMA-fill stand-in)
    uint4 v = make_uint4(1, 2, 3, 4);
    for (int t = 0; t < tiles * 64; ++t) {
      uint4* dst = reinterpret_cast<uint4*>(smem + 48 * 1024) + ((t * 64 + (threadIdx.x - 64)) & 1023);
      *dst = v;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run(const char* name, long long* d, int tiles) {
  cudaFuncSetAttribute(mma_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  mma_bench<MODE><<<148, 128, 80 * 1024>>>(d, tiles);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double groups = (MODE == 2 || MODE == 3) ? 2.0 : 1.0;
  printf("%-34s cycles/tile=%.1f  (ideal 512 per 8-MMA group -> %.0f)  frac=%.3f\n", name,
         (double)mx / tiles, 512 * groups, 512 * groups * tiles / (double)mx);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int tiles = 2000;
  run<0>("SS  (QK^T pattern)", d, tiles);
  run<1>("TS  (PV pattern, A in TMEM)", d, tiles);
  run<2>("SS + TS alternating", d, tiles);
  run<3>("SS + TS + smem write stream", d, tiles);
  return 0;
}
