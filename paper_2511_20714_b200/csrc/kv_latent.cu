// kv_latent.cu — K2L / K7L: the KV cache's latent mode (kvcache.py:26-31,201-203,323-325,
// MLA-style: rows are stored down-projected, k . down [d, L], and expanded at fetch time,
// lat . up [L, d]) fused into the page write and the gather, in fp32 like the reference.
//
// One CTA = RB rows of K or V (blockIdx.y = 0 / 1): the rows are staged in shared memory as
// fp32, and each thread owns output columns j, j + 256, ...: out[r][j] = sum_i x[r][i] w[i][j]
// with w read once per RB rows (coalesced across the threads' j) and the row values
// broadcast from shared memory. Summation runs over i in order, in fp32 FMA.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device_state.h"
#include "kv_kernels.h"

namespace ifx {
namespace {

constexpr int kThreads = 256;

struct LatPool {
  uint8_t* dev_k;
  uint8_t* dev_v;
  uint8_t* host_k;
  uint8_t* host_v;
  int64_t row_b;  // bytes per stored row
  int page_len;
  int bf16;       // element type of the pool
};

__device__ __forceinline__ uint8_t* lat_row(const LatPool& p, bool is_v, int32_t code, int in_page) {
  const int64_t r = (int64_t)(code >= 0 ? code : -1 - code) * p.page_len + in_page;
  uint8_t* base = code >= 0 ? (is_v ? p.dev_v : p.dev_k) : (is_v ? p.host_v : p.host_k);
  return base + r * p.row_b;
}

__device__ __forceinline__ float load_elem(const void* base, int64_t i, int bf16) {
  return bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(base)[i])
              : static_cast<const float*>(base)[i];
}
__device__ __forceinline__ void store_elem(void* base, int64_t i, float x, int bf16) {
  if (bf16) static_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16(x);
  else static_cast<float*>(base)[i] = x;
}

// K2L: rows [0, t) of K / V (tokens token0 + r) -> (row . down) into their page slots;
// pool columns [L, width) are written as zeros (16-byte row padding)
template <int RB>
__global__ void __launch_bounds__(kThreads) latent_append_kernel(
    const void* __restrict__ ks, const void* __restrict__ vs, int64_t src_ld, int src_bf16,
    int d_in, const float* __restrict__ down, int L, int width, LatPool pool,
    const int32_t* __restrict__ slots, int64_t rel0, int64_t t) {
  extern __shared__ float xs[];  // [RB][d_in]
  const bool is_v = blockIdx.y == 1;
  const void* src = is_v ? vs : ks;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nr = (int)(t - r0 < RB ? t - r0 : RB);
  for (int idx = threadIdx.x; idx < RB * d_in; idx += kThreads) {
    const int r = idx / d_in, i = idx - r * d_in;
    xs[idx] = r < nr ? load_elem(src, (r0 + r) * src_ld + i, src_bf16) : 0.f;
  }
  __syncthreads();
  uint8_t* dst[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    dst[r] = nullptr;
    if (r < nr) {
      const int64_t rel = rel0 + r0 + r;
      const int pg = (int)(rel / pool.page_len);
      dst[r] = lat_row(pool, is_v, __ldg(slots + pg), (int)(rel - (int64_t)pg * pool.page_len));
    }
  }
  for (int j = threadIdx.x; j < width; j += kThreads) {
    float acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = 0.f;
    if (j < L) {
      for (int i = 0; i < d_in; ++i) {
        const float w = __ldg(down + (int64_t)i * L + j);
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r] = fmaf(xs[r * d_in + i], w, acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (dst[r] != nullptr) store_elem(dst[r], j, acc[r], pool.bf16);
  }
}

// K7L: out row i = (stored row of token tokens[i] (or token0 + i)) . up, columns [0, d_out)
template <int RB>
__global__ void __launch_bounds__(kThreads) latent_gather_kernel(
    LatPool pool, const int32_t* __restrict__ slots, const int64_t* __restrict__ tokens,
    int64_t rel0, int64_t n, int L, const float* __restrict__ up, int d_out, void* ko, void* vo,
    int64_t out_ld, int out_bf16) {
  extern __shared__ float xs[];  // [RB][L]
  const bool is_v = blockIdx.y == 1;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nr = (int)(n - r0 < RB ? n - r0 : RB);
  for (int idx = threadIdx.x; idx < RB * L; idx += kThreads) {
    const int r = idx / L, i = idx - r * L;
    float x = 0.f;
    if (r < nr) {
      const int64_t rel = tokens ? tokens[r0 + r] - rel0 : rel0 + r0 + r;
      const int pg = (int)(rel / pool.page_len);
      const uint8_t* row = lat_row(pool, is_v, __ldg(slots + pg), (int)(rel - (int64_t)pg * pool.page_len));
      x = load_elem(row, i, pool.bf16);
    }
    xs[idx] = x;
  }
  __syncthreads();
  void* out = is_v ? vo : ko;
  for (int j = threadIdx.x; j < d_out; j += kThreads) {
    float acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = 0.f;
    for (int i = 0; i < L; ++i) {
      const float w = __ldg(up + (int64_t)i * d_out + j);
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = fmaf(xs[r * L + i], w, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (r < nr) store_elem(out, (r0 + r) * out_ld + j, acc[r], out_bf16);
  }
}

LatPool lat_pool(void* dk, void* dv, void* hk, void* hv, int64_t width, int bf16, int64_t page_len) {
  LatPool p;
  p.dev_k = static_cast<uint8_t*>(dk);
  p.dev_v = static_cast<uint8_t*>(dv);
  p.host_k = static_cast<uint8_t*>(hk);
  p.host_v = static_cast<uint8_t*>(hv);
  p.row_b = width * (bf16 ? 2 : 4);
  p.page_len = (int)page_len;
  p.bf16 = bf16;
  return p;
}

// rows per CTA: 8 while the staged rows fit 96 KB of shared memory
template <typename F8, typename F1>
int with_rb(int64_t cols, F8 f8, F1 f1) {
  return cols * 8 * 4 <= 96 * 1024 ? f8() : f1();
}

}  // namespace

int kv_append_latent_launch(const void* ks, const void* vs, int64_t src_ld, int src_bf16,
                            int64_t d_in, const float* down, int64_t L, void* dk, void* dv,
                            void* hk, void* hv, int pool_bf16, int64_t width, int64_t page_len,
                            const int32_t* slots, int64_t rel0, int64_t t, cudaStream_t st) {
  const LatPool pool = lat_pool(dk, dv, hk, hv, width, pool_bf16, page_len);
  return with_rb(
      d_in,
      [&] {
        const size_t smem = 8 * d_in * 4;
        if (smem > 48 * 1024)
          cudaFuncSetAttribute(latent_append_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        latent_append_kernel<8><<<dim3((unsigned)((t + 7) / 8), 2), kThreads, smem, st>>>(
            ks, vs, src_ld, src_bf16, (int)d_in, down, (int)L, (int)width, pool, slots, rel0, t);
        return (int)cudaGetLastError();
      },
      [&] {
        const size_t smem = d_in * 4;
        if (smem > 48 * 1024)
          cudaFuncSetAttribute(latent_append_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        latent_append_kernel<1><<<dim3((unsigned)t, 2), kThreads, smem, st>>>(
            ks, vs, src_ld, src_bf16, (int)d_in, down, (int)L, (int)width, pool, slots, rel0, t);
        return (int)cudaGetLastError();
      });
}

int kv_gather_latent_launch(void* dk, void* dv, void* hk, void* hv, int pool_bf16, int64_t width,
                            int64_t page_len, const int32_t* slots, const int64_t* tokens,
                            int64_t rel0, int64_t n, int64_t L, const float* up, int64_t d_out,
                            void* ko, void* vo, int64_t out_ld, int out_bf16, cudaStream_t st) {
  const LatPool pool = lat_pool(dk, dv, hk, hv, width, pool_bf16, page_len);
  return with_rb(
      L,
      [&] {
        const size_t smem = 8 * L * 4;
        if (smem > 48 * 1024)
          cudaFuncSetAttribute(latent_gather_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        latent_gather_kernel<8><<<dim3((unsigned)((n + 7) / 8), 2), kThreads, smem, st>>>(
            pool, slots, tokens, rel0, n, (int)L, up, (int)d_out, ko, vo, out_ld, out_bf16);
        return (int)cudaGetLastError();
      },
      [&] {
        const size_t smem = L * 4;
        if (smem > 48 * 1024)
          cudaFuncSetAttribute(latent_gather_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        latent_gather_kernel<1><<<dim3((unsigned)n, 2), kThreads, smem, st>>>(
            pool, slots, tokens, rel0, n, (int)L, up, (int)d_out, ko, vo, out_ld, out_bf16);
        return (int)cudaGetLastError();
      });
}

}  // namespace ifx
