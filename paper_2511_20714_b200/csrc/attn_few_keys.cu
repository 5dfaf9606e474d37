// attn_few_keys.cu — K1s: attention over a handful of keys (cross-attention to the prompt).
//
// Same semantics as K1 (engine.py:211-215 cross-attention through `_mha`, attention.py:
// 74-94: softmax(q k^T * scale) v, every key visible) for n_keys <= kMaxKeys. With 3 prompt
// tokens a 128x128 tcgen05 tile is 98 % padding and K1's fixed per-CTA cost (TMEM alloc,
// barrier setup, Q tile load, epilogue) dominates (~30 us per launch at the c2 shape);
// this is a memory-bound SIMT kernel instead: the keys/values of every head are staged in
// shared memory once per CTA, one warp per (query row, head) with head_dim/32 dims per
// lane, dot products reduced with warp shuffles, fp32 softmax, bf16 out. Traffic = read Q +
// write O (~29 MB at the c2 shape).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn_kernel.h"

namespace ifx {
namespace {

constexpr int kMaxKeys = 32;

template <int HD>
__global__ void __launch_bounds__(256) attn_few_keys_kernel(FewKeysArgs a) {
  constexpr int PER = HD / 32;  // dims per lane (2 or 4)
  extern __shared__ __nv_bfloat16 kv[];  // [2][n_keys][heads*HD]
  const int width = a.heads * HD;
  const int nk = a.n_ctx + a.n_cur;
  // stage K and V of all heads (rows from the two segments), 16-byte vectors
  const int vec_per_row = width / 8;
  for (int i = threadIdx.x; i < 2 * nk * vec_per_row; i += blockDim.x) {
    const int which = i / (nk * vec_per_row);
    const int r = (i / vec_per_row) % nk;
    const int c = i % vec_per_row;
    const __nv_bfloat16* src =
        r < a.n_ctx ? (which ? a.v_ctx : a.k_ctx) + (int64_t)r * a.ctx_ld
                    : (which ? a.v_cur : a.k_cur) + (int64_t)(r - a.n_ctx) * a.cur_ld;
    reinterpret_cast<uint4*>(kv + ((int64_t)which * nk + r) * width)[c] =
        reinterpret_cast<const uint4*>(src)[c];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t n_tasks = (int64_t)a.n_q * a.heads;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < n_tasks;
       t += warps) {
    const int64_t row = t / a.heads;
    const int head = (int)(t % a.heads);
    const int col = head * HD + lane * PER;
    float q[PER];
    const __nv_bfloat16* qp = a.q + row * a.q_ld + col;
#pragma unroll
    for (int e = 0; e < PER; e += 2) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qp + e));
      q[e] = f.x;
      q[e + 1] = f.y;
    }
    float s[kMaxKeys];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j) {
      if (j < nk) {
        const __nv_bfloat16* kp = kv + (int64_t)j * width + col;
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < PER; e += 2) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(kp + e));
          d = fmaf(q[e], f.x, fmaf(q[e + 1], f.y, d));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        s[j] = d * a.scale_log2;
        m = fmaxf(m, s[j]);
      }
    }
    float acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
    float l = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j) {
      if (j < nk) {
        const float p = exp2f(s[j] - m);
        l += p;
        const __nv_bfloat16* vp = kv + ((int64_t)nk + j) * width + col;
#pragma unroll
        for (int e = 0; e < PER; e += 2) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vp + e));
          acc[e] = fmaf(p, f.x, acc[e]);
          acc[e + 1] = fmaf(p, f.y, acc[e + 1]);
        }
      }
    }
    const float inv = 1.f / l;
    __nv_bfloat16* op = a.o + row * a.o_ld + col;
#pragma unroll
    for (int e = 0; e < PER; e += 2)
      *reinterpret_cast<__nv_bfloat162*>(op + e) = __floats2bfloat162_rn(acc[e] * inv, acc[e + 1] * inv);
  }
}

}  // namespace

int attn_few_keys_max() { return kMaxKeys; }

int attn_few_keys_launch(const FewKeysArgs& a, int head_dim, cudaStream_t st) {
  const int nk = a.n_ctx + a.n_cur;
  if (nk < 1 || nk > kMaxKeys || (head_dim != 64 && head_dim != 128)) return -1;
  const size_t smem = (size_t)2 * nk * a.heads * head_dim * sizeof(__nv_bfloat16);
  const int64_t tasks = (int64_t)a.n_q * a.heads;
  int blocks = (int)((tasks + 7) / 8);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  if (head_dim == 128) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(attn_few_keys_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_few_keys_kernel<128><<<blocks, 256, smem, st>>>(a);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(attn_few_keys_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_few_keys_kernel<64><<<blocks, 256, smem, st>>>(a);
  }
  return (int)cudaGetLastError();
}

}  // namespace ifx
