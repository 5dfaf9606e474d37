// attn_few_keys.cu — K1s: attention over a handful of keys (cross-attention to the prompt).
//
// Same semantics as K1 (engine.py:211-215 cross-attention through `_mha`, attention.py:
// 74-94: softmax(q k^T * scale) v, every key visible) for n_keys <= kMaxKeys. With 3 prompt
// tokens a 128x128 tcgen05 tile is 98 % padding and K1's fixed per-CTA cost (TMEM alloc,
// barrier setup, Q tile load, epilogue) dominates (~30 us per launch at the c2 shape);
// this is a memory-bound SIMT kernel instead: the keys/values of every head are staged in
// shared memory (fp32) once per CTA, one thread per (query row, head), fp32 softmax, bf16
// out. Traffic = read Q + write O (~29 MB at the c2 shape).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn_kernel.h"

namespace ifx {
namespace {

constexpr int kMaxKeysAll = 32;

// One THREAD per (query row, head); the 32 threads of a warp take 32 consecutive rows of the
// same head, so every K / V read from shared memory is a broadcast. Each thread streams its
// q row (head_dim bf16, 16-byte loads) once for the dot products, then writes its output
// row; no cross-lane reductions, many independent loads in flight per thread.
template <int HD, int kMaxKeys>
__global__ void __launch_bounds__(256) attn_few_keys_kernel(FewKeysArgs a) {
  extern __shared__ float kvf[];  // [2][n_keys][heads*HD] fp32
  const int width = a.heads * HD;
  const int nk = a.n_ctx + a.n_cur;
  for (int i = threadIdx.x; i < 2 * nk * width / 2; i += blockDim.x) {
    const int e = 2 * i;
    const int which = e / (nk * width);
    const int r = (e / width) % nk;
    const int c = e % width;
    const __nv_bfloat16* src =
        r < a.n_ctx ? (which ? a.v_ctx : a.k_ctx) + (int64_t)r * a.ctx_ld
                    : (which ? a.v_cur : a.k_cur) + (int64_t)(r - a.n_ctx) * a.cur_ld;
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(src + c));
    kvf[e] = f.x;
    kvf[e + 1] = f.y;
  }
  __syncthreads();
  const int64_t n_tasks = (int64_t)a.n_q * a.heads;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tasks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int head = (int)(t / a.n_q);
    const int64_t row = t - (int64_t)head * a.n_q;
    const uint4* qp = reinterpret_cast<const uint4*>(a.q + row * a.q_ld + head * HD);
    const float* kh = kvf + head * HD;
    const float* vh = kvf + (int64_t)nk * width + head * HD;
    float s[kMaxKeys];
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j) s[j] = 0.f;
#pragma unroll 2
    for (int c = 0; c < HD / 8; ++c) {  // 8 dims per 16-byte load
      const uint4 u = qp[c];
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
      float q[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
        q[2 * e] = f.x;
        q[2 * e + 1] = f.y;
      }
#pragma unroll
      for (int j = 0; j < kMaxKeys; ++j) {
        if (j < nk) {
          const float4 k0 = *reinterpret_cast<const float4*>(kh + (int64_t)j * width + c * 8);
          const float4 k1 = *reinterpret_cast<const float4*>(kh + (int64_t)j * width + c * 8 + 4);
          s[j] = fmaf(q[0], k0.x, fmaf(q[1], k0.y, fmaf(q[2], k0.z, fmaf(q[3], k0.w, s[j]))));
          s[j] = fmaf(q[4], k1.x, fmaf(q[5], k1.y, fmaf(q[6], k1.z, fmaf(q[7], k1.w, s[j]))));
        }
      }
    }
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j)
      if (j < nk) {
        s[j] *= a.scale_log2;
        m = fmaxf(m, s[j]);
      }
    float l = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j)
      if (j < nk) {
        s[j] = exp2f(s[j] - m);
        l += s[j];
      }
    const float inv = 1.f / l;
    uint4* op = reinterpret_cast<uint4*>(a.o + row * a.o_ld + head * HD);
#pragma unroll 2
    for (int c = 0; c < HD / 8; ++c) {
      float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < kMaxKeys; ++j) {
        if (j < nk) {
          const float4 v0 = *reinterpret_cast<const float4*>(vh + (int64_t)j * width + c * 8);
          const float4 v1 = *reinterpret_cast<const float4*>(vh + (int64_t)j * width + c * 8 + 4);
          o[0] = fmaf(s[j], v0.x, o[0]);
          o[1] = fmaf(s[j], v0.y, o[1]);
          o[2] = fmaf(s[j], v0.z, o[2]);
          o[3] = fmaf(s[j], v0.w, o[3]);
          o[4] = fmaf(s[j], v1.x, o[4]);
          o[5] = fmaf(s[j], v1.y, o[5]);
          o[6] = fmaf(s[j], v1.z, o[6]);
          o[7] = fmaf(s[j], v1.w, o[7]);
        }
      }
      uint4 w;
      __nv_bfloat162 b0 = __floats2bfloat162_rn(o[0] * inv, o[1] * inv);
      __nv_bfloat162 b1 = __floats2bfloat162_rn(o[2] * inv, o[3] * inv);
      __nv_bfloat162 b2 = __floats2bfloat162_rn(o[4] * inv, o[5] * inv);
      __nv_bfloat162 b3 = __floats2bfloat162_rn(o[6] * inv, o[7] * inv);
      w.x = *reinterpret_cast<uint32_t*>(&b0);
      w.y = *reinterpret_cast<uint32_t*>(&b1);
      w.z = *reinterpret_cast<uint32_t*>(&b2);
      w.w = *reinterpret_cast<uint32_t*>(&b3);
      op[c] = w;
    }
  }
}

}  // namespace

int attn_few_keys_max() { return kMaxKeysAll; }

template <int HD, int MAXK>
static int launch_fk(const FewKeysArgs& a, size_t smem, int blocks, cudaStream_t st) {
  auto* fn = attn_few_keys_kernel<HD, MAXK>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  fn<<<blocks, 256, smem, st>>>(a);
  return (int)cudaGetLastError();
}

template <int HD>
static int launch_fk_hd(const FewKeysArgs& a, size_t smem, int blocks, cudaStream_t st) {
  const int nk = a.n_ctx + a.n_cur;
  if (nk <= 4) return launch_fk<HD, 4>(a, smem, blocks, st);  // registers scale with the cap
  if (nk <= 8) return launch_fk<HD, 8>(a, smem, blocks, st);
  if (nk <= 16) return launch_fk<HD, 16>(a, smem, blocks, st);
  return launch_fk<HD, 32>(a, smem, blocks, st);
}

int attn_few_keys_launch(const FewKeysArgs& a, int head_dim, cudaStream_t st) {
  const int nk = a.n_ctx + a.n_cur;
  if (nk < 1 || nk > kMaxKeysAll || (head_dim != 64 && head_dim != 128)) return -1;
  const size_t smem = (size_t)2 * nk * a.heads * head_dim * sizeof(float);
  const int64_t tasks = (int64_t)a.n_q * a.heads;
  int blocks = (int)((tasks + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  return head_dim == 128 ? launch_fk_hd<128>(a, smem, blocks, st) : launch_fk_hd<64>(a, smem, blocks, st);
}

}  // namespace ifx
