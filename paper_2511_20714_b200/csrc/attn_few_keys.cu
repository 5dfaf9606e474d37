// attn_few_keys.cu — K1s: attention over a handful of keys (cross-attention to the prompt).
//
// Same semantics as K1 (engine.py:211-215 cross-attention through `_mha`, attention.py:
// 74-94: softmax(q k^T * scale) v, every key visible) for n_keys <= kMaxKeys. With 3 prompt
// tokens a 128x128 tcgen05 tile is 98 % padding and K1's fixed per-CTA cost (TMEM alloc,
// barrier setup, Q tile load, epilogue) dominates (~30 us per launch at the c2 shape);
// this is a memory-bound SIMT kernel instead: four threads per (query row, head), the few
// K/V rows read through L1 as broadcasts, fp32 softmax, bf16 out. Traffic = read Q + write
// O (~29 MB at the c2 shape).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn_kernel.h"
#include "launch.cuh"

namespace ifx {
namespace {

constexpr int kMaxKeysAll = 32;

__device__ __forceinline__ void bf16x8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}

// FOUR threads per (query row, head), each owning head_dim/4 contiguous dims (fully
// unrolled 16-byte loads: all of a thread's q bytes are in flight at once); partial dot
// products are combined with two xor-shuffles inside the 4-lane group. A warp covers 8
// consecutive rows of one head, so its K / V reads (a few hundred bytes per head, read
// through L1) are 8-way broadcasts.
template <int HD, int kMaxKeys>
__global__ void __launch_bounds__(256) attn_few_keys_kernel(FewKeysArgs a) {
  pdl_wait();
  constexpr int DPT = HD / 4;      // dims per thread
  constexpr int VPT = DPT / 8;     // 16-byte vectors per thread
  const int nk = a.n_ctx + a.n_cur;
  const int sub = threadIdx.x & 3;
  const int64_t n_tasks = (int64_t)a.n_q * a.heads;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 2);
  // the 4 threads of a group iterate the same tasks: group-masked shuffles stay converged
  const unsigned gmask = 0xFu << (threadIdx.x & 28);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 2) + (threadIdx.x >> 2); t < n_tasks;
       t += stride) {
    const int head = (int)(t / a.n_q);
    const int64_t row = t - (int64_t)head * a.n_q;
    const int d0 = head * HD + sub * DPT;
    const uint4* qp = reinterpret_cast<const uint4*>(a.q + row * a.q_ld + d0);
    uint4 u[VPT];
#pragma unroll
    for (int c = 0; c < VPT; ++c) u[c] = __ldg(qp + c);
    float s[kMaxKeys];
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j) s[j] = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j) {
      if (j < nk) {
        const __nv_bfloat16* kr = (j < a.n_ctx ? a.k_ctx + (int64_t)j * a.ctx_ld
                                              : a.k_cur + (int64_t)(j - a.n_ctx) * a.cur_ld) + d0;
#pragma unroll
        for (int c = 0; c < VPT; ++c) {
          float q[8], k[8];
          bf16x8(u[c], q);
          bf16x8(__ldg(reinterpret_cast<const uint4*>(kr) + c), k);
#pragma unroll
          for (int e = 0; e < 8; ++e) s[j] = fmaf(q[e], k[e], s[j]);
        }
      }
    }
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j)
      if (j < nk) {
        s[j] += __shfl_xor_sync(gmask, s[j], 1);
        s[j] += __shfl_xor_sync(gmask, s[j], 2);
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
    uint4* op = reinterpret_cast<uint4*>(a.o + row * a.o_ld + d0);
#pragma unroll
    for (int c = 0; c < VPT; ++c) {
      float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < kMaxKeys; ++j) {
        if (j < nk) {
          const __nv_bfloat16* vr = (j < a.n_ctx ? a.v_ctx + (int64_t)j * a.ctx_ld
                                                : a.v_cur + (int64_t)(j - a.n_ctx) * a.cur_ld) + d0;
          float v[8];
          bf16x8(__ldg(reinterpret_cast<const uint4*>(vr) + c), v);
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = fmaf(s[j], v[e], o[e]);
        }
      }
      __nv_bfloat162 b[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) b[e] = __floats2bfloat162_rn(o[2 * e] * inv, o[2 * e + 1] * inv);
      op[c] = *reinterpret_cast<const uint4*>(b);
    }
  }
}

}  // namespace

int attn_few_keys_max() { return kMaxKeysAll; }

template <int HD, int MAXK>
static int launch_fk(const FewKeysArgs& a, size_t, int blocks, cudaStream_t st) {
  launch_pdl(attn_few_keys_kernel<HD, MAXK>, dim3(blocks), dim3(256), 0, st, 1, a);
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
  int blocks = (int)((tasks + 63) / 64);  // 64 (row, head) tasks per 256-thread CTA
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  return head_dim == 128 ? launch_fk_hd<128>(a, smem, blocks, st) : launch_fk_hd<64>(a, smem, blocks, st);
}

}  // namespace ifx
