// attn_kernel.h — device-side argument block of K1 (attn_fwd_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ifx {

struct AttnKernelArgs {
  CUtensorMap tm_q;   // Q       [n_q, H*dh]   box 64 x 128, SW128
  CUtensorMap tm_kc;  // K slab  [rows, H*dh]
  CUtensorMap tm_vc;  // V slab
  CUtensorMap tm_kn;  // K of the current block [n_cur, H*dh]
  CUtensorMap tm_vn;  // V of the current block
  int n_q, n_ctx, n_cur, ctx_row0;
  float scale_log2;   // scale * log2(e)
  int pad_;
  __nv_bfloat16* o;
  int64_t o_ld;
  const uint8_t* mask;
  int64_t mask_ld;
  float* row_max;
  float* row_sum;
};

// Grid (ceil(n_q/128), heads) x 320 threads. Returns cudaError_t.
int attn_fwd_launch(const AttnKernelArgs& a, int head_dim, int n_q, int heads, cudaStream_t st);

}  // namespace ifx
