// attn_kernel.h — device-side argument block of K1 (attn_fwd_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ifx {

struct AttnKernelArgs {
  CUtensorMap tm_q;   // Q       [n_q, H*dh]   box 64 x 128, SW128
  CUtensorMap tm_kc;  // K context [rows, H*dh] (contiguous: box 128 rows; paged: box page_len)
  CUtensorMap tm_vc;  // V context
  CUtensorMap tm_ks;  // paged only: K staging pool (slot codes < 0), box page_len
  CUtensorMap tm_vs;  // V staging pool
  CUtensorMap tm_kc_run;  // paged only: the pools again with 128-row boxes, for tiles whose
  CUtensorMap tm_vc_run;  // pages are one consecutive run of slots
  CUtensorMap tm_ks_run;
  CUtensorMap tm_vs_run;
  CUtensorMap tm_kn;  // K of the current block [n_cur, H*dh]
  CUtensorMap tm_vn;  // V of the current block
  int n_q, n_ctx, n_cur, ctx_row0;
  float scale_log2;   // scale * log2(e)
  // paged context (ctx_slots != nullptr): context rows [0, n_ctx) counted from the start of
  // the first page; row r lives in slot code c = ctx_slots[r / page_len]: c >= 0 slot c of
  // the pool (tm_kc/tm_vc), c < 0 slot -1-c of the staging pool (tm_ks/tm_vs); rows
  // [0, ctx_lo) precede the addressable window and are masked
  int ctx_lo;
  const int32_t* ctx_slots;
  const int32_t* ctx_tile_runs;  // optional: per 128-key tile, run start code or INT32_MIN
  int ctx_page_len;
  int pad_;
  __nv_bfloat16* o;
  int64_t o_ld;
  const uint8_t* mask;
  int64_t mask_ld;
  float* row_max;
  float* row_sum;
  // split-KV (grid.z = n_splits > 1): partials merged by the K4 combine kernel
  int heads, n_splits;
  __nv_bfloat16* part_o;  // [n_splits, n_q, part_ld] normalised partial outputs
  int64_t part_ld;
  float* part_m;          // [n_splits, heads, n_q] max (log2 units)
  float* part_l;          // [n_splits, heads, n_q] denominator w.r.t. part_m
  // O scatter over peer memory (o_peer_rows > 0; the Ulysses head->sequence re-shard fused
  // into the epilogue): output row r is sequence row g = o_row0 + r, stored at row
  // g % o_peer_rows of o_peer[g / o_peer_rows] (row stride o_ld)
  __nv_bfloat16* o_peer[8];
  int o_peer_rows, o_row0;
};

// Destination of output row `r` (before the head's column offset).
__device__ __forceinline__ __nv_bfloat16* attn_out_row(const AttnKernelArgs& a, int r) {
  if (a.o_peer_rows > 0) {
    const int g = a.o_row0 + r;
    const int p = g / a.o_peer_rows;
    return a.o_peer[p] + (int64_t)(g - p * a.o_peer_rows) * a.o_ld;
  }
  return a.o + (int64_t)r * a.o_ld;
}

// K1s (attn_few_keys.cu): attention over <= attn_few_keys_max() keys, SIMT
struct FewKeysArgs {
  const __nv_bfloat16* q;
  int64_t q_ld;
  const __nv_bfloat16 *k_ctx, *v_ctx;
  int64_t ctx_ld;
  const __nv_bfloat16 *k_cur, *v_cur;
  int64_t cur_ld;
  __nv_bfloat16* o;
  int64_t o_ld;
  int n_q, n_ctx, n_cur, heads;
  float scale_log2;
};
int attn_few_keys_max();
int attn_few_keys_launch(const FewKeysArgs& a, int head_dim, cudaStream_t st);

// Grid (ceil(n_q/128), heads, n_splits) x 320 threads (+ K4 combine when n_splits > 1).
// Returns cudaError_t.
int attn_fwd_launch(const AttnKernelArgs& a, int head_dim, int n_q, int heads, cudaStream_t st);
// K4 alone over a.n_splits partials (part_o / part_m / part_l) into a.o.
int attn_combine_launch(const AttnKernelArgs& a, int head_dim, cudaStream_t st);

}  // namespace ifx
