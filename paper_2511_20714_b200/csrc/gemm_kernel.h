// gemm_kernel.h — device-side argument block of G1 (gemm_sm100.cu), the engine's dense
// projections as a persistent tcgen05/TMA GEMM with the work either side fused into its
// epilogue (RMS row scale, ReLU, fp32 residual, next-norm statistics, 3D RoPE, page write).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ifx {

struct GemmArgs {
  CUtensorMap tm_a;  // A bf16 [M, K] row-major (K-major operand), box 64 x 128, SW128
  CUtensorMap tm_b;  // B bf16 [K, N] row-major (MN-major operand), box 64 (N) x 64 (K), SW128
  int M, N, K;
  int tiles_m, tiles_n;
  // ---- output: C[M, N] = epi(acc) (bf16), or fp32 C = beta * C + epi(acc)
  void* c;
  int64_t ldc;
  int c_f32;
  float beta;
  int relu;
  // ---- row scale (the consumer side of the RMS norm, engine.py:171-173): acc row r is
  // multiplied by rsqrt(sum_p rs_part[r * rs_ld + p] * rs_inv_d + rs_eps); rs_part holds the
  // producer's per-column-tile sums of squares of the fp32 row whose bf16 copy is A
  const float* rs_part;
  int rs_parts;
  int64_t rs_ld;
  float rs_inv_d, rs_eps;
  // ---- next-norm statistics (fp32 output only): the new fp32 row is also written as bf16
  // to emit_b (the next GEMM's A) and its sum of squares over this tile's columns to
  // emit_ss[r * emit_ss_ld + tile_n] (no atomics: the consumer sums tiles in a fixed order)
  __nv_bfloat16* emit_b;
  int64_t emit_ld;
  float* emit_ss;
  int64_t emit_ss_ld;
  // ---- 3D RoPE on column ranges [q0, q0 + heads*hs) and [k0, k0 + heads*hs): pair (2i,
  // 2i+1) of a head (i < pairs) rotated by row r's angle i: cos/sin [(row0 + r) * pairs + i]
  const float* rope_cos;
  const float* rope_sin;
  int64_t rope_row0, rope_q0, rope_k0;
  int rope_pairs, rope_hs, rope_heads, rope_vec;  // rope_vec: tables 16-byte aligned rows
  // ---- page write (KvCache.append_block, kvcache.py:179-234, fused): columns
  // [pk_col0, pk_col0 + pwidth) of row r are token (rel0 + r) of the K stream, columns
  // [pv_col0, ...) of the V stream; its page's slot code slots[(rel0 + r) / page_len]
  // (>= 0 device slot, < 0 host slot -1-c of the mapped pinned pool), rows of prow_b bytes
  const int32_t* slots;
  uint8_t* pk_dev;
  uint8_t* pv_dev;
  uint8_t* pk_host;
  uint8_t* pv_host;
  int64_t prow_b, rel0, pk_col0, pv_col0, pwidth;
  int page_len, pad1_;
  // ---- peer scatter (bf16 output; the Ulysses sequence->head re-shard fused): column block
  // b = col / scat_w goes to <= 2 destinations scat[(b*2 + e)*4 + {addr, row stride bytes,
  // row_lo, row_hi}]; rows outside [row_lo, row_hi) skipped. c may be null then.
  const int64_t* scat;
  int scat_w, scat_blocks;
};

// Persistent launch (<= one CTA per SM), BN in {64, 128, 192, 256}; mode 1: one CTA per
// 128 x BN tile; 2: clusters of two column tiles sharing A by multicast (tm_a box 64 rows);
// 3: cta_group::2 CTA pairs per 256 x BN tile (BN 128 / 256; tiles_m counts 256-row
// tiles). Returns cudaError_t.
int gemm_launch(const GemmArgs& a, int bn, int mode, cudaStream_t st);
void gemm_plan(int64_t M, int64_t N, int64_t K, int n_sm, int* bn_out, int* mode_out);

}  // namespace ifx
