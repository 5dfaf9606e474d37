// kv_kernels.h — launchers of the HBM-bound kernels in kv_ops.cu (return cudaError_t).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ifx {
int kv_append_launch(const void* ks, const void* vs, int64_t src_ld, int src_bf16, void* dk,
                     void* dv, void* hk, void* hv, int pool_bf16, int64_t width, int64_t page_len,
                     const int32_t* slots, int64_t rel0, int64_t t, cudaStream_t st);
int kv_gather_launch(void* dk, void* dv, void* hk, void* hv, int esz, int64_t width,
                     int64_t page_len, const int32_t* slots, const int64_t* tokens, int64_t rel0,
                     int64_t n, void* ko, void* vo, cudaStream_t st);
int kv_append_latent_launch(const void* ks, const void* vs, int64_t src_ld, int src_bf16,
                            int64_t d_in, const float* down, int64_t L, void* dk, void* dv,
                            void* hk, void* hv, int pool_bf16, int64_t width, int64_t page_len,
                            const int32_t* slots, int64_t rel0, int64_t t, cudaStream_t st);
int kv_gather_latent_launch(void* dk, void* dv, void* hk, void* hv, int pool_bf16, int64_t width,
                            int64_t page_len, const int32_t* slots, const int64_t* tokens,
                            int64_t rel0, int64_t n, int64_t L, const float* up, int64_t d_out,
                            void* ko, void* vo, int64_t out_ld, int out_bf16, cudaStream_t st);
int kv_move_launch(void* dk, void* dv, void* hk, void* hv, int esz, int64_t width,
                   int64_t page_len, const int64_t* moves, int64_t n, int dir, cudaStream_t st);
int copy_blocks_launch(const void* src, void* dst, const int64_t* desc, int64_t n_blocks,
                       int64_t max_rows, cudaStream_t st);
int group_softmax_launch(const float* s, int64_t rows, int groups, int gs, int64_t ld,
                         float scale_log2, void* p, int64_t p_ld, const float* rs_part,
                         int rs_parts, int64_t rs_ld, float rs_inv_d, float rs_eps,
                         cudaStream_t st);
int rms_launch(const float* x, int64_t rows, int64_t width, const float* tvec, float t,
               float* x_out, void* y, cudaStream_t st);
int rope_launch(void* qkv, int64_t rows, int64_t ld, int heads, int64_t head_stride, int pairs,
                int64_t q_col0, int64_t k_col0, const float* cos_t, const float* sin_t,
                int64_t tab_row0, cudaStream_t st);
int ulysses_launch(const void* src, void* dst, int64_t n, int64_t groups, int64_t world,
                   int64_t chunk_bytes, int64_t ld_bytes, bool pack, cudaStream_t st);
}  // namespace ifx
