/*
 * ifx_abi.h — C-ABI of libinferix_b200.so, the B200-native (sm_100a) block-diffusion
 * decode hot path. Plain pointers, sizes and opaque handles only: no torch types.
 *
 * The reference (/root/reference/pkg/src/inferix) is pure Python, so it has no FFI of its
 * own; each entry point below names the Python interface it replaces (file:line). The
 * Python façade in paper_2511_20714_b200/ binds these with ctypes.
 *
 * Conventions
 *   - Every function returns int status: IFX_OK (0) or one of IFX_E* below. The message of
 *     the last failure on the calling thread is available from ifx_last_error().
 *   - Status codes map 1:1 onto the reference exception classes (errors.py:4-33).
 *   - `stream` is a cudaStream_t passed as void*; kernels are enqueued on it, never synced.
 *   - Device pointers are borrowed for the duration of the enqueued work.
 *   - Token/row counts are int64.
 */
#ifndef IFX_ABI_H
#define IFX_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-33) -------------------------------------------------- */
#define IFX_OK 0
#define IFX_EDIM 1      /* DimensionError  (errors.py:8)  */
#define IFX_EMASK 2     /* MaskError       (errors.py:12) */
#define IFX_ECAPACITY 3 /* CapacityError   (errors.py:16) */
#define IFX_ERANGE 4    /* OutOfRangeError (errors.py:20) */
#define IFX_ECONFIG 5   /* ConfigError     (errors.py:24) */
#define IFX_ECUDA 16    /* CUDA runtime/driver failure (no reference equivalent) */
#define IFX_EUNSUPPORTED 17
#define IFX_ENCCL 18    /* NCCL failure, or NCCL not loadable (ifx_comm_*) */

/* stream kinds (kvcache.py:75-76) */
#define IFX_SELF_ATTN 0
#define IFX_CROSS_ATTN 1

/* element types of device buffers */
#define IFX_F32 0
#define IFX_BF16 1

const char* ifx_last_error(void);
int ifx_version(void);

/* =====================================================================================
 * Page table: bit-exact bookkeeping of KvCache (kvcache.py:105-404), host C++.
 * It decides ids, tiers, LRU, eviction and block entries exactly as the reference does,
 * and the physical slot of every page in the device / pinned-host pools (below).
 * ===================================================================================*/
typedef struct ifx_pagetable ifx_pagetable;

/* KvCache.__init__ / KvConfig.validate (kvcache.py:33-58,108-122) */
int ifx_pt_create(int64_t num_layers, int64_t head_dim, int64_t page_len,
                  int64_t capacity_pages_device, int64_t capacity_pages_host,
                  ifx_pagetable** out);
void ifx_pt_destroy(ifx_pagetable* pt);

/* KvCache.append_block bookkeeping (kvcache.py:205-234).
 * On success *out_written == t and the block entry is returned through the out params
 * (page ids into out_pages[0..*out_npages), capacity page_cap). On IFX_ECAPACITY the
 * reference has already packed *out_written tokens into pages (kvcache.py:210-223); the
 * caller must still copy those rows. */
int ifx_pt_append(ifx_pagetable* pt, int64_t layer, int kind, int64_t t, int64_t chunk_index,
                  int64_t* out_block_id, int64_t* out_start, int64_t* out_written,
                  int64_t* out_pages, int64_t page_cap, int64_t* out_npages);
/* KvCache.offload_blocks (kvcache.py:236-256) */
int ifx_pt_offload(ifx_pagetable* pt, const int64_t* block_ids, int64_t n, int64_t* out_moved);
/* KvCache.evict_window (kvcache.py:258-285) */
int ifx_pt_evict_window(ifx_pagetable* pt, int64_t keep_last_n_tokens, int64_t* out_freed);
/* KvCache.clear_cross_attention (kvcache.py:287-299) */
int ifx_pt_clear_cross(ifx_pagetable* pt, int64_t* out_cleared);
/* fetch_range bookkeeping: restore-on-read + per-token access clock (kvcache.py:303-339) */
int ifx_pt_touch_range(ifx_pagetable* pt, int64_t layer, int kind, int64_t start, int64_t end);
/* fetch_indices bookkeeping (kvcache.py:341-353) */
int ifx_pt_touch_indices(ifx_pagetable* pt, int64_t layer, int kind, const int64_t* idx,
                         int64_t n);
/* KvCache.addressable_range (kvcache.py:355-357) */
int ifx_pt_range(const ifx_pagetable* pt, int64_t layer, int kind, int64_t* base,
                 int64_t* total);
/* KvCache.memory_stats counters (kvcache.py:359-372): out[0]=device pages, out[1]=host
 * pages, out[2]=addressable tokens, out[3+l]=block entries of layer l */
int ifx_pt_stats(const ifx_pagetable* pt, int64_t* out, int64_t out_cap);
/* Full canonical state as a flat int64 record (layout in pagetable.cpp header comment);
 * *out_len receives the needed length; call with out=NULL to size. */
int ifx_pt_snapshot(const ifx_pagetable* pt, int64_t* out, int64_t cap, int64_t* out_len);

/* ---- physical placement (B200): every page owns a slot of page_len rows in the device
 * pool (tier device) or the mapped pinned host pool (tier host) of its kind. Tier changes
 * made by a call (restore-on-read, LRU demotion, offload) are logged as page moves. */

/* Drain the logged page moves as records of 5 int64 (epoch, kind, dir, device slot, host
 * slot); dir 0 = device -> host, 1 = host -> device. Records are in execution order: per
 * logging call, all dir-0 moves then all dir-1 moves (each group is hazard-free, so it is
 * one ifx_kv_move_pages launch). out == NULL: only *n_records is set, nothing drained.
 * Fails with IFX_ECONFIG while a batch is open (its pages still index the move log). */
int ifx_pt_drain_moves(ifx_pagetable* pt, int64_t* out, int64_t cap, int64_t* n_records);
/* Group the following calls into one move batch (one epoch): a page restored by one call
 * and demoted again by a later one before the drain (the LRU churn of fetching a whole
 * context that exceeds the device tier) cancels instead of moving twice. Batches nest;
 * drain after the outermost end, before reading the data. */
int ifx_pt_batch_begin(ifx_pagetable* pt);
int ifx_pt_batch_end(ifx_pagetable* pt);
/* Pending work of the open epoch: out3[0] = live moves, out3[1] = demotions still waiting
 * for a host slot (each needs one at the drain, on top of the slots in use), out3[2] = those
 * of them on self-attention streams of layers <= max_layer (in a layer-ordered context fetch
 * they will not be restored again before the batch ends). A caller whose host pool cannot
 * absorb the committed ones closes the batch early (drain, run, reopen). */
int ifx_pt_pending(const ifx_pagetable* pt, int64_t max_layer, int64_t* out3);
/* slots ever used per pool: out4[kind*2 + tier] (tier 0 device, 1 host) */
int ifx_pt_pool_extent(const ifx_pagetable* pt, int64_t* out4);
/* Slot codes of the pages covering tokens [start, end) of a stream (within its stored
 * pages, which may begin below the addressable base after window eviction), in order:
 * code >= 0 = device slot, code < 0 = host slot -1-code. *first_token = start token of the
 * first page (page k covers [first_token + k*page_len, ...)); out == NULL sizes *n. */
int ifx_pt_slots(ifx_pagetable* pt, int64_t layer, int kind, int64_t start, int64_t end,
                 int32_t* out, int64_t cap, int64_t* first_token, int64_t* n);

/* =====================================================================================
 * KV data kernels (HBM-bound) over the two pools
 * ===================================================================================*/
typedef struct ifx_kv_pool {
  void* dev_k;    /* device pool [device slots * page_len, width] */
  void* dev_v;
  void* host_k;   /* mapped pinned host pool [host slots * page_len, width] (ifx_host_alloc) */
  void* host_v;
  int64_t width;  /* elements per row */
  int64_t page_len;
  int type;       /* IFX_F32 or IFX_BF16 */
} ifx_kv_pool;

/* K2 — page write for KvCache.append_block (kvcache.py:215-218): rows [0, t) of K and V
 * (src row stride in elements) are tokens [token0, token0 + t) of a stream whose pages,
 * starting at first_token, have the slot codes `slots` (device int32 array, ifx_pt_slots).
 * 128-bit vectorised; src/pool types F32->F32, F32->BF16, BF16->BF16. */
int ifx_kv_append(const void* k_src, const void* v_src, int64_t src_ld, int src_type,
                  const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                  int64_t token0, int64_t t, void* stream);
/* K7 — gather for fetch_range / fetch_indices (kvcache.py:303-353): out row i = token
 * tokens[i] (device int64 array) or, tokens == NULL, token0 + i. Same dtype as the pool. */
int ifx_kv_gather(const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                  const int64_t* tokens, int64_t token0, int64_t n, void* k_out, void* v_out,
                  void* stream);
/* K2L / K7L — latent mode (kvcache.py:26-31,201-203,323-325, MLA-style): the page write
 * stores row . down (down fp32 [d_in, latent_dim] row-major; pool width >= latent_dim, the
 * rest zero) and the gather returns stored_row . up (up fp32 [latent_dim, d_out]) into
 * k_out / v_out (row stride out_ld, IFX_F32 or IFX_BF16), both in fp32 arithmetic inside the
 * copy kernels. Tokens / slots as ifx_kv_append / ifx_kv_gather. */
int ifx_kv_append_latent(const void* k_src, const void* v_src, int64_t src_ld, int src_type,
                         int64_t d_in, const float* down, int64_t latent_dim,
                         const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                         int64_t token0, int64_t t, void* stream);
int ifx_kv_gather_latent(const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                         const int64_t* tokens, int64_t token0, int64_t n, int64_t latent_dim,
                         const float* up, int64_t d_out, void* k_out, void* v_out, int64_t out_ld,
                         int out_type, void* stream);
/* K6 — whole-page copies between the pools (tier moves of ifx_pt_drain_moves, staging of
 * host pages for attention): moves = device int64 [n][2] (device slot, host slot);
 * dir 0 device -> host, 1 host -> device. */
int ifx_kv_move_pages(const ifx_kv_pool* pool, const int64_t* moves, int64_t n, int dir,
                      void* stream);
/* The same page copies on the DMA copy engines instead of SMs: runs = HOST int64
 * [n][3] (device slot, host slot, page count) of consecutive slots on both sides, one
 * cudaMemcpyAsync per run and K/V. Used to stage host pages for attention while K1 holds
 * every SM (a copy kernel would wait for free SMs). */
int ifx_kv_copy_runs(const ifx_kv_pool* pool, const int64_t* runs, int64_t n, int dir,
                     void* stream);
/* pinned host memory mapped into the device address space (cudaHostAllocMapped; under UVA
 * the device address equals the host address) for the host pools */
int ifx_host_alloc(int64_t bytes, void** out);
int ifx_host_free(void* p);
/* Device buffers outside the caller's caching allocator (the host-tier staging buffers:
 * tens of GB allocated and grown rarely; cudaFree synchronises the device). */
int ifx_dev_alloc(int64_t bytes, void** out);
int ifx_dev_free(void* p);

/* =====================================================================================
 * K1 — fused attention of a block's queries over [cached context ∥ the block's own K/V]
 * (engine.py:176-182,206-210 + attention.py:74-94), tcgen05/TMEM/TMA, bf16 in, fp32
 * accumulate. All heads of one [n_q, H*dh] Q matrix in one launch.
 * ===================================================================================*/
typedef struct ifx_attn_params {
  /* Q: [n_q, heads*head_dim] bf16, row stride q_ld elements */
  const void* q;
  int64_t q_ld;
  int64_t n_q;
  /* segment 0 (cached context): rows [ctx_row0, ctx_row0 + n_ctx) of K/V slabs */
  const void* k_ctx;
  const void* v_ctx;
  int64_t ctx_ld;    /* row stride (elements) of the context slabs */
  int64_t ctx_rows;  /* physical rows of the context slabs (TMA extent) */
  int64_t ctx_row0;
  int64_t n_ctx;
  /* segment 1 (the block's own K/V): rows [0, n_cur) */
  const void* k_cur;
  const void* v_cur;
  int64_t cur_ld;
  int64_t n_cur;
  /* output [n_q, heads*head_dim] bf16, row stride o_ld */
  void* o;
  int64_t o_ld;
  int64_t heads;
  int64_t head_dim;  /* 64 or 128 */
  float scale;       /* usually 1/sqrt(head_dim) (attention.py:87) */
  /* optional dense visibility mask, uint8 [n_q, n_ctx + n_cur] row stride mask_ld
   * (attention.py:89); NULL = every key visible (engine.py:209) */
  const uint8_t* mask;
  int64_t mask_ld;
  /* optional partial-softmax statistics (attention.py:127-154): when row_max != NULL the
   * kernel also writes per (head, row) the exact row max (log2 units, [heads, n_q]) and
   * the denominator relative to it, so callers can merge partials (attention.py:157-173) */
  float* row_max;
  float* row_sum;
  /* paged context: when ctx_slots != NULL, k_ctx/v_ctx are device pools [ctx_rows, width]
   * of ctx_page_len-row slots (ifx_kv_pool.dev_k/dev_v) and the context is tokens
   * [ctx_row0, ctx_row0 + n_ctx) of a stream whose pages, from ctx_first_token on, are in
   * slots ctx_slots[] (device int32): code c >= 0 is slot c of the pool, c < 0 is slot
   * -1-c of the staging pool k_stage/v_stage [stage_rows, width] (same row stride), where
   * the caller copied host-tier pages (ifx_kv_move_pages). ctx_page_len must divide 128
   * and be a multiple of 8 (whole 1 KB swizzle atoms per TMA box). */
  const int32_t* ctx_slots;
  int64_t ctx_page_len;
  int64_t ctx_first_token;
  const void* k_stage;
  const void* v_stage;
  int64_t stage_rows;
  /* optional (paged): per 128-key tile of the context, counted from ctx_first_token, the
   * code of its first page when the tile's pages are consecutive slots of one pool (device
   * codes ascending or staging codes descending), else INT32_MIN. Lets K1 load such a
   * tile as one 128-row box with one table read; NULL = K1 checks the slots itself. */
  const int32_t* ctx_tile_runs;
  /* optional device scratch for split-KV (size from ifx_attn_workspace_bytes). When given
   * and (query tiles x heads) would leave the SMs under-filled (e.g. a Ulysses rank holding
   * few heads), the key range is split across CTAs and merged by a combine kernel
   * (attention.py:157-180 semantics). NULL = never split. Not combined with row_max. */
  void* workspace;
  int64_t workspace_bytes;
  /* optional O scatter over peer memory (the Ulysses head->sequence re-shard fused into
   * the epilogue, replaces parallel.py:164-169's output all-to-all): when o_peer_rows > 0,
   * output row r is sequence row g = o_row0 + r, stored at row g % o_peer_rows of
   * o_peer[g / o_peer_rows] (a peer's buffer mapped into this process, ifx_ipc_open; row
   * stride o_ld, head h at column h*head_dim from that pointer); `o` is then unused */
  void* o_peer[8];
  int64_t o_peer_rows;
  int64_t o_row0;
} ifx_attn_params;

int ifx_attn_fwd(const ifx_attn_params* p, void* stream);
/* bytes of `workspace` that allow ifx_attn_fwd to split the key range up to 8 ways */
int ifx_attn_workspace_bytes(const ifx_attn_params* p, int64_t* bytes);

/* K4 alone — merge n_splits attention partials over disjoint key shards (attention.py:
 * 157-180; the ring strategies, parallel.py:172-298): part_o [n_splits, n_q, part_ld] bf16
 * normalised outputs (heads*head_dim columns), part_m / part_l [n_splits, heads, n_q] fp32
 * row max (log2 units, -inf = no visible key) and denominator w.r.t. it — exactly what
 * ifx_attn_fwd writes with row_max / row_sum set. o = sum_s w_s O_s / sum_s w_s, w_s =
 * l_s 2^(m_s - max m); if row_max != NULL the merged max / denominator are written too
 * (denominator 0 = the row saw no key in any shard). n_splits <= 32. */
int ifx_attn_combine(const void* part_o, int64_t part_ld, const float* part_m,
                     const float* part_l, int64_t n_splits, int64_t n_q, int64_t heads,
                     int64_t head_dim, void* o, int64_t o_ld, float* row_max, float* row_sum,
                     void* stream);

/* Fused RMS-norm (engine.py:171-173) + optional time conditioning, fp32 in, bf16 out:
 * y = bf16( (x + t*tvec) / sqrt(mean((x + t*tvec)^2) + eps) ). If x_out != NULL the
 * conditioned fp32 row is also written there. tvec may be NULL. */
int ifx_rms_bf16(const float* x, int64_t rows, int64_t width, const float* tvec, float t,
                 float* x_out, void* y, void* stream);

/* Folded cross-attention (engine.py:211-215 with the prompt's few keys): the logits of all
 * heads come from one GEMM, s = rms(x) @ (cq . K^T) [rows, groups*group_size] fp32 (row
 * stride ld); this writes p = bf16(softmax over each group of group_size logits * scale)
 * (row stride p_ld), which then meets (V . co) in one more GEMM. */
int ifx_group_softmax(const float* s, int64_t rows, int64_t groups, int64_t group_size,
                      int64_t ld, float scale, void* p, int64_t p_ld, void* stream);
/* The same with the logits' RMS row scale still to apply (s = bf16(x) . W rather than
 * rms(x) . W): row r's logits are scaled by rsqrt(sum_p rs_part[r * rs_ld + p] / rs_dim +
 * 1e-6) first (the statistics G1's residual epilogue emitted, engine.py:171-173). */
int ifx_group_softmax_rs(const float* s, int64_t rows, int64_t groups, int64_t group_size,
                         int64_t ld, float scale, void* p, int64_t p_ld, const float* rs_part,
                         int64_t rs_ld, int64_t rs_parts, int64_t rs_dim, void* stream);

/* 3D RoPE (B200 extension; the reference has no positional encoding, attention.py:6):
 * rotate, in place, the interleaved pairs (2k, 2k+1), k < pairs, of every head of the Q
 * columns [q_col0 + h*head_stride, ...) and K columns [k_col0 + ...) of `rows` bf16 rows
 * (row stride ld) by the angle whose cos/sin are tables[(tab_row0 + r) * pairs + k] (fp32).
 * Applied once after the QKV projection, so cached K is stored post-RoPE. Semantics:
 * oracle/rope.py (Wan2.1-style frame/row/column split of the head dims). */
int ifx_rope_qk(void* qkv, int64_t rows, int64_t ld, int64_t heads, int64_t head_stride,
                int64_t pairs, int64_t q_col0, int64_t k_col0, const float* cos_t,
                const float* sin_t, int64_t tab_row0, void* stream);

/* Ulysses head<->sequence re-shard (parallel.py:150-169). A row-major [n][groups][world]
 * [chunk] activation (e.g. groups=3 for fused Q|K|V, each split into per-peer head chunks)
 * is packed as [world][n][groups][chunk] so one all-to-all moves every peer's heads
 * contiguously; unpack is the inverse. Element type F32 or BF16; chunk*size % 16 == 0. */
int ifx_ulysses_pack(const void* src, int64_t n, int64_t groups, int64_t world, int64_t chunk,
                     int64_t src_ld, int type, void* dst, void* stream);
int ifx_ulysses_unpack(const void* src, int64_t n, int64_t groups, int64_t world, int64_t chunk,
                       int type, void* dst, int64_t dst_ld, void* stream);

/* K5b — Ulysses re-shard when heads do not divide the ranks (balanced query split): copy
 * n_blocks 2-D byte blocks from src to dst in one launch. desc = DEVICE int64 [n][6]:
 * (src offset, src row stride, dst offset, dst row stride, rows, row bytes), all in bytes,
 * row bytes a multiple of 16; max_rows = the largest block's row count. */
int ifx_copy_blocks(const void* src, void* dst, const int64_t* desc, int64_t n_blocks,
                    int64_t max_rows, void* stream);

/* Peer memory over NVLink / NVSwitch (the Ulysses exchange without NCCL on the data
 * path). ifx_ipc_handle: the 64-byte CUDA IPC handle of a buffer from ifx_dev_alloc (the
 * ranks exchange them through torch.distributed: plumbing only); ifx_ipc_open maps a
 * peer's handle into this process (peer access enabled lazily), ifx_ipc_close unmaps. */
int ifx_ipc_handle(const void* dev_ptr, void* handle_out);
int ifx_ipc_open(const void* handle, void** dev_ptr_out);
int ifx_ipc_close(void* dev_ptr);
/* Strided copy by the DMA copy engines (any direction; peers' mapped buffers included):
 * `rows` rows of width_bytes from src (pitch spitch bytes) to dst (pitch dpitch). */
int ifx_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                 int64_t rows, void* stream);
/* Barrier across the ranks of a peer mesh, enqueued on `stream` (graph-capturable): every
 * store this GPU issued before it (earlier kernels on the stream, e.g. a scatter epilogue
 * into peers' buffers) is visible to every peer after it, and vice versa. pads = host
 * array of `world` device pointers, pads[p] = peer p's signal pad (uint32[8], zeroed
 * before first use); counter = this rank's own device uint32 epoch (starts at 0). A peer
 * that does not arrive within ~timeout_ms traps (a CUDA error instead of a hang). */
int ifx_peer_barrier(void* const* pads, int world, int rank, uint32_t* counter, int timeout_ms,
                     void* stream);

/* NCCL communicator for hosts that run the Ulysses exchange without torch.distributed
 * (SURVEY §8(b) `ifx_comm_init`; replaces the reference's WorkerGroup / all_to_all,
 * parallel.py:63-111, with a real collective over NVLink / NVSwitch). NCCL is loaded on
 * first use (dlopen libnccl.so.2); IFX_ENCCL when it is absent or a call fails.
 * ifx_comm_unique_id: 128 opaque bytes, made on rank 0 and sent to every rank out of band.
 * ifx_comm_init: this rank's communicator on the CURRENT CUDA device (collective over the
 * `world` ranks). ifx_comm_all_to_all: the variable-size byte all-to-all of the Ulysses
 * re-shard (what UlyssesComm.a2a_var does over torch.distributed): host arrays of `world`
 * byte offsets / sizes into the DEVICE buffers send / recv, enqueued on `stream`.
 * ifx_comm_all_gather: `bytes` from every rank into recv[rank * bytes] (e.g. the 64-byte
 * CUDA IPC handles a peer mesh needs, copied to device first). */
typedef struct ifx_comm ifx_comm;
int ifx_comm_unique_id(void* id_out);
int ifx_comm_init(const void* id, int world, int rank, ifx_comm** out);
int ifx_comm_destroy(ifx_comm* comm);
int ifx_comm_size(const ifx_comm* comm, int* world, int* rank);
int ifx_comm_all_to_all(ifx_comm* comm, const void* send, const int64_t* send_off,
                        const int64_t* send_bytes, void* recv, const int64_t* recv_off,
                        const int64_t* recv_bytes, void* stream);
int ifx_comm_all_gather(ifx_comm* comm, const void* send, int64_t bytes, void* recv, void* stream);

/* Dense projection on cuBLASLt (a plain library GEMM; per-shape algorithm choice timed on
 * the first call outside a CUDA-graph capture): D[M,N] = relu?(A[M,K] . B[K,N] + beta * D),
 * row-major bf16 A (row stride lda) and B (ldb), fp32 accumulate, D fp32 or bf16 (ldd). */
int ifx_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                  int d_type, int64_t M, int64_t N, int64_t K, float beta, int relu, void* stream);

/* G1 — the dense projections as a hand-written persistent tcgen05/TMA GEMM with fused
 * epilogues (engine.py:202-205 h @ wq/wk/wv, :210 @ wo, :215 cross, :217-218 FFN, :220
 * eps; the page write of kvcache.py:179-234 on the clean pass, engine.py:303-306):
 *   C[m, n] = f(A[m, :] . B[:, n]) with A bf16 [M, K] (row stride lda), B bf16 [K, N]
 *   (ldb), fp32 accumulation; C bf16, or fp32 with C = beta * C + f(.) (the residual).
 * f, in order: row scale (rs_part != NULL: x rsqrt(sum_p rs_part[m * rs_ld + p] / rs_dim +
 * rs_eps), the RMS norm of the fp32 row A was copied from, engine.py:171-173), ReLU, 3D RoPE
 * (rope_cos != NULL: pairs (2i, 2i+1), i < rope_pairs, of each head (stride rope_hs) of
 * the column blocks at rope_q0 and rope_k0, rotated by row m's angle i, tables
 * [(rope_row0 + m) * rope_pairs + i]). With fp32 C and emit_b != NULL the new row is also
 * written as bf16 to emit_b and partial sums of its squares (one per half column tile) to
 * emit_ss[m * emit_ss_ld + part] (*out_tiles_n = parts per row: the consumer's rs_parts).
 * page_pool != NULL (bf16 C only): columns [page_k_col0, +pool width) of row m are also
 * written to token page_token0 + m of the K stream whose pages start at page_first_token
 * with slot codes page_slots (device int32, as ifx_kv_append), [page_v_col0, ...) to V.
 * N % 8 == 0; 16-byte aligned operands. */
typedef struct ifx_gemm_params {
  const void* a; int64_t lda;
  const void* b; int64_t ldb;
  void* c; int64_t ldc; int c_type;
  int relu;
  int64_t m, n, k;
  float beta;
  float rs_eps;
  const float* rs_part; int64_t rs_ld; int64_t rs_parts; int64_t rs_dim;
  void* emit_b; int64_t emit_ld;
  float* emit_ss; int64_t emit_ss_ld;
  const float* rope_cos; const float* rope_sin;
  int64_t rope_row0, rope_q0, rope_k0, rope_pairs, rope_hs, rope_heads;
  const ifx_kv_pool* page_pool; const int32_t* page_slots;
  int64_t page_first_token, page_token0, page_k_col0, page_v_col0;
  /* optional peer scatter of the bf16 output (the Ulysses sequence->head re-shard fused
   * into the epilogue, replaces parallel.py:150-160's all-to-all): column block
   * b = col / scatter_w (scatter_blocks of them) goes to up to two destinations, DEVICE
   * int64 scatter[(b*2 + e)*4 + {0,1,2,3}] = {address, row stride in bytes, row_lo,
   * row_hi}: row r in [row_lo, row_hi) is stored at address + r*stride + (col % scatter_w)*2
   * (rows outside are skipped; row_hi = 0 marks an unused entry); scatter_w is a multiple
   * of 32. Addresses are this
   * process's mappings of peers' buffers (ifx_ipc_open). c may then be NULL. */
  const int64_t* scatter; int64_t scatter_w; int64_t scatter_blocks;
} ifx_gemm_params;
int ifx_gemm_fused(const ifx_gemm_params* p, int64_t* out_tiles_n, void* stream);
/* sum-of-squares parts per row G1 emits for an [M, N] = [M, K] . [K, N] output (the
 * emit_ss width needed) */
int ifx_gemm_tiles_n(int64_t m, int64_t n, int64_t k, int64_t* out_tiles_n);

/* Initial block noise, host side (engine.py:280-282): writes the first n values of
 * np.random.default_rng([seed, chunk]).standard_normal(...).astype(float32) into `out`
 * (host memory, e.g. pinned), bit-identically, using `threads` host threads (0 = all).
 * pcg_state = {state_hi, state_lo, inc_hi, inc_lo} of the seeded PCG64 bit generator
 * (Generator.bit_generator.state["state"]). Ziggurat = numpy 2.3's own routine. */
int ifx_noise_normal_f32(const uint64_t pcg_state[4], int64_t n, float* out, int threads);

#ifdef __cplusplus
}
#endif
#endif /* IFX_ABI_H */
