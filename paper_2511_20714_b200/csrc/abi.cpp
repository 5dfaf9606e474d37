// abi.cpp — extern "C" entry points of libinferix_b200.so (declared in include/ifx_abi.h):
// argument validation, TMA tensor-map encoding, status-code / last-error plumbing.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/ifx_abi.h"
#include "attn_kernel.h"
#include "common_host.h"
#include "device_state.h"
#include "gemm_kernel.h"
#include "kv_kernels.h"

namespace ifx {

static thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static int cuda_fail(int err, const char* what) {
  if (err == 0) return IFX_OK;
  return fail(IFX_ECUDA, std::string(what) + ": " + cudaGetErrorString((cudaError_t)err));
}

static int check_pool(const ifx_kv_pool* p) {
  if (p == nullptr || p->width <= 0 || p->page_len <= 0) return fail(IFX_EDIM, "bad pool");
  const int esz = p->type == IFX_BF16 ? 2 : 4;
  if ((p->width * esz) % 16) return fail(IFX_EDIM, "row width must be a multiple of 16 bytes");
  if ((reinterpret_cast<uintptr_t>(p->dev_k) | reinterpret_cast<uintptr_t>(p->dev_v) |
       reinterpret_cast<uintptr_t>(p->host_k) | reinterpret_cast<uintptr_t>(p->host_v)) & 15)
    return fail(IFX_EDIM, "pools must be 16-byte aligned");
  return IFX_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// bf16 matrix [rows, cols] with row stride ld (elements); box = 64 cols x box_rows, SW128.
static int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld,
                    int box_rows = 128) {
  std::memset(m, 0, sizeof(*m));
  if (base == nullptr || rows <= 0) return IFX_OK;  // unused segment
  auto fn = encode_fn();
  if (!fn) return fail(IFX_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 2) & 15))
    return fail(IFX_EDIM, "TMA operands need 16-byte aligned base and row stride");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(IFX_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return IFX_OK;
}

int num_sms();
int64_t split_workspace_bytes(const ifx_attn_params* p, int splits);
int choose_splits(const ifx_attn_params* p);

int attn_fwd(const ifx_attn_params* p, void* stream) {
  if (p->head_dim != 64 && p->head_dim != 128)
    return fail(IFX_EUNSUPPORTED, "head_dim must be 64 or 128");
  if (p->heads < 1 || p->n_q < 0 || p->n_ctx < 0 || p->n_cur < 0)
    return fail(IFX_EDIM, "bad attention sizes");
  if (p->n_ctx + p->n_cur == 0 && p->n_q > 0) return fail(IFX_EMASK, "query row with no allowed key");
  if (p->n_q == 0) return IFX_OK;
  const bool paged = p->ctx_slots != nullptr && p->n_ctx > 0;
  if (paged) {
    const int64_t pl = p->ctx_page_len;
    if (pl < 8 || pl > 128 || 128 % pl || pl % 8)
      return fail(IFX_EUNSUPPORTED, "paged attention needs page_len in {8, 16, 32, 64, 128}");
    if (p->ctx_row0 < p->ctx_first_token) return fail(IFX_ERANGE, "context before its first page");
    if (p->mask != nullptr) return fail(IFX_EUNSUPPORTED, "dense masks need a contiguous context");
    if (p->ctx_rows % pl) return fail(IFX_EDIM, "pool rows must be whole slots");
  } else if (p->n_ctx > 0 && p->ctx_row0 + p->n_ctx > p->ctx_rows) {
    return fail(IFX_ERANGE, "context rows outside the slab");
  }
  const int64_t width = p->heads * p->head_dim;
  if (p->n_q > INT32_MAX || p->ctx_rows > INT32_MAX || p->n_cur > INT32_MAX)
    return fail(IFX_EDIM, "attention extents must fit int32");
  // a handful of keys (cross-attention to the prompt): K1s, SIMT, no tensor-core tile
  static const bool few_keys_off = std::getenv("IFX_NO_FEW_KEYS") != nullptr;  // A/B probes
  const bool scatter = p->o_peer_rows > 0;
  if (scatter) {
    const int64_t n_peers = (p->o_row0 + p->n_q + p->o_peer_rows - 1) / p->o_peer_rows;
    if (p->o_row0 < 0 || n_peers > 8 || p->o_row0 + p->n_q > INT32_MAX)
      return fail(IFX_EDIM, "O scatter rows outside the 8 peers");
    for (int64_t i = p->o_row0 / p->o_peer_rows; i < n_peers; ++i)
      if (p->o_peer[i] == nullptr || (reinterpret_cast<uintptr_t>(p->o_peer[i]) & 15))
        return fail(IFX_EDIM, "O scatter needs a 16-byte aligned buffer for every peer it reaches");
    if ((p->o_ld * 2) % 16) return fail(IFX_EDIM, "O scatter row stride must be 16-byte aligned");
  }
  if (!few_keys_off && !scatter && !paged && p->mask == nullptr && p->row_max == nullptr &&
      p->n_ctx + p->n_cur <= attn_few_keys_max() && p->n_q * p->heads >= 1024 &&
      ((p->q_ld | p->ctx_ld | p->cur_ld | p->o_ld | width) % 8) == 0 &&
      ((reinterpret_cast<uintptr_t>(p->k_ctx) | reinterpret_cast<uintptr_t>(p->v_ctx) |
        reinterpret_cast<uintptr_t>(p->k_cur) | reinterpret_cast<uintptr_t>(p->v_cur) |
        reinterpret_cast<uintptr_t>(p->q) | reinterpret_cast<uintptr_t>(p->o)) & 15) == 0) {
    FewKeysArgs f;
    f.q = static_cast<const __nv_bfloat16*>(p->q);
    f.q_ld = p->q_ld;
    f.k_ctx = static_cast<const __nv_bfloat16*>(p->k_ctx) + p->ctx_row0 * p->ctx_ld;
    f.v_ctx = static_cast<const __nv_bfloat16*>(p->v_ctx) + p->ctx_row0 * p->ctx_ld;
    f.ctx_ld = p->ctx_ld;
    f.k_cur = static_cast<const __nv_bfloat16*>(p->k_cur);
    f.v_cur = static_cast<const __nv_bfloat16*>(p->v_cur);
    f.cur_ld = p->cur_ld;
    f.o = static_cast<__nv_bfloat16*>(p->o);
    f.o_ld = p->o_ld;
    f.n_q = (int)p->n_q;
    f.n_ctx = (int)p->n_ctx;
    f.n_cur = (int)p->n_cur;
    f.heads = (int)p->heads;
    f.scale_log2 = p->scale * 1.4426950408889634f;
    return cuda_fail(attn_few_keys_launch(f, (int)p->head_dim, static_cast<cudaStream_t>(stream)),
                     "attn_few_keys launch");
  }
  AttnKernelArgs a;
  std::memset(&a, 0, sizeof(a));
  int rc;
  if ((rc = make_map(&a.tm_q, p->q, p->n_q, width, p->q_ld))) return rc;
  if (p->n_ctx > 0) {
    const int box = paged ? (int)p->ctx_page_len : 128;
    if ((rc = make_map(&a.tm_kc, p->k_ctx, p->ctx_rows, width, p->ctx_ld, box))) return rc;
    if ((rc = make_map(&a.tm_vc, p->v_ctx, p->ctx_rows, width, p->ctx_ld, box))) return rc;
    if (paged) {
      if ((rc = make_map(&a.tm_kc_run, p->k_ctx, p->ctx_rows, width, p->ctx_ld))) return rc;
      if ((rc = make_map(&a.tm_vc_run, p->v_ctx, p->ctx_rows, width, p->ctx_ld))) return rc;
    }
    if (paged && p->k_stage != nullptr && p->stage_rows > 0) {
      if (p->stage_rows % p->ctx_page_len) return fail(IFX_EDIM, "staging rows must be whole slots");
      if ((rc = make_map(&a.tm_ks, p->k_stage, p->stage_rows, width, p->ctx_ld, box))) return rc;
      if ((rc = make_map(&a.tm_vs, p->v_stage, p->stage_rows, width, p->ctx_ld, box))) return rc;
      if ((rc = make_map(&a.tm_ks_run, p->k_stage, p->stage_rows, width, p->ctx_ld))) return rc;
      if ((rc = make_map(&a.tm_vs_run, p->v_stage, p->stage_rows, width, p->ctx_ld))) return rc;
    }
  }
  if (p->n_cur > 0) {
    if ((rc = make_map(&a.tm_kn, p->k_cur, p->n_cur, width, p->cur_ld))) return rc;
    if ((rc = make_map(&a.tm_vn, p->v_cur, p->n_cur, width, p->cur_ld))) return rc;
  }
  a.n_q = (int)p->n_q;
  a.n_ctx = (int)p->n_ctx;
  a.n_cur = (int)p->n_cur;
  a.ctx_row0 = (int)p->ctx_row0;
  if (paged) {
    const int64_t lo = p->ctx_row0 - p->ctx_first_token;
    if (lo + p->n_ctx > INT32_MAX) return fail(IFX_EDIM, "attention extents must fit int32");
    a.ctx_slots = p->ctx_slots;
    a.ctx_tile_runs = p->ctx_tile_runs;
    a.ctx_page_len = (int)p->ctx_page_len;
    a.ctx_lo = (int)lo;
    a.n_ctx = (int)(lo + p->n_ctx);  // rows from the first page's start
    a.ctx_row0 = 0;
  }
  a.scale_log2 = p->scale * 1.4426950408889634f;
  a.o = static_cast<__nv_bfloat16*>(p->o);
  a.o_ld = p->o_ld;
  if (scatter) {
    for (int i = 0; i < 8; ++i) a.o_peer[i] = static_cast<__nv_bfloat16*>(p->o_peer[i]);
    a.o_peer_rows = (int)p->o_peer_rows;
    a.o_row0 = (int)p->o_row0;
  }
  a.mask = p->mask;
  a.mask_ld = p->mask_ld;
  a.row_max = p->row_max;
  a.row_sum = p->row_sum;
  a.heads = (int)p->heads;
  a.n_splits = p->row_max != nullptr ? 1 : choose_splits(p);
  if (a.n_splits > 1) {
    char* ws = static_cast<char*>(p->workspace);
    a.part_o = reinterpret_cast<__nv_bfloat16*>(ws);
    a.part_ld = width;
    a.part_m = reinterpret_cast<float*>(ws + a.n_splits * p->n_q * width * 2);
    a.part_l = a.part_m + a.n_splits * p->heads * p->n_q;
  }
  int e = attn_fwd_launch(a, (int)p->head_dim, (int)p->n_q, (int)p->heads,
                          static_cast<cudaStream_t>(stream));
  return cuda_fail(e, "attn_fwd launch");
}

int num_sms() {  // of the CURRENT device (a process may drive several)
  int dev = 0;
  cudaGetDevice(&dev);
  return device_sms(dev);
}

int64_t split_workspace_bytes(const ifx_attn_params* p, int splits) {
  const int64_t width = p->heads * p->head_dim;
  return splits * p->n_q * width * 2 + 2 * splits * p->heads * p->n_q * 4 + 256;
}

// Split the key range only when (query tiles x heads) CTAs leave the SMs under-filled:
// pick the split count with the best wave efficiency (ctas*s / sms / ceil(ctas*s / sms)),
// at least 16 key tiles per split, within the caller's workspace.
int choose_splits(const ifx_attn_params* p) {
  if (p->workspace == nullptr) return 1;
  const int sms = num_sms();
  const int64_t ctas = ((p->n_q + 127) / 128) * p->heads;
  if (ctas >= 3 * sms) return 1;
  const int64_t lo = p->ctx_slots != nullptr ? p->ctx_row0 - p->ctx_first_token : 0;
  const int64_t tiles = (lo + p->n_ctx + 127) / 128 + (p->n_cur + 127) / 128;
  auto eff = [&](int s) {
    const double w = (double)(ctas * s) / sms;
    return w / std::ceil(w);
  };
  static const int min_tiles = [] {  // key tiles per split at least (A/B: IFX_K1_MIN_SPLIT_TILES)
    const char* e = std::getenv("IFX_K1_MIN_SPLIT_TILES");
    return e ? std::max(1, std::atoi(e)) : 16;
  }();
  int best = 1;
  double best_eff = eff(1);
  for (int s = 2; s <= 8 && tiles / s >= min_tiles; ++s) {
    if (p->workspace_bytes < split_workspace_bytes(p, s)) break;
    if (eff(s) > best_eff + 0.05) {
      best = s;
      best_eff = eff(s);
    }
  }
  return best;
}

// G1 (gemm_sm100.cu): validation + tensor maps; the epilogue options are documented at
// ifx_gemm_params in include/ifx_abi.h.
int gemm_fused(const ifx_gemm_params* p, int64_t* out_tiles_n, void* stream) {
  const bool scat = p->scatter != nullptr;
  if (p->m < 0 || p->n < 1 || p->k < 1 || p->lda < p->k || p->ldb < p->n ||
      (p->c != nullptr && p->ldc < p->n) || (p->c == nullptr && !scat))
    return fail(IFX_EDIM, "bad GEMM sizes");
  if (scat && (p->c_type != IFX_BF16 || p->scatter_w < 32 || p->scatter_w % 32 ||
               p->scatter_w * p->scatter_blocks < p->n || p->scatter_w > INT32_MAX ||
               p->scatter_blocks > INT32_MAX))
    return fail(IFX_EDIM, "peer scatter needs a bf16 output in 32-column-aligned blocks covering N");
  if (p->n % 8) return fail(IFX_EDIM, "GEMM N must be a multiple of 8");
  if (p->m > INT32_MAX || p->n > INT32_MAX || p->k > INT32_MAX)
    return fail(IFX_EDIM, "GEMM extents must fit int32");
  const bool f32 = p->c_type == IFX_F32;
  if (!f32 && p->c_type != IFX_BF16) return fail(IFX_EUNSUPPORTED, "C must be fp32 or bf16");
  const int esz = f32 ? 4 : 2;
  auto mis = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) != 0; };
  if (mis(p->c) || (p->ldc * esz) % 16) return fail(IFX_EDIM, "C must be 16-byte aligned");
  if (!f32 && (p->beta != 0.f || p->emit_b != nullptr))
    return fail(IFX_EUNSUPPORTED, "beta / emit need an fp32 C");
  if (p->emit_b != nullptr && (mis(p->emit_b) || (p->emit_ld * 2) % 16 || p->emit_ss == nullptr))
    return fail(IFX_EDIM, "emit needs a 16-byte aligned bf16 row buffer and a sum-of-squares buffer");
  const int n_sm = num_sms();
  int bn = 0, mode = 0;
  gemm_plan(p->m, p->n, p->k, n_sm, &bn, &mode);
  GemmArgs a;
  std::memset(&a, 0, sizeof(a));
  a.M = (int)p->m;
  a.N = (int)p->n;
  a.K = (int)p->k;
  a.tiles_m = (int)(mode == 3 ? (p->m + 255) / 256 : (p->m + 127) / 128);
  a.tiles_n = (int)((p->n + bn - 1) / bn);
  // sums of squares per row: one per (column tile, epilogue half)
  if (out_tiles_n) *out_tiles_n = 2 * a.tiles_n;
  if (p->emit_b != nullptr && p->emit_ss_ld < 2 * a.tiles_n)
    return fail(IFX_EDIM, "emit_ss_ld smaller than the sum-of-squares part count");
  if (p->m == 0) return IFX_OK;
  int rc;
  if ((rc = make_map(&a.tm_a, p->a, p->m, p->k, p->lda, mode == 2 ? 64 : 128))) return rc;
  if ((rc = make_map(&a.tm_b, p->b, p->k, p->n, p->ldb, 64))) return rc;
  a.c = p->c;
  a.ldc = p->ldc;
  a.c_f32 = f32;
  if (scat) {
    a.scat = p->scatter;
    a.scat_w = (int)p->scatter_w;
    a.scat_blocks = (int)p->scatter_blocks;
  }
  a.beta = p->beta;
  a.relu = p->relu;
  if (p->rs_part != nullptr) {
    if (p->rs_parts < 1 || p->rs_ld < p->rs_parts || p->rs_dim < 1)
      return fail(IFX_EDIM, "bad row-scale statistics");
    a.rs_part = p->rs_part;
    a.rs_parts = (int)p->rs_parts;
    a.rs_ld = p->rs_ld;
    a.rs_inv_d = 1.f / (float)p->rs_dim;
    a.rs_eps = p->rs_eps;
  }
  a.emit_b = static_cast<__nv_bfloat16*>(p->emit_b);
  a.emit_ld = p->emit_ld;
  a.emit_ss = p->emit_b != nullptr ? p->emit_ss : nullptr;
  a.emit_ss_ld = p->emit_ss_ld;
  if (p->rope_cos != nullptr) {
    if (p->rope_hs % 32 || p->rope_q0 % 32 || p->rope_k0 % 32 || p->rope_pairs * 2 > p->rope_hs ||
        p->rope_heads < 1 || p->rope_sin == nullptr)
      return fail(IFX_EDIM, "RoPE heads must be 32-column aligned");
    a.rope_cos = p->rope_cos;
    a.rope_sin = p->rope_sin;
    a.rope_row0 = p->rope_row0;
    a.rope_q0 = p->rope_q0;
    a.rope_k0 = p->rope_k0;
    a.rope_pairs = (int)p->rope_pairs;
    a.rope_hs = (int)p->rope_hs;
    a.rope_heads = (int)p->rope_heads;
    a.rope_vec = (p->rope_pairs % 4 == 0 && ((reinterpret_cast<uintptr_t>(p->rope_cos) |
                                               reinterpret_cast<uintptr_t>(p->rope_sin)) & 15) == 0);
  }
  if (p->page_pool != nullptr) {
    const ifx_kv_pool* pool = p->page_pool;
    if (int r2 = check_pool(pool)) return r2;
    if (f32 || pool->type != IFX_BF16) return fail(IFX_EUNSUPPORTED, "fused page write is bf16 -> bf16");
    if (pool->width % 32 || p->page_k_col0 % 32 || p->page_v_col0 % 32 ||
        p->page_k_col0 + pool->width > p->n || p->page_v_col0 + pool->width > p->n)
      return fail(IFX_EDIM, "page-write columns must be 32-aligned blocks inside C");
    if (p->page_token0 < p->page_first_token || p->page_slots == nullptr)
      return fail(IFX_EDIM, "bad page-write tokens");
    a.slots = p->page_slots;
    a.pk_dev = static_cast<uint8_t*>(pool->dev_k);
    a.pv_dev = static_cast<uint8_t*>(pool->dev_v);
    a.pk_host = static_cast<uint8_t*>(pool->host_k);
    a.pv_host = static_cast<uint8_t*>(pool->host_v);
    a.prow_b = pool->width * 2;
    a.rel0 = p->page_token0 - p->page_first_token;
    a.pk_col0 = p->page_k_col0;
    a.pv_col0 = p->page_v_col0;
    a.pwidth = pool->width;
    a.page_len = (int)pool->page_len;
  }
  return cuda_fail(gemm_launch(a, bn, mode, static_cast<cudaStream_t>(stream)), "gemm launch");
}

}  // namespace ifx

extern "C" {

const char* ifx_last_error(void) { return ifx::g_last_error.c_str(); }
int ifx_version(void) { return 1; }

int ifx_attn_fwd(const ifx_attn_params* p, void* stream) { return ifx::attn_fwd(p, stream); }

int ifx_attn_combine(const void* part_o, int64_t part_ld, const float* part_m,
                     const float* part_l, int64_t n_splits, int64_t n_q, int64_t heads,
                     int64_t head_dim, void* o, int64_t o_ld, float* row_max, float* row_sum,
                     void* stream) {
  if (head_dim != 64 && head_dim != 128) return ifx::fail(IFX_EUNSUPPORTED, "head_dim must be 64 or 128");
  if (n_splits < 1 || n_splits > 32 || n_q < 0 || heads < 1 || part_ld < heads * head_dim ||
      o_ld < heads * head_dim ||
      n_q > INT32_MAX || n_splits > INT32_MAX)
    return ifx::fail(IFX_EDIM, "bad combine sizes");
  if (part_o == nullptr || part_m == nullptr || part_l == nullptr || o == nullptr ||
      (row_max == nullptr) != (row_sum == nullptr))
    return ifx::fail(IFX_EDIM, "combine: null operand");
  if (n_q == 0) return IFX_OK;
  ifx::AttnKernelArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_q = (int)n_q;
  a.heads = (int)heads;
  a.n_splits = (int)n_splits;
  a.part_o = static_cast<__nv_bfloat16*>(const_cast<void*>(part_o));
  a.part_ld = part_ld;
  a.part_m = const_cast<float*>(part_m);
  a.part_l = const_cast<float*>(part_l);
  a.o = static_cast<__nv_bfloat16*>(o);
  a.o_ld = o_ld;
  a.row_max = row_max;
  a.row_sum = row_sum;
  return ifx::cuda_fail(ifx::attn_combine_launch(a, (int)head_dim, static_cast<cudaStream_t>(stream)),
                        "attn_combine launch");
}

int ifx_attn_workspace_bytes(const ifx_attn_params* p, int64_t* bytes) {
  *bytes = ifx::split_workspace_bytes(p, 8);
  return IFX_OK;
}


int ifx_kv_append(const void* k_src, const void* v_src, int64_t src_ld, int src_type,
                  const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                  int64_t token0, int64_t t, void* stream) {
  if (int rc = ifx::check_pool(pool)) return rc;
  if (t < 0 || token0 < first_token) return ifx::fail(IFX_EDIM, "bad append sizes");
  if (t == 0) return IFX_OK;
  if (src_type == IFX_BF16 && pool->type == IFX_F32)
    return ifx::fail(IFX_EUNSUPPORTED, "bf16 -> fp32 append not supported");
  const int ssz = src_type == IFX_BF16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(k_src) | reinterpret_cast<uintptr_t>(v_src)) & 15 ||
      (src_ld * ssz) % 16)
    return ifx::fail(IFX_EDIM, "append operands must be 16-byte aligned");
  int e = ifx::kv_append_launch(k_src, v_src, src_ld, src_type == IFX_BF16, pool->dev_k,
                                pool->dev_v, pool->host_k, pool->host_v, pool->type == IFX_BF16,
                                pool->width, pool->page_len, slots, token0 - first_token, t,
                                static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "kv_append launch");
}

int ifx_kv_append_latent(const void* k_src, const void* v_src, int64_t src_ld, int src_type,
                         int64_t d_in, const float* down, int64_t latent_dim,
                         const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                         int64_t token0, int64_t t, void* stream) {
  if (int rc = ifx::check_pool(pool)) return rc;
  if (t < 0 || token0 < first_token || d_in < 1 || latent_dim < 1 || latent_dim > pool->width ||
      src_ld < d_in || down == nullptr)
    return ifx::fail(IFX_EDIM, "bad latent append sizes");
  if (t == 0) return IFX_OK;
  int e = ifx::kv_append_latent_launch(k_src, v_src, src_ld, src_type == IFX_BF16, d_in, down,
                                       latent_dim, pool->dev_k, pool->dev_v, pool->host_k,
                                       pool->host_v, pool->type == IFX_BF16, pool->width,
                                       pool->page_len, slots, token0 - first_token, t,
                                       static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "kv_append_latent launch");
}

int ifx_kv_gather_latent(const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                         const int64_t* tokens, int64_t token0, int64_t n, int64_t latent_dim,
                         const float* up, int64_t d_out, void* k_out, void* v_out, int64_t out_ld,
                         int out_type, void* stream) {
  if (int rc = ifx::check_pool(pool)) return rc;
  if (n < 0 || latent_dim < 1 || latent_dim > pool->width || d_out < 1 || out_ld < d_out ||
      up == nullptr)
    return ifx::fail(IFX_EDIM, "bad latent gather sizes");
  if (n == 0) return IFX_OK;
  int e = ifx::kv_gather_latent_launch(pool->dev_k, pool->dev_v, pool->host_k, pool->host_v,
                                       pool->type == IFX_BF16, pool->width, pool->page_len, slots,
                                       tokens, tokens ? first_token : token0 - first_token, n,
                                       latent_dim, up, d_out, k_out, v_out, out_ld,
                                       out_type == IFX_BF16, static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "kv_gather_latent launch");
}

int ifx_kv_gather(const ifx_kv_pool* pool, const int32_t* slots, int64_t first_token,
                  const int64_t* tokens, int64_t token0, int64_t n, void* k_out, void* v_out,
                  void* stream) {
  if (int rc = ifx::check_pool(pool)) return rc;
  if (n < 0) return ifx::fail(IFX_EDIM, "bad gather sizes");
  if (n == 0) return IFX_OK;
  const int esz = pool->type == IFX_BF16 ? 2 : 4;
  int e = ifx::kv_gather_launch(pool->dev_k, pool->dev_v, pool->host_k, pool->host_v, esz,
                                pool->width, pool->page_len, slots, tokens,
                                tokens ? first_token : token0 - first_token, n, k_out, v_out,
                                static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "kv_gather launch");
}

int ifx_kv_move_pages(const ifx_kv_pool* pool, const int64_t* moves, int64_t n, int dir,
                      void* stream) {
  if (int rc = ifx::check_pool(pool)) return rc;
  if (n < 0 || (dir != 0 && dir != 1)) return ifx::fail(IFX_EDIM, "bad page move batch");
  if (n == 0) return IFX_OK;
  const int esz = pool->type == IFX_BF16 ? 2 : 4;
  int e = ifx::kv_move_launch(pool->dev_k, pool->dev_v, pool->host_k, pool->host_v, esz,
                              pool->width, pool->page_len, moves, n, dir,
                              static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "kv_move_pages launch");
}

int ifx_kv_copy_runs(const ifx_kv_pool* pool, const int64_t* runs, int64_t n, int dir,
                     void* stream) {
  if (int rc = ifx::check_pool(pool)) return rc;
  if (n < 0 || (dir != 0 && dir != 1)) return ifx::fail(IFX_EDIM, "bad page run batch");
  const int esz = pool->type == IFX_BF16 ? 2 : 4;
  const int64_t slot_b = pool->page_len * pool->width * esz;
  auto st = static_cast<cudaStream_t>(stream);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t ds = runs[3 * i], hs = runs[3 * i + 1], cnt = runs[3 * i + 2];
    if (ds < 0 || hs < 0 || cnt < 1) return ifx::fail(IFX_EDIM, "bad page run");
    for (int kv = 0; kv < 2; ++kv) {
      char* dev = static_cast<char*>(kv ? pool->dev_v : pool->dev_k) + ds * slot_b;
      char* host = static_cast<char*>(kv ? pool->host_v : pool->host_k) + hs * slot_b;
      cudaError_t e = dir == 1 ? cudaMemcpyAsync(dev, host, cnt * slot_b, cudaMemcpyHostToDevice, st)
                               : cudaMemcpyAsync(host, dev, cnt * slot_b, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return ifx::cuda_fail((int)e, "kv_copy_runs");
    }
  }
  return IFX_OK;
}

int ifx_host_alloc(int64_t bytes, void** out) {
  *out = nullptr;
  if (bytes <= 0) return IFX_OK;
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable | cudaHostAllocMapped);
  if (e != cudaSuccess) return ifx::cuda_fail((int)e, "cudaHostAlloc");
  void* d = nullptr;
  e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess || d != p) {  // UVA: the mapped device address is the host address
    cudaFreeHost(p);
    return ifx::fail(IFX_ECUDA, "pinned host pool is not mapped at its host address (no UVA?)");
  }
  *out = p;
  return IFX_OK;
}

int ifx_host_free(void* p) {
  if (p == nullptr) return IFX_OK;
  return ifx::cuda_fail((int)cudaFreeHost(p), "cudaFreeHost");
}

int ifx_dev_alloc(int64_t bytes, void** out) {
  *out = nullptr;
  if (bytes <= 0) return IFX_OK;
  return ifx::cuda_fail((int)cudaMalloc(out, (size_t)bytes), "cudaMalloc");
}

int ifx_dev_free(void* p) {
  if (p == nullptr) return IFX_OK;
  return ifx::cuda_fail((int)cudaFree(p), "cudaFree");
}

int ifx_rms_bf16(const float* x, int64_t rows, int64_t width, const float* tvec, float t,
                 float* x_out, void* y, void* stream) {
  if (rows < 0 || width <= 0 || width % 4) return ifx::fail(IFX_EDIM, "rms width must be a multiple of 4");
  if (rows == 0) return IFX_OK;
  int e = ifx::rms_launch(x, rows, width, tvec, t, x_out, y, static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "rms launch");
}

int ifx_copy_blocks(const void* src, void* dst, const int64_t* desc, int64_t n_blocks,
                    int64_t max_rows, void* stream) {
  if (n_blocks < 0 || max_rows < 0 || n_blocks > 65535) return ifx::fail(IFX_EDIM, "bad block copy");
  if (n_blocks == 0 || max_rows == 0) return IFX_OK;
  int e = ifx::copy_blocks_launch(src, dst, desc, n_blocks, max_rows,
                                  static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "copy_blocks launch");
}

int ifx_group_softmax(const float* s, int64_t rows, int64_t groups, int64_t group_size,
                      int64_t ld, float scale, void* p, int64_t p_ld, void* stream) {
  return ifx_group_softmax_rs(s, rows, groups, group_size, ld, scale, p, p_ld, nullptr, 0, 0, 1,
                              stream);
}

int ifx_group_softmax_rs(const float* s, int64_t rows, int64_t groups, int64_t group_size,
                         int64_t ld, float scale, void* p, int64_t p_ld, const float* rs_part,
                         int64_t rs_ld, int64_t rs_parts, int64_t rs_dim, void* stream) {
  if (rows < 0 || groups < 1 || group_size < 1 || ld < groups * group_size || p_ld < groups * group_size)
    return ifx::fail(IFX_EDIM, "bad group softmax sizes");
  if (rs_part != nullptr && (rs_parts < 1 || rs_ld < rs_parts || rs_dim < 1))
    return ifx::fail(IFX_EDIM, "bad row-scale statistics");
  if (rows == 0) return IFX_OK;
  int e = ifx::group_softmax_launch(s, rows, (int)groups, (int)group_size, ld,
                                    scale * 1.4426950408889634f, p, p_ld, rs_part, (int)rs_parts,
                                    rs_ld, 1.f / (float)rs_dim, 1e-6f,
                                    static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "group softmax launch");
}

int ifx_rope_qk(void* qkv, int64_t rows, int64_t ld, int64_t heads, int64_t head_stride,
                int64_t pairs, int64_t q_col0, int64_t k_col0, const float* cos_t,
                const float* sin_t, int64_t tab_row0, void* stream) {
  if (rows < 0 || heads < 1 || pairs < 1 || 2 * pairs > head_stride)
    return ifx::fail(IFX_EDIM, "bad rope sizes");
  if ((ld | head_stride | q_col0 | k_col0) & 1)
    return ifx::fail(IFX_EDIM, "rope pairs must be 4-byte aligned");
  if (rows == 0) return IFX_OK;
  int e = ifx::rope_launch(qkv, rows, ld, (int)heads, head_stride, (int)pairs, q_col0, k_col0,
                           cos_t, sin_t, tab_row0, static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "rope launch");
}

int ifx_ulysses_pack(const void* src, int64_t n, int64_t groups, int64_t world, int64_t chunk,
                     int64_t src_ld, int type, void* dst, void* stream) {
  const int esz = type == IFX_BF16 ? 2 : 4;
  if (world < 1 || groups < 1 || chunk < 1 || n < 0) return ifx::fail(IFX_EDIM, "bad re-shard sizes");
  if ((chunk * esz) % 16 || (src_ld * esz) % 16 || src_ld < groups * world * chunk)
    return ifx::fail(IFX_EDIM, "re-shard chunks must be 16-byte multiples inside the row");
  if (n == 0) return IFX_OK;
  int e = ifx::ulysses_launch(src, dst, n, groups, world, chunk * esz, src_ld * esz, true,
                              static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "ulysses pack");
}

int ifx_ulysses_unpack(const void* src, int64_t n, int64_t groups, int64_t world, int64_t chunk,
                       int type, void* dst, int64_t dst_ld, void* stream) {
  const int esz = type == IFX_BF16 ? 2 : 4;
  if (world < 1 || groups < 1 || chunk < 1 || n < 0) return ifx::fail(IFX_EDIM, "bad re-shard sizes");
  if ((chunk * esz) % 16 || (dst_ld * esz) % 16 || dst_ld < groups * world * chunk)
    return ifx::fail(IFX_EDIM, "re-shard chunks must be 16-byte multiples inside the row");
  if (n == 0) return IFX_OK;
  int e = ifx::ulysses_launch(src, dst, n, groups, world, chunk * esz, dst_ld * esz, false,
                              static_cast<cudaStream_t>(stream));
  return ifx::cuda_fail(e, "ulysses unpack");
}

int ifx_gemm_fused(const ifx_gemm_params* p, int64_t* out_tiles_n, void* stream) {
  return ifx::gemm_fused(p, out_tiles_n, stream);
}

int ifx_gemm_tiles_n(int64_t m, int64_t n, int64_t k, int64_t* out_tiles_n) {
  if (m < 0 || n < 1 || out_tiles_n == nullptr) return ifx::fail(IFX_EDIM, "bad GEMM sizes");
  int bn = 0, mode = 0;
  ifx::gemm_plan(m, n, k, ifx::num_sms(), &bn, &mode);
  *out_tiles_n = 2 * ((n + bn - 1) / bn);
  return IFX_OK;
}

}  // extern "C"
