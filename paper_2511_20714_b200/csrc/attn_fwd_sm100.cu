// attn_fwd_sm100.cu — K1: attention of one block's queries over [cached context ∥ own K/V].
//
// Replaces the reference's per-head numpy loop `_mha` -> `scaled_dot_attention`
// (/root/reference/pkg/src/inferix/engine.py:176-182,206-210, attention.py:74-94) and the
// context concat it needs. softmax(Q K^T * scale) V with online (flash) softmax; every key
// is visible (engine.py:209) unless a dense mask is given (API parity, attention.py:89).
//
// Blackwell structure (one CTA = one 128-query tile of one head, 1 CTA/SM):
//   warp 0      TMA producer: Q once, then K_j / V_j tiles (128 keys x head_dim) into a
//               2-stage smem ring, 128B-swizzled, completion on mbarriers (tx bytes)
//   warp 1      MMA issuer (one elected lane): S_j = Q K_j^T into TMEM (double-buffered),
//               then O += P_{j-1} V_{j-1} into TMEM; tcgen05.commit frees smem / signals
//   warps 2-5   softmax: thread r owns query row r (TMEM lane r): tcgen05.ld the S row,
//               row max / exp2 / row sum in fp32, lazy O rescale (only when the running
//               max grows by > 2^8), P as bf16 -> smem (SW128, K-major) or TMEM, epilogue
//               O / l -> bf16 -> global.
// Keys come from two segments so the block's own K/V never need to be copied next to the
// cache: segment 0 = slab rows [ctx_row0, ctx_row0 + n_ctx), segment 1 = rows [0, n_cur)
// of the fresh QKV projection. Ragged tails are masked in softmax (TMA zero-fills rows past
// a tensor's extent; rows past a segment end inside the slab are finite and masked).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn_kernel.h"
#include "sm100_ptx.cuh"

namespace ifx {
namespace {

using namespace ptx;

constexpr int BM = 128;          // query rows per CTA (= TMEM lanes)
constexpr int BN = 128;          // keys per tile
constexpr int NS = 2;            // smem stages for K and for V
constexpr int NTHREADS = 192;    // 6 warps
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale O only if max grows > 2^8
constexpr int kPolyEvery = 4;              // every 4th exp2 of a full tile runs on the FMA pipe

// 2^x on the FMA/ALU pipes (round-to-nearest split, cubic on [-0.5, 0.5], exponent add):
// rel. error < 5e-4, far below bf16 P rounding. x is clamped to >= -125 (result ~0).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: low mantissa bits = round(x)
  const float r = t - 12582912.f;
  const float f = x - r;
  const float p = fmaf(fmaf(fmaf(0.0555041087f, f, 0.2402265070f), f, 0.6931471806f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int HD, bool kPInTmem>
struct Layout {
  static constexpr int KCH = HD / 64;                 // 64-column (128 B) chunks of head_dim
  static constexpr int Q_BYTES = BM * HD * 2;
  static constexpr int KV_BYTES = BN * HD * 2;
  static constexpr int P_BYTES = kPInTmem ? 0 : BM * BN * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * KV_BYTES;
  static constexpr int OFF_P = OFF_V + NS * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int NBAR = 1 + 4 * NS + 2 * 4;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;  // + align slack
  // TMEM columns: S0 [0,128) S1 [128,256) O [256, 256+HD); P (TS mode) aliases S[b] cols [64,128)
  static constexpr uint32_t TM_O = 256;
  static constexpr uint32_t TM_P_OFF = 64;
};

struct Tile {
  int seg;    // 0 ctx, 1 cur
  int row;    // first row inside the segment's tensor
  int kv0;    // logical key index of column 0
  int valid;  // valid keys in this tile
};

__device__ __forceinline__ Tile tile_of(const AttnKernelArgs& a, int j, int n0) {
  Tile t;
  if (j < n0) {
    t.seg = 0;
    t.row = a.ctx_row0 + j * BN;
    t.kv0 = j * BN;
    t.valid = min(BN, a.n_ctx - j * BN);
  } else {
    t.seg = 1;
    t.row = (j - n0) * BN;
    t.kv0 = a.n_ctx + (j - n0) * BN;
    t.valid = min(BN, a.n_cur - (j - n0) * BN);
  }
  return t;
}

template <int HD, bool kPInTmem>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_fwd_kernel(const __grid_constant__ AttnKernelArgs a) {
  using L = Layout<HD, kPInTmem>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sP = smem + L::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;
  uint64_t* v_empty = v_full + NS;
  uint64_t* s_full = v_empty + NS;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* pv_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NBAR);

  const int warp = warp_id();
  const int lane = lane_id();
  const int head = blockIdx.y;
  const int q0 = blockIdx.x * BM;
  const int n0 = (a.n_ctx + BN - 1) / BN;
  const int n_tiles = n0 + (a.n_cur + BN - 1) / BN;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(s_empty + b, 128);
      mbar_init(p_full + b, 128);
      mbar_init(pv_done + b, 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&a.tm_q);
      if (n0 > 0) {
        tma_prefetch_desc(&a.tm_kc);
        tma_prefetch_desc(&a.tm_vc);
      }
      if (n_tiles > n0) {
        tma_prefetch_desc(&a.tm_kn);
        tma_prefetch_desc(&a.tm_vn);
      }
      mbar_expect_tx(q_full, L::Q_BYTES);
      for (int c = 0; c < L::KCH; ++c)
        tma_load_2d(sQ + c * BM * 128, &a.tm_q, q_full, head * HD + c * 64, q0);
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % NS;
        const uint32_t ph = (j / NS) & 1;
        const Tile t = tile_of(a, j, n0);
        const CUtensorMap* mk = t.seg == 0 ? &a.tm_kc : &a.tm_kn;
        const CUtensorMap* mv = t.seg == 0 ? &a.tm_vc : &a.tm_vn;
        mbar_wait(k_empty + s, ph ^ 1);
        mbar_expect_tx(k_full + s, L::KV_BYTES);
        for (int c = 0; c < L::KCH; ++c)
          tma_load_2d(sK + s * L::KV_BYTES + c * BN * 128, mk, k_full + s, head * HD + c * 64,
                      t.row);
        mbar_wait(v_empty + s, ph ^ 1);
        mbar_expect_tx(v_full + s, L::KV_BYTES);
        for (int c = 0; c < L::KCH; ++c)
          tma_load_2d(sV + s * L::KV_BYTES + c * BN * 128, mv, v_full + s, head * HD + c * 64,
                      t.row);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, 0, 0);  // Q, K both K-major
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, HD, 0, 1);  // P K-major, V MN-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      const uint32_t q_base = smem_u32(sQ);
      for (int j = 0; j <= n_tiles; ++j) {
        if (j < n_tiles) {
          const int s = j % NS;
          const int b = j & 1;
          mbar_wait(k_full + s, (j / NS) & 1);
          mbar_wait(s_empty + b, ((j >> 1) & 1) ^ 1);
          if (kPInTmem && j >= 2) mbar_wait(pv_done + b, ((j >> 1) & 1) ^ 1);  // P_{j-2} read
          tc_fence_after();
          const uint32_t k_base = smem_u32(sK + s * L::KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (BM * 128) + (kk & 3) * 32;
            const uint32_t offk = (kk >> 2) * (BN * 128) + (kk & 3) * 32;
            mma_bf16_ss(tmem + b * 128, smem_desc_sw128(q_base + off, 16, 1024),
                        smem_desc_sw128(k_base + offk, 16, 1024), idesc_qk, kk > 0);
          }
          mma_commit(k_empty + s);
          mma_commit(s_full + b);
        }
        if (j >= 1) {
          const int jp = j - 1;
          const int s = jp % NS;
          const int b = jp & 1;
          mbar_wait(p_full + b, (jp >> 1) & 1);
          mbar_wait(v_full + s, (jp / NS) & 1);
          tc_fence_after();
          const uint32_t v_base = smem_u32(sV + s * L::KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            // V tile: KCH chunks [BN keys x 64 dims], rows of 128 B; MN-major B operand:
            // LBO = stride between 64-dim chunks, SBO = 8 key rows; K step = 16 rows.
            const uint64_t bdesc = smem_desc_sw128(v_base + kk * 16 * 128, BN * 128, 1024);
            if constexpr (kPInTmem) {
              mma_bf16_ts(tmem + L::TM_O, tmem + b * 128 + L::TM_P_OFF + kk * 8, bdesc, idesc_pv,
                          (jp > 0 || kk > 0));
            } else {
              const uint32_t p_base = smem_u32(sP + b * L::P_BYTES);
              const uint32_t off = (kk >> 2) * (BM * 128) + (kk & 3) * 32;
              mma_bf16_ss(tmem + L::TM_O, smem_desc_sw128(p_base + off, 16, 1024), bdesc,
                          idesc_pv, (jp > 0 || kk > 0));
            }
          }
          mma_commit(v_empty + s);
          mma_commit(pv_done + b);
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== softmax / correction / epilogue =====================
    const int q4 = warp & 3;            // TMEM lane quarter this warp may access
    const int row = q4 * 32 + lane;     // query row within the tile
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int grow = q0 + row;
    const float sl2 = a.scale_log2;
    float m_run = -INFINITY;  // running max, log2-scaled units
    float l_run = 0.f;
    float m_exact = -INFINITY;  // true running max (only for the partial-stats output)
    bool o_live = false;      // some PV has accumulated into O
    const uint8_t* mrow = (a.mask != nullptr && grow < a.n_q) ? a.mask + (int64_t)grow * a.mask_ld
                                                              : nullptr;
    for (int j = 0; j < n_tiles; ++j) {
      const int b = j & 1;
      const Tile t = tile_of(a, j, n0);
      mbar_wait(s_full + b, (j >> 1) & 1);
      tc_fence_after();
      float sv[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + b * 128 + c * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[i]);
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_empty + b);

      // visibility: ragged tile tail, optional dense mask
      if (t.valid < BN || mrow != nullptr) {
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          bool ok = i < t.valid;
          if (ok && mrow != nullptr) ok = mrow[t.kv0 + i] != 0;
          if (!ok) sv[i] = -INFINITY;
        }
      }
      // 8 independent chains: one softmax warp per SM sub-partition has no other warp to
      // hide FMNMX/FADD latency behind, so the reductions must carry their own ILP
      float m8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) m8[i] = sv[i];
#pragma unroll
      for (int i = 8; i < BN; ++i) m8[i & 7] = fmaxf(m8[i & 7], sv[i]);
      const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                             fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      const float m_tile = mx * sl2;  // -inf if nothing visible
      m_exact = fmaxf(m_exact, m_tile);
      float alpha = 1.f;
      bool rescale_o = false;
      if (m_tile > m_run + kRescaleThreshold || (m_run == -INFINITY && m_tile > -INFINITY)) {
        alpha = (m_run == -INFINITY) ? 0.f : ex2(m_run - m_tile);
        rescale_o = o_live && m_run != -INFINITY;
        m_run = m_tile;
      }
      const float m_sub = (m_run == -INFINITY) ? 0.f : m_run;
      float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (t.valid == BN && mrow == nullptr) {
        // full unmasked tile: 1 in kPolyEvery exponentials on the FMA pipe (MUFU offload)
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          const float x = fmaf(sv[i], sl2, -m_sub);
          const float p = (i % kPolyEvery == kPolyEvery - 1) ? ex2_poly(x) : ex2(x);
          sv[i] = p;
          s8[i & 7] += p;
        }
      } else {
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          const float p = ex2(fmaf(sv[i], sl2, -m_sub));  // exp2(-inf) = 0 for masked keys
          sv[i] = p;
          s8[i & 7] += p;
        }
      }
      const float sum = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
      l_run = l_run * alpha + sum;

      // tcgen05.ld/st are warp-collective: rescale if any row of this warp needs it
      if (__any_sync(0xffffffffu, rescale_o)) {  // O *= alpha once PV_{j-1} has landed
        const float f = rescale_o ? alpha : 1.f;
        const int jp = j - 1;
        mbar_wait(pv_done + (jp & 1), (jp >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_off + L::TM_O + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
          tmem_st32(tmem + lane_off + L::TM_O + c * 32, r);
        }
        tmem_wait_st();
      }

      if constexpr (kPInTmem) {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = pack_bf16(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]);
          tmem_st16(tmem + lane_off + b * 128 + L::TM_P_OFF + c * 16, r);
        }
        tmem_wait_st();
      } else {
        // P[b] was last read by PV_{j-2}
        mbar_wait(pv_done + b, ((j >> 1) & 1) ^ 1);
        uint8_t* pb = sP + b * L::P_BYTES;
#pragma unroll
        for (int c16 = 0; c16 < BN / 8; ++c16) {
          uint4 v;
          v.x = pack_bf16(sv[c16 * 8 + 0], sv[c16 * 8 + 1]);
          v.y = pack_bf16(sv[c16 * 8 + 2], sv[c16 * 8 + 3]);
          v.z = pack_bf16(sv[c16 * 8 + 4], sv[c16 * 8 + 5]);
          v.w = pack_bf16(sv[c16 * 8 + 6], sv[c16 * 8 + 7]);
          const int chunk = c16 & 7;
          uint8_t* dst = pb + (c16 >> 3) * (BM * 128) + row * 128 + ((chunk ^ (row & 7)) << 4);
          *reinterpret_cast<uint4*>(dst) = v;
        }
        fence_proxy_async_smem();
      }
      tc_fence_before();
      mbar_arrive(p_full + b);
      o_live = true;
    }

    // ---------------- epilogue: O / l -> bf16 -> global ----------------
    if (n_tiles > 0) {
      const int jl = n_tiles - 1;
      mbar_wait(pv_done + (jl & 1), (jl >> 1) & 1);
      tc_fence_after();
    }
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    __nv_bfloat16* orow = a.o + (int64_t)grow * a.o_ld + head * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + L::TM_O + c * 32, r);
      tmem_wait_ld();
      if (grow < a.n_q) {
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(r[v4 * 8 + 0]) * inv, __uint_as_float(r[v4 * 8 + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(r[v4 * 8 + 2]) * inv, __uint_as_float(r[v4 * 8 + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(r[v4 * 8 + 4]) * inv, __uint_as_float(r[v4 * 8 + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(r[v4 * 8 + 6]) * inv, __uint_as_float(r[v4 * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + v4 * 8) = w;
        }
      }
    }
    if (a.row_max != nullptr && grow < a.n_q) {
      // re-reference the denominator to the exact max (attention.py:140-154 convention)
      const bool live = m_exact > -INFINITY;
      a.row_max[(int64_t)head * a.n_q + grow] = m_exact;
      a.row_sum[(int64_t)head * a.n_q + grow] = live ? l_run * ex2(m_run - m_exact) : 0.f;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int HD, bool kPInTmem>
int launch(const AttnKernelArgs& a, int n_q, int heads, cudaStream_t st) {
  using L = Layout<HD, kPInTmem>;
  auto* fn = attn_fwd_kernel<HD, kPInTmem>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  dim3 grid((n_q + BM - 1) / BM, heads);
  fn<<<grid, NTHREADS, L::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace

int attn_fwd_launch(const AttnKernelArgs& a, int head_dim, int variant, int n_q, int heads,
                    cudaStream_t st) {
  const bool p_tmem = variant == 1;
  if (head_dim == 128) return p_tmem ? launch<128, true>(a, n_q, heads, st) : launch<128, false>(a, n_q, heads, st);
  if (head_dim == 64) return p_tmem ? launch<64, true>(a, n_q, heads, st) : launch<64, false>(a, n_q, heads, st);
  return -1;
}

}  // namespace ifx
