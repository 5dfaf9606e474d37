// attn_fwd_sm100.cu — K1: attention of one block's queries over [cached context ∥ own K/V].
//
// Replaces the reference's per-head numpy loop `_mha` -> `scaled_dot_attention`
// (/root/reference/pkg/src/inferix/engine.py:176-182,206-210, attention.py:74-94) and the
// context concat it needs: softmax(Q K^T * scale) V with online (flash) softmax; every key
// is visible (engine.py:209) unless a dense mask is given (API parity, attention.py:89).
//
// Work item = one 128-query tile of one head (and key split): 37 tiles x 12 heads = 444 =
// 3 x 148 at the Wan-1.3B shape. Persistent CTAs (one per SM, 320 threads) walk items
// blockIdx.x, blockIdx.x + gridDim.x, ...:
//   warp 0      TMA producer: Q per item (double-buffered), then K_j / V_j tiles (128 keys x
//               head_dim, SW128)
//               into 2-stage smem rings; mbarrier tx completion
//   warp 1      MMA issuer (one elected lane): S_j = Q K_j^T into TMEM (double-buffered S),
//               then per key half h: O_h += P_h V_h (P read from TMEM, TS form) as soon as
//               that half's P is published; tcgen05.commit frees smem stages / signals
//   warps 2-9   softmax, TWO warps per TMEM lane quarter: warp (q4, h) owns query rows
//               32*q4..+31 and key columns 64h..64h+63 of every S tile and runs its OWN
//               online softmax over them (own running max / denominator, own accumulator
//               O_h), so the two warps of a sub-partition never synchronise per tile and
//               overlap freely (one in TMEM loads while the other is on MUFU/FMA). 64
//               exponentials per warp per tile, 2 pairs in 8 as a cubic on the FMA pipe,
//               FFMA2/FADD2 packed math; P (bf16) overwrites the S columns it came from;
//               lazy O rescale (only when the running max grows by > 2^8). The epilogue
//               merges (O_0, m_0, l_0) and (O_1, m_1, l_1) (attention.py:157-180) and each
//               warp stores half of the head dims.
// Design study with the measurements behind each choice: profiles/r02_attn_variants.md.
// Keys come from two segments so the block's own K/V never need to be copied next to the
// cache: segment 0 = slab rows [ctx_row0, ctx_row0 + n_ctx), segment 1 = rows [0, n_cur)
// of the fresh QKV projection. Ragged tails are masked in softmax (TMA zero-fills rows past
// a tensor's extent; rows past a segment end inside the slab are finite and masked).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "attn_kernel.h"
#include "device_state.h"
#include "launch.cuh"
#include "sm100_ptx.cuh"

namespace ifx {
namespace {

using namespace ptx;

constexpr int BM = 128;          // query rows per CTA (= TMEM lanes)
constexpr int BN = 128;          // keys per tile
constexpr int HALF = BN / 2;     // key columns per softmax warp
constexpr int NS = 2;            // smem stages for K and for V
constexpr int NB = 2;            // S buffers in TMEM (P aliases S)
constexpr int NTHREADS = 320;    // 10 warps
constexpr int NSOFT = 256;       // softmax threads
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale O only if max grows > 2^8
#ifndef IFX_POLY_PAIRS_OF_8
#define IFX_POLY_PAIRS_OF_8 2  // r03 power-capped bench: 1-2 beat 3 (profiles/r03_attn_poly.md)
#endif
// exp2 pairs (out of every 8 pairs) evaluated as a cubic on the FMA pipe instead of MUFU
constexpr int kPolyPairsOf8 = IFX_POLY_PAIRS_OF_8;

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

// the same on a pair with packed fp32x2 ops (FADD2 / FFMA2)
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 p = __ffma2_rn(make_float2(0.0555041087f, 0.0555041087f), f,
                        make_float2(0.2402265070f, 0.2402265070f));
  p = __ffma2_rn(p, f, make_float2(0.6931471806f, 0.6931471806f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int HD>
struct Layout {
  static constexpr int KCH = HD / 64;
  static constexpr int Q_BYTES = BM * HD * 2;
  static constexpr int KV_BYTES = BN * HD * 2;
  static constexpr int OFF_Q = 0;                      // two Q buffers (item parity)
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * KV_BYTES;
  static constexpr int OFF_RED = OFF_V + NS * KV_BYTES;  // float [2 halves][3][BM] merge swap
  static constexpr int OFF_BAR = OFF_RED + 2 * 3 * BM * 4;
  // q_full[2] q_empty[2] k_full k_empty v_full v_empty s_full s_empty p_full[2] pv_done o_free
  static constexpr int NBAR = 4 + 4 * NS + 5 * NB + 1;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
  // TMEM columns: S0 [0,128) S1 [128,256) O_lo [256, 256+HD) O_hi [384, 384+HD).
  // Key half h of S_b (columns 64h..64h+63) is overwritten in place by its packed bf16 P
  // (32 columns at 64h): each softmax warp only ever writes the S columns it read.
  __host__ __device__ static constexpr uint32_t TM_O(int h) { return 256 + 128 * h; }
  __host__ __device__ static constexpr uint32_t TM_P(int h) { return 64 * h; }
};

struct Tile {
  int seg, row, kv0, lo, valid;  // keys [lo, valid) of the tile are visible
};

__device__ __forceinline__ Tile tile_of(const AttnKernelArgs& a, int j, int n0) {
  Tile t;
  if (j < n0) {
    t.seg = 0;
    t.row = a.ctx_row0 + j * BN;  // paged: row relative to the first page (ctx_row0 = 0)
    t.kv0 = j * BN;
    t.lo = j == 0 ? a.ctx_lo : 0;
    t.valid = min(BN, a.n_ctx - j * BN);
  } else {
    t.seg = 1;
    t.row = (j - n0) * BN;
    t.kv0 = a.n_ctx + (j - n0) * BN;
    t.lo = 0;
    t.valid = min(BN, a.n_cur - (j - n0) * BN);
  }
  return t;
}

// A work item = (128-query tile, head, key split). CTAs are persistent: CTA c runs items
// c, c + gridDim.x, ... in order, so the next item's Q load and first S tiles overlap the
// previous item's epilogue (and the per-CTA setup is paid once per SM, not per item).
struct Item {
  int head, q0, split, t0, n_tiles;
};

__device__ __forceinline__ Item item_of(const AttnKernelArgs& a, int it, int n_total) {
  const int gx = (a.n_q + BM - 1) / BM;
  Item r;
  r.q0 = (it % gx) * BM;
  r.head = (it / gx) % a.heads;
  r.split = it / (gx * a.heads);
  // split-KV: this item walks key tiles [t0, t0 + n_tiles) and, when the key range is
  // split, writes a partial (normalised O, max, denominator) merged by K4
  r.t0 = (int)(((int64_t)r.split * n_total) / a.n_splits);
  r.n_tiles = (int)(((int64_t)(r.split + 1) * n_total) / a.n_splits) - r.t0;
  return r;
}

template <int HD, bool PAGED>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_fwd_kernel(const __grid_constant__ AttnKernelArgs a) {
  using L = Layout<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  float* red = reinterpret_cast<float*>(smem + L::OFF_RED);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;       // [2]
  uint64_t* q_empty = bars + 2;  // [2]
  uint64_t* k_full = bars + 4;
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;
  uint64_t* v_empty = v_full + NS;
  uint64_t* s_full = v_empty + NS;
  uint64_t* s_empty = s_full + NB;
  uint64_t* p_full = s_empty + NB;   // [NB][2 key halves]
  uint64_t* pv_done = p_full + 2 * NB;
  uint64_t* o_free = pv_done + NB;  // the softmax warps have read O of their current item
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NBAR);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n0 = (a.n_ctx + BN - 1) / BN;
  const int n_total = n0 + (a.n_cur + BN - 1) / BN;
  const int n_items = ((a.n_q + BM - 1) / BM) * a.heads * a.n_splits;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
    }
    mbar_init(o_free, NSOFT);
    for (int s = 0; s < NS; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(s_empty + b, NSOFT);
      mbar_init(p_full + 2 * b, NSOFT / 2);
      mbar_init(p_full + 2 * b + 1, NSOFT / 2);
      mbar_init(pv_done + b, 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // setup above overlapped the previous kernel (launch.cuh)

  if (warp == 0 && !PAGED) {
    // ===================== TMA producer (contiguous context) =====================
    if (elect_one()) {
      tma_prefetch_desc(&a.tm_q);
      if (n0 > 0) {
        tma_prefetch_desc(&a.tm_kc);
        tma_prefetch_desc(&a.tm_vc);
      }
      if (n_total > n0) {
        tma_prefetch_desc(&a.tm_kn);
        tma_prefetch_desc(&a.tm_vn);
      }
      int g = 0;  // key tiles loaded so far by this CTA (smem ring position)
      for (int it = blockIdx.x, k = 0; it < n_items; it += gridDim.x, ++k) {
      const Item im = item_of(a, it, n_total);
      const int head = im.head, t0 = im.t0, n_tiles = im.n_tiles;
      const int ib = k & 1;
      if (k >= 2) mbar_wait(q_empty + ib, ((k >> 1) - 1) & 1);
      mbar_expect_tx(q_full + ib, L::Q_BYTES);
      for (int c = 0; c < L::KCH; ++c)
        tma_load_2d(sQ + ib * L::Q_BYTES + c * BM * 128, &a.tm_q, q_full + ib,
                    head * HD + c * 64, im.q0);
      for (int j = 0; j < n_tiles; ++j, ++g) {
        const int s = g % NS;
        const uint32_t ph = (g / NS) & 1;
        const Tile t = tile_of(a, t0 + j, n0);
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
    }
    __syncwarp();
  } else if (warp == 0) {
    // ===================== TMA producer (paged context) =====================
    // One elected thread, like the contiguous path (its instructions share sub-partition 0
    // with two softmax warps, so it is kept lean). A context tile whose pages sit in
    // consecutive slots of one pool (the common case: a block's appends take consecutive
    // slots) is one 128-row box per 64-column chunk; otherwise every page is its own
    // page_len-row box from its slot. The caller's per-tile run codes (ctx_tile_runs)
    // make the common case one table load per tile, prefetched a tile ahead; without
    // them the tile's page slots are loaded and compared here.
    if (elect_one()) {
      constexpr int MAXP = BN / 8;  // pages per tile at the smallest page_len
      constexpr int32_t kNoRun = INT32_MIN;
      const int ppt = BN / a.ctx_page_len;
      const int prow_b = a.ctx_page_len * 128;  // smem bytes of one page box
      const int n_pages = (a.n_ctx + a.ctx_page_len - 1) / a.ctx_page_len;
      const int32_t* runs = a.ctx_tile_runs;
      tma_prefetch_desc(&a.tm_q);
      if (n0 > 0) {
        tma_prefetch_desc(&a.tm_kc_run);
        tma_prefetch_desc(&a.tm_vc_run);
      }
      if (n_total > n0) {
        tma_prefetch_desc(&a.tm_kn);
        tma_prefetch_desc(&a.tm_vn);
      }
      int g = 0;  // key tiles loaded so far by this CTA (smem ring position)
      for (int it = blockIdx.x, k = 0; it < n_items; it += gridDim.x, ++k) {
      const Item im = item_of(a, it, n_total);
      const int head = im.head, t0 = im.t0, n_tiles = im.n_tiles;
      const int ib = k & 1;
      if (k >= 2) mbar_wait(q_empty + ib, ((k >> 1) - 1) & 1);
      mbar_expect_tx(q_full + ib, L::Q_BYTES);
      for (int c = 0; c < L::KCH; ++c)
        tma_load_2d(sQ + ib * L::Q_BYTES + c * BM * 128, &a.tm_q, q_full + ib,
                    head * HD + c * 64, im.q0);
      int32_t rnext = (runs != nullptr && n_tiles > 0 && t0 < n0) ? __ldg(runs + t0) : kNoRun;
      for (int j = 0; j < n_tiles; ++j, ++g) {
        const int s = g % NS;
        const uint32_t ph = (g / NS) & 1;
        const Tile t = tile_of(a, t0 + j, n0);
        int32_t rc = rnext;
        if (runs != nullptr && j + 1 < n_tiles && t0 + j + 1 < n0) rnext = __ldg(runs + t0 + j + 1);
        int32_t sl[MAXP];
        if (t.seg == 0 && rc == kNoRun) {  // page by page (or detect the run here)
#pragma unroll
          for (int i = 0; i < MAXP; ++i)
            if (i < ppt) sl[i] = __ldg(a.ctx_slots + min((t0 + j) * ppt + i, n_pages - 1));
          if (runs == nullptr) {
            bool run = true;
#pragma unroll
            for (int i = 1; i < MAXP; ++i)
              if (i < ppt) run = run && sl[i] == sl[0] + (sl[0] >= 0 ? i : -i);
            if (run) rc = sl[0];
          }
        }
        if (t.seg != 0) {
          mbar_wait(k_empty + s, ph ^ 1);
          mbar_expect_tx(k_full + s, L::KV_BYTES);
          for (int c = 0; c < L::KCH; ++c)
            tma_load_2d(sK + s * L::KV_BYTES + c * BN * 128, &a.tm_kn, k_full + s,
                        head * HD + c * 64, t.row);
          mbar_wait(v_empty + s, ph ^ 1);
          mbar_expect_tx(v_full + s, L::KV_BYTES);
          for (int c = 0; c < L::KCH; ++c)
            tma_load_2d(sV + s * L::KV_BYTES + c * BN * 128, &a.tm_vn, v_full + s,
                        head * HD + c * 64, t.row);
        } else if (rc != kNoRun) {
          const bool dev = rc >= 0;
          const int row = (dev ? rc : -1 - rc) * a.ctx_page_len;
          mbar_wait(k_empty + s, ph ^ 1);
          mbar_expect_tx(k_full + s, L::KV_BYTES);
          for (int c = 0; c < L::KCH; ++c)
            tma_load_2d(sK + s * L::KV_BYTES + c * BN * 128, dev ? &a.tm_kc_run : &a.tm_ks_run,
                        k_full + s, head * HD + c * 64, row);
          mbar_wait(v_empty + s, ph ^ 1);
          mbar_expect_tx(v_full + s, L::KV_BYTES);
          for (int c = 0; c < L::KCH; ++c)
            tma_load_2d(sV + s * L::KV_BYTES + c * BN * 128, dev ? &a.tm_vc_run : &a.tm_vs_run,
                        v_full + s, head * HD + c * 64, row);
        } else {
          for (int kv = 0; kv < 2; ++kv) {
            uint64_t* full = (kv == 0 ? k_full : v_full) + s;
            uint8_t* dst = (kv == 0 ? sK : sV) + s * L::KV_BYTES;
            mbar_wait((kv == 0 ? k_empty : v_empty) + s, ph ^ 1);
            mbar_expect_tx(full, L::KV_BYTES);
#pragma unroll
            for (int i = 0; i < MAXP; ++i) {
              if (i < ppt) {
                const bool dev = sl[i] >= 0;
                const CUtensorMap* m = dev ? (kv == 0 ? &a.tm_kc : &a.tm_vc)
                                           : (kv == 0 ? &a.tm_ks : &a.tm_vs);
                const int row = (dev ? sl[i] : -1 - sl[i]) * a.ctx_page_len;
                for (int c = 0; c < L::KCH; ++c)
                  tma_load_2d(dst + c * BN * 128 + i * prow_b, m, full, head * HD + c * 64, row);
              }
            }
          }
        }
      }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, 0, 0);  // Q, K both K-major
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, HD, 0, 1);  // P (TMEM), V MN-major
      int g0 = 0;  // key tiles of earlier items (ring / S-buffer position)
      for (int it = blockIdx.x, k = 0; it < n_items; it += gridDim.x, ++k) {
        const int n_tiles = item_of(a, it, n_total).n_tiles;
        const int ib = k & 1;
        mbar_wait(q_full + ib, (k >> 1) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ + ib * L::Q_BYTES);
        for (int j = 0; j <= n_tiles; ++j) {
          if (j < n_tiles) {
            const int gj = g0 + j;
            const int s = gj % NS;
            const int b = gj % NB;
            const uint32_t bph = (gj / NB) & 1;
            mbar_wait(k_full + s, (gj / NS) & 1);
            mbar_wait(s_empty + b, bph ^ 1);                    // S_b of tile gj-NB read
            // P_b aliases S_b: explicit wait for PV(gj-NB) before QK(gj) overwrites it. The
            // PTX guarantees in-order execution only between MMAs on the same accumulator,
            // and PV and QK^T use different ones; dropping the wait measured +0.3 % in the
            // bench (profiles/r03_k1_persistent.md), not worth a possible WAR race.
            if (gj >= NB) mbar_wait(pv_done + b, bph ^ 1);
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
          if (k >= 1 && j == (n_tiles > 0 ? 1 : 0)) {
            // O is overwritten by this item's first PV: the previous item's epilogue must
            // have read it (this item's first two S tiles, issued above, overlap it)
            mbar_wait(o_free, (k - 1) & 1);
          }
          if (j >= 1) {
            const int gp = g0 + j - 1;
            const int s = gp % NS;
            const int b = gp % NB;
            mbar_wait(v_full + s, (gp / NS) & 1);
            const uint32_t v_base = smem_u32(sV + s * L::KV_BYTES);
            // O_h += P_h V[64h .. 64h+63]: each key half has its own running max, so its own
            // accumulator; issued as soon as that half's softmax warps published P_h
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              mbar_wait(p_full + 2 * b + h, (gp / NB) & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < HALF / 16; ++kk) {
                // V tile: KCH chunks [BN keys x 64 dims], rows of 128 B; MN-major B operand:
                // LBO = stride between 64-dim chunks, SBO = 8 key rows; K step = 16 rows.
                const uint64_t bdesc =
                    smem_desc_sw128(v_base + (h * (HALF / 16) + kk) * 16 * 128, BN * 128, 1024);
                mma_bf16_ts(tmem + L::TM_O(h), tmem + b * 128 + L::TM_P(h) + kk * 8, bdesc,
                            idesc_pv, (j > 1 || kk > 0) ? 1u : 0u);
              }
            }
            mma_commit(v_empty + s);
            mma_commit(pv_done + b);
          }
        }
        mma_commit(q_empty + ib);  // this item's QK^T MMAs have read its Q buffer
        g0 += n_tiles;
      }
    }
    __syncwarp();
  } else {
    // ===================== softmax (2 warps per TMEM lane quarter) =====================
    const int q4 = warp & 3;                  // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;         // key-column half of every S tile
    const int row = q4 * 32 + lane;           // query row within the tile
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const float sl2 = a.scale_log2;
    const int pair_bar = 1 + q4;              // named barrier of the two warps of quarter q4
    int g0 = 0;                               // key tiles of earlier items (S-buffer position)
    for (int it = blockIdx.x, k = 0; it < n_items; it += gridDim.x, ++k) {
    const Item im = item_of(a, it, n_total);
    const int head = im.head, split = im.split, t0 = im.t0, n_tiles = im.n_tiles;
    const int grow = im.q0 + row;
    float m_run = -INFINITY;                  // running max used for exponents (log2 units)
    float l_half = 0.f;                       // denominator over this warp's columns
    float m_exact = -INFINITY;                // true running max (partial-stats output)
    const uint8_t* mrow = (a.mask != nullptr && grow < a.n_q) ? a.mask + (int64_t)grow * a.mask_ld
                                                              : nullptr;
    // the only tiles with invisible keys: a window start inside the first context tile,
    // and the ragged last tile of each segment (everything else skips the masking)
    const int part0 = (n0 > 0 && a.ctx_lo > 0) ? 0 : -1;
    const int part1 = (a.n_ctx % BN) ? n0 - 1 : -1;
    const int part2 = (a.n_cur % BN) ? n_total - 1 : -1;
    for (int j = 0; j < n_tiles; ++j) {
      const int gj = g0 + j;
      const int b = gj % NB;
      const int jt = t0 + j;
      const int c0 = half * HALF;  // first key column of this warp
      mbar_wait(s_full + b, (gj / NB) & 1);
      tc_fence_after();
      float sv[HALF];
      {  // the warp's 64 score columns in ONE load (vs two x32: +0.7 % K1, r05_k1_softmax_variants.md)
        static_assert(HALF == 64, "one 32x32b.x64 load per key half");
        uint32_t r[64];
        tmem_ld64(tmem + lane_off + b * 128 + c0, r);
#pragma unroll
        for (int i = 0; i < 64; ++i) sv[i] = __uint_as_float(r[i]);
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_empty + b);

      const bool full = mrow == nullptr && jt != part0 && jt != part1 && jt != part2;
      if (!full) {
        const Tile t = tile_of(a, jt, n0);
#pragma unroll
        for (int i = 0; i < HALF; ++i) {
          bool ok = c0 + i < t.valid && c0 + i >= t.lo;
          if (ok && mrow != nullptr) ok = mrow[t.kv0 + c0 + i] != 0;
          if (!ok) sv[i] = -INFINITY;
        }
      }
      float m4[8];  // 8 independent max chains (ILP; +0.5 % in the bench, r03_attn_poly.md)
#pragma unroll
      for (int i = 0; i < 8; ++i) m4[i] = sv[i];
#pragma unroll
      for (int i = 8; i < HALF; ++i) m4[i & 7] = fmaxf(m4[i & 7], sv[i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) m4[i] = fmaxf(m4[i], m4[i + 4]);
      // this key half's own online softmax: no per-tile exchange with the other half
      const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      const float m_tile = mx * sl2;  // -inf if nothing visible
      m_exact = fmaxf(m_exact, m_tile);
      float alpha = 1.f;
      bool rescale_o = false;
      if (m_tile > m_run + kRescaleThreshold) {
        alpha = (m_run == -INFINITY) ? 0.f : ex2(m_run - m_tile);
        rescale_o = j > 0 && m_run != -INFINITY;
        m_run = m_tile;
      }
      const float m_sub = (m_run == -INFINITY) ? 0.f : m_run;
      // packed fp32x2 arithmetic (FFMA2 / FADD2) halves the FMA-pipe instruction count;
      // MUFU.EX2 stays scalar (the bf16x2/f16x2 forms issue two MUFU ops on sm_100)
      const float2 sl2v = make_float2(sl2, sl2);
      const float2 negm = make_float2(-m_sub, -m_sub);
      float2 acc[8];  // 8 independent sum chains (ILP)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
      if (full) {
#pragma unroll
        for (int i = 0; i < HALF / 2; ++i) {
          const float2 x = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), sl2v, negm);
          float2 p;
          if ((i & 7) >= 8 - kPolyPairsOf8) {
            p = ex2_poly2(x);  // kPolyPairsOf8 of every 8 pairs on the FMA pipe
          } else {
            p.x = ex2(x.x);
            p.y = ex2(x.y);
          }
          sv[2 * i] = p.x;
          sv[2 * i + 1] = p.y;
          acc[i & 7] = __fadd2_rn(acc[i & 7], p);
        }
      } else {
#pragma unroll
        for (int i = 0; i < HALF / 2; ++i) {
          const float2 x = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), sl2v, negm);
          const float2 p = make_float2(ex2(x.x), ex2(x.y));  // exp2(-inf) = 0 for masked keys
          sv[2 * i] = p.x;
          sv[2 * i + 1] = p.y;
          acc[i & 7] = __fadd2_rn(acc[i & 7], p);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = __fadd2_rn(acc[i], acc[i + 4]);
      const float2 a01 = __fadd2_rn(acc[0], acc[1]), a23 = __fadd2_rn(acc[2], acc[3]);
      const float2 a4 = __fadd2_rn(a01, a23);
      l_half = l_half * alpha + (a4.x + a4.y);

      // tcgen05.ld/st are warp-collective: rescale if any row of this warp needs it
      if (__any_sync(0xffffffffu, rescale_o)) {  // O_half *= alpha once PV_{j-1} landed
        const float f = rescale_o ? alpha : 1.f;
        const int jp = gj - 1;
        mbar_wait(pv_done + (jp % NB), (jp / NB) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t r[32];
          const uint32_t ta = tmem + lane_off + L::TM_O(half) + c * 32;
          tmem_ld32(ta, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
          tmem_st32(ta, r);
        }
      }
      {  // P (64 bf16 = 32 packed columns) in ONE store
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = pack_bf16(sv[2 * i], sv[2 * i + 1]);
        tmem_st32(tmem + lane_off + b * 128 + L::TM_P(half), r);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + 2 * b + half);
    }

    // ---------------- epilogue: O / l -> bf16 -> global (this warp's half of O) --------
    if (n_tiles > 0) {
      const int jl = g0 + n_tiles - 1;
      mbar_wait(pv_done + (jl % NB), (jl / NB) & 1);
      tc_fence_after();
    }
    g0 += n_tiles;
    // merge the two key halves' partials (attention.py:157-180): swap (max, denominator,
    // exact max) with the partner warp, then each warp stores half of the head dims
    float* me = red + half * 3 * BM;
    me[row] = m_run;
    me[BM + row] = l_half;
    me[2 * BM + row] = m_exact;
    named_sync(pair_bar, 64);
    const float* ot = red + (half ^ 1) * 3 * BM;
    const float m_o = ot[row], l_o = ot[BM + row], mx_o = ot[2 * BM + row];
    const float M = fmaxf(m_run, m_o);
    const float w_me = (m_run == -INFINITY) ? 0.f : ex2(m_run - M);
    const float w_ot = (m_o == -INFINITY) ? 0.f : ex2(m_o - M);
    const float den = l_half * w_me + l_o * w_ot;
    const float inv = den > 0.f ? 1.f / den : 0.f;
    const float w_lo = (half == 0 ? w_me : w_ot) * inv;  // weight of O_lo
    const float w_hi = (half == 0 ? w_ot : w_me) * inv;  // weight of O_hi
    const bool partial = a.n_splits > 1;
    __nv_bfloat16* orow =
        partial ? a.part_o + ((int64_t)split * a.n_q + grow) * a.part_ld + head * HD + half * (HD / 2)
                : attn_out_row(a, grow < a.n_q ? grow : 0) + head * HD + half * (HD / 2);
    // read and merge all of this warp's O columns first, so the next item's first PV
    // (waiting on o_free) is not held up by the global stores
    uint32_t packed[HD / 64][16];
#pragma unroll
    for (int c = 0; c < HD / 64; ++c) {
      uint32_t r0[32], r1[32];
      const uint32_t col = half * (HD / 2) + c * 32;
      tmem_ld32(tmem + lane_off + L::TM_O(0) + col, r0);
      tmem_ld32(tmem + lane_off + L::TM_O(1) + col, r1);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        // a half that saw no key has weight 0 and an undefined accumulator
        float o2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float x0 = w_lo != 0.f ? __uint_as_float(r0[2 * i + e]) * w_lo : 0.f;
          const float x1 = w_hi != 0.f ? __uint_as_float(r1[2 * i + e]) * w_hi : 0.f;
          o2[e] = x0 + x1;
        }
        packed[c][i] = pack_bf16(o2[0], o2[1]);
      }
    }
    tc_fence_before();
    mbar_arrive(o_free);  // O read: the next item's first PV may overwrite it
    if (grow < a.n_q) {
#pragma unroll
      for (int c = 0; c < HD / 64; ++c)
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4)
          *reinterpret_cast<uint4*>(orow + c * 32 + v4 * 8) =
              make_uint4(packed[c][4 * v4], packed[c][4 * v4 + 1], packed[c][4 * v4 + 2],
                         packed[c][4 * v4 + 3]);
    }
    if (partial && grow < a.n_q && half == 0) {  // K4 merges these (attention.py:157-173)
      const int64_t k = ((int64_t)split * a.heads + head) * a.n_q + grow;
      a.part_m[k] = M;
      a.part_l[k] = den;
    }
    if (!partial && a.row_max != nullptr && grow < a.n_q && half == 0) {
      // exact max over both halves, denominator re-referenced to it (attention.py:140-154)
      const float mx = fmaxf(m_exact, mx_o);
      const bool live = mx > -INFINITY;
      a.row_max[(int64_t)head * a.n_q + grow] = mx;
      a.row_sum[(int64_t)head * a.n_q + grow] = live ? den * ex2(M - mx) : 0.f;
    }
    named_sync(pair_bar, 64);  // the partner has read `red` before the next item rewrites it
    }
  }

  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  // peer stores (O scatter, or partials written into a peer's arena) out before the barrier
  // that publishes them: one system fence per CTA, cumulative over the CTA's stores
  if (threadIdx.x == 0 && (a.o_peer_rows > 0 || a.row_max != nullptr)) __threadfence_system();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// K4 — merge split-KV partials (attention.py:157-180 semantics), one warp per (row, head):
// out = sum_s w_s O_s / sum_s w_s with w_s = l_s * 2^(m_s - max_s m_s).
template <int HD>
__global__ void attn_combine_kernel(const AttnKernelArgs a) {
  pdl_wait();
  constexpr int PER = HD / 32;  // head dims per lane: one 8-byte (HD 128) / 4-byte load
  using Vec = typename std::conditional<PER == 4, uint2, uint32_t>::type;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  const int S = a.n_splits;  // <= 32: lane s holds split s's statistics
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
       w < (int64_t)a.n_q * a.heads; w += n_warps) {
    const int row = (int)(w / a.heads), head = (int)(w % a.heads);
    float ms = -INFINITY, ls = 0.f;
    if (lane < S) {
      const int64_t k = ((int64_t)lane * a.heads + head) * a.n_q + row;
      ms = a.part_m[k];
      ls = a.part_l[k];
    }
    float M = ms;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float wl = (ms == -INFINITY) ? 0.f : ls * exp2f(ms - M);
    float den = wl;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    float acc[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) acc[i] = 0.f;
    for (int s = 0; s < S; ++s) {
      const float wgt = __shfl_sync(0xffffffffu, wl, s);
      const Vec v = *reinterpret_cast<const Vec*>(
          a.part_o + ((int64_t)s * a.n_q + row) * a.part_ld + head * HD + lane * PER);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int i = 0; i < PER / 2; ++i) {
        const float2 f = __bfloat1622float2(h2[i]);
        acc[2 * i] = fmaf(wgt, f.x, acc[2 * i]);
        acc[2 * i + 1] = fmaf(wgt, f.y, acc[2 * i + 1]);
      }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    Vec out;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
    for (int i = 0; i < PER / 2; ++i) o2[i] = __floats2bfloat162_rn(acc[2 * i] * inv, acc[2 * i + 1] * inv);
    *reinterpret_cast<Vec*>(attn_out_row(a, row) + head * HD + lane * PER) = out;
    if (a.row_max != nullptr && lane == 0) {
      a.row_max[(int64_t)head * a.n_q + row] = M;
      a.row_sum[(int64_t)head * a.n_q + row] = den;
    }
  }
  if (a.o_peer_rows > 0 || a.row_max != nullptr) {  // peer stores out before the barrier:
    __syncthreads();                                  // one system fence per CTA, cumulative
    if (threadIdx.x == 0) __threadfence_system();     // over the CTA's stores (bar.sync)
  }
}

template <int HD>
int launch(const AttnKernelArgs& a, int n_q, int heads, cudaStream_t st) {
  using L = Layout<HD>;
  auto* fn = a.ctx_slots != nullptr ? attn_fwd_kernel<HD, true> : attn_fwd_kernel<HD, false>;
  static DeviceFlags attr_set;  // the smem attribute is per device context
  const int dev = current_device();
  if (attr_set.first(dev)) {
    for (auto* f : {attn_fwd_kernel<HD, true>, attn_fwd_kernel<HD, false>}) {
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
      if (e != cudaSuccess) return (int)e;
    }
    attr_set.set(dev);
  }
  // persistent CTAs: at most one per SM, each walking items blockIdx.x + i * gridDim.x
  // (IFX_K1_GRID=items launches one CTA per item, the pre-persistent schedule, for A/B)
  const int n_sm = device_sms(dev);
  static const bool per_item = [] {
    const char* env = std::getenv("IFX_K1_GRID");
    return env != nullptr && std::string(env) == "items";
  }();
  const int64_t items = (int64_t)((n_q + BM - 1) / BM) * heads * a.n_splits;
  const int grid = (int)(per_item || items < n_sm ? items : n_sm);
  cudaError_t e = launch_pdl(fn, dim3(grid), dim3(NTHREADS), L::SMEM, st, 1, a);
  if (e != cudaSuccess || a.n_splits == 1) return (int)e;
  const int64_t warps = (int64_t)n_q * heads;
  const int blocks = (int)((warps + 7) / 8 < n_sm * 16 ? (warps + 7) / 8 : n_sm * 16);
  return (int)launch_pdl(attn_combine_kernel<HD>, dim3(blocks), dim3(256), 0, st, 1, a);
}

}  // namespace

// K4 alone: merge n_splits partials a.part_o / part_m / part_l into a.o (the ring
// strategies' partials, computed by separate K1 launches over key shards).
int attn_combine_launch(const AttnKernelArgs& a, int head_dim, cudaStream_t st) {
  const int64_t warps = (int64_t)a.n_q * a.heads;
  const int n_sm = device_sms(current_device());
  const int blocks = (int)((warps + 7) / 8 < n_sm * 16 ? (warps + 7) / 8 : n_sm * 16);
  if (blocks == 0) return 0;
  if (head_dim == 128) return (int)launch_pdl(attn_combine_kernel<128>, dim3(blocks), dim3(256), 0, st, 1, a);
  if (head_dim == 64) return (int)launch_pdl(attn_combine_kernel<64>, dim3(blocks), dim3(256), 0, st, 1, a);
  return -1;
}

int attn_fwd_launch(const AttnKernelArgs& a, int head_dim, int n_q, int heads, cudaStream_t st) {
  if (head_dim == 128) return launch<128>(a, n_q, heads, st);
  if (head_dim == 64) return launch<64>(a, n_q, heads, st);
  return -1;
}

}  // namespace ifx
