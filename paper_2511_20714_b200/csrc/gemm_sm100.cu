// gemm_sm100.cu — G1: the engine's dense projections (engine.py:202-205 q/k/v = h @ W, :210
// @ wo, :215 cross, :217 FFN, :220 eps) as one persistent tcgen05/TMA GEMM with the work on
// either side of each projection fused into its epilogue.
//
// C[M, N] = A[M, K] . B[K, N]: A bf16 row-major (K-major operand), B bf16 row-major weights
// (MN-major operand, the layout cuBLASLt used too), fp32 accumulation in TMEM.
//
// Persistent CTAs (one per SM, 320 threads) walk output tiles blockIdx.x, +gridDim.x, ...
// (row tile fastest, so CTAs running at the same time share the weight tile in L2):
//   warp 0     TMA producer: per 64-wide K step, A box 128 x 64 and BN/64 B boxes 64 x 64
//              (SW128) into an NST-deep smem ring; mbarrier tx completion
//   warp 1     MMA issuer (one elected lane): 4 x tcgen05.mma kind::f16 M=128 N=BN K=16 per
//              stage into one of TWO TMEM accumulators (tile parity), so the epilogue of
//              tile i overlaps the MMAs of tile i+1; tcgen05.commit frees smem stages
//   warps 2-9  epilogue, two warps per TMEM lane quarter (warp % 4), each one thread per
//              output row over half of the tile's columns; the fp32 residual's old values
//              are loaded while the tile's MMAs still run; 32 columns per tcgen05.ld, then
//              in registers:
//                row scale   x rsqrt(mean(x^2) + eps) of the fp32 row A was copied from —
//                            the RMS norm (engine.py:171-173) applied AFTER the product
//                            (diag(s) X W = diag(s) (X W)), so no norm kernel runs between
//                            GEMMs; the producer GEMM wrote A and the row's sum of squares
//                relu        FFN up-projection (engine.py:217)
//                rope        3D RoPE on the Q / K column blocks (north_star (1))
//                store       bf16, or fp32 C = beta C + acc (the fp32 residual stream)
//                emit        with fp32 output: the new row as bf16 (next GEMM's A) and its
//                            sum of squares per (tile, half) (the next row scale)
//                page write  the clean pass's K / V columns also go straight into their
//                            KV-cache page slots (kvcache.py:179-234; K2 fused, either tier)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cmath>
#include <cstdlib>

#include "device_state.h"
#include "launch.cuh"
#include "gemm_kernel.h"
#include "sm100_ptx.cuh"

namespace ifx {
namespace {

using namespace ptx;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NTHREADS = 320;  // producer, MMA, 8 epilogue warps
constexpr int NEPI = 256;

template <int BN, int BNL>  // BNL: B columns held per CTA (BN, or BN / 2 for a CTA pair)
struct GLayout {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BK * BNL * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STG = 8 * 4096;  // epilogue staging, 4 KB per epilogue warp
  static constexpr int NST0 = (224 * 1024 - STG) / STAGE;
  static constexpr int NST = NST0 > 8 ? 8 : NST0;
  static constexpr int OFF_STG = NST * STAGE;
  static constexpr int OFF_BAR = OFF_STG + STG;
  static constexpr int NBAR = 2 * NST + 4;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr uint32_t TM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA 2D load multicast to the CTAs of `mask` (same smem offset, their own mbarrier)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar,
                                               int32_t c0, int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// arrive on the mbarrier at this offset in every CTA of `mask` once this thread's MMAs finish
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// ---- CTA pair (cta_group::2): one MMA of M = 256 over the two SMs of a TPC -------------
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// TMA load into this CTA's smem whose completion is counted on the LEADER CTA's barrier
// (the peer bit of the shared::cluster address cleared), which the pair MMA waits on
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar,
                                                 int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
// arrive on the barrier at the same offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// CL = CTAs per cluster along N (1 or 2). With CL = 2 the two CTAs of a cluster compute
// the tiles (m, 2p) and (m, 2p + 1): they need the same A tile, so each loads half of its
// rows and multicasts it to both (A's L2 -> SM traffic halves), and a stage is refilled
// only when BOTH CTAs' MMAs have read it (the MMA commit arrives in both CTAs).
//
// PAIR (CL = 2): the two CTAs of a cluster are a cta_group::2 pair computing one 256 x BN
// tile: CTA r holds A rows [128 r, 128 r + 128) and B columns [r BN/2, (r + 1) BN/2) of it;
// the leader (rank 0) issues M = 256 MMAs that read both CTAs' shared memory and write each
// CTA's 128 rows into that CTA's TMEM. Per SM a K step moves A 16 KB + B BN/2 x 128 B
// through shared memory instead of A + B BN x 128 B: with the TMA fill and the tensor
// core's reads sharing the shared-memory bandwidth this is what lets the MMAs run back to
// back (profiles/r04_g1_ncu.md). tiles_m counts 256-row tiles in this mode.
template <int BN, int CL, bool PAIR>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_kernel(const __grid_constant__ GemmArgs a) {
  static_assert(!PAIR || CL == 2, "a CTA pair is a cluster of 2");
  constexpr int BNL = PAIR ? BN / 2 : BN;
  using L = GLayout<BN, BNL>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + L::NST;
  uint64_t* tfull = bars + 2 * L::NST;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NBAR);

  const int warp = warp_id();
  const int lane = lane_id();
  const int k_iters = (a.K + BK - 1) / BK;
  // work units: u = (row tile u % tiles_m, column tile(s) u / tiles_m): one tile per CTA
  // (CL = 1), a column-tile pair sharing A (CL = 2), one 256-row tile per CTA pair (PAIR)
  const int rank = CL > 1 ? (int)cluster_rank() : 0;
  const int unit0 = blockIdx.x / CL, unit_step = gridDim.x / CL;
  const int n_units = PAIR ? a.tiles_m * a.tiles_n : a.tiles_m * ((a.tiles_n + CL - 1) / CL);
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1);
  constexpr int kEpiWarps = NEPI / 32;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < L::NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, PAIR ? 1 : CL);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, PAIR ? 2 * kEpiWarps : kEpiWarps);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair(tmem_slot, L::TM_COLS);
    else tmem_alloc<L::TM_COLS>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // the peer's barriers exist before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // setup above overlapped the previous kernel (launch.cuh)

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (elect_one()) {
      tma_prefetch_desc(&a.tm_a);
      tma_prefetch_desc(&a.tm_b);
      int g = 0;
      for (int u = unit0; u < n_units; u += unit_step) {
        const int m0 = PAIR ? (u % a.tiles_m) * 2 * BM + rank * BM : (u % a.tiles_m) * BM;
        const int n0 = PAIR ? (u / a.tiles_m) * BN + rank * BNL : ((u / a.tiles_m) * CL + rank) * BN;
        for (int kb = 0; kb < k_iters; ++kb, ++g) {
          const int s = g % L::NST;
          mbar_wait(empty + s, ((g / L::NST) & 1) ^ 1);
          uint8_t* st = smem + s * L::STAGE;
          if (PAIR) {  // both CTAs' bytes complete on the leader's barrier
            if (rank == 0) mbar_expect_tx(full + s, 2 * L::STAGE);
            tma_load_2d_pair(st, &a.tm_a, full + s, kb * BK, m0);
#pragma unroll
            for (int c = 0; c < BNL / 64; ++c)
              tma_load_2d_pair(st + L::A_BYTES + c * (BK * 128), &a.tm_b, full + s, n0 + c * 64, kb * BK);
            continue;
          }
          mbar_expect_tx(full + s, L::STAGE);
          if (CL == 1) {
            tma_load_2d(st, &a.tm_a, full + s, kb * BK, m0);
          } else {  // this CTA's share of the A rows, to every CTA of the cluster
            constexpr int RA = BM / CL;
            tma_load_2d_mc(st + rank * RA * 128, &a.tm_a, full + s, kb * BK, m0 + rank * RA, kMask);
          }
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_2d(st + L::A_BYTES + c * (BK * 128), &a.tm_b, full + s, n0 + c * 64, kb * BK);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if ((!PAIR || rank == 0) && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * BM : BM, BN, 0, 1);  // A K-major, B MN-major
      int g = 0, i = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++i) {
        const int acc = i & 1;
        mbar_wait(tempty + acc, ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < k_iters; ++kb, ++g) {
          const int s = g % L::NST;
          mbar_wait(full + s, (g / L::NST) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * L::STAGE);
          const uint32_t b_base = a_base + L::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // A: rows of 128 B, K step 16 = 32 B inside the swizzle atom.
            // B: BN/64 chunks [64 K rows x 128 B]; K step 16 = 16 rows; LBO = chunk stride
            const uint64_t ad = smem_desc_sw128(a_base + kk * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(b_base + kk * 16 * 128, BK * 128, 1024);
            if (PAIR) mma_bf16_pair(d, ad, bd, idesc, (kb | kk) != 0);
            else mma_bf16_ss(d, ad, bd, idesc, (kb | kk) != 0);
          }
          if (PAIR) mma_commit_pair(empty + s, kMask);
          else if (CL == 1) mma_commit(empty + s);
          else mma_commit_mc(empty + s, kMask);
        }
        if (PAIR) mma_commit_pair(tfull + acc, kMask);
        else mma_commit(tfull + acc);
      }
    }
    __syncwarp();
  } else {
    // ============================ epilogue ============================
    // Two warps per TMEM lane quarter: warp (q, half) owns rows 32q..32q+31 and columns
    // [half * BN/2, (half + 1) * BN/2) of each tile. Per 32-column chunk: tcgen05.ld gives
    // one thread one row (row scale / ReLU / RoPE there), the chunk goes through a 4 KB
    // swizzled shared-memory stage, and global memory is read and written coalesced: fp32
    // 8 lanes x 16 B = one 128 B row segment (4 rows per instruction), bf16 4 lanes x 16 B
    // (8 rows per instruction).
    constexpr int HC = BN / 2;      // columns per warp
    constexpr int NCH = HC / 32;    // 32-column chunks per warp
    constexpr int PD = NCH < 2 ? NCH : 2;  // residual chunks prefetched ahead
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool beta_on = a.c_f32 && a.beta != 0.f;
    // one arrive per warp on the accumulator's barrier in the MMA-issuing CTA
    auto release_acc = [&](uint64_t* bar) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_cta(bar, 0);
        else mbar_arrive(bar);
      }
    };
    uint8_t* stg = smem + L::OFF_STG + (warp - 2) * 4096;
    const uint32_t stg_u = smem_u32(stg);
    // coalesced-domain coordinates: fp32 rows k*4 + (lane >> 3), 16 B column piece lane & 7;
    // bf16 rows k*8 + (lane >> 2), piece lane & 3
    const int fr = lane >> 3, fj = lane & 7;
    const int br = lane >> 2, bj = lane & 3;
    int i = 0;
    for (int u = unit0; u < n_units; u += unit_step, ++i) {
      const int acc = i & 1;
      const int tm = u % a.tiles_m;
      const int tn = PAIR ? u / a.tiles_m : (u / a.tiles_m) * CL + rank;
      const int64_t r0 = (PAIR ? (int64_t)tm * 2 * BM + rank * BM : (int64_t)tm * BM) + q * 32;
      const int64_t grow = r0 + lane;
      const int c0 = tn * BN + half * HC;
      const bool live = grow < a.M;
      // the residual's old values are read while the MMAs of this tile still run
      float4 cb[PD][8];
      if (beta_on) {
#pragma unroll
        for (int c = 0; c < PD; ++c)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int64_t rr = r0 + k * 4 + fr;
            const int col = c0 + c * 32 + 4 * fj;
            if (rr < a.M && col < a.N)
              cb[c][k] = *reinterpret_cast<const float4*>(static_cast<const float*>(a.c) + rr * a.ldc + col);
          }
      }
      float scale = 1.f;
      if (a.rs_part != nullptr && live) {
        float ss = 0.f;
        for (int p = 0; p < a.rs_parts; ++p) ss += __ldg(a.rs_part + grow * a.rs_ld + p);
        scale = rsqrtf(ss * a.rs_inv_d + a.rs_eps);
      }
      float ssum[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) ssum[k] = 0.f;
      bool released = false;
      mbar_wait(tfull + acc, (i >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col0 = c0 + c * 32;
        if (col0 >= a.N) break;  // warp-uniform
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + acc * BN + half * HC + c * 32, r);
        tmem_wait_ld();
        if (c == NCH - 1) {  // every TMEM column of this warp is read: release the buffer
          release_acc(tempty + acc);
          released = true;
        }
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) * scale;
        if (a.relu) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = fmaxf(v[e], 0.f);
        }
        if (a.rope_cos != nullptr && live) {
          const int64_t span = (int64_t)a.rope_heads * a.rope_hs;
          int64_t base = -1;
          if (col0 >= a.rope_q0 && col0 < a.rope_q0 + span) base = a.rope_q0;
          else if (col0 >= a.rope_k0 && col0 < a.rope_k0 + span) base = a.rope_k0;
          if (base >= 0) {
            const int k0 = (int)(((col0 - base) % a.rope_hs) >> 1);
            const int64_t tab = (a.rope_row0 + grow) * a.rope_pairs + k0;
            if (a.rope_vec && k0 + 16 <= a.rope_pairs) {  // 16 pairs as 4 x float4 per table
#pragma unroll
              for (int e4 = 0; e4 < 4; ++e4) {
                const float4 cs = __ldg(reinterpret_cast<const float4*>(a.rope_cos + tab) + e4);
                const float4 sn = __ldg(reinterpret_cast<const float4*>(a.rope_sin + tab) + e4);
                const float cv[4] = {cs.x, cs.y, cs.z, cs.w}, sv[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int e = 4 * e4 + u;
                  const float x0 = v[2 * e], x1 = v[2 * e + 1];
                  v[2 * e] = x0 * cv[u] - x1 * sv[u];
                  v[2 * e + 1] = x0 * sv[u] + x1 * cv[u];
                }
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                if (k0 + e < a.rope_pairs) {
                  const float cs = __ldg(a.rope_cos + tab + e), sn = __ldg(a.rope_sin + tab + e);
                  const float x0 = v[2 * e], x1 = v[2 * e + 1];
                  v[2 * e] = x0 * cs - x1 * sn;
                  v[2 * e + 1] = x0 * sn + x1 * cs;
                }
              }
            }
          }
        }
        if (a.c_f32) {
          // stage: row `lane` as 8 x 16 B, piece j at (j ^ (row & 7)) (conflict-free)
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                             stg_u + lane * 128 + ((jj ^ (lane & 7)) << 4)),
                         "f"(v[4 * jj]), "f"(v[4 * jj + 1]), "f"(v[4 * jj + 2]), "f"(v[4 * jj + 3])
                         : "memory");
          __syncwarp();
          const int col = col0 + 4 * fj;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rl = k * 4 + fr;
            float4 o;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(o.x), "=f"(o.y), "=f"(o.z), "=f"(o.w)
                         : "r"(stg_u + rl * 128 + ((fj ^ (rl & 7)) << 4)));
            const int64_t rr = r0 + rl;
            if (rr < a.M && col < a.N) {
              if (beta_on) {
                const float4 p = cb[c % PD][k];
                o.x = fmaf(a.beta, p.x, o.x);
                o.y = fmaf(a.beta, p.y, o.y);
                o.z = fmaf(a.beta, p.z, o.z);
                o.w = fmaf(a.beta, p.w, o.w);
              }
              *reinterpret_cast<float4*>(static_cast<float*>(a.c) + rr * a.ldc + col) = o;
              if (a.emit_b != nullptr) {
                ssum[k] = fmaf(o.x, o.x, fmaf(o.y, o.y, fmaf(o.z, o.z, fmaf(o.w, o.w, ssum[k]))));
                *reinterpret_cast<uint2*>(a.emit_b + rr * a.emit_ld + col) =
                    make_uint2(pack_bf16(o.x, o.y), pack_bf16(o.z, o.w));
              }
            }
            if (beta_on && c + PD < NCH) {  // refill this ring slot with chunk c + PD
              if (rr < a.M && col + PD * 32 < a.N)
                cb[c % PD][k] = *reinterpret_cast<const float4*>(static_cast<const float*>(a.c) +
                                                                rr * a.ldc + col + PD * 32);
            }
          }
          __syncwarp();
        } else {
          // stage: row `lane` as 4 x 16 B (64 B rows), piece j at (j ^ ((row >> 1) & 3))
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             stg_u + lane * 64 + ((jj ^ ((lane >> 1) & 3)) << 4)),
                         "r"(pack_bf16(v[8 * jj], v[8 * jj + 1])), "r"(pack_bf16(v[8 * jj + 2], v[8 * jj + 3])),
                         "r"(pack_bf16(v[8 * jj + 4], v[8 * jj + 5])), "r"(pack_bf16(v[8 * jj + 6], v[8 * jj + 7]))
                         : "memory");
          __syncwarp();
          const int col = col0 + 8 * bj;
          // peer scatter: a 32-column chunk lies in one column block (scat_w % 32 == 0), so
          // its (<= 2) destinations are read once per chunk, not per store
          uint8_t* sc_base[2] = {nullptr, nullptr};
          int64_t sc_ld[2] = {0, 0}, sc_lo[2] = {0, 0}, sc_hi[2] = {0, 0};
          if (a.scat != nullptr && col0 < a.N) {
            const int blk = col0 / a.scat_w;
            const int64_t* d = a.scat + (int64_t)blk * 8;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              sc_ld[e] = __ldg(d + 4 * e + 1);
              sc_lo[e] = __ldg(d + 4 * e + 2);
              sc_hi[e] = __ldg(d + 4 * e + 3);
              sc_base[e] = reinterpret_cast<uint8_t*>(__ldg(d + 4 * e)) +
                           (int64_t)(col - blk * a.scat_w) * 2;
            }
          }
          int pstream = -1;  // page write: 0 = K stream, 1 = V stream of this chunk
          int64_t poff = 0;
          if (a.slots != nullptr) {
            if (col0 >= a.pk_col0 && col0 < a.pk_col0 + a.pwidth) {
              pstream = 0;
              poff = (int64_t)(col - a.pk_col0) * 2;
            } else if (col0 >= a.pv_col0 && col0 < a.pv_col0 + a.pwidth) {
              pstream = 1;
              poff = (int64_t)(col - a.pv_col0) * 2;
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int rl = k * 8 + br;
            uint4 o;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w)
                         : "r"(stg_u + rl * 64 + ((bj ^ ((rl >> 1) & 3)) << 4)));
            const int64_t rr = r0 + rl;
            if (rr < a.M && col < a.N) {
              if (a.c != nullptr)
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.c) + rr * a.ldc + col) = o;
              if (a.scat != nullptr) {  // straight into the consumer rank's buffer (NVLink)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                  if (rr >= sc_lo[e] && rr < sc_hi[e])
                    *reinterpret_cast<uint4*>(sc_base[e] + rr * sc_ld[e]) = o;
              }
              if (pstream >= 0) {
                const int64_t rel = a.rel0 + rr;
                const int pg = (int)(rel / a.page_len);
                const int32_t code = __ldg(a.slots + pg);
                const int64_t prow = (int64_t)(code >= 0 ? code : -1 - code) * a.page_len +
                                     (rel - (int64_t)pg * a.page_len);
                uint8_t* dst = (code >= 0 ? (pstream ? a.pv_dev : a.pk_dev)
                                          : (pstream ? a.pv_host : a.pk_host)) +
                               prow * a.prow_b + poff;
                *reinterpret_cast<uint4*>(dst) = o;
              }
            }
          }
          __syncwarp();
        }
      }
      if (!released) release_acc(tempty + acc);  // ragged N: last columns past the edge
      if (a.emit_ss != nullptr) {  // per-row sums of this warp's columns (8 lanes per row)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float sk = ssum[k];
          sk += __shfl_xor_sync(0xffffffffu, sk, 1);
          sk += __shfl_xor_sync(0xffffffffu, sk, 2);
          sk += __shfl_xor_sync(0xffffffffu, sk, 4);
          const int64_t rr = r0 + k * 4 + fr;
          if (fj == 0 && rr < a.M && tn < a.tiles_n) a.emit_ss[rr * a.emit_ss_ld + 2 * tn + half] = sk;
        }
      }
    }
  }

  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  // peer-scatter stores out before the barrier that publishes them (one system fence per
  // CTA, cumulative over the CTA's stores through the bar.sync above)
  if (threadIdx.x == 0 && a.scat != nullptr) __threadfence_system();
  if (CL > 1) cluster_sync_all();  // no multicast or remote arrive still targets this CTA
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tmem, L::TM_COLS);
    else tmem_dealloc<L::TM_COLS>(tmem);
  }
}

template <int BN, int CL, bool PAIR = false>
int launch(const GemmArgs& a, cudaStream_t st) {
  using L = GLayout<BN, PAIR ? BN / 2 : BN>;
  static DeviceFlags attr_set;
  const int dev = current_device();
  if (attr_set.first(dev)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, CL, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set.set(dev);
  }
  const int units = PAIR ? a.tiles_m * a.tiles_n : a.tiles_m * ((a.tiles_n + CL - 1) / CL);
  const int n_sm = device_sms(dev);
  const int per = n_sm / CL;
  const int grid = (units < per ? units : per) * CL;
  if (CL == 1) {
    return (int)launch_pdl(gemm_kernel<BN, 1, false>, dim3(grid), dim3(NTHREADS), L::SMEM, st, 1, a);
  }
  return (int)launch_pdl(gemm_kernel<BN, CL, PAIR>, dim3(grid), dim3(NTHREADS), L::SMEM, st, CL, a);
}

}  // namespace

// Tile plan: output tile width BN and mode (1: one CTA per 128 x BN tile; 2: a cluster of
// two column tiles sharing A by multicast; 3: a cta_group::2 CTA pair per 256 x BN tile).
// Modelled time = waves x (K steps x 2 BN / util + 2,500) clk, with the tensor-pipe
// utilisation of each main loop and the per-tile ramp / exposed epilogue fitted to the
// c2 / c4 projection shapes (tools/gemm_probe.py, profiles/r04_g1.md): one CTA reaches
// ~0.78 at BN 192-256 (its K step moves A + B through shared memory twice, TMA fill and
// tensor-core read, against 2 BN clk of MMA), a CTA pair ~0.91 at BN 256 (each SM holds
// only half of B). Mode 2 (L2 traffic only) is kept for A/B (IFX_G1_MODE=2).
void gemm_plan(int64_t M, int64_t N, int64_t K, int n_sm, int* bn_out, int* mode_out) {
  static const int forced_bn = [] {
    const char* e = std::getenv("IFX_G1_BN");
    return e ? std::atoi(e) : 0;
  }();
  static const int forced_mode = [] {
    const char* e = std::getenv("IFX_G1_MODE");
    return e ? std::atoi(e) : 0;
  }();
  const int64_t k_iters = (K + BK - 1) / BK;
  double best = 1e300;
  int bn_best = 64, mode_best = 1;
  for (int mode : {1, 3}) {
    if (forced_mode && mode != (forced_mode == 2 ? 1 : forced_mode)) continue;
    for (int bn : {256, 192, 128, 64}) {
      if (forced_bn && bn != forced_bn) continue;
      if (mode == 3 && bn != 256 && bn != 128) continue;
      const int64_t rows = mode == 3 ? 2 * BM : BM;
      const int64_t units = ((M + rows - 1) / rows) * ((N + bn - 1) / bn);
      const int64_t slots = mode == 3 ? n_sm / 2 : n_sm;
      const int64_t waves = (units + slots - 1) / slots;
      const double util = mode == 3 ? (bn == 256 ? 0.91 : 0.80)
                                    : (bn >= 192 ? 0.78 : (bn == 128 ? 0.70 : 0.55));
      const double cost = (double)waves * ((double)k_iters * 2.0 * bn / util + 2500.0);
      if (cost < best * (1 - 1e-9)) {
        best = cost;
        bn_best = bn;
        mode_best = mode;
      }
    }
  }
  if (forced_mode == 2 && ((N + bn_best - 1) / bn_best) % 2 == 0) mode_best = 2;
  *bn_out = bn_best;
  *mode_out = mode_best;
}

int gemm_launch(const GemmArgs& a, int bn, int cl, cudaStream_t st) {
  if (cl == 3) {  // CTA pair
    switch (bn) {
      case 128: return launch<128, 2, true>(a, st);
      case 256: return launch<256, 2, true>(a, st);
      default: return (int)cudaErrorInvalidValue;
    }
  }
  if (cl == 2) {
    switch (bn) {
      case 64: return launch<64, 2>(a, st);
      case 128: return launch<128, 2>(a, st);
      case 192: return launch<192, 2>(a, st);
      case 256: return launch<256, 2>(a, st);
      default: return (int)cudaErrorInvalidValue;
    }
  }
  switch (bn) {
    case 64: return launch<64, 1>(a, st);
    case 128: return launch<128, 1>(a, st);
    case 192: return launch<192, 1>(a, st);
    case 256: return launch<256, 1>(a, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace ifx
