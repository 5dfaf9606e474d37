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
#include <cstdlib>

#include "device_state.h"
#include "gemm_kernel.h"
#include "sm100_ptx.cuh"

namespace ifx {
namespace {

using namespace ptx;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NTHREADS = 320;  // producer, MMA, 8 epilogue warps
constexpr int NEPI = 256;

template <int BN>
struct GLayout {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BK * BN * 2;
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

__device__ __forceinline__ void st_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  *reinterpret_cast<uint4*>(p) = make_uint4(a, b, c, d);
}

template <int BN>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_kernel(const __grid_constant__ GemmArgs a) {
  using L = GLayout<BN>;
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
  const int n_tiles = a.tiles_m * a.tiles_n;
  const int k_iters = (a.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < L::NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, NEPI);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<L::TM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (elect_one()) {
      tma_prefetch_desc(&a.tm_a);
      tma_prefetch_desc(&a.tm_b);
      int g = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int m0 = (t % a.tiles_m) * BM, n0 = (t / a.tiles_m) * BN;
        for (int kb = 0; kb < k_iters; ++kb, ++g) {
          const int s = g % L::NST;
          mbar_wait(empty + s, ((g / L::NST) & 1) ^ 1);
          uint8_t* st = smem + s * L::STAGE;
          mbar_expect_tx(full + s, L::STAGE);
          tma_load_2d(st, &a.tm_a, full + s, kb * BK, m0);
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_2d(st + L::A_BYTES + c * (BK * 128), &a.tm_b, full + s, n0 + c * 64, kb * BK);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, 0, 1);  // A K-major, B MN-major
      int g = 0, i = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
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
            mma_bf16_ss(d, smem_desc_sw128(a_base + kk * 32, 16, 1024),
                        smem_desc_sw128(b_base + kk * 16 * 128, BK * 128, 1024), idesc,
                        (kb | kk) != 0);
          }
          mma_commit(empty + s);
        }
        mma_commit(tfull + acc);
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
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool beta_on = a.c_f32 && a.beta != 0.f;
    uint8_t* stg = smem + L::OFF_STG + (warp - 2) * 4096;
    const uint32_t stg_u = smem_u32(stg);
    // coalesced-domain coordinates: fp32 rows k*4 + (lane >> 3), 16 B column piece lane & 7;
    // bf16 rows k*8 + (lane >> 2), piece lane & 3
    const int fr = lane >> 3, fj = lane & 7;
    const int br = lane >> 2, bj = lane & 3;
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      const int tm = t % a.tiles_m, tn = t / a.tiles_m;
      const int64_t r0 = (int64_t)tm * BM + q * 32;  // first row of this warp
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
          tc_fence_before();
          mbar_arrive(tempty + acc);
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
            const int64_t tab = (a.rope_row0 + grow) * a.rope_pairs;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              if (k0 + e < a.rope_pairs) {
                const float cs = __ldg(a.rope_cos + tab + k0 + e), sn = __ldg(a.rope_sin + tab + k0 + e);
                const float x0 = v[2 * e], x1 = v[2 * e + 1];
                v[2 * e] = x0 * cs - x1 * sn;
                v[2 * e + 1] = x0 * sn + x1 * cs;
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
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.c) + rr * a.ldc + col) = o;
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
      if (!released) {  // ragged N: this warp's last columns were past the edge
        tc_fence_before();
        mbar_arrive(tempty + acc);
      }
      if (a.emit_ss != nullptr) {  // per-row sums of this warp's columns (8 lanes per row)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float sk = ssum[k];
          sk += __shfl_xor_sync(0xffffffffu, sk, 1);
          sk += __shfl_xor_sync(0xffffffffu, sk, 2);
          sk += __shfl_xor_sync(0xffffffffu, sk, 4);
          const int64_t rr = r0 + k * 4 + fr;
          if (fj == 0 && rr < a.M) a.emit_ss[rr * a.emit_ss_ld + 2 * tn + half] = sk;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<L::TM_COLS>(tmem);
  }
}

template <int BN>
int launch(const GemmArgs& a, cudaStream_t st) {
  using L = GLayout<BN>;
  static DeviceFlags attr_set;
  const int dev = current_device();
  if (attr_set.first(dev)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set.set(dev);
  }
  const int tiles = a.tiles_m * a.tiles_n;
  const int n_sm = device_sms(dev);
  const int grid = tiles < n_sm ? tiles : n_sm;
  gemm_kernel<BN><<<grid, NTHREADS, L::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace

// Output tile width: fewest waves x per-tile cost on n_sm SMs (a tile's cost ~ BN + a fixed
// ramp / epilogue share). At T = 4,680 rows (37 row tiles, 148 = 4 x 37) BN = 192 makes
// every c2 projection whole waves: N = 1,536 / 3,072 / 4,608 -> 296 / 592 / 888 tiles.
int gemm_pick_bn(int64_t M, int64_t N, int n_sm) {
  static const int forced = [] {
    const char* e = std::getenv("IFX_G1_BN");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 64 || forced == 128 || forced == 192 || forced == 256) return forced;
  const int64_t tm = (M + BM - 1) / BM;
  int best = 64;
  int64_t best_cost = INT64_MAX;
  for (int bn : {256, 192, 128, 64}) {
    const int64_t tiles = tm * ((N + bn - 1) / bn);
    const int64_t waves = (tiles + n_sm - 1) / n_sm;
    const int64_t cost = waves * (bn + 48);
    if (cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

int gemm_launch(const GemmArgs& a, int bn, cudaStream_t st) {
  switch (bn) {
    case 64: return launch<64>(a, st);
    case 128: return launch<128>(a, st);
    case 192: return launch<192>(a, st);
    case 256: return launch<256>(a, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace ifx
