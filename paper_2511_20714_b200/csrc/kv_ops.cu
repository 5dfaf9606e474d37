// kv_ops.cu — HBM-bound kernels around the attention: K2 page write (append), K7 gather,
// fused RMS-norm -> bf16, Ulysses pack/unpack. All use 16-byte vector accesses and grids
// sized in multiples of the SM count (grid-stride loops), per the B200 rules in DESIGN.md.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "device_state.h"
#include "kv_kernels.h"
#include "launch.cuh"

namespace ifx {
namespace {

// grid caps scale with the SM count of the current device (148 on B200)
inline int kSMs_now() { return ifx::device_sms(ifx::current_device()); }

__device__ __forceinline__ uint4 ld_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_na(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w));
}
__device__ __forceinline__ uint32_t f2_to_bf2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// ---- K2: page write / K7: gather. One WARP per (K|V, row): lanes stride the row's 16-byte
// vectors, all loads of a row issued before its stores (up to 8 in flight per lane); no
// 64-bit divisions in the hot loop. Grid-stride over 2*rows row units.
template <int UNROLL>
__device__ __forceinline__ void copy_row(const uint8_t* __restrict__ s, uint8_t* __restrict__ d,
                                         int64_t row_vecs, int lane) {
  for (int64_t c0 = lane; c0 < row_vecs; c0 += 32 * UNROLL) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (c0 + u * 32 < row_vecs) v[u] = ld_nc(s + (c0 + u * 32) * 16);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (c0 + u * 32 < row_vecs) st_na(d + (c0 + u * 32) * 16, v[u]);
  }
}

// Pool addressing: a page slot code c >= 0 is device slot c, c < 0 is host slot -1-c; a
// slot is page_len consecutive rows of `width` elements. Host pools are mapped pinned
// memory, so the same kernels read and write both tiers (host traffic crosses PCIe).
struct PoolPtrs {
  uint8_t* dev_k;
  uint8_t* dev_v;
  uint8_t* host_k;
  uint8_t* host_v;
  int64_t row_b;  // bytes per row (= width * esz; rows are dense inside a slot)
  int page_len;
};

__device__ __forceinline__ uint8_t* pool_row(const PoolPtrs& p, bool is_v, int32_t code,
                                             int in_page) {
  const int64_t r = (int64_t)(code >= 0 ? code : -1 - code) * p.page_len + in_page;
  uint8_t* base = code >= 0 ? (is_v ? p.dev_v : p.dev_k) : (is_v ? p.host_v : p.host_k);
  return base + r * p.row_b;
}

// K2 same-type: row r of K / V (token token0 + r) -> its page slot row
__global__ void append_same(const uint8_t* __restrict__ ks, const uint8_t* __restrict__ vs,
                            int64_t src_ld_b, PoolPtrs pool, const int32_t* __restrict__ slots,
                            int64_t rel0, int64_t t, int64_t row_vecs) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < 2 * t;
       u += n_warps) {
    const bool is_v = u >= t;
    const int64_t r = is_v ? u - t : u;
    const int64_t rel = rel0 + r;  // token - first page's start token
    const int pg = (int)(rel / pool.page_len);
    uint8_t* d = pool_row(pool, is_v, __ldg(slots + pg), (int)(rel - (int64_t)pg * pool.page_len));
    copy_row<8>((is_v ? vs : ks) + r * src_ld_b, d, row_vecs, lane);
  }
}
// fp32 -> bf16: per 16-byte destination vector, 32 source bytes
__global__ void append_f32_bf16(const float* __restrict__ ks, const float* __restrict__ vs,
                                int64_t src_ld, PoolPtrs pool, const int32_t* __restrict__ slots,
                                int64_t rel0, int64_t t, int64_t row_vecs) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < 2 * t;
       u += n_warps) {
    const bool is_v = u >= t;
    const int64_t r = is_v ? u - t : u;
    const int64_t rel = rel0 + r;
    const int pg = (int)(rel / pool.page_len);
    const float* srow = (is_v ? vs : ks) + r * src_ld;
    uint8_t* drow =
        pool_row(pool, is_v, __ldg(slots + pg), (int)(rel - (int64_t)pg * pool.page_len));
    for (int64_t c = lane; c < row_vecs; c += 32) {
      const uint4 a = ld_nc(srow + c * 8), b = ld_nc(srow + c * 8 + 4);
      uint4 o;
      o.x = f2_to_bf2(__uint_as_float(a.x), __uint_as_float(a.y));
      o.y = f2_to_bf2(__uint_as_float(a.z), __uint_as_float(a.w));
      o.z = f2_to_bf2(__uint_as_float(b.x), __uint_as_float(b.y));
      o.w = f2_to_bf2(__uint_as_float(b.z), __uint_as_float(b.w));
      st_na(drow + c * 16, o);
    }
  }
}

// K2 (same type, TMA bulk): each warp streams rows through a 2-deep shared-memory ring with
// the bulk-copy engine — cp.async.bulk global->shared completing on an mbarrier, then
// cp.async.bulk shared->global into the page slot — so a row costs a handful of
// instructions and the copy engine, not registers, keeps the bytes in flight. Rows whose
// page is on the host tier are written by the warp's lanes from shared memory instead.
constexpr int kBulkMaxRowBytes = 12288;  // 2 buffers x 8 warps fit 192 KB of smem

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256) append_bulk(const uint8_t* __restrict__ ks,
                                                   const uint8_t* __restrict__ vs,
                                                   int64_t src_ld_b, PoolPtrs pool,
                                                   const int32_t* __restrict__ slots, int64_t rel0,
                                                   int64_t t, int row_b) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  __shared__ __align__(8) uint64_t bars[8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf[2] = {bulk_smem + (warp * 2) * row_b, bulk_smem + (warp * 2 + 1) * row_b};
  if (lane == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[warp][i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t u0 = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp;
  auto src_of = [&](int64_t u) {
    const bool is_v = u >= t;
    return (is_v ? vs : ks) + (is_v ? u - t : u) * src_ld_b;
  };
  auto issue_load = [&](int64_t u, int k) {
    const uint32_t bar = smem_addr(&bars[warp][k]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(row_b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(buf[k])), "l"(src_of(u)), "r"(row_b), "r"(bar) : "memory");
  };
  uint32_t phase[2] = {0, 0};
  if (lane == 0 && u0 < 2 * t) issue_load(u0, 0);
  int k = 0;
  for (int64_t u = u0; u < 2 * t; u += n_warps, k ^= 1) {
    const int64_t un = u + n_warps;
    if (lane == 0 && un < 2 * t) {
      // the other buffer is free once its previous bulk store finished reading it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue_load(un, k ^ 1);
    }
    // wait for this row's bytes
    const uint32_t bar = smem_addr(&bars[warp][k]);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                   "selp.b32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(bar), "r"(phase[k]) : "memory");
    phase[k] ^= 1;
    const bool is_v = u >= t;
    const int64_t rel = rel0 + (is_v ? u - t : u);
    const int pg = (int)(rel / pool.page_len);
    const int32_t code = __ldg(slots + pg);
    uint8_t* d = pool_row(pool, is_v, code, (int)(rel - (int64_t)pg * pool.page_len));
    if (code >= 0) {
      if (lane == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(d), "r"(smem_addr(buf[k])), "r"(row_b) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {  // host tier (mapped pinned memory): the lanes write it
      for (int c = lane; c < row_b / 16; c += 32)
        reinterpret_cast<uint4*>(d)[c] = reinterpret_cast<const uint4*>(buf[k])[c];
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// K7: out[i] = pool row of token tokens[i] (tokens == NULL: token0 + i), K and V; tokens
// are given relative to the first page's start token
__global__ void gather_rows(PoolPtrs pool, const int32_t* __restrict__ slots,
                            const int64_t* __restrict__ tokens, int64_t rel0, int64_t n,
                            int64_t row_vecs, uint8_t* __restrict__ ko, uint8_t* __restrict__ vo) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < 2 * n;
       u += n_warps) {
    const bool is_v = u >= n;
    const int64_t i = is_v ? u - n : u;
    const int64_t rel = tokens ? tokens[i] - rel0 : rel0 + i;
    const int pg = (int)(rel / pool.page_len);
    const uint8_t* src =
        pool_row(pool, is_v, __ldg(slots + pg), (int)(rel - (int64_t)pg * pool.page_len));
    copy_row<8>(src, (is_v ? vo : ko) + i * pool.row_b, row_vecs, lane);
  }
}

// K6: whole-page copies between the device and host pools (tier moves, staging). moves[i]
// = (device slot, host slot); dir 0 device -> host, 1 host -> device. One warp per
// (move, K|V, 4 KB piece) so a batch of large pages spreads over every SM.
__global__ void move_pages(PoolPtrs pool, const int64_t* __restrict__ moves, int64_t n, int dir,
                           int64_t page_vecs, int64_t piece_vecs) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t pieces = (page_vecs + piece_vecs - 1) / piece_vecs;
  const int64_t units = n * 2 * pieces;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t page_b = page_vecs * 16;
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < units;
       u += n_warps) {
    const int64_t piece = u % pieces;
    const int64_t mv = u / pieces;
    const int64_t m = mv >> 1;
    const bool is_v = mv & 1;
    const int64_t ds = moves[2 * m], hs = moves[2 * m + 1];
    uint8_t* dev = (is_v ? pool.dev_v : pool.dev_k) + ds * page_b;
    uint8_t* host = (is_v ? pool.host_v : pool.host_k) + hs * page_b;
    const int64_t off = piece * piece_vecs * 16;
    const int64_t nv = min(piece_vecs, page_vecs - piece * piece_vecs);
    if (dir == 0)
      copy_row<8>(dev + off, host + off, nv, lane);
    else
      copy_row<8>(host + off, dev + off, nv, lane);
  }
}

// ---- fused RMS norm (engine.py:171-173), one warp per row ------------------------------
__global__ void rms_bf16_kernel(const float* __restrict__ x, int64_t rows, int64_t width,
                                const float* __restrict__ tvec, float t, float* __restrict__ x_out,
                                __nv_bfloat16* __restrict__ y) {
  pdl_wait();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += warps) {
    const float* xr = x + r * width;
    float ss = 0.f;
#pragma unroll 4  // several row loads in flight per warp
    for (int c = lane * 4; c < (int)width; c += 128) {
      float4 v = *reinterpret_cast<const float4*>(xr + c);
      if (tvec) {
        const float4 tv = *reinterpret_cast<const float4*>(tvec + c);
        v.x += t * tv.x; v.y += t * tv.y; v.z += t * tv.z; v.w += t * tv.w;
      }
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = rsqrtf(ss / (float)width + 1e-6f);
#pragma unroll 4
    for (int c = lane * 4; c < (int)width; c += 128) {
      float4 v = *reinterpret_cast<const float4*>(xr + c);
      if (tvec) {
        const float4 tv = *reinterpret_cast<const float4*>(tvec + c);
        v.x += t * tv.x; v.y += t * tv.y; v.z += t * tv.z; v.w += t * tv.w;
        if (x_out) *reinterpret_cast<float4*>(x_out + r * width + c) = v;
      }
      uint2 o;
      o.x = f2_to_bf2(v.x * inv, v.y * inv);
      o.y = f2_to_bf2(v.z * inv, v.w * inv);
      *reinterpret_cast<uint2*>(y + r * width + c) = o;
    }
  }
}

// One CTA of kRmsThreads per row, the row held in registers (x read once): rows up to
// kRmsThreads * 4 * VPT floats. Block reduction of the sum of squares through shared memory.
template <int kRmsThreads, int VPT>
__global__ void __launch_bounds__(kRmsThreads) rms_row_kernel(
    const float* __restrict__ x, int64_t rows, int width, const float* __restrict__ tvec, float t,
    float* __restrict__ x_out, __nv_bfloat16* __restrict__ y) {
  pdl_wait();
  __shared__ float part[kRmsThreads / 32];
  const int tid = threadIdx.x;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* xr = x + r * width;
    float4 v[VPT];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int c = (tid + i * kRmsThreads) * 4;
      if (c < width) {
        v[i] = *reinterpret_cast<const float4*>(xr + c);
        if (tvec) {
          const float4 tv = *reinterpret_cast<const float4*>(tvec + c);
          v[i].x += t * tv.x; v[i].y += t * tv.y; v[i].z += t * tv.z; v[i].w += t * tv.w;
        }
        ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((tid & 31) == 0) part[tid >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < kRmsThreads / 32; ++w) tot += part[w];
    __syncthreads();  // part is rewritten by the next row
    const float inv = rsqrtf(tot / (float)width + 1e-6f);
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int c = (tid + i * kRmsThreads) * 4;
      if (c < width) {
        if (tvec && x_out) *reinterpret_cast<float4*>(x_out + r * width + c) = v[i];
        uint2 o;
        o.x = f2_to_bf2(v[i].x * inv, v[i].y * inv);
        o.y = f2_to_bf2(v[i].z * inv, v[i].w * inv);
        *reinterpret_cast<uint2*>(y + r * width + c) = o;
      }
    }
  }
}

// ---- Ulysses re-shard (parallel.py:150-169): row-major [n][G][W][c] <-> packed [W][n][G][c]
// (G column groups, e.g. Q|K|V, each split into W per-peer chunks of c elements), so one
// all-to-all moves every peer's chunk contiguously. 16-byte vectors.
__global__ void ulysses_transpose(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                  int64_t n, int64_t groups, int64_t world, int64_t chunk_vecs,
                                  int64_t ld_b, bool pack) {
  pdl_wait();
  const int64_t total = n * groups * world * chunk_vecs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % chunk_vecs;
    int64_t rest = i / chunk_vecs;
    const int64_t g = rest % groups;
    rest /= groups;
    const int64_t r = rest % n, p = rest / n;  // packed order: p, r, g, c
    const int64_t packed = i * 16;
    const int64_t rowmaj = r * ld_b + ((g * world + p) * chunk_vecs + c) * 16;
    if (pack)
      *reinterpret_cast<uint4*>(dst + packed) = ld_nc(src + rowmaj);
    else
      *reinterpret_cast<uint4*>(dst + rowmaj) = ld_nc(src + packed);
  }
}

// ---- 3D RoPE on the Q and K column blocks of a fused QKV buffer, in place (bf16) --------
// One thread per (row, head, pair): rotates the interleaved pair (2k, 2k+1) of q and of k by
// the row's angle k (cos/sin tables [tab_rows, pairs], fp32). Semantics: oracle/rope.py.
__global__ void rope_qk_kernel(__nv_bfloat16* __restrict__ qkv, int64_t rows, int64_t ld,
                               int heads, int64_t head_stride, int pairs, int64_t q_col0,
                               int64_t k_col0, const float* __restrict__ cos_t,
                               const float* __restrict__ sin_t, int64_t tab_row0) {
  pdl_wait();
  const int64_t total = rows * heads * pairs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % pairs);
    const int64_t rest = i / pairs;
    const int h = (int)(rest % heads);
    const int64_t r = rest / heads;
    const int64_t t = (tab_row0 + r) * pairs + k;
    const float c = __ldg(cos_t + t), s = __ldg(sin_t + t);
    const int64_t off = r * ld + h * head_stride + 2 * k;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      __nv_bfloat162* p =
          reinterpret_cast<__nv_bfloat162*>(qkv + off + (which == 0 ? q_col0 : k_col0));
      const float2 v = __bfloat1622float2(*p);
      *p = __floats2bfloat162_rn(v.x * c - v.y * s, v.x * s + v.y * c);
    }
  }
}

// ---- gather / scatter of 2-D byte blocks between two buffers (Ulysses re-shard with
// uneven head splits): desc[b] = (src offset, src row stride, dst offset, dst row stride,
// rows, row bytes) in bytes, row bytes a multiple of 16. grid.x = block, grid.y = row chunk.
__global__ void copy_blocks_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                   const int64_t* __restrict__ desc, int rows_per_cta) {
  pdl_wait();
  const int64_t* d = desc + 6 * blockIdx.x;
  const int64_t rows = d[4];
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  if (r0 >= rows) return;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  const int64_t vecs = d[5] / 16;
  const int lane = threadIdx.x & 31;
  for (int64_t r = r0 + (threadIdx.x >> 5); r < r1; r += blockDim.x >> 5)
    copy_row<4>(src + d[0] + r * d[1], dst + d[2] + r * d[3], vecs, lane);
}

// ---- softmax over groups of a few logits (the folded cross-attention, engine.py:211-215):
// p[r, g*gs + j] = bf16(softmax_j(s[r, g*gs + j] * scale)), one thread per (row, group)
// rs_part != nullptr: the logits are (bf16 x) . W rows whose RMS norm (engine.py:171-173)
// is still to be applied: row r is scaled by rsqrt(sum_p rs_part[r, p] * inv_d + eps) (the
// statistics G1's residual epilogue left, see gemm_sm100.cu)
__global__ void group_softmax_kernel(const float* __restrict__ s, int64_t rows, int groups,
                                     int gs, int64_t ld, float scale_log2_in,
                                     __nv_bfloat16* __restrict__ p, int64_t p_ld,
                                     const float* __restrict__ rs_part, int rs_parts,
                                     int64_t rs_ld, float rs_inv_d, float rs_eps) {
  pdl_wait();
  const int64_t total = rows * groups;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / groups;
    const int g = (int)(i - r * groups);
    float scale_log2 = scale_log2_in;
    if (rs_part != nullptr) {
      float ss = 0.f;
      for (int q = 0; q < rs_parts; ++q) ss += __ldg(rs_part + r * rs_ld + q);
      scale_log2 *= rsqrtf(ss * rs_inv_d + rs_eps);
    }
    const float* sr = s + r * ld + (int64_t)g * gs;
    __nv_bfloat16* pr = p + r * p_ld + (int64_t)g * gs;
    float m = -INFINITY;
    for (int j = 0; j < gs; ++j) m = fmaxf(m, sr[j] * scale_log2);
    float l = 0.f;
    for (int j = 0; j < gs; ++j) l += exp2f(sr[j] * scale_log2 - m);
    const float inv = 1.f / l;
    for (int j = 0; j < gs; ++j) pr[j] = __float2bfloat16(exp2f(sr[j] * scale_log2 - m) * inv);
  }
}

int grid_for(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)kSMs_now() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace

static PoolPtrs pool_ptrs(void* dk, void* dv, void* hk, void* hv, int64_t width, int esz,
                          int64_t page_len) {
  return PoolPtrs{static_cast<uint8_t*>(dk), static_cast<uint8_t*>(dv), static_cast<uint8_t*>(hk),
                  static_cast<uint8_t*>(hv), width * esz, (int)page_len};
}

int kv_append_launch(const void* ks, const void* vs, int64_t src_ld, int src_bf16, void* dk,
                     void* dv, void* hk, void* hv, int pool_bf16, int64_t width, int64_t page_len,
                     const int32_t* slots, int64_t rel0, int64_t t, cudaStream_t st) {
  const int threads = 256;
  const PoolPtrs pool = pool_ptrs(dk, dv, hk, hv, width, pool_bf16 ? 2 : 4, page_len);
  if (!src_bf16 && pool_bf16) {
    launch_pdl(append_f32_bf16, dim3(grid_for(2 * t * 32, threads)), dim3(threads), 0, st, 1,
        static_cast<const float*>(ks), static_cast<const float*>(vs), src_ld, pool, slots, rel0, t,
        width / 8);
  } else if ((width * (pool_bf16 ? 2 : 4)) <= kBulkMaxRowBytes && !std::getenv("IFX_K2_SIMT")) {
    const int row_b = (int)(width * (pool_bf16 ? 2 : 4));
    const size_t smem = (size_t)16 * row_b;  // 8 warps x 2 buffers
    static DeviceFlags attr;  // per device context
    const int dev = current_device();
    if (attr.first(dev)) {
      cudaFuncSetAttribute(append_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           16 * kBulkMaxRowBytes);
      attr.set(dev);
    }
    int blocks = (int)((2 * t + 7) / 8);
    const int cap = kSMs_now() * (row_b <= 4096 ? 4 : 1);
    if (blocks > cap) blocks = cap;
    launch_pdl(append_bulk, dim3(blocks), dim3(threads), smem, st, 1, static_cast<const uint8_t*>(ks),
                                               static_cast<const uint8_t*>(vs),
                                               src_ld * (pool_bf16 ? 2 : 4), pool, slots, rel0, t,
                                               row_b);
  } else {
    const int esz = pool_bf16 ? 2 : 4;
    launch_pdl(append_same, dim3(grid_for(2 * t * 32, threads)), dim3(threads), 0, st, 1,
        static_cast<const uint8_t*>(ks), static_cast<const uint8_t*>(vs), src_ld * esz, pool, slots,
        rel0, t, width * esz / 16);
  }
  return (int)cudaGetLastError();
}

int kv_gather_launch(void* dk, void* dv, void* hk, void* hv, int esz, int64_t width,
                     int64_t page_len, const int32_t* slots, const int64_t* tokens, int64_t rel0,
                     int64_t n, void* ko, void* vo, cudaStream_t st) {
  const int threads = 256;
  const PoolPtrs pool = pool_ptrs(dk, dv, hk, hv, width, esz, page_len);
  gather_rows<<<grid_for(2 * n * 32, threads), threads, 0, st>>>(
      pool, slots, tokens, rel0, n, width * esz / 16, static_cast<uint8_t*>(ko),
      static_cast<uint8_t*>(vo));
  return (int)cudaGetLastError();
}

int kv_move_launch(void* dk, void* dv, void* hk, void* hv, int esz, int64_t width,
                   int64_t page_len, const int64_t* moves, int64_t n, int dir, cudaStream_t st) {
  const int threads = 256;
  const PoolPtrs pool = pool_ptrs(dk, dv, hk, hv, width, esz, page_len);
  const int64_t page_vecs = page_len * width * esz / 16;
  const int64_t piece = 256;  // 4 KB per warp task
  const int64_t units = n * 2 * ((page_vecs + piece - 1) / piece);
  move_pages<<<grid_for(units * 32, threads), threads, 0, st>>>(pool, moves, n, dir, page_vecs,
                                                                piece);
  return (int)cudaGetLastError();
}

int copy_blocks_launch(const void* src, void* dst, const int64_t* desc, int64_t n_blocks,
                       int64_t max_rows, cudaStream_t st) {
  const int rows_per_cta = 64;
  dim3 grid((unsigned)n_blocks, (unsigned)((max_rows + rows_per_cta - 1) / rows_per_cta));
  launch_pdl(copy_blocks_kernel, dim3(grid), dim3(256), 0, st, 1, static_cast<const uint8_t*>(src),
                                           static_cast<uint8_t*>(dst), desc, rows_per_cta);
  return (int)cudaGetLastError();
}

int group_softmax_launch(const float* s, int64_t rows, int groups, int gs, int64_t ld,
                         float scale_log2, void* p, int64_t p_ld, const float* rs_part,
                         int rs_parts, int64_t rs_ld, float rs_inv_d, float rs_eps,
                         cudaStream_t st) {
  const int threads = 256;
  launch_pdl(group_softmax_kernel, dim3(grid_for(rows * groups, threads)), dim3(threads), 0, st, 1,
      s, rows, groups, gs, ld, scale_log2, static_cast<__nv_bfloat16*>(p), p_ld, rs_part,
      rs_parts, rs_ld, rs_inv_d, rs_eps);
  return (int)cudaGetLastError();
}

int rms_launch(const float* x, int64_t rows, int64_t width, const float* tvec, float t,
               float* x_out, void* y, cudaStream_t st) {
  auto* yb = static_cast<__nv_bfloat16*>(y);
  const int64_t v128 = (width / 4 + 127) / 128;  // float4 per thread at 128 threads
  const int gr = (int)(rows < (int64_t)kSMs_now() * 64 ? rows : (int64_t)kSMs_now() * 64);
  if (v128 <= 24 && gr > 0) {  // wider rows: the warp-per-row kernel (two passes)
    if (v128 <= 3)
      launch_pdl(rms_row_kernel<128, 3>, dim3(gr), dim3(128), 0, st, 1, x, rows, (int)width, tvec, t, x_out, yb);
    else if (v128 <= 6)
      launch_pdl(rms_row_kernel<128, 6>, dim3(gr), dim3(128), 0, st, 1, x, rows, (int)width, tvec, t, x_out, yb);
    else if (v128 <= 12)  // e.g. 5,120 (Wan-14B): 256 threads x 5 vectors
      launch_pdl(rms_row_kernel<256, 6>, dim3(gr), dim3(256), 0, st, 1, x, rows, (int)width, tvec, t, x_out, yb);
    else
      launch_pdl(rms_row_kernel<512, 6>, dim3(gr), dim3(512), 0, st, 1, x, rows, (int)width, tvec, t, x_out, yb);
    return (int)cudaGetLastError();
  }
  const int threads = 256;
  const int64_t blocks = (rows + 7) / 8;
  const int g = (int)(blocks < (int64_t)kSMs_now() * 16 ? blocks : (int64_t)kSMs_now() * 16);
  launch_pdl(rms_bf16_kernel, dim3(g), dim3(threads), 0, st, 1, x, rows, width, tvec, t, x_out, yb);
  return (int)cudaGetLastError();
}

int rope_launch(void* qkv, int64_t rows, int64_t ld, int heads, int64_t head_stride, int pairs,
                int64_t q_col0, int64_t k_col0, const float* cos_t, const float* sin_t,
                int64_t tab_row0, cudaStream_t st) {
  const int threads = 256;
  launch_pdl(rope_qk_kernel, dim3(grid_for(rows * heads * pairs, threads)), dim3(threads), 0, st, 1,
      static_cast<__nv_bfloat16*>(qkv), rows, ld, heads, head_stride, pairs, q_col0, k_col0, cos_t,
      sin_t, tab_row0);
  return (int)cudaGetLastError();
}

int ulysses_launch(const void* src, void* dst, int64_t n, int64_t groups, int64_t world,
                   int64_t chunk_bytes, int64_t ld_bytes, bool pack, cudaStream_t st) {
  const int threads = 256;
  const int64_t cv = chunk_bytes / 16;
  launch_pdl(ulysses_transpose, dim3(grid_for(n * groups * world * cv, threads)), dim3(threads), 0, st, 1,
      static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), n, groups, world, cv, ld_bytes,
      pack);
  return (int)cudaGetLastError();
}

}  // namespace ifx
