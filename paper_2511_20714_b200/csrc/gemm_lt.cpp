// gemm_lt.cpp — the engine's dense projections on cuBLASLt with per-shape algorithm choice.
//
// Plain library GEMMs (QKV, wo / co / w2 with the fp32 residual as C, w1 + ReLU, eps):
// D[M,N] = A[M,K] . B[K,N] (+ beta * C), row-major bf16 operands, fp32 accumulate, D fp32 or
// bf16. cuBLASLt's first heuristic is not always its fastest algorithm on these shapes
// (tools/lt_algo_probe: w2 4680x1536x3072 runs 19 % faster with the 7th candidate), so the
// first call of each shape outside a CUDA-graph capture times the top candidates on scratch
// outputs and keeps the fastest. A shape first seen inside a capture keeps the first
// heuristic for good, so captured and later eager calls of one shape run the same algorithm
// (bit-identical results). Handles, workspaces and plans are per device.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ifx_abi.h"
#include "common_host.h"

namespace {

using Key =
    std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, int, int, int64_t>;

struct Plan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulAlgo_t algo{};
  bool tuned = false;
};

struct Lt {
  cublasLtHandle_t h = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 32u << 20;
  std::map<Key, Plan> plans;
  std::mutex mu;
};

constexpr int kMaxDevices = 64;

Lt& lt(int dev) {
  static Lt s[kMaxDevices];
  return s[dev];
}

int lt_fail(const char* what, int st) {
  return ifx::fail(IFX_ECUDA, std::string(what) + " failed: status " + std::to_string(st));
}

}  // namespace

extern "C" int ifx_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* D,
                             int64_t ldd, int d_type, int64_t M, int64_t N, int64_t K, float beta,
                             int relu, void* stream) {
  if (M < 0 || N < 0 || K < 1 || lda < K || ldb < N || ldd < N)
    return ifx::fail(IFX_EDIM, "bad gemm sizes");
  if (M == 0 || N == 0) return IFX_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return ifx::fail(IFX_ECUDA, "gemm: no current CUDA device");
  Lt& L = lt(dev);
  std::lock_guard<std::mutex> g(L.mu);
  auto st = static_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) return ifx::fail(IFX_ECUDA, "gemm stream");
  if (!L.h && cap != cudaStreamCaptureStatusNone)  // cudaMalloc is illegal inside a capture
    return ifx::fail(IFX_ECUDA, "gemm: first call inside a CUDA graph capture (run it eagerly once)");
  if (!L.h) {
    if (int s = cublasLtCreate(&L.h)) return lt_fail("cublasLtCreate", s);
    if (cudaMalloc(&L.ws, L.ws_bytes) != cudaSuccess) return ifx::fail(IFX_ECUDA, "gemm workspace");
  }
  const cudaDataType_t dt = d_type == IFX_F32 ? CUDA_R_32F : CUDA_R_16BF;
  // pointer alignment is part of the plan: an algorithm chosen for 256-byte aligned operands
  // may refuse a column block of a wider buffer
  auto align = [](const void* ptr) {
    uint32_t a = 256;
    while (a > 2 && (reinterpret_cast<uintptr_t>(ptr) % a)) a >>= 1;
    return a;
  };
  const uint32_t al_a = align(A), al_b = align(B), al_d = align(D);
  const Key key{M, N, K, lda, ldb, ldd, d_type, relu, beta != 0.f,
                (int64_t)al_a << 20 | (int64_t)al_b << 10 | al_d};
  Plan& p = L.plans[key];
  if (!p.op) {  // row-major D = A B  <=>  col-major D^T[N,M] = B^T[N,K] A^T[K,M]
    cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
    cublasLtEpilogue_t epi = relu ? CUBLASLT_EPILOGUE_RELU : CUBLASLT_EPILOGUE_DEFAULT;
    cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi));
    cublasLtMatrixLayoutCreate(&p.la, CUDA_R_16BF, N, K, ldb);
    cublasLtMatrixLayoutCreate(&p.lb, CUDA_R_16BF, K, M, lda);
    cublasLtMatrixLayoutCreate(&p.lc, dt, N, M, ldd);
  }
  const float alpha = 1.f;
  if (!p.tuned) {
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &L.ws_bytes,
                                         sizeof(L.ws_bytes));
    // cuBLASLt's A is our B^T and its B is our A^T
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_A_BYTES, &al_b,
                                         sizeof(al_b));
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_B_BYTES, &al_a,
                                         sizeof(al_a));
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_C_BYTES, &al_d,
                                         sizeof(al_d));
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_D_BYTES, &al_d,
                                         sizeof(al_d));
#ifndef IFX_LT_CANDIDATES
#define IFX_LT_CANDIDATES 8
#endif
    std::vector<cublasLtMatmulHeuristicResult_t> res(IFX_LT_CANDIDATES);
    int got = 0;
    int s = cublasLtMatmulAlgoGetHeuristic(L.h, p.op, p.la, p.lb, p.lc, p.lc, pref, IFX_LT_CANDIDATES, res.data(), &got);
    cublasLtMatmulPreferenceDestroy(pref);
    if (s || got == 0) return lt_fail("cublasLtMatmulAlgoGetHeuristic", s);
    p.algo = res[0].algo;
    if (cap != cudaStreamCaptureStatusNone || got == 1) p.tuned = true;  // frozen (see top)
    if (!p.tuned) {
      // time the candidates on a scratch output (the real D may be the residual C)
      const size_t esz = d_type == IFX_F32 ? 4 : 2;
      void* scratch = nullptr;
      // same offset from a 256-byte boundary as D, so the timed candidates see D's alignment
      const size_t off = reinterpret_cast<uintptr_t>(D) % 256;
      const size_t bytes = ((size_t)(M - 1) * ldd + N) * esz;
      if (cudaMalloc(&scratch, bytes + off) != cudaSuccess) {
        cudaGetLastError();  // no memory to time candidates: keep heuristic #0, clear the error
        p.tuned = true;
      } else {
        void* sd = static_cast<char*>(scratch) + off;
        cudaMemcpyAsync(sd, D, bytes, cudaMemcpyDeviceToDevice, st);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int i = 0; i < got; ++i) {
          bool ok = true;
          for (int r = 0; r < 4 && ok; ++r) {  // 1 warm-up + 3 timed
            if (r == 1) cudaEventRecord(e0, st);
            ok = cublasLtMatmul(L.h, p.op, &alpha, B, p.la, A, p.lb, &beta, sd, p.lc, sd, p.lc,
                                &res[i].algo, L.ws, L.ws_bytes, st) == CUBLAS_STATUS_SUCCESS;
          }
          cudaEventRecord(e1, st);
          cudaEventSynchronize(e1);
          float ms = 0.f;
          if (ok && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess && ms < best) {
            best = ms;
            p.algo = res[i].algo;
          }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamSynchronize(st);
        cudaFree(scratch);
        p.tuned = true;
      }
    }
  }
  int s = cublasLtMatmul(L.h, p.op, &alpha, B, p.la, A, p.lb, &beta, D, p.lc, D, p.lc, &p.algo,
                         L.ws, L.ws_bytes, st);
  if (s) return lt_fail("cublasLtMatmul", s);
  return IFX_OK;
}
