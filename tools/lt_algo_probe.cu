// lt_algo_probe.cu — how far from the best cuBLASLt algorithm is the default heuristic for
// the engine's GEMM shapes? D[fp32, M x N] (+)= A[bf16, M x K] . B[bf16, K x N], row-major
// (torch layout; cuBLASLt sees the column-major transposes). Times the top-N heuristic
// results with CUDA events. Build: nvcc -O2 -arch=sm_100a lt_algo_probe.cu -lcublasLt
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void fill_rand(__nv_bfloat16* p, size_t n, unsigned seed, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    p[i] = __float2bfloat16(((h & 0xFFFF) / 65535.f - 0.5f) * scale);
  }
}

#define CK(x) do { auto e = (x); if (e != 0) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); return 1; } } while (0)

int run(cublasLtHandle_t lt, int M, int N, int K, bool beta1, const char* name) {
  // row-major C[M,N] = A[M,K] B[K,N]  <=>  col-major C^T[N,M] = B^T[N,K] A^T[K,M]
  __nv_bfloat16 *A, *B;
  float* C;
  CK(cudaMalloc(&A, (size_t)M * K * 2));
  CK(cudaMalloc(&B, (size_t)K * N * 2));
  CK(cudaMalloc(&C, (size_t)M * N * 4));
  fill_rand<<<1184, 256>>>(A, (size_t)M * K, 1u, 4.f);  // random operands: realistic power
  fill_rand<<<1184, 256>>>(B, (size_t)K * N, 2u, 0.1f);
  cudaMemset(C, 0, (size_t)M * N * 4);
  void* ws;
  size_t ws_bytes = 64 << 20;
  CK(cudaMalloc(&ws, ws_bytes));
  cublasLtMatmulDesc_t op;
  CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  cublasLtMatrixLayout_t la, lb, lc;
  CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, N, K, N));  // B^T as col-major [N,K]
  CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, M, K));  // A^T as col-major [K,M]
  CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, N, M, N));
  cublasLtMatmulPreference_t pref;
  CK(cublasLtMatmulPreferenceCreate(&pref));
  CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof(ws_bytes)));
  const int want = 32;
  std::vector<cublasLtMatmulHeuristicResult_t> res(want);
  int got = 0;
  CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, want, res.data(), &got));
  float alpha = 1.f, beta = beta1 ? 1.f : 0.f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double flops = 2.0 * M * N * K;
  printf("%s M=%d N=%d K=%d: %d algos\n", name, M, N, K, got);
  for (int i = 0; i < got; ++i) {
    auto launch = [&]() {
      return cublasLtMatmul(lt, op, &alpha, B, la, A, lb, &beta, C, lc, C, lc, &res[i].algo, ws,
                            ws_bytes, 0);
    };
    if (launch() != CUBLAS_STATUS_SUCCESS) continue;
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    printf("  algo %2d: %8.1f us  %7.1f TFLOP/s%s\n", i, ms * 1e3, flops / ms / 1e9, i == 0 ? "  (heuristic #0)" : "");
  }
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(ws);
  return 0;
}

int main(int argc, char** argv) {
  cublasLtHandle_t lt;
  cublasLtCreate(&lt);
  const int M = argc > 1 ? atoi(argv[1]) : 4680;
  run(lt, M, 4608, 1536, false, "QKV");
  run(lt, M, 1536, 1536, true, "wo (residual)");
  run(lt, M, 3072, 1536, false, "w1");
  run(lt, M, 1536, 3072, true, "w2 (residual)");
  run(lt, M, 15360, 5120, false, "QKV 14B");
  run(lt, M, 5120, 5120, true, "wo 14B (residual)");
  run(lt, M, 10240, 5120, false, "w1 14B");
  run(lt, M, 5120, 10240, true, "w2 14B (residual)");
  return 0;
}
