// K7: the dense per-layer transform (the only GEMM-shaped work on the path).
// Round-1 implementation: cuBLAS fp32 SGEMM in pedantic math mode (no TF32
// down-conversion, so the 1e-3 fp32 tolerance of the north star holds), with
// the bias folded into the operand layout (see hg_layer.cu). Row-major
// wrappers over the column-major library.
#include "hgb200.h"
#include <cublas_v2.h>

#include <mutex>

#include "hg_common.cuh"

namespace hg {
namespace {

std::mutex g_mu;
cublasHandle_t g_handles[64] = {};

int handle_for(cublasHandle_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail("cublas", kCuda, cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_handles[dev]) {
    if (cublasCreate(&g_handles[dev]) != CUBLAS_STATUS_SUCCESS) return fail("cublas", kCublas, "cublasCreate failed");
    cublasSetMathMode(g_handles[dev], CUBLAS_PEDANTIC_MATH);
  }
  *out = g_handles[dev];
  return kOk;
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

// Row-major C[M x N] = alpha * op(A)[M x K] * op(B)[K x N] + beta * C.
int hg_gemm_rm(int transA, int transB, long long M, long long N, long long K, const float* A, long long lda,
               const float* B, long long ldb, float beta, float* C, long long ldc, cudaStream_t stream) {
  if (M == 0 || N == 0) return kOk;
  cublasHandle_t h;
  int st = handle_for(&h);
  if (st) return st;
  if (cublasSetStream(h, stream) != CUBLAS_STATUS_SUCCESS) return fail("hg_gemm_rm", kCublas, "setStream");
  const float alpha = 1.f;
  if (K == 0) beta = beta;  // C = beta*C handled by cuBLAS
  cublasStatus_t s = cublasSgemm(h, transB ? CUBLAS_OP_T : CUBLAS_OP_N, transA ? CUBLAS_OP_T : CUBLAS_OP_N, (int)N,
                                 (int)M, (int)K, &alpha, B, (int)ldb, A, (int)lda, &beta, C, (int)ldc);
  if (s != CUBLAS_STATUS_SUCCESS) return fail("hg_gemm_rm", kCublas, "cublasSgemm failed");
  return kOk;
}

}  // extern "C"
