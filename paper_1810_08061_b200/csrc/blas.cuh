// blas.cuh — the plain library GEMMs of libskb (cuBLAS), shared by the decoder
// (beam.cu) and the TreeLSTM levels (tree.cu).  Row-major C[M,N] = A[M,K] @ B[K,N]
// via column-major C^T = B^T A^T.  math 0: fp32 (no TF32), 1: TF32 tensor cores.
#pragma once
#include <cublas_v2.h>
#include <cuda_runtime.h>

namespace skb {

inline cublasHandle_t blas_handle(cudaStream_t stream) {
  static cublasHandle_t h = nullptr;
  if (!h && cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  cublasSetStream(h, stream);
  return h;
}

inline bool gemm_f32(cublasHandle_t h, int math, const float* A, int lda, const float* B, int ldb, float* C,
                     int ldc, int M, int N, int K, float beta = 0.f) {
  const float one = 1.f;
  const cublasComputeType_t ct = math == 1 ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F_PEDANTIC;
  return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, B, CUDA_R_32F, ldb, A, CUDA_R_32F, lda, &beta, C,
                      CUDA_R_32F, ldc, ct, CUBLAS_GEMM_DEFAULT) == CUBLAS_STATUS_SUCCESS;
}

}  // namespace skb
