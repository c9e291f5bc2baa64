// Plain library GEMMs through cuBLAS DGEMM (FP64 DMMA, ~35 TF/s on B200 for
// well-shaped products).  Used only where a product is a plain GEMM into a
// scratch operand outside the speculative predicate chain: the inner product
// G = Y^T C when it is not overlapped with the fast panel (b = 128, TRQRCP,
// the noise-floor tail), the blocked QRs' inner products, and TUXV's A V and
// U^T A.  Everything fused or SM-shared stays in the hand-written kernels.
#include <cublas_v2.h>

#include "runtime.hpp"

namespace rq {

bool gemm_lib(Handle& h, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
              int64_t ldc, cudaStream_t s, int cat) {
  if (!h.use_cublas || m <= 0 || n <= 0 || k <= 0) return false;
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX || lda > INT32_MAX || ldb > INT32_MAX ||
      ldc > INT32_MAX)
    return false;
  if (h.cublas == nullptr) {
    cublasHandle_t ch;
    if (cublasCreate(&ch) != CUBLAS_STATUS_SUCCESS) {
      h.use_cublas = false;
      return false;
    }
    h.cublas = ch;
  }
  cublasHandle_t ch = (cublasHandle_t)h.cublas;
  if (cublasSetStream(ch, s) != CUBLAS_STATUS_SUCCESS) return false;
  (void)cat;   // timed as its own family: not one of this library's kernels
  ProfScope prof(h, kProfLibGemm, 2.0 * m * n * k, 8.0 * ((double)m * k + (double)k * n + 2.0 * m * n), s);
  const cublasStatus_t st =
      cublasDgemm(ch, ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb ? CUBLAS_OP_T : CUBLAS_OP_N, (int)m,
                  (int)n, (int)k, &alpha, A, (int)lda, B, (int)ldb, &beta, C, (int)ldc);
  if (st != CUBLAS_STATUS_SUCCESS) throw std::runtime_error("cublasDgemm failed");
  RQ_CHECK_LAUNCH();
  return true;
}

void release_blas(Handle& h) {
  if (h.cublas != nullptr) cublasDestroy((cublasHandle_t)h.cublas);
  h.cublas = nullptr;
}

}  // namespace rq
