// Plain library GEMMs through cuBLAS for the fp32 reference-precision API path
// and the fp32 training GEMMs (the bf16 hot path runs on the hand-written
// tcgen05 GEMM, gemm_tc.cu).  Row-major C[m,n] = A[m,k] @ B[k,n] is issued as
// the column-major product C^T = B^T A^T.  fp32 mode never uses TF32 unless
// asked.  The cuBLAS handle is per thread and device (thread_local), so
// concurrent callers on different streams share no state.
#include "common.cuh"

#include <cublas_v2.h>

namespace lsrm {

struct HandleSlot {
  int device = -1;
  cublasHandle_t h = nullptr;
};
static thread_local HandleSlot g_handles[16];

static int get_handle(cublasHandle_t* out) {
  int dev = 0;
  LSRM_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) return set_error(LSRM_E_CUDA, "device id %d out of range", dev);
  HandleSlot& s = g_handles[dev];
  if (!s.h) {
    if (cublasCreate(&s.h) != CUBLAS_STATUS_SUCCESS)
      return set_error(LSRM_E_CUDA, "cublasCreate failed");
    cublasSetMathMode(s.h, CUBLAS_DEFAULT_MATH);
    s.device = dev;
  }
  *out = s.h;
  return LSRM_OK;
}

}  // namespace lsrm

using namespace lsrm;

extern "C" int lsrm_gemm(int dtype, int64_t m, int64_t n, int64_t k, const void* a,
                         int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc,
                         void* stream) {
  LSRM_REQUIRE(dtype >= 0 && dtype <= 2, "gemm: bad dtype %d", dtype);
  if (m == 0 || n == 0) return LSRM_OK;
  cublasHandle_t h;
  int rc = get_handle(&h);
  if (rc) return rc;
  cublasSetStream(h, as_stream(stream));
  const float one = 1.f, zero = 0.f;
  cublasStatus_t s;
  if (dtype == 0) {
    s = cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)m, (int)k, &one,
                    (const float*)b, (int)ldb, (const float*)a, (int)lda, &zero, (float*)c,
                    (int)ldc);
  } else {
    cudaDataType_t ct = dtype == 1 ? CUDA_R_16BF : CUDA_R_32F;
    s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)m, (int)k, &one, b,
                     CUDA_R_16BF, (int)ldb, a, CUDA_R_16BF, (int)lda, &zero, c, ct, (int)ldc,
                     CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  }
  if (s != CUBLAS_STATUS_SUCCESS) return set_error(LSRM_E_CUDA, "cublas gemm failed: %d", (int)s);
  return LSRM_OK;
}

// Row-major fp32 C[m,n] = alpha op(A) op(B) + beta C, op = transpose when
// trans_* != 0 (op(A) is [m,k], op(B) is [k,n]; lda/ldb are the row strides of
// the stored A/B).  The backward's weight / input gradients.
extern "C" int lsrm_gemm_f32_ex(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                                float alpha, const float* a, int64_t lda, const float* b,
                                int64_t ldb, float beta, float* c, int64_t ldc, int tf32,
                                void* stream) {
  if (m == 0 || n == 0) return LSRM_OK;
  cublasHandle_t h;
  int rc = get_handle(&h);
  if (rc) return rc;
  cublasSetStream(h, as_stream(stream));
  // column-major: C^T (n x m) = op(B)^T op(A)^T; a row-major stored matrix is
  // its own transpose in column-major, so the flags carry over unchanged.
  const cublasOperation_t ob = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t oa = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;
  if (tf32) cublasSetMathMode(h, CUBLAS_TF32_TENSOR_OP_MATH);
  cublasStatus_t s = cublasSgemm(h, ob, oa, (int)n, (int)m, (int)k, &alpha, b, (int)ldb, a,
                                 (int)lda, &beta, c, (int)ldc);
  if (tf32) cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);
  if (s != CUBLAS_STATUS_SUCCESS) return set_error(LSRM_E_CUDA, "cublas gemm_ex failed: %d", (int)s);
  return LSRM_OK;
}
