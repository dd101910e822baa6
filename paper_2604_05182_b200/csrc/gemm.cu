// Plain projection GEMMs through cuBLAS (library GEMM; the fused hot ops are
// hand-written).  Row-major C[m,n] = A[m,k] @ B[k,n] is issued as the
// column-major product C^T = B^T A^T.  fp32 mode never uses TF32.
#include "common.cuh"

#include <cublas_v2.h>
#include <cublasLt.h>

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

// cuBLASLt (bias epilogue): one handle + 32 MiB workspace per device, made
// on first use (the documented exception to "no hidden allocation").
struct LtSlot {
  cublasLtHandle_t h = nullptr;
  void* ws = nullptr;
};
static LtSlot g_lt[16];
constexpr size_t kLtWorkspace = 32u << 20;

static int get_lt(int dev, LtSlot** out) {
  if (dev < 0 || dev >= 16) return set_error(LSRM_E_CUDA, "device id %d out of range", dev);
  LtSlot& s = g_lt[dev];
  if (!s.h) {
    if (cublasLtCreate(&s.h) != CUBLAS_STATUS_SUCCESS)
      return set_error(LSRM_E_CUDA, "cublasLtCreate failed");
    LSRM_CUDA(cudaMalloc(&s.ws, kLtWorkspace));
  }
  *out = &s;
  return LSRM_OK;
}

}  // namespace lsrm

using namespace lsrm;

// Row-major D[m,n] = A[m,k] @ B[k,n] (bf16 in, fp32 accumulate) + bias[n]
// (optional) + beta * C, issued as the column-major D^T = B^T A^T with a row
// bias.  C may alias D.
static int lt_gemm(int64_t m, int64_t n, int64_t k, const void* a, int64_t lda, const void* b,
                   int64_t ldb, const void* bias, cudaDataType_t bias_t, float beta,
                   const void* c, int64_t ldc, void* d, int64_t ldd, cudaDataType_t cd_t,
                   void* stream) {
  if (m == 0 || n == 0) return LSRM_OK;
  int dev = 0;
  LSRM_CUDA(cudaGetDevice(&dev));
  LtSlot* lt;
  int rc = get_lt(dev, &lt);
  if (rc) return rc;
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr, ld = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  int status = LSRM_OK;
  cublasOperation_t tn = CUBLAS_OP_N;
  cublasLtEpilogue_t epi = bias ? CUBLASLT_EPILOGUE_BIAS : CUBLASLT_EPILOGUE_DEFAULT;
  size_t wsz = kLtWorkspace;
  cublasLtMatmulHeuristicResult_t heur = {};
  int n_res = 0;
  const float one = 1.f;
  bool ok = cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tn, sizeof(tn)) == 0;
  ok = ok && cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tn, sizeof(tn)) == 0;
  ok = ok && cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)) == 0;
  if (bias) {
    ok = ok && cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias,
                                              sizeof(bias)) == 0;
    ok = ok && cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bias_t,
                                              sizeof(bias_t)) == 0;
  }
  // column-major view: D (n x m) = B^T (n x k) . A^T (k x m)
  ok = ok && cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, n, k, ldb) == 0;
  ok = ok && cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, k, m, lda) == 0;
  ok = ok && cublasLtMatrixLayoutCreate(&lc, cd_t, n, m, c ? ldc : ldd) == 0;
  ok = ok && cublasLtMatrixLayoutCreate(&ld, cd_t, n, m, ldd) == 0;
  ok = ok && cublasLtMatmulPreferenceCreate(&pref) == 0;
  ok = ok && cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                                  &wsz, sizeof(wsz)) == 0;
  ok = ok && cublasLtMatmulAlgoGetHeuristic(lt->h, op, la, lb, lc, ld, pref, 1, &heur, &n_res) == 0 &&
       n_res > 0;
  ok = ok && cublasLtMatmul(lt->h, op, &one, b, la, a, lb, &beta, c ? c : d, lc, d, ld,
                            &heur.algo, lt->ws, kLtWorkspace,
                            as_stream(stream)) == CUBLAS_STATUS_SUCCESS;
  if (!ok) status = set_error(LSRM_E_CUDA, "cublasLt GEMM failed (m=%lld n=%lld k=%lld)",
                              (long long)m, (long long)n, (long long)k);
  if (pref) cublasLtMatmulPreferenceDestroy(pref);
  if (ld) cublasLtMatrixLayoutDestroy(ld);
  if (lc) cublasLtMatrixLayoutDestroy(lc);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (op) cublasLtMatmulDescDestroy(op);
  return status;
}

// C[m,n] = A[m,k] @ B[k,n] + bias[n], bf16 in / fp32 accumulate / bf16 out.
extern "C" int lsrm_gemm_bias_bf16(int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
                                   const void* b, int64_t ldb, const void* bias, void* c,
                                   int64_t ldc, void* stream) {
  return lt_gemm(m, n, k, a, lda, b, ldb, bias, CUDA_R_16BF, 0.f, nullptr, 0, c, ldc,
                 CUDA_R_16BF, stream);
}

// D[m,n] = A[m,k] @ B[k,n] + bias[n] + R[m,n], bf16 in, f32 bias / residual /
// out (the FFN's second GEMM with its bias and residual in the epilogue).
extern "C" int lsrm_gemm_bias_res_f32(int64_t m, int64_t n, int64_t k, const void* a,
                                      int64_t lda, const void* b, int64_t ldb, const float* bias,
                                      const float* res, int64_t ldr, float* d, int64_t ldd,
                                      void* stream) {
  return lt_gemm(m, n, k, a, lda, b, ldb, bias, CUDA_R_32F, res ? 1.f : 0.f, res, ldr, d, ldd,
                 CUDA_R_32F, stream);
}

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
