// Stage-2 sparse residual block around the four NSA uses
// (lsrm/recon_pipeline.py:461-497): injection + pre-norm, the two-gate
// mixture of the self/cross NSA outputs with the residual, and the FFN
// (affine-gelu-affine) with its residual.  The GEMMs are library GEMMs
// (lsrm_gemm); these kernels are the fused row-wise / element-wise steps.
//
// exact = 1 reproduces the reference's f32 storage with f64 arithmetic (the
// reference-API path, parity <= 1e-5); exact = 0 is the bf16 engine's fp32
// arithmetic.
#include "common.cuh"

namespace lsrm {

__device__ __forceinline__ double ld_any(const void* p, int bf16, int64_t i) {
  return bf16 ? (double)__bfloat162float(((const __nv_bfloat16*)p)[i])
              : (double)((const float*)p)[i];
}
__device__ __forceinline__ void st_any(void* p, int bf16, int64_t i, float v) {
  if (bf16)
    ((__nv_bfloat16*)p)[i] = __float2bfloat16_rn(v);
  else
    ((float*)p)[i] = v;
}
// sigmoid in f64, branch on sign as tensor_core.py:89-94
__device__ __forceinline__ double sigmoid64(double x) {
  return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
}

// Warp per row: LayerNorm of the f32 row r (already in `row`, length d) with
// f64 statistics (tensor_core.py:139-146) -> y.
__device__ __forceinline__ void ln_row(const float* row, int d, const float* gamma,
                                       const float* beta, float eps, int out_bf16, void* y,
                                       int64_t yoff, int lane) {
  double s = 0.0;
  for (int c = lane; c < d; c += 32) s += (double)row[c];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const double mu = s / d;
  double v = 0.0;
  for (int c = lane; c < d; c += 32) {
    const double t = (double)row[c] - mu;
    v += t * t;
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const double inv = 1.0 / sqrt(v / d + (double)eps);
  for (int c = lane; c < d; c += 32)
    st_any(y, out_bf16, yoff + c,
           (float)(((double)row[c] - mu) * inv * (double)gamma[c] + (double)beta[c]));
}

// sum = f32(a + b) (b optional), y = LayerNorm(sum)
__global__ void add_ln_kernel(const float* __restrict__ a, const void* __restrict__ b,
                              int b_bf16, int64_t n, int d, const float* __restrict__ gamma,
                              const float* __restrict__ beta, float eps,
                              float* __restrict__ sum_out, int out_bf16, void* y) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  float* row = sum_out + r * d;
  for (int c = lane; c < d; c += 32)
    row[c] = b ? (float)((double)a[r * d + c] + ld_any(b, b_bf16, r * d + c)) : a[r * d + c];
  __syncwarp();
  ln_row(row, d, gamma, beta, eps, out_bf16, y, r * d, lane);
}

// Two-gate mixture with the residual (recon_pipeline.py:474-490):
//   g_self, g_cross = f32(sigmoid(f32(logit + bias)))     (logits [n, 2d])
//   x1 = f32(xe + g_self * o_self + g_cross * o_cross)     (f64 sums)
// then h = LayerNorm(x1) for the FFN.
__global__ void gate_mix_ln_kernel(int exact, const float* __restrict__ xe,
                                   const void* __restrict__ gl, int64_t ld_gl, int gl_bf16,
                                   const float* __restrict__ gate_b,
                                   const void* __restrict__ o_self,
                                   const void* __restrict__ o_cross, int o_bf16, int64_t n,
                                   int d, float* __restrict__ x1,
                                   const float* __restrict__ gamma,
                                   const float* __restrict__ beta, float eps, int out_bf16,
                                   void* h) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  float* row = x1 + r * d;
  for (int c = lane; c < d; c += 32) {
    const double zs = (double)(float)(ld_any(gl, gl_bf16, r * ld_gl + c) + (double)gate_b[c]);
    const double zc =
        (double)(float)(ld_any(gl, gl_bf16, r * ld_gl + d + c) + (double)gate_b[d + c]);
    double gs, gc;
    if (exact) {
      gs = (double)(float)sigmoid64(zs);
      gc = (double)(float)sigmoid64(zc);
    } else {
      gs = (double)(1.f / (1.f + __expf(-(float)zs)));
      gc = (double)(1.f / (1.f + __expf(-(float)zc)));
    }
    const double o = gs * ld_any(o_self, o_bf16, r * d + c) + gc * ld_any(o_cross, o_bf16, r * d + c);
    row[c] = (float)((double)xe[r * d + c] + o);
  }
  __syncwarp();
  ln_row(row, d, gamma, beta, eps, out_bf16, h, r * d, lane);
}

// out = f32(act(f32(h + bias)) [+ residual])   act: 0 identity, 1 exact-erf gelu
__global__ void bias_act_kernel(int exact, const void* __restrict__ hin, int h_bf16, int64_t ld,
                                const float* __restrict__ bias, int64_t n, int cols, int act,
                                const float* __restrict__ residual, void* out, int out_bf16,
                                int64_t ld_out) {
  const int64_t total = n * (int64_t)cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e % cols);
    float v = (float)(ld_any(hin, h_bf16, r * ld + c) + (bias ? (double)bias[c] : 0.0));
    if (act == 1) {
      if (exact) {
        const double x = (double)v;
        v = (float)(0.5 * x * (1.0 + erf(x * 0.70710678118654752440)));
      } else {
        v = 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
      }
    }
    if (residual) v = (float)((double)residual[r * cols + c] + (double)v);
    st_any(out, out_bf16, r * ld_out + c, v);
  }
}

// Fast path of bias_act (exact = 0) for bf16 rows: 8 columns per thread,
// 16-byte loads/stores, fp32 arithmetic.
__global__ void bias_act_fast_kernel(const __nv_bfloat16* __restrict__ hin, int64_t ld,
                                     const float* __restrict__ bias, int64_t n, int cols, int act,
                                     const float* __restrict__ residual, void* out, int out_bf16,
                                     int64_t ld_out) {
  const int c8 = cols / 8;
  const int64_t total = n * (int64_t)c8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / c8;
    const int c = (int)(e % c8) * 8;
    const uint4 raw = *reinterpret_cast<const uint4*>(hin + r * ld + c);
    const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&raw);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float x = __bfloat162float(hv[j]) + (bias ? __ldg(bias + c + j) : 0.f);
      if (act == 1) x = 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
      if (residual) x += residual[r * cols + c + j];
      v[j] = x;
    }
    if (out_bf16) {
      uint4 w;
      uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        wp[j] = *reinterpret_cast<uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>((__nv_bfloat16*)out + r * ld_out + c) = w;
    } else {
      float* o = (float*)out + r * ld_out + c;
      *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(o + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

// ---- fast row kernels (exact = 0, the bf16 engine): warp per row, the row
// kept in registers (CH chunks of 8 columns per lane, d = 256*CH), 16-byte
// loads/stores, fp32 arithmetic and two-pass fp32 LayerNorm statistics.
__device__ __forceinline__ void ld8(const void* p, int bf16, int64_t i, float* v) {
  if (bf16) {
    const uint4 raw = *reinterpret_cast<const uint4*>((const __nv_bfloat16*)p + i);
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(h[j]);
  } else {
    const float4 a = *reinterpret_cast<const float4*>((const float*)p + i);
    const float4 b = *reinterpret_cast<const float4*>((const float*)p + i + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}
__device__ __forceinline__ void st8(void* p, int bf16, int64_t i, const float* v) {
  if (bf16) {
    uint4 w;
    uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      wp[j] = *reinterpret_cast<uint32_t*>(&h2);
    }
    *reinterpret_cast<uint4*>((__nv_bfloat16*)p + i) = w;
  } else {
    *reinterpret_cast<float4*>((float*)p + i) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>((float*)p + i + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
}

template <int CH>
__device__ __forceinline__ void ln_regs(float (&x)[CH][8], int d, const float* __restrict__ gamma,
                                        const float* __restrict__ beta, float eps, int out_bf16,
                                        void* y, int64_t yoff, int lane) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < CH; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[k][j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s / d;
  float v = 0.f;
#pragma unroll
  for (int k = 0; k < CH; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float t = x[k][j] - mu;
      v = fmaf(t, t, v);
    }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const float inv = rsqrtf(v / d + eps);
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = k * 256 + lane * 8;
    float g[8], b[8], o[8];
    ld8(gamma, 0, c, g);
    ld8(beta, 0, c, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = fmaf((x[k][j] - mu) * inv, g[j], b[j]);
    st8(y, out_bf16, yoff + c, o);
  }
}

template <int CH>
__global__ void add_ln_fast_kernel(const float* __restrict__ a, const void* __restrict__ b,
                                   int b_bf16, int64_t n, const float* __restrict__ gamma,
                                   const float* __restrict__ beta, float eps,
                                   float* __restrict__ sum_out, int out_bf16, void* y) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  constexpr int d = 256 * CH;
  float x[CH][8];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int64_t i = r * d + k * 256 + lane * 8;
    ld8(a, 0, i, x[k]);
    if (b) {
      float t[8];
      ld8(b, b_bf16, i, t);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[k][j] += t[j];
    }
    st8(sum_out, 0, i, x[k]);
  }
  ln_regs<CH>(x, d, gamma, beta, eps, out_bf16, y, r * d, lane);
}

template <int CH>
__global__ void gate_mix_ln_fast_kernel(const float* __restrict__ xe, const void* __restrict__ gl,
                                        int64_t ld_gl, int gl_bf16,
                                        const float* __restrict__ gate_b,
                                        const void* __restrict__ o_self,
                                        const void* __restrict__ o_cross, int o_bf16, int64_t n,
                                        float* __restrict__ x1, const float* __restrict__ gamma,
                                        const float* __restrict__ beta, float eps, int out_bf16,
                                        void* h) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  constexpr int d = 256 * CH;
  float x[CH][8];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = k * 256 + lane * 8;
    float zs[8], zc[8], bs[8], bc[8], os[8], oc[8];
    ld8(xe, 0, r * d + c, x[k]);
    ld8(gl, gl_bf16, r * ld_gl + c, zs);
    ld8(gl, gl_bf16, r * ld_gl + d + c, zc);
    ld8(gate_b, 0, c, bs);
    ld8(gate_b, 0, d + c, bc);
    ld8(o_self, o_bf16, r * d + c, os);
    ld8(o_cross, o_bf16, r * d + c, oc);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float gs = 1.f / (1.f + __expf(-(zs[j] + bs[j])));
      const float gc = 1.f / (1.f + __expf(-(zc[j] + bc[j])));
      x[k][j] += fmaf(gs, os[j], gc * oc[j]);
    }
    st8(x1, 0, r * d + c, x[k]);
  }
  ln_regs<CH>(x, d, gamma, beta, eps, out_bf16, h, r * d, lane);
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_add_layer_norm(int exact, const float* a, const void* b, int b_bf16, int64_t n, int d,
                        const float* gamma, const float* beta, float eps, float* sum_out,
                        int out_bf16, void* y, void* stream) {
  LSRM_REQUIRE(d > 0, "add_layer_norm: d must be positive");
  if (n == 0) return LSRM_OK;
  const bool al = ((uintptr_t)a % 16) == 0 && ((uintptr_t)b % 16) == 0 &&
                  ((uintptr_t)sum_out % 16) == 0 && ((uintptr_t)y % 16) == 0;
  if (!exact && d == 1024 && al) {
    add_ln_fast_kernel<4><<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(
        a, b, b_bf16, n, gamma, beta, eps, sum_out, out_bf16, y);
    LSRM_LAUNCHED();
    return LSRM_OK;
  }
  add_ln_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(
      a, b, b_bf16, n, d, gamma, beta, eps, sum_out, out_bf16, y);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_gate_mix_layer_norm(int exact, const float* xe, const void* gate_logits, int64_t ld_gl,
                             int gl_bf16, const float* gate_b, const void* o_self,
                             const void* o_cross, int o_bf16, int64_t n, int d, float* x1,
                             const float* gamma, const float* beta, float eps, int out_bf16,
                             void* h, void* stream) {
  LSRM_REQUIRE(d > 0 && ld_gl >= 2 * d, "gate_mix: logits need 2*d columns");
  if (n == 0) return LSRM_OK;
  const bool al = (ld_gl % 8) == 0 && ((uintptr_t)gate_logits % 16) == 0 &&
                  ((uintptr_t)o_self % 16) == 0 && ((uintptr_t)o_cross % 16) == 0;
  if (!exact && d == 1024 && al) {
    gate_mix_ln_fast_kernel<4><<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(
        xe, gate_logits, ld_gl, gl_bf16, gate_b, o_self, o_cross, o_bf16, n, x1, gamma, beta,
        eps, out_bf16, h);
    LSRM_LAUNCHED();
    return LSRM_OK;
  }
  gate_mix_ln_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(
      exact, xe, gate_logits, ld_gl, gl_bf16, gate_b, o_self, o_cross, o_bf16, n, d, x1, gamma,
      beta, eps, out_bf16, h);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_bias_act(int exact, const void* h, int h_bf16, int64_t ld, const float* bias, int64_t n,
                  int cols, int act, const float* residual, void* out, int out_bf16,
                  int64_t ld_out, void* stream) {
  LSRM_REQUIRE(act == 0 || act == 1, "bias_act: act must be 0 (identity) or 1 (gelu)");
  if (n == 0 || cols == 0) return LSRM_OK;
  int64_t total = n * (int64_t)cols;
  const bool fast = !exact && h_bf16 && cols % 8 == 0 && ld % 8 == 0 && ld_out % 8 == 0 &&
                    ((uintptr_t)h % 16) == 0 && ((uintptr_t)out % 16) == 0;
  if (fast) {
    const int64_t t8 = total / 8;
    unsigned grid = (unsigned)(ceil_div(t8, 256) < 148 * 32 ? ceil_div(t8, 256) : 148 * 32);
    bias_act_fast_kernel<<<grid, 256, 0, as_stream(stream)>>>(
        (const __nv_bfloat16*)h, ld, bias, n, cols, act, residual, out, out_bf16, ld_out);
    LSRM_LAUNCHED();
    return LSRM_OK;
  }
  unsigned grid = (unsigned)(ceil_div(total, 256) < 148 * 16 ? ceil_div(total, 256) : 148 * 16);
  bias_act_kernel<<<grid, 256, 0, as_stream(stream)>>>(exact, h, h_bf16, ld, bias, n, cols, act,
                                                       residual, out, out_bf16, ld_out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
