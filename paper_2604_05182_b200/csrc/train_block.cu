// Backward of the Stage-2 block around the NSA uses (
// the reference block is lsrm/recon_pipeline.py:461-497, inference only):
//
//   xe  = x + x_inj;  x_hat = LN_a(xe)                          (add + LayerNorm)
//   g   = sigmoid(x_hat W_g + b_g) = [g_self | g_cross]          (use gates)
//   x1  = xe + g_self * O_self + g_cross * O_cross               (gated mixture)
//   h   = LN_f(x1);  x2 = x1 + gelu(h W1 + b1) W2 + b2           (FFN)
//
// Kernels (fp32, deterministic: fixed reduction orders, no float atomics):
//   layer_norm_bwd   dx (+)= rstd (g - mean(g) - x_hat mean(g x_hat)), g = dy gamma;
//                    per-CTA partial column sums of dy x_hat (dgamma) and dy
//                    (dbeta), warp partials combined in warp order
//   gate_mix_bwd     d O_self / d O_cross / d logits of the gated mixture
//   gelu_bwd         dt = du (Phi(t) + t phi(t)) (exact erf gelu)
//   colsum           column sums of a row block (bias gradients): per-CTA
//                    partials over fixed row ranges, then the partials in CTA
//                    order
#include "common.cuh"

namespace lsrm {
namespace tb {

constexpr int kRowsPerCta = 64;     // row range of one CTA's partial column sums
constexpr int kWarps = 8;

// dx (+)= rstd (g - mean(g) - x_hat mean(g x_hat)), g = dy gamma: one warp
// per row, float4 columns (lane owns columns 4 lane + 128 j), the row's mean
// and rstd written for the column sums below.  V4 = d / 128 float4 per lane.
template <int V4>
__global__ void __launch_bounds__(256) layer_norm_bwd_rows_kernel(
    const float* __restrict__ x, int64_t ld_x, int64_t n, int d,
    const float* __restrict__ gamma, float eps, const float* __restrict__ dy, int64_t ld_dy,
    float* __restrict__ dx, int64_t ld_dx, int accumulate, float2* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n) return;
  float4 xv[V4], gv[V4];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    xv[j] = __ldg(reinterpret_cast<const float4*>(x + r * ld_x) + lane + 32 * j);
    s += (xv[j].x + xv[j].y) + (xv[j].z + xv[j].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / (float)d;
  float v = 0.f;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const float a = xv[j].x - mean, b = xv[j].y - mean, c = xv[j].z - mean, e = xv[j].w - mean;
    v += (a * a + b * b) + (c * c + e * e);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const float rstd = rsqrtf(v / (float)d + eps);
  float sg = 0.f, sgx = 0.f;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const float4 g = __ldg(reinterpret_cast<const float4*>(dy + r * ld_dy) + lane + 32 * j);
    const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma) + lane + 32 * j);
    xv[j] = make_float4((xv[j].x - mean) * rstd, (xv[j].y - mean) * rstd,
                        (xv[j].z - mean) * rstd, (xv[j].w - mean) * rstd);
    gv[j] = make_float4(g.x * gm.x, g.y * gm.y, g.z * gm.z, g.w * gm.w);
    sg += (gv[j].x + gv[j].y) + (gv[j].z + gv[j].w);
    sgx += (gv[j].x * xv[j].x + gv[j].y * xv[j].y) + (gv[j].z * xv[j].z + gv[j].w * xv[j].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sg += __shfl_xor_sync(0xffffffffu, sg, o);
    sgx += __shfl_xor_sync(0xffffffffu, sgx, o);
  }
  const float mg = sg / (float)d, mgx = sgx / (float)d;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    float4* o = reinterpret_cast<float4*>(dx + r * ld_dx) + lane + 32 * j;
    float4 g = make_float4(rstd * (gv[j].x - mg - xv[j].x * mgx),
                           rstd * (gv[j].y - mg - xv[j].y * mgx),
                           rstd * (gv[j].z - mg - xv[j].z * mgx),
                           rstd * (gv[j].w - mg - xv[j].w * mgx));
    if (accumulate) {
      const float4 p = *o;
      g = make_float4(p.x + g.x, p.y + g.y, p.z + g.z, p.w + g.w);
    }
    *o = g;
  }
  if (lane == 0) stats[r] = make_float2(mean, rstd);
}

// per-CTA partial column sums of dy x_hat (dgamma) and dy (dbeta) over rows
// [kRowsPerCta * blockIdx.x, +kRowsPerCta), rows in order
__global__ void layer_norm_bwd_cols_kernel(const float* __restrict__ x, int64_t ld_x, int64_t n,
                                           int d, const float* __restrict__ dy, int64_t ld_dy,
                                           const float2* __restrict__ stats,
                                           float* __restrict__ dgamma_part,
                                           float* __restrict__ dbeta_part) {
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta;
  const int64_t r1 = r0 + kRowsPerCta < n ? r0 + kRowsPerCta : n;
  float a = 0.f, b = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    const float2 st = stats[r];
    const float g = dy[r * ld_dy + c];
    a += g * ((x[r * ld_x + c] - st.x) * st.y);
    b += g;
  }
  dgamma_part[(int64_t)blockIdx.x * d + c] = a;
  dbeta_part[(int64_t)blockIdx.x * d + c] = b;
}

// (the previous single-kernel form: one warp per row with per-lane column
// partials held in registers; kept for d not a multiple of 128)
// one warp per row (rows r0 + warp, r0 + warp + 8, ... < r0 + kRowsPerCta);
// lane owns columns lane, lane + 32, ... (D / 32 of them, D <= 4096)
template <int PER>
__global__ void __launch_bounds__(kWarps * 32) layer_norm_bwd_kernel(
    const float* __restrict__ x, int64_t ld_x, int64_t n, int d, const float* __restrict__ gamma,
    float eps, const float* __restrict__ dy, int64_t ld_dy, float* __restrict__ dx,
    int64_t ld_dx, int accumulate, float* __restrict__ dgamma_part,
    float* __restrict__ dbeta_part) {
  extern __shared__ float tb_smem[];   // [kWarps][2][d]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta;
  float pg[PER], pb[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) pg[j] = pb[j] = 0.f;
  for (int64_t r = r0 + warp; r < r0 + kRowsPerCta && r < n; r += kWarps) {
    float xv[PER], gv[PER];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int c = lane + 32 * j;
      xv[j] = c < d ? x[r * ld_x + c] : 0.f;
      s += xv[j];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s / (float)d;
    float v = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int c = lane + 32 * j;
      const float t = c < d ? xv[j] - mean : 0.f;
      v += t * t;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const float rstd = rsqrtf(v / (float)d + eps);
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int c = lane + 32 * j;
      if (c < d) {
        const float xh = (xv[j] - mean) * rstd, g = dy[r * ld_dy + c];
        pg[j] += g * xh;
        pb[j] += g;
        gv[j] = g * gamma[c];
        sg += gv[j];
        sgx += gv[j] * xh;
        xv[j] = xh;
      } else {
        gv[j] = 0.f;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sg += __shfl_xor_sync(0xffffffffu, sg, o);
      sgx += __shfl_xor_sync(0xffffffffu, sgx, o);
    }
    const float mg = sg / (float)d, mgx = sgx / (float)d;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int c = lane + 32 * j;
      if (c < d) {
        const float g = rstd * (gv[j] - mg - xv[j] * mgx);
        float* o = dx + r * ld_dx + c;
        *o = accumulate ? *o + g : g;
      }
    }
  }
  // CTA partials: warps in order
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int c = lane + 32 * j;
    if (c < d) {
      tb_smem[(warp * 2) * d + c] = pg[j];
      tb_smem[(warp * 2 + 1) * d + c] = pb[j];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < kWarps; ++w) {
      a += tb_smem[(w * 2) * d + c];
      b += tb_smem[(w * 2 + 1) * d + c];
    }
    dgamma_part[(int64_t)blockIdx.x * d + c] = a;
    dbeta_part[(int64_t)blockIdx.x * d + c] = b;
  }
}

// partial rows [n_part][d] -> out[d]: CTA = 32 columns x 32 warps; warp w
// sums parts w, w + 32, ... (two accumulators, in order), then warp 0 adds
// the 32 warp sums in warp order (a fixed order: deterministic)
__global__ void __launch_bounds__(1024) sum_parts_kernel(const float* __restrict__ part,
                                                         int64_t n_part, int d,
                                                         float* __restrict__ out) {
  __shared__ float red[32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + lane;
  float a0 = 0.f, a1 = 0.f;
  if (c < d) {
    int64_t p = warp;
    for (; p + 32 < n_part; p += 64) {
      a0 += part[p * d + c];
      a1 += part[(p + 32) * d + c];
    }
    if (p < n_part) a0 += part[p * d + c];
  }
  red[warp][lane] = a0 + a1;
  __syncthreads();
  if (warp == 0 && c < d) {
    float t = 0.f;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    out[c] = t;
  }
}

// column partial sums of rows [kRowsPerCta * blockIdx.x, +kRowsPerCta)
__global__ void colsum_part_kernel(const float* __restrict__ x, int64_t ld, int64_t n, int d,
                                   float* __restrict__ part) {
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta;
  const int64_t r1 = r0 + kRowsPerCta < n ? r0 + kRowsPerCta : n;
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += x[r * ld + c];
  part[(int64_t)blockIdx.x * d + c] = s;
}

__device__ __forceinline__ float sigm(float z) { return 1.f / (1.f + __expf(-z)); }

// x1 = xe + s(l_s) o_s + s(l_c) o_c  (l = logits + bias):
//   do_s = dx1 s(l_s); dl_s = dx1 o_s s(l_s)(1 - s(l_s)); likewise cross
__global__ void gate_mix_bwd_kernel(const float* __restrict__ logits, int64_t ld_l,
                                    const float* __restrict__ bias, const float* __restrict__ o_s,
                                    const float* __restrict__ o_c, const float* __restrict__ dx1,
                                    int64_t n, int d, float* __restrict__ do_s,
                                    float* __restrict__ do_c, float* __restrict__ dl) {
  const int64_t total = n * (int64_t)d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d;
    const int c = (int)(i % d);
    const float gs = sigm(logits[r * ld_l + c] + bias[c]);
    const float gc = sigm(logits[r * ld_l + d + c] + bias[d + c]);
    const float g = dx1[i];
    do_s[i] = g * gs;
    do_c[i] = g * gc;
    dl[r * 2 * d + c] = g * o_s[i] * gs * (1.f - gs);
    dl[r * 2 * d + d + c] = g * o_c[i] * gc * (1.f - gc);
  }
}

// dt = du * gelu'(z + b), gelu(t) = t Phi(t)
__global__ void gelu_bwd_kernel(const float* __restrict__ z, const float* __restrict__ bias,
                                const float* __restrict__ du, int64_t n, int d,
                                float* __restrict__ dt) {
  const int64_t total = n * (int64_t)d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float t = z[i] + bias[i % d];
    const float cdf = 0.5f * (1.f + erff(t * 0.70710678118654752f));
    const float pdf = 0.3989422804014327f * __expf(-0.5f * t * t);
    dt[i] = du[i] * (cdf + t * pdf);
  }
}

// dst[c][r] = bf16(src[r][c]) for r < rows, 0 for rows <= r < rows_pad:
// 32 x 32 tiles through shared memory (coalesced both ways)
__global__ void transpose_cast_kernel(const float* __restrict__ src, int64_t ld, int64_t rows,
                                      int64_t cols, __nv_bfloat16* __restrict__ dst,
                                      int64_t rows_pad) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? src[r * ld + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows_pad) dst[c * rows_pad + r] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

// out = (accumulate ? out : 0) + parts[0] + ... + parts[n_slices - 1]
// (split-K partial products, summed in slice order), float4 per thread
__global__ void sum_slices_kernel(const float4* __restrict__ parts, int n_slices, int64_t n4,
                                  float4* __restrict__ out, int accumulate) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = accumulate ? out[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < n_slices; ++s) {
      const float4 p = __ldcs(parts + (int64_t)s * n4 + i);
      a.x += p.x; a.y += p.y; a.z += p.z; a.w += p.w;
    }
    out[i] = a;
  }
}

}  // namespace tb
}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_sum_slices_f32(const float* parts, int n_slices, int64_t n, float* out, int accumulate,
                        void* stream) {
  LSRM_REQUIRE(n_slices >= 1 && n % 4 == 0 && ((uintptr_t)parts % 16) == 0 &&
                   ((uintptr_t)out % 16) == 0,
               "sum_slices: n %% 4 == 0 and 16-byte aligned buffers required");
  if (n == 0) return LSRM_OK;
  const int64_t n4 = n / 4;
  tb::sum_slices_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n4, 256), 148 * 8), 256, 0,
                          as_stream(stream)>>>(reinterpret_cast<const float4*>(parts), n_slices,
                                               n4, reinterpret_cast<float4*>(out), accumulate);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int64_t lsrm_colsum_parts(int64_t n) { return (n + tb::kRowsPerCta - 1) / tb::kRowsPerCta; }

int lsrm_layer_norm_bwd_f32(const float* x, int64_t ld_x, int64_t n, int d, const float* gamma,
                            float eps, const float* dy, int64_t ld_dy, float* dx, int64_t ld_dx,
                            int accumulate, float* part, float* dgamma, float* dbeta,
                            void* stream) {
  LSRM_REQUIRE(d >= 1 && d <= 4096, "layer_norm_bwd: d must be in 1..4096, got %d", d);
  if (n == 0) {
    LSRM_CUDA(cudaMemsetAsync(dgamma, 0, d * sizeof(float), as_stream(stream)));
    LSRM_CUDA(cudaMemsetAsync(dbeta, 0, d * sizeof(float), as_stream(stream)));
    return LSRM_OK;
  }
  const int64_t n_part = lsrm_colsum_parts(n);
  cudaStream_t st = as_stream(stream);
  const size_t smem = (size_t)tb::kWarps * 2 * d * sizeof(float);
  float* pg = part;
  float* pb = part + n_part * d;
  const bool vec = d % 128 == 0 && d <= 1024 && ((uintptr_t)x % 16) == 0 &&
                   ((uintptr_t)dy % 16) == 0 && ((uintptr_t)dx % 16) == 0 &&
                   ((uintptr_t)gamma % 16) == 0 && ld_x % 4 == 0 && ld_dy % 4 == 0 &&
                   ld_dx % 4 == 0;
  if (vec) {
    // row pass (dx, per-row mean / rstd) then fixed-order column partials; the
    // row stats live in the workspace after the partials (2 n floats)
    float2* stats = reinterpret_cast<float2*>(part + 2 * n_part * d);
#define LSRM_LNR(V)                                                                         \
  if (d == 128 * V) {                                                                       \
    tb::layer_norm_bwd_rows_kernel<V><<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(            \
        x, ld_x, n, d, gamma, eps, dy, ld_dy, dx, ld_dx, accumulate, stats);                \
  } else
    LSRM_LNR(1) LSRM_LNR(2) LSRM_LNR(4) LSRM_LNR(8) {}
#undef LSRM_LNR
    LSRM_LAUNCHED();
    tb::layer_norm_bwd_cols_kernel<<<dim3((unsigned)n_part, (unsigned)ceil_div(d, 256)), 256, 0,
                                     st>>>(x, ld_x, n, d, dy, ld_dy, stats, pg, pb);
    LSRM_LAUNCHED();
  } else {
#define LSRM_LNB(PER)                                                                       \
  if ((d + 31) / 32 <= PER) {                                                               \
    LSRM_CUDA(cudaFuncSetAttribute(tb::layer_norm_bwd_kernel<PER>,                          \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    tb::layer_norm_bwd_kernel<PER><<<(unsigned)n_part, tb::kWarps * 32, smem, st>>>(        \
        x, ld_x, n, d, gamma, eps, dy, ld_dy, dx, ld_dx, accumulate, pg, pb);               \
  } else
  LSRM_LNB(2) LSRM_LNB(8) LSRM_LNB(32) LSRM_LNB(128) {
    return set_error(LSRM_E_CONFIG, "layer_norm_bwd: d too large");
  }
#undef LSRM_LNB
  LSRM_LAUNCHED();
  }
  tb::sum_parts_kernel<<<(unsigned)ceil_div(d, 32), 1024, 0, st>>>(pg, n_part, d, dgamma);
  LSRM_LAUNCHED();
  tb::sum_parts_kernel<<<(unsigned)ceil_div(d, 32), 1024, 0, st>>>(pb, n_part, d, dbeta);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_colsum_f32(const float* x, int64_t ld, int64_t n, int d, float* part, float* out,
                    void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    LSRM_CUDA(cudaMemsetAsync(out, 0, d * sizeof(float), st));
    return LSRM_OK;
  }
  const int64_t n_part = lsrm_colsum_parts(n);
  tb::colsum_part_kernel<<<dim3((unsigned)n_part, (unsigned)ceil_div(d, 256)), 256, 0, st>>>(
      x, ld, n, d, part);
  LSRM_LAUNCHED();
  tb::sum_parts_kernel<<<(unsigned)ceil_div(d, 32), 1024, 0, st>>>(part, n_part, d, out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_gate_mix_bwd_f32(const float* logits, int64_t ld_l, const float* bias, const float* o_s,
                          const float* o_c, const float* dx1, int64_t n, int d, float* do_s,
                          float* do_c, float* dlogits, void* stream) {
  if (n == 0) return LSRM_OK;
  const int64_t total = n * (int64_t)d;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  tb::gate_mix_bwd_kernel<<<grid, 256, 0, as_stream(stream)>>>(logits, ld_l, bias, o_s, o_c, dx1,
                                                               n, d, do_s, do_c, dlogits);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_transpose_cast_bf16(const float* src, int64_t ld, int64_t rows, int64_t cols,
                             void* dst, int64_t rows_pad, void* stream) {
  LSRM_REQUIRE(rows_pad >= rows && ld >= cols, "transpose_cast: bad shape");
  if (cols == 0 || rows_pad == 0) return LSRM_OK;
  const dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows_pad, 32));
  tb::transpose_cast_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(
      src, ld, rows, cols, (__nv_bfloat16*)dst, rows_pad);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_gelu_bwd_f32(const float* z, const float* bias, const float* du, int64_t n, int d,
                      float* dt, void* stream) {
  if (n == 0) return LSRM_OK;
  const int64_t total = n * (int64_t)d;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  tb::gelu_bwd_kernel<<<grid, 256, 0, as_stream(stream)>>>(z, bias, du, n, d, dt);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
