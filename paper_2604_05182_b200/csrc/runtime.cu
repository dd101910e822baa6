// Runtime plumbing of the C ABI: per-thread error buffer, launch counter,
// generic row permutation / cast / LayerNorm kernels.
#include "common.cuh"

#include <math.h>

namespace lsrm {

static thread_local char g_err[1024] = "";
static thread_local int64_t g_launches = 0;

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

void count_launch() { ++g_launches; }

// ---------------------------------------------------------------------------
// row gather/scatter: dst[i] = src[index[i]]  /  dst[index[i]] = src[i]
// 16-byte vectorised when rows are 16B aligned.

template <typename V, bool kScatter>
__global__ void permute_rows_kernel(const V* __restrict__ src, int64_t ld_src,
                                    const int64_t* __restrict__ index, int64_t n,
                                    int64_t row_vecs, V* __restrict__ dst,
                                    int64_t ld_dst) {
  int64_t total = n * row_vecs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / row_vecs, c = t - i * row_vecs;
    int64_t j = index[i];
    if (kScatter)
      dst[j * ld_dst + c] = src[i * ld_src + c];
    else
      dst[i * ld_dst + c] = src[j * ld_src + c];
  }
}

template <bool kScatter>
static int permute_rows(int elem_bytes, const void* src, int64_t ld_src,
                        const int64_t* index, int64_t n, int64_t row_elems,
                        void* dst, int64_t ld_dst, void* stream) {
  if (n == 0 || row_elems == 0) return LSRM_OK;
  int64_t row_b = row_elems * elem_bytes, lds_b = ld_src * elem_bytes,
          ldd_b = ld_dst * elem_bytes;
  int blocks = (int)std::min<int64_t>(ceil_div(n * std::max<int64_t>(row_b / 16, 1), 256), 148 * 16);
  auto aligned = [&](int64_t a) {
    return (a % 16) == 0;
  };
  if (aligned(row_b) && aligned(lds_b) && aligned(ldd_b) &&
      ((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0) {
    permute_rows_kernel<int4, kScatter><<<blocks, 256, 0, as_stream(stream)>>>(
        (const int4*)src, lds_b / 16, index, n, row_b / 16, (int4*)dst, ldd_b / 16);
  } else if ((row_b % 4) == 0 && (lds_b % 4) == 0 && (ldd_b % 4) == 0) {
    permute_rows_kernel<int, kScatter><<<blocks, 256, 0, as_stream(stream)>>>(
        (const int*)src, lds_b / 4, index, n, row_b / 4, (int*)dst, ldd_b / 4);
  } else {
    permute_rows_kernel<uint16_t, kScatter><<<blocks, 256, 0, as_stream(stream)>>>(
        (const uint16_t*)src, lds_b / 2, index, n, row_b / 2, (uint16_t*)dst, ldd_b / 2);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}

__global__ void cast_kernel(int to_bf16, const void* src, void* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (to_bf16)
      ((__nv_bfloat16*)dst)[i] = __float2bfloat16_rn(((const float*)src)[i]);
    else
      ((float*)dst)[i] = __bfloat162float(((const __nv_bfloat16*)src)[i]);
  }
}

// 8 elements per thread and step: 32-byte f32 side, 16-byte bf16 side
// (both pointers 16-byte aligned, n % 8 == 0)
__global__ void cast8_kernel(int to_bf16, const void* __restrict__ src, void* __restrict__ dst,
                             int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (to_bf16) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(src) + 2 * i);
      const float4 b = __ldcs(reinterpret_cast<const float4*>(src) + 2 * i + 1);
      __nv_bfloat162 h[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                             __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
      reinterpret_cast<uint4*>(dst)[i] = *reinterpret_cast<const uint4*>(h);
    } else {
      const uint4 w = __ldcs(reinterpret_cast<const uint4*>(src) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
      float4* o = reinterpret_cast<float4*>(dst) + 2 * i;
      o[0] = make_float4(__low2float(h[0]), __high2float(h[0]), __low2float(h[1]),
                         __high2float(h[1]));
      o[1] = make_float4(__low2float(h[2]), __high2float(h[2]), __low2float(h[3]),
                         __high2float(h[3]));
    }
  }
}

// LayerNorm, one warp per row, f64 statistics (tensor_core.py:139-146).
__global__ void layer_norm_kernel(int in_bf16, const void* x, int64_t n, int d,
                                  const float* __restrict__ gamma,
                                  const float* __restrict__ beta, float eps,
                                  int out_bf16, void* y) {
  int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (row >= n) return;
  auto ld = [&](int c) -> double {
    return in_bf16 ? (double)__bfloat162float(((const __nv_bfloat16*)x)[row * d + c])
                   : (double)((const float*)x)[row * d + c];
  };
  double s = 0.0;
  for (int c = lane; c < d; c += 32) s += ld(c);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  double mu = s / d;
  double v = 0.0;
  for (int c = lane; c < d; c += 32) {
    double t = ld(c) - mu;
    v += t * t;
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  double inv = 1.0 / sqrt(v / d + (double)eps);
  for (int c = lane; c < d; c += 32) {
    float r = (float)((ld(c) - mu) * inv * (double)gamma[c] + (double)beta[c]);
    if (out_bf16)
      ((__nv_bfloat16*)y)[row * d + c] = __float2bfloat16_rn(r);
    else
      ((float*)y)[row * d + c] = r;
  }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_abi_version(void) { return 1; }
const char* lsrm_last_error(void) { return g_err; }
int64_t lsrm_launch_count(void) { return g_launches; }
void lsrm_reset_launch_count(void) { g_launches = 0; }

int lsrm_gather_rows(int elem_bytes, const void* src, int64_t ld_src,
                     const int64_t* index, int64_t n, int64_t row_elems,
                     void* dst, int64_t ld_dst, void* stream) {
  LSRM_REQUIRE(elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
               "gather_rows: elem_bytes must be 2, 4 or 8");
  return permute_rows<false>(elem_bytes, src, ld_src, index, n, row_elems, dst,
                             ld_dst, stream);
}

int lsrm_scatter_rows(int elem_bytes, const void* src, int64_t ld_src,
                      const int64_t* index, int64_t n, int64_t row_elems,
                      void* dst, int64_t ld_dst, void* stream) {
  LSRM_REQUIRE(elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
               "scatter_rows: elem_bytes must be 2, 4 or 8");
  return permute_rows<true>(elem_bytes, src, ld_src, index, n, row_elems, dst,
                            ld_dst, stream);
}

int lsrm_cast(int to_bf16, const void* src, void* dst, int64_t n, void* stream) {
  if (n == 0) return LSRM_OK;
  if (n % 8 == 0 && ((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0) {
    const int blocks = (int)std::min<int64_t>(ceil_div(n / 8, 256), 148 * 8);
    cast8_kernel<<<blocks, 256, 0, as_stream(stream)>>>(to_bf16, src, dst, n / 8);
    LSRM_LAUNCHED();
    return LSRM_OK;
  }
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 16);
  cast_kernel<<<blocks, 256, 0, as_stream(stream)>>>(to_bf16, src, dst, n);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_layer_norm(int in_bf16, const void* x, int64_t n, int d,
                    const float* gamma, const float* beta, float eps,
                    int out_bf16, void* y, void* stream) {
  if (n == 0) return LSRM_OK;
  LSRM_REQUIRE(d > 0, "layer_norm: d must be positive");
  int64_t blocks = ceil_div(n, 8);
  layer_norm_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      in_bf16, x, n, d, gamma, beta, eps, out_bf16, y);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Segment copy: dst[d_off : d_off + n] = src[s_off : s_off + n] for a list of
// byte segments (16-byte aligned).  Used to place all-gathered per-rank KV
// shards into the canonical block-major layout (W-invariant attention input).
namespace lsrm {
__global__ void copy_segments_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                     const int64_t* __restrict__ segs, int64_t n_segs) {
  for (int64_t sg = blockIdx.x; sg < n_segs; sg += gridDim.x) {
    const int64_t so = segs[3 * sg], dof = segs[3 * sg + 1], nb = segs[3 * sg + 2];
    const int4* s4 = reinterpret_cast<const int4*>(src + so);
    int4* d4 = reinterpret_cast<int4*>(dst + dof);
    for (int64_t i = threadIdx.x; i < nb / 16; i += blockDim.x) d4[i] = s4[i];
  }
}
}  // namespace lsrm

extern "C" int lsrm_copy_segments(const void* src, void* dst, const int64_t* segs,
                                  int64_t n_segs, void* stream) {
  using namespace lsrm;
  if (n_segs == 0) return LSRM_OK;
  LSRM_REQUIRE(((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0,
               "copy_segments: buffers must be 16-byte aligned");
  int blocks = (int)std::min<int64_t>(n_segs, 148 * 8);
  copy_segments_kernel<<<blocks, 128, 0, as_stream(stream)>>>((const uint8_t*)src, (uint8_t*)dst,
                                                              segs, n_segs);
  LSRM_LAUNCHED();
  return LSRM_OK;
}
