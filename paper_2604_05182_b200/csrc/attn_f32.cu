// fp32 NSA attention branches on CUDA cores (lsrm/nsa_attention.py:84-207)
// and the fp32 gated merge (nsa_attention.py:266-284).
//
// This is the exact-precision path (BASELINE config C1 "fp32 fwd", and the
// reference API's f32 contract): S lanes per (query, q-head) (S a power of
// two chosen so the launch fills the GPU), lane j walking every S-th key of
// the query's key sequence in block order with an fp32 online softmax
// (accurate expf) and FFMA dot products; the lanes' (max, sum, acc) states
// are merged by a fixed xor-shuffle tree (deterministic).  Keys/values are in
// the KV partition's block-major order so each selected block is one
// contiguous row range.
#include "common.cuh"

namespace lsrm {

// LSRM_F32_FASTEXP: __expf (ex2.approx based) instead of the accurate expf
#ifdef LSRM_F32_FASTEXP
#define F32_EXP(x) __expf(x)
#else
#define F32_EXP(x) expf(x)
#endif

// keys lo, lo+S, ... of [lo, hi) after the first `skip` (this lane's share)
template <int DH>
__device__ __forceinline__ void attend_range(const float* __restrict__ k,
                                             const float* __restrict__ v, int hkv,
                                             int kvh, int64_t lo, int64_t hi,
                                             const float (&q)[DH], float scale, float& m,
                                             float& l, float (&acc)[DH], int step = 1) {
  for (int64_t j = lo; j < hi; j += step) {
    const float* kr = k + (j * hkv + kvh) * DH;
    const float* vr = v + (j * hkv + kvh) * DH;
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < DH; ++c) s = fmaf(q[c], kr[c], s);
    s *= scale;
    if (s > m) {
      float corr = F32_EXP(m - s);  // m = -inf -> 0
      l *= corr;
#pragma unroll
      for (int c = 0; c < DH; ++c) acc[c] *= corr;
      m = s;
    }
    float p = F32_EXP(s - m);
    l += p;
#pragma unroll
    for (int c = 0; c < DH; ++c) acc[c] = fmaf(p, vr[c], acc[c]);
  }
}

template <int DH>
__global__ void attention_f32_kernel(int mode, const float* __restrict__ q, int64_t nq,
                                     int hq, int hkv, const float* __restrict__ k,
                                     const float* __restrict__ v, int64_t nk,
                                     const int64_t* __restrict__ offs,
                                     const int32_t* __restrict__ rows,
                                     const int32_t* __restrict__ count, int kmax,
                                     const int32_t* __restrict__ own_row,
                                     const int64_t* __restrict__ ids,
                                     const int64_t* __restrict__ lengths, int64_t width,
                                     float* __restrict__ out, int split) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t t = gt / split;            // (query, head) of this lane group
  const int sl = (int)(gt % split);        // lane within the group (groups are aligned)
  const bool valid = t < nq * hq;
  const int64_t tt = valid ? t : 0;
  const int64_t i = tt / hq;
  const int h = (int)(tt % hq);
  const int kvh = h / (hq / hkv);
  float qr[DH], acc[DH];
#pragma unroll
  for (int c = 0; c < DH; ++c) { qr[c] = q[tt * DH + c]; acc[c] = 0.f; }
  const float scale = 1.0f / sqrtf((float)DH);
  float m = -__builtin_huge_valf(), l = 0.f;
  // this lane takes the keys whose position in the query's key sequence is
  // = sl (mod split); `seen` counts the keys of the ranges walked so far
  int64_t seen = 0;
  auto range = [&](int64_t lo, int64_t hi) {
    const int64_t first = lo + ((sl - seen) % split + split) % split;
    attend_range<DH>(k, v, hkv, kvh, first, hi, qr, scale, m, l, acc, split);
    seen += hi - lo;
  };
  if (valid) {
    if (mode == 0) {
      range(0, nk);
    } else if (mode == 1) {
      const int c = count[i];
      for (int s = 0; s < c; ++s) {
        const int r = rows[i * kmax + s];
        range(offs[r], offs[r + 1]);
      }
    } else if (mode == 2) {
      const int r = own_row[i];
      range(offs[r], offs[r + 1]);
    } else {
      const int64_t len = lengths[i];
      for (int64_t s = 0; s < len; ++s) {
        const int64_t j = ids[i * width + s];
        range(j, j + 1);
      }
    }
  }
  // merge the group's lane states (fixed xor tree: deterministic)
  for (int o = 1; o < split; o <<= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, o);
    const float lo_ = __shfl_xor_sync(0xffffffffu, l, o);
    const float mn = fmaxf(m, mo);
    const float a = m == mn ? 1.f : expf(m - mn), b = mo == mn ? 1.f : expf(mo - mn);
    l = l * a + lo_ * b;
#pragma unroll
    for (int c = 0; c < DH; ++c) {
      const float ao = __shfl_xor_sync(0xffffffffu, acc[c], o);
      acc[c] = acc[c] * a + ao * b;
    }
    m = mn;
  }
  if (!valid) return;
  const float inv = 1.0f / l;
  // lane sl writes columns sl, sl + split, ... of the row
#pragma unroll
  for (int c = 0; c < DH; ++c)
    if (c % split == sl) out[tt * DH + c] = acc[c] * inv;
}

__global__ void gated_merge_f32_kernel(const float* __restrict__ gl, int64_t ld,
                                       const float* __restrict__ gb, int ng,
                                       const float* __restrict__ o0,
                                       const float* __restrict__ o1,
                                       const float* __restrict__ o2, int64_t n, int d,
                                       float* __restrict__ merged) {
  int64_t total = n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / d;
    int c = (int)(e % d);
    const float* ob[3] = {o0, o1, o2};
    double acc = 0.0;
    for (int b = 0; b < ng; ++b) {
      // gate = f32(sigmoid_f64(f32(logit + bias)))   (tensor_core.py:89-94)
      float z = gl[i * ld + b * d + c] + (gb ? gb[b * d + c] : 0.f);
      double x = (double)z;
      double g = x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
      acc += (double)(float)g * (double)ob[b][e];
    }
    merged[e] = (float)acc;
  }
}

__device__ __forceinline__ float sigmoid_ref(float z) {
  double x = (double)z;
  return (float)(x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x)));
}

__global__ void sigmoid_f32_kernel(const float* __restrict__ gl, int64_t ld,
                                   const float* __restrict__ gb, int64_t n, int cols,
                                   float* __restrict__ out) {
  int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols;
    int c = (int)(e % cols);
    out[e] = sigmoid_ref(gl[i * ld + c] + (gb ? gb[c] : 0.f));
  }
}

// The reference's score is np.einsum("xhd,yhd->xy", q64, k64) over C-contiguous
// operands (nsa_attention.py:226-227).  NumPy's einsum coalesces (h, d) into
// one contiguous inner loop of n = h_q*d_h products and reduces it with its
// baseline-SIMD sum-of-products kernel (x86-64 baseline SSE2: 2 f64 lanes, no
// FMA): per group of 8 elements each lane l adds the products of elements
// 6+l, 4+l, 2+l, l in that order, the tail is added pair by pair, then lane 0
// + lane 1.  Restated here with explicit round-to-nearest mul/add so the f64
// scores -- and therefore the ranked block ids, ties included -- are bit-equal.
__device__ __forceinline__ double einsum_score(const float* __restrict__ qi,
                                               const float* __restrict__ kb, int hq, int g,
                                               int dh) {
  const int n = hq * dh;
  auto prod = [&](int e) {
    int h = e / dh, c = e - h * dh;
    return __dmul_rn((double)qi[e], (double)kb[(h / g) * dh + c]);
  };
  double v0 = 0.0, v1 = 0.0;
  int i = 0;
  for (; n - i >= 8; i += 8) {
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      v0 = __dadd_rn(prod(i + 2 * j), v0);
      v1 = __dadd_rn(prod(i + 2 * j + 1), v1);
    }
  }
  for (; i < n; i += 2) {
    v0 = __dadd_rn(prod(i), v0);
    if (i + 1 < n) v1 = __dadd_rn(prod(i + 1), v1);
  }
  return __dadd_rn(0.0, __dadd_rn(v0, v1));
}

// Vanilla selection (nsa_attention.py:210-232): score = sum_h sum_d q.k_cmp in
// f64, unscaled, in einsum's order; stable descending top-b_sel ==
// lexicographic (-score, col).
__global__ void score_topk_kernel(const float* __restrict__ q, int64_t nq, int hq, int hkv,
                                  int dh, const float* __restrict__ kc, int nb, int b_sel,
                                  int32_t* __restrict__ out_rows,
                                  int32_t* __restrict__ out_count) {
  int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (i >= nq) return;
  int g = hq / hkv;
  int take = min(b_sel, nb);
  double last_v = -__builtin_huge_val();
  int last_i = -1;
  for (int s = 0; s < take; ++s) {
    double best = __builtin_huge_val();
    int bi = 0x7fffffff;
    for (int b = lane; b < nb; b += 32) {
      double key = -einsum_score(q + i * hq * dh, kc + (int64_t)b * hkv * dh, hq, g, dh);
      if (lex_less(last_v, last_i, key, b) && lex_less(key, b, best, bi)) { best = key; bi = b; }
    }
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (lex_less(ov, oi, best, bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) out_rows[i * b_sel + s] = bi;
    last_v = best;
    last_i = bi;
  }
  if (lane == 0) {
    for (int s = take; s < b_sel; ++s) out_rows[i * b_sel + s] = -1;
    out_count[i] = take;
  }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_sigmoid_f32(const float* logits, int64_t ld, const float* bias, int64_t n, int cols,
                     float* out, void* stream) {
  if (n == 0) return LSRM_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(n * cols, 256), 148 * 16);
  sigmoid_f32_kernel<<<blocks, 256, 0, as_stream(stream)>>>(logits, ld, bias, n, cols, out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_score_topk(const float* q, int64_t nq, int hq, int hkv, int dh, const float* k_cmp,
                    int64_t n_blocks, int b_sel, int32_t* out_rows, int32_t* out_count,
                    void* stream) {
  LSRM_REQUIRE(b_sel >= 1, "b_sel must be at least 1");
  if (n_blocks == 0) return set_error(LSRM_E_EMPTY_CONTEXT, "scoring against zero compressed blocks");
  if (nq == 0) return LSRM_OK;
  score_topk_kernel<<<(unsigned)ceil_div(nq, 8), 256, 0, as_stream(stream)>>>(
      q, nq, hq, hkv, dh, k_cmp, (int)n_blocks, b_sel, out_rows, out_count);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_attention_f32(int mode, const float* q, int64_t nq, int hq, int hkv, int dh,
                       const float* k, const float* v, int64_t nk,
                       const int64_t* block_offsets, const int32_t* rows,
                       const int32_t* count, int kmax_rows, const int32_t* own_row,
                       const int64_t* ids, const int64_t* lengths, int64_t width,
                       float* out, void* stream) {
  LSRM_REQUIRE(mode >= 0 && mode <= 3, "attention_f32: bad mode %d", mode);
  LSRM_REQUIRE(hq >= 1 && hkv >= 1 && hq % hkv == 0,
               "n_q_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  if (nq == 0) return LSRM_OK;
  if (nk == 0) return set_error(LSRM_E_EMPTY_CONTEXT, "attention over an empty key set");
  // lanes per (query, head): fill ~148 SMs x LSRM_F32_FILL threads, at most 32
#ifndef LSRM_F32_FILL
#define LSRM_F32_FILL 1024
#endif
  int split = 1;
  while (split < 32 && nq * hq * split * 2 <= 148LL * LSRM_F32_FILL) split *= 2;
  unsigned blocks = (unsigned)ceil_div(nq * hq * split, 128);
  cudaStream_t st = as_stream(stream);
#define LSRM_ATTN_CASE(D)                                                              \
  case D:                                                                              \
    attention_f32_kernel<D><<<blocks, 128, 0, st>>>(mode, q, nq, hq, hkv, k, v, nk,    \
                                                    block_offsets, rows, count,        \
                                                    kmax_rows, own_row, ids, lengths,  \
                                                    width, out, split);                \
    break;
  switch (dh) {
    LSRM_ATTN_CASE(4)
    LSRM_ATTN_CASE(8)
    LSRM_ATTN_CASE(16)
    LSRM_ATTN_CASE(32)
    LSRM_ATTN_CASE(64)
    LSRM_ATTN_CASE(128)
    default:
      return set_error(LSRM_E_CONFIG, "attention_f32: head_dim %d not in {4,8,16,32,64,128}", dh);
  }
#undef LSRM_ATTN_CASE
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_gated_merge_f32(const float* gate_logits, int64_t ld_gl, const float* gate_bias,
                         int n_gates, const float* o0, const float* o1, const float* o2,
                         int64_t n, int d, float* merged, void* stream) {
  LSRM_REQUIRE(n_gates >= 1 && n_gates <= 3, "gated_merge: 1..3 gates");
  if (n == 0) return LSRM_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(n * d, 256), 148 * 16);
  gated_merge_f32_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      gate_logits, ld_gl, gate_bias, n_gates, o0, o1, o2, n, d, merged);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
