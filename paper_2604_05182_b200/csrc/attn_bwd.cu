// Backward of one gated NSA use, fp32 on CUDA cores (SURVEY.md §8f rank 2:
// the reference has no backward; the oracle is a float64 torch autograd
// restatement, oracle/torch_nsa.py).
//
//   * attention_bwd: a query-major pass (thread per (query, q-head), the key
//     set walked like the forward in attn_f32.cu) recomputes the softmax
//     statistics and accumulates dQ; a key-major pass (CTA per 64-key tile,
//     thread per key) streams the queries whose key set holds that tile and
//     accumulates dK, dV in registers: dS = P (dO.V - rowsum(dO O)).
//   * gate_merge_bwd: merged = sum_b sigmoid(z_b) * O_b  ->  dO_b, dz_b.
//   * res_block_bwd: the compression's per-token ResBlock under the block
//     mean, r = x + gelu(x W1 + b1) W2 + b2, k_cmp[b] = mean_{t in b} r_t;
//     emits dx (accumulated), dz1 and h for the weight-gradient GEMMs.
// No float atomics: every gradient is summed in a fixed order, so a run's
// bytes are reproducible.
#include "common.cuh"

namespace lsrm {

template <int DH>
__device__ __forceinline__ void range_stats(const float* __restrict__ k, int hkv, int kvh,
                                            int64_t lo, int64_t hi, const float (&q)[DH],
                                            float scale, float& m, float& l) {
  for (int64_t j = lo; j < hi; ++j) {
    const float* kr = k + (j * hkv + kvh) * DH;
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < DH; ++c) s = fmaf(q[c], kr[c], s);
    s *= scale;
    if (s > m) {
      l *= expf(m - s);
      m = s;
    }
    l += expf(s - m);
  }
}

template <int DH>
__device__ __forceinline__ void range_dq(const float* __restrict__ k, const float* __restrict__ v,
                                        int hkv, int kvh, int64_t lo, int64_t hi,
                                        const float (&q)[DH], const float (&dout)[DH],
                                        float dsum, float scale, float lse, float (&dq)[DH]) {
  for (int64_t j = lo; j < hi; ++j) {
    const int64_t base = (j * hkv + kvh) * DH;
    const float* kr = k + base;
    const float* vr = v + base;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int c = 0; c < DH; ++c) {
      s = fmaf(q[c], __ldg(kr + c), s);
      dp = fmaf(dout[c], __ldg(vr + c), dp);
    }
    const float ds = expf(s * scale - lse) * (dp - dsum) * scale;
#pragma unroll
    for (int c = 0; c < DH; ++c) dq[c] = fmaf(ds, __ldg(kr + c), dq[c]);
  }
}

// Query-major pass: thread per (query, q-head).  Recomputes the softmax
// statistics, writes lse = m + log(l) and D = dO . O for the key pass, and
// accumulates dQ.
template <int DH>
__global__ void attention_bwd_dq_kernel(int mode, const float* __restrict__ q,
                                        const float* __restrict__ dO,
                                        const float* __restrict__ O, int64_t nq, int hq,
                                        int hkv, const float* __restrict__ k,
                                        const float* __restrict__ v, int64_t nk,
                                        const int64_t* __restrict__ offs,
                                        const int32_t* __restrict__ rows,
                                        const int32_t* __restrict__ count, int kmax,
                                        const int32_t* __restrict__ own_row,
                                        float* __restrict__ dq, float* __restrict__ lse_out,
                                        float* __restrict__ dsum_out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nq * hq) return;
  const int64_t i = t / hq;
  const int h = (int)(t % hq);
  const int kvh = h / (hq / hkv);
  float qr[DH], dor[DH], dqa[DH];
  float dsum = 0.f;
#pragma unroll
  for (int c = 0; c < DH; ++c) {
    qr[c] = q[t * DH + c];
    dor[c] = dO[t * DH + c];
    dsum = fmaf(dor[c], O[t * DH + c], dsum);
    dqa[c] = 0.f;
  }
  const float scale = 1.0f / sqrtf((float)DH);
  float m = -__builtin_huge_valf(), l = 0.f;
  auto walk = [&](auto&& f) {
    if (mode == 0) {
      f((int64_t)0, nk);
    } else if (mode == 1) {
      const int cnt = count[i];
      for (int s = 0; s < cnt; ++s) {
        const int r = rows[i * kmax + s];
        f(offs[r], offs[r + 1]);
      }
    } else {
      const int r = own_row[i];
      f(offs[r], offs[r + 1]);
    }
  };
  walk([&](int64_t lo, int64_t hi) { range_stats<DH>(k, hkv, kvh, lo, hi, qr, scale, m, l); });
  const float lse = m + logf(l);
  walk([&](int64_t lo, int64_t hi) {
    range_dq<DH>(k, v, hkv, kvh, lo, hi, qr, dor, dsum, scale, lse, dqa);
  });
#pragma unroll
  for (int c = 0; c < DH; ++c) dq[t * DH + c] += dqa[c];
  lse_out[t] = lse;
  dsum_out[t] = dsum;
}

// Key-major pass, deterministic (no atomics): CTA per (64-key tile of one
// block row, kv head, query slice).  Each thread owns one key and keeps k, v,
// dk, dv in registers.  The CTA scans its query slice in order, compacts the
// queries whose key set contains this row (sel: the row is in the query's
// resolved list; win: it is the query's own row; cmp: every query), and
// streams their (query, head) pairs through shared memory 16 at a time.
// Partial dK/dV per slice go to part[slice]; a fixed-order reduction sums
// them.
constexpr int kBwdKeys = 64;
constexpr int kBwdPairs = 16;

template <int DH>
__global__ void __launch_bounds__(kBwdKeys)
attention_bwd_dkdv_kernel(int mode, const float* __restrict__ q, const float* __restrict__ dO,
                          const float* __restrict__ lse, const float* __restrict__ dsum,
                          int64_t nq, int hq, int hkv, const float* __restrict__ k,
                          const float* __restrict__ v, int64_t nk,
                          const int64_t* __restrict__ offs, int n_rows, int tiles_per_row,
                          const int32_t* __restrict__ rows, const int32_t* __restrict__ count,
                          int kmax, const int32_t* __restrict__ own_row, int n_slices,
                          float* __restrict__ part_dk, float* __restrict__ part_dv) {
  __shared__ int qlist[kBwdKeys];
  __shared__ int wsum[2];
  __shared__ float qs[kBwdPairs][DH];
  __shared__ float dos[kBwdPairs][DH];
  __shared__ float ls[kBwdPairs], ds_[kBwdPairs];
  const int tid = threadIdx.x;
  const int row = mode == 0 ? -1 : (int)(blockIdx.x / tiles_per_row);
  const int tile = mode == 0 ? (int)blockIdx.x : (int)(blockIdx.x % tiles_per_row);
  const int g = blockIdx.y;
  const int slice = blockIdx.z;
  const int64_t r_lo = mode == 0 ? 0 : offs[row];
  const int64_t r_hi = mode == 0 ? nk : offs[row + 1];
  const int64_t key0 = r_lo + (int64_t)tile * kBwdKeys;
  if (key0 >= r_hi) return;
  const int64_t j = key0 + tid;
  const bool valid = j < r_hi;
  const int group = hq / hkv;
  const float scale = 1.0f / sqrtf((float)DH);
  float kr[DH], vr[DH], dk[DH], dv[DH];
#pragma unroll
  for (int c = 0; c < DH; ++c) {
    kr[c] = valid ? k[(j * hkv + g) * DH + c] : 0.f;
    vr[c] = valid ? v[(j * hkv + g) * DH + c] : 0.f;
    dk[c] = 0.f;
    dv[c] = 0.f;
  }
  const int64_t q_lo = nq * slice / n_slices, q_hi = nq * (slice + 1) / n_slices;
  for (int64_t base = q_lo; base < q_hi; base += kBwdKeys) {
    const int64_t i = base + tid;
    bool match = false;
    if (i < q_hi) {
      if (mode == 0) {
        match = true;
      } else if (mode == 1) {
        const int cnt = count[i];
        for (int s = 0; s < cnt; ++s) match |= rows[i * kmax + s] == row;
      } else {
        match = own_row[i] == row;
      }
    }
    // in-order compaction (two warps)
    const unsigned bal = __ballot_sync(0xffffffffu, match);
    const int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    const int before = (warp ? wsum[0] : 0) + __popc(bal & ((1u << lane) - 1u));
    const int n_match = wsum[0] + wsum[1];
    if (match) qlist[before] = (int)(i - base);
    __syncthreads();
    const int n_pairs = n_match * group;
    for (int p0 = 0; p0 < n_pairs; p0 += kBwdPairs) {
      const int np = min(kBwdPairs, n_pairs - p0);
      for (int e = tid; e < np * DH; e += kBwdKeys) {
        const int pp = e / DH, c = e % DH;
        const int pair = p0 + pp;
        const int64_t qi = base + qlist[pair / group];
        const int64_t th = qi * hq + (int64_t)g * group + pair % group;
        qs[pp][c] = q[th * DH + c];
        dos[pp][c] = dO[th * DH + c];
        if (c == 0) {
          ls[pp] = lse[th];
          ds_[pp] = dsum[th];
        }
      }
      __syncthreads();
      if (valid) {
        for (int pp = 0; pp < np; ++pp) {
          float s = 0.f, dp = 0.f;
#pragma unroll
          for (int c = 0; c < DH; ++c) {
            s = fmaf(qs[pp][c], kr[c], s);
            dp = fmaf(dos[pp][c], vr[c], dp);
          }
          const float pr = expf(s * scale - ls[pp]);
          const float dsv = pr * (dp - ds_[pp]) * scale;
#pragma unroll
          for (int c = 0; c < DH; ++c) {
            dv[c] = fmaf(pr, dos[pp][c], dv[c]);
            dk[c] = fmaf(dsv, qs[pp][c], dk[c]);
          }
        }
      }
      __syncthreads();
    }
  }
  if (valid) {
    const int64_t o = ((int64_t)slice * nk * hkv + j * hkv + g) * DH;
#pragma unroll
    for (int c = 0; c < DH; ++c) {
      part_dk[o + c] = dk[c];
      part_dv[o + c] = dv[c];
    }
  }
}

// out[e] += sum_{s < n_slices} part[s][e] in slice order (both dK and dV).
__global__ void bwd_reduce_kernel(const float* __restrict__ pk, const float* __restrict__ pv,
                                  int n_slices, int64_t n, float* __restrict__ dk,
                                  float* __restrict__ dv) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int s = 0; s < n_slices; ++s) {
      a += pk[(int64_t)s * n + e];
      b += pv[(int64_t)s * n + e];
    }
    dk[e] += a;
    dv[e] += b;
  }
}

__device__ __forceinline__ double sigmoid_d(double x) {
  return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
}

// merged = sum_b g_b * O_b, g_b = sigmoid(z_b + bias_b):  dO_b = dM g_b,
// dz_b = dM O_b g_b (1 - g_b)
template <int NG>
__device__ __forceinline__ float gate_sig(float z, int fast) {
  return fast ? 1.f / (1.f + __expf(-z)) : (float)sigmoid_d((double)z);
}

// dO_b = dM g_b, dz_b = dM O_b g_b (1 - g_b); fast = fp32 sigmoid (training)
template <int NG>
__global__ void gate_merge_bwd_kernel(const float* __restrict__ gl, int64_t ld,
                                      const float* __restrict__ gb,
                                      const float* __restrict__ o0, const float* __restrict__ o1,
                                      const float* __restrict__ o2,
                                      const float* __restrict__ dm, int64_t n, int d, int fast,
                                      float* __restrict__ do0, float* __restrict__ do1,
                                      float* __restrict__ do2, float* __restrict__ dz) {
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int c = (int)(e % d);
    const float g_m = dm[e];
#pragma unroll
    for (int b = 0; b < NG; ++b) {
      const float* ob = b == 0 ? o0 : (b == 1 ? o1 : o2);
      float* dob = b == 0 ? do0 : (b == 1 ? do1 : do2);
      const float z = gl[i * ld + b * d + c] + (gb ? gb[b * d + c] : 0.f);
      const float g = gate_sig<NG>(z, fast);
      dob[e] = g_m * g;
      dz[i * (int64_t)NG * d + b * d + c] = g_m * ob[e] * g * (1.f - g);
    }
  }
}

// training forward of the gated merge in fp32: merged = sum_b sigmoid(z_b) O_b
template <int NG>
__global__ void gated_merge_fast_kernel(const float* __restrict__ gl, int64_t ld,
                                        const float* __restrict__ gb,
                                        const float* __restrict__ o0,
                                        const float* __restrict__ o1,
                                        const float* __restrict__ o2, int64_t n, int d,
                                        float* __restrict__ merged) {
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int c = (int)(e % d);
    float acc = 0.f;
#pragma unroll
    for (int b = 0; b < NG; ++b) {
      const float* ob = b == 0 ? o0 : (b == 1 ? o1 : o2);
      const float z = gl[i * ld + b * d + c] + (gb ? gb[b * d + c] : 0.f);
      acc = fmaf(1.f / (1.f + __expf(-z)), ob[e], acc);
    }
    merged[e] = acc;
  }
}

// kTokB tokens per CTA (w threads each), W1 / W2 staged in shared memory:
// r = x + gelu(z1) W2 + b2, z1 = x W1 + b1.
// dr = dcmp[row(t)] / occ[row(t)];  dz1 = (dr W2^T) * gelu'(z1);
// dx += dr + dz1 W1^T;  dR, dZ1, H (= gelu(z1)) rows for the weight GEMMs.
constexpr int kTokB = 4;

__global__ void res_block_bwd_kernel(const float* __restrict__ x, int64_t n, int w,
                                     const float* __restrict__ w1, const float* __restrict__ b1,
                                     const float* __restrict__ w2,
                                     const float* __restrict__ dcmp,
                                     const int32_t* __restrict__ row_of_token,
                                     const int64_t* __restrict__ occupancy,
                                     float* __restrict__ dx, float* __restrict__ dr_out,
                                     float* __restrict__ dz1_out, float* __restrict__ h_out) {
  extern __shared__ float sm[];
  const int ws = w + 1;           // padded row stride: row and column walks conflict-free
  float* W1 = sm;                 // [w][w + 1]
  float* W2 = W1 + w * ws;        // [w][w + 1]
  float* xs = W2 + w * ws;        // [kTokB][w]
  float* drs = xs + kTokB * w;    // [kTokB][w]
  float* dz1s = drs + kTokB * w;  // [kTokB][w]
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    W1[(e / w) * ws + e % w] = w1[e];
    W2[(e / w) * ws + e % w] = w2[e];
  }
  const int tl = threadIdx.x / w, o = threadIdx.x % w;
  const int64_t t = (int64_t)blockIdx.x * kTokB + tl;
  const bool ok = tl < kTokB && t < n;
  if (ok) {
    const int r = row_of_token[t];
    xs[tl * w + o] = x[t * w + o];
    drs[tl * w + o] = dcmp[(int64_t)r * w + o] / (float)occupancy[r];
  }
  __syncthreads();
  if (ok) {
    const float* xr = xs + tl * w;
    const float* dr = drs + tl * w;
    float z = b1[o];
    for (int i = 0; i < w; ++i) z = fmaf(xr[i], W1[i * ws + o], z);
    const float cdf = 0.5f * (1.f + erff(z * 0.70710678118654752f));
    const float pdf = 0.39894228040143268f * expf(-0.5f * z * z);
    h_out[t * w + o] = z * cdf;
    // (dr W2^T)[o] = sum_j dr[j] W2[o][j]
    float dh = 0.f;
    for (int j = 0; j < w; ++j) dh = fmaf(dr[j], W2[o * ws + j], dh);
    const float dz = dh * (cdf + z * pdf);
    dz1s[tl * w + o] = dz;
    dz1_out[t * w + o] = dz;
    dr_out[t * w + o] = dr[o];
  }
  __syncthreads();
  if (ok) {
    const float* dz = dz1s + tl * w;
    float acc = drs[tl * w + o];
    for (int j = 0; j < w; ++j) acc = fmaf(dz[j], W1[o * ws + j], acc);
    dx[t * w + o] += acc;
  }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t lsrm_attention_bwd_workspace(int64_t nq, int hq, int64_t nk, int hkv, int dh,
                                    int n_slices) {
  return 2 * align256((size_t)nq * hq * sizeof(float)) +
         2 * align256((size_t)n_slices * nk * hkv * dh * sizeof(float));
}

int lsrm_attention_bwd_f32(int mode, const float* q, const float* dO, const float* O, int64_t nq,
                           int hq, int hkv, int dh, const float* k, const float* v, int64_t nk,
                           const int64_t* block_offsets, int n_rows, int max_row_keys,
                           const int32_t* rows, const int32_t* count, int kmax_rows,
                           const int32_t* own_row, int n_slices, float* dq, float* dk, float* dv,
                           void* workspace, size_t ws_bytes, void* stream) {
  LSRM_REQUIRE(mode >= 0 && mode <= 2, "attention_bwd: mode must be 0 (cmp), 1 (sel), 2 (win)");
  LSRM_REQUIRE(hq % hkv == 0, "n_q_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  LSRM_REQUIRE(n_slices >= 1 && n_slices <= 65535, "attention_bwd: n_slices out of range");
  LSRM_REQUIRE(ws_bytes >= lsrm_attention_bwd_workspace(nq, hq, nk, hkv, dh, n_slices),
               "attention_bwd: workspace too small");
  LSRM_REQUIRE(mode == 0 || (block_offsets && n_rows >= 1),
               "attention_bwd: sel/win need block offsets");
  if (nq == 0 || nk == 0) return LSRM_OK;
  char* ws = (char*)workspace;
  float* lse = (float*)ws;
  float* dsum = (float*)(ws + align256((size_t)nq * hq * sizeof(float)));
  float* pk = (float*)(ws + 2 * align256((size_t)nq * hq * sizeof(float)));
  float* pv = (float*)((char*)pk + align256((size_t)n_slices * nk * hkv * dh * sizeof(float)));
  cudaStream_t st = as_stream(stream);
  const int64_t threads = nq * hq;
  const unsigned grid = (unsigned)ceil_div(threads, 128);
  const int tiles_per_row = mode == 0 ? 0 : (int)ceil_div(max_row_keys, kBwdKeys);
  LSRM_REQUIRE(mode == 0 || tiles_per_row >= 1, "attention_bwd: max_row_keys must be positive");
  const dim3 g2(mode == 0 ? (unsigned)ceil_div(nk, kBwdKeys) : (unsigned)(n_rows * tiles_per_row),
                (unsigned)hkv, (unsigned)n_slices);
  if (mode != 0) {
    // a tile that starts past its row's end returns early; rows without
    // queries leave their partials untouched, so clear them first
    LSRM_CUDA(cudaMemsetAsync(pk, 0, (size_t)n_slices * nk * hkv * dh * sizeof(float), st));
    LSRM_CUDA(cudaMemsetAsync(pv, 0, (size_t)n_slices * nk * hkv * dh * sizeof(float), st));
  }
#define LSRM_BWD_CASE(D)                                                                     \
  case D:                                                                                    \
    attention_bwd_dq_kernel<D><<<grid, 128, 0, st>>>(mode, q, dO, O, nq, hq, hkv, k, v, nk,  \
                                                     block_offsets, rows, count, kmax_rows,  \
                                                     own_row, dq, lse, dsum);                \
    attention_bwd_dkdv_kernel<D><<<g2, kBwdKeys, 0, st>>>(                                   \
        mode, q, dO, lse, dsum, nq, hq, hkv, k, v, nk, block_offsets, n_rows, tiles_per_row, \
        rows, count, kmax_rows, own_row, n_slices, pk, pv);                                  \
    break;
  switch (dh) {
    LSRM_BWD_CASE(4)
    LSRM_BWD_CASE(8)
    LSRM_BWD_CASE(16)
    LSRM_BWD_CASE(32)
    LSRM_BWD_CASE(64)
    default:
      return set_error(LSRM_E_CONFIG, "attention_bwd: head_dim %d not in {4,8,16,32,64}", dh);
  }
#undef LSRM_BWD_CASE
  LSRM_LAUNCHED();
  const int64_t n = nk * hkv * dh;
  const unsigned g3 = (unsigned)(ceil_div(n, 256) < 148 * 8 ? ceil_div(n, 256) : 148 * 8);
  bwd_reduce_kernel<<<g3, 256, 0, st>>>(pk, pv, n_slices, n, dk, dv);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_gate_merge_bwd_f32(const float* gate_logits, int64_t ld_gl, const float* gate_bias,
                            int n_gates, const float* o0, const float* o1, const float* o2,
                            const float* dmerged, int64_t n, int d, int fast, float* do0,
                            float* do1, float* do2, float* dz, void* stream) {
  LSRM_REQUIRE(n_gates >= 1 && n_gates <= 3, "n_gates must be 1..3");
  if (n == 0) return LSRM_OK;
  const int64_t total = n * d;
  const unsigned grid = (unsigned)(ceil_div(total, 256) < 148 * 16 ? ceil_div(total, 256) : 148 * 16);
  cudaStream_t st = as_stream(stream);
  if (n_gates == 3)
    gate_merge_bwd_kernel<3><<<grid, 256, 0, st>>>(gate_logits, ld_gl, gate_bias, o0, o1, o2,
                                                   dmerged, n, d, fast, do0, do1, do2, dz);
  else if (n_gates == 2)
    gate_merge_bwd_kernel<2><<<grid, 256, 0, st>>>(gate_logits, ld_gl, gate_bias, o0, o1, o2,
                                                   dmerged, n, d, fast, do0, do1, do2, dz);
  else
    gate_merge_bwd_kernel<1><<<grid, 256, 0, st>>>(gate_logits, ld_gl, gate_bias, o0, o1, o2,
                                                   dmerged, n, d, fast, do0, do1, do2, dz);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_gated_merge_fast_f32(const float* gate_logits, int64_t ld_gl, const float* gate_bias,
                              int n_gates, const float* o0, const float* o1, const float* o2,
                              int64_t n, int d, float* merged, void* stream) {
  LSRM_REQUIRE(n_gates >= 1 && n_gates <= 3, "n_gates must be 1..3");
  if (n == 0) return LSRM_OK;
  const int64_t total = n * d;
  const unsigned grid = (unsigned)(ceil_div(total, 256) < 148 * 16 ? ceil_div(total, 256) : 148 * 16);
  cudaStream_t st = as_stream(stream);
  if (n_gates == 3)
    gated_merge_fast_kernel<3><<<grid, 256, 0, st>>>(gate_logits, ld_gl, gate_bias, o0, o1, o2,
                                                     n, d, merged);
  else if (n_gates == 2)
    gated_merge_fast_kernel<2><<<grid, 256, 0, st>>>(gate_logits, ld_gl, gate_bias, o0, o1, o2,
                                                     n, d, merged);
  else
    gated_merge_fast_kernel<1><<<grid, 256, 0, st>>>(gate_logits, ld_gl, gate_bias, o0, o1, o2,
                                                     n, d, merged);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_res_block_bwd_f32(const float* x, int64_t n, int width, const float* w1,
                           const float* b1, const float* w2, const float* dcmp,
                           const int32_t* row_of_token, const int64_t* occupancy, float* dx,
                           float* dr_out, float* dz1_out, float* h_out, void* stream) {
  LSRM_REQUIRE(width >= 1 && width <= 256, "res_block_bwd: width %d out of range", width);
  if (n == 0) return LSRM_OK;
  LSRM_REQUIRE(width * kTokB <= 1024, "res_block_bwd: width %d too large", width);
  const size_t smem = (2 * (size_t)width * (width + 1) + 3 * kTokB * (size_t)width) * sizeof(float);
  if (smem > 48 * 1024)
    LSRM_CUDA(cudaFuncSetAttribute(res_block_bwd_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  res_block_bwd_kernel<<<(unsigned)ceil_div(n, kTokB), kTokB * width, smem, as_stream(stream)>>>(
      x, n, width, w1, b1, w2, dcmp, row_of_token, occupancy, dx, dr_out, dz1_out, h_out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
