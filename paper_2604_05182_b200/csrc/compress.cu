// K6 per-block KV compression (lsrm/block_partition.py:141-167).
//
// Pass 1 (token-parallel): ResBlock r = x + W2 gelu(W1 x + b1) + b2 per token,
// evaluated in f64 with the reference's f32 roundings after each affine/gelu.
// Pass 2 (block-parallel): mean over the block's tokens in ascending token id
// order with an f64 running sum (fixed order: bit-stable across workers).
#include "common.cuh"

namespace lsrm {

constexpr int kTokTile = 16;

__device__ __forceinline__ double load_elem(const void* x, int bf16, int64_t idx) {
  return bf16 ? (double)__bfloat162float(((const __nv_bfloat16*)x)[idx])
              : (double)((const float*)x)[idx];
}

// smem: W1, W2 as f32 [w*w] each, x tile f64 [kTokTile*w], h tile f64 [kTokTile*w]
__global__ void res_block_kernel(int src_bf16, const void* __restrict__ x, int64_t ld_x,
                                 int64_t n, int w, const float* __restrict__ w1,
                                 const float* __restrict__ b1, const float* __restrict__ w2,
                                 const float* __restrict__ b2, float* __restrict__ r_out) {
  extern __shared__ double sm[];
  double* xt = sm;                       // [kTokTile][w]
  double* ht = xt + kTokTile * w;        // [kTokTile][w]
  float* W1 = (float*)(ht + kTokTile * w);
  float* W2 = W1 + w * w;
  for (int i = threadIdx.x; i < w * w; i += blockDim.x) { W1[i] = w1[i]; W2[i] = w2[i]; }
  int64_t t0 = (int64_t)blockIdx.x * kTokTile;
  int nt = (int)(n - t0 < kTokTile ? n - t0 : kTokTile);
  for (int e = threadIdx.x; e < kTokTile * w; e += blockDim.x) {
    int t = e / w, c = e % w;
    xt[e] = t < nt ? (double)(float)load_elem(x, src_bf16, (t0 + t) * ld_x + c) : 0.0;
  }
  __syncthreads();
  // h = f32(gelu(f32(x W1 + b1)))
  for (int e = threadIdx.x; e < nt * w; e += blockDim.x) {
    int t = e / w, o = e % w;
    double acc = 0.0;
    for (int i = 0; i < w; ++i) acc += xt[t * w + i] * (double)W1[i * w + o];
    float a = (float)(acc + (double)b1[o]);
    double a64 = (double)a;
    ht[e] = (double)(float)(0.5 * a64 * (1.0 + erf(a64 * 0.70710678118654752440)));
  }
  __syncthreads();
  // r = f32(x + f32(h W2 + b2))
  for (int e = threadIdx.x; e < nt * w; e += blockDim.x) {
    int t = e / w, o = e % w;
    double acc = 0.0;
    for (int i = 0; i < w; ++i) acc += ht[t * w + i] * (double)W2[i * w + o];
    float h2 = (float)(acc + (double)b2[o]);
    r_out[(t0 + t) * w + o] = (float)(xt[e] + (double)h2);
  }
}

// fp32 ResBlock for the bf16 engine (its K/V are bf16 already): 32 tokens
// per CTA, W1/W2 and the x/h tiles in smem, thread = (token group, output).
constexpr int kTokTileF = 32;
__global__ void __launch_bounds__(256)
res_block_f32_kernel(int src_bf16, const void* __restrict__ x, int64_t ld_x, int64_t n, int w,
                     const float* __restrict__ w1, const float* __restrict__ b1,
                     const float* __restrict__ w2, const float* __restrict__ b2,
                     float* __restrict__ r_out) {
  extern __shared__ float smf[];
  float* W1 = smf;
  float* W2 = W1 + w * w;
  float* xt = W2 + w * w;                 // [kTokTileF][w + 1]
  float* ht = xt + kTokTileF * (w + 1);   // [kTokTileF][w + 1]
  const int ldt = w + 1;
  for (int i = threadIdx.x; i < w * w; i += blockDim.x) { W1[i] = w1[i]; W2[i] = w2[i]; }
  const int64_t t0 = (int64_t)blockIdx.x * kTokTileF;
  const int nt = (int)(n - t0 < kTokTileF ? n - t0 : kTokTileF);
  for (int e = threadIdx.x; e < kTokTileF * w; e += blockDim.x) {
    int t = e / w, c = e % w;
    xt[t * ldt + c] = t < nt ? (float)load_elem(x, src_bf16, (t0 + t) * ld_x + c) : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nt * w; e += blockDim.x) {
    int t = e / w, o = e % w;
    float acc = b1[o];
    for (int i = 0; i < w; ++i) acc = fmaf(xt[t * ldt + i], W1[i * w + o], acc);
    ht[t * ldt + o] = 0.5f * acc * (1.f + erff(acc * 0.70710678118654752f));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nt * w; e += blockDim.x) {
    int t = e / w, o = e % w;
    float acc = b2[o];
    for (int i = 0; i < w; ++i) acc = fmaf(ht[t * ldt + i], W2[i * w + o], acc);
    r_out[(t0 + t) * w + o] = xt[t * ldt + o] + acc;
  }
}

// CTA per block; thread (column c, slice s) sums the block's tokens
// s, s+S, s+2S, ... in ascending order in f64, then slice partials are
// combined in fixed slice order: deterministic, coalesced, and no single
// serial chain of dependent loads over a 512-token block.
__global__ void block_mean_kernel(const float* __restrict__ r, int w,
                                  const int64_t* __restrict__ tok,
                                  const int64_t* __restrict__ offs, int64_t nb,
                                  float* __restrict__ out) {
  extern __shared__ double part[];
  const int64_t b = blockIdx.x;
  const int S = blockDim.x / w;
  const int c = threadIdx.x % w, s = threadIdx.x / w;
  const int64_t lo = offs[b], hi = offs[b + 1];
  if (s < S) {
    double acc = 0.0;
    for (int64_t j = lo + s; j < hi; j += S) acc += (double)r[tok[j] * w + c];
    part[s * w + c] = acc;
  }
  __syncthreads();
  if (s == 0) {
    double tot = 0.0;
    for (int k = 0; k < S; ++k) tot += part[k * w + c];
    out[b * w + c] = (float)(tot / (double)(hi - lo));
  }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_compress_block(int src_bf16, const void* x, int64_t ld_x, int64_t n, int width,
                        const float* w1, const float* b1, const float* w2,
                        const float* b2, const int64_t* block_token_ids,
                        const int64_t* block_offsets, int64_t n_blocks, float* out,
                        float* scratch, void* stream) {
  LSRM_REQUIRE(width >= 1 && width <= 128, "compress: width %d outside [1,128]", width);
  if (n == 0 || n_blocks == 0) return LSRM_OK;
  cudaStream_t st = as_stream(stream);
  const int bf16_src = src_bf16 & 1, fast = (src_bf16 >> 1) & 1;
  if (fast) {
    size_t smem = (2 * width * width + 2 * kTokTileF * (width + 1)) * sizeof(float);
    if (smem > 48 * 1024)
      LSRM_CUDA(cudaFuncSetAttribute(res_block_f32_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    res_block_f32_kernel<<<(unsigned)ceil_div(n, kTokTileF), 256, smem, st>>>(
        bf16_src, x, ld_x, n, width, w1, b1, w2, b2, scratch);
  } else {
    size_t smem = 2 * kTokTile * width * sizeof(double) + 2 * width * width * sizeof(float);
    if (smem > 48 * 1024)
      LSRM_CUDA(cudaFuncSetAttribute(res_block_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    res_block_kernel<<<(unsigned)ceil_div(n, kTokTile), 256, smem, st>>>(
        bf16_src, x, ld_x, n, width, w1, b1, w2, b2, scratch);
  }
  LSRM_LAUNCHED();
  int threads = width >= 256 ? width : (256 / width) * width;
  block_mean_kernel<<<(unsigned)n_blocks, threads, threads * sizeof(double), st>>>(
      scratch, width, block_token_ids, block_offsets, n_blocks, out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Fused K/V preparation for the bf16 engine (one launch per K or V tensor):
// reads 64 token rows [hkv*dh] (bf16, block-major), writes them into the
// padded core-matrix interleaved layout consumed by the tcgen05 attention
// (plus the 16 "ones" columns for V), and evaluates the fp32 ResBlock of the
// KV compression with 4x4 register tiles (W1/W2 and the x/h tiles in smem).
namespace lsrm {

constexpr int kPrepTok = 64;

__global__ void __launch_bounds__(256)
kv_prepare_kernel(const __nv_bfloat16* __restrict__ src, int64_t ld, int64_t n, int hkv, int dh,
                  const int32_t* __restrict__ pad_row, int64_t n_rows_pad,
                  __nv_bfloat16* __restrict__ il, int ones_cols, const float* __restrict__ w1,
                  const float* __restrict__ b1, const float* __restrict__ w2,
                  const float* __restrict__ b2, float* __restrict__ r_out) {
  extern __shared__ float smp[];
  const int w = hkv * dh;                 // ResBlock width (<= 128)
  const int ldt = w + 4;                  // padded tile row (16B aligned, fewer conflicts)
  float* W1 = smp;
  float* W2 = W1 + w * w;
  float* xt = W2 + w * w;                 // [kPrepTok][ldt]
  float* ht = xt + kPrepTok * ldt;        // [kPrepTok][ldt]
  for (int i = threadIdx.x; i < w * w; i += blockDim.x) { W1[i] = w1[i]; W2[i] = w2[i]; }
  const int64_t t0 = (int64_t)blockIdx.x * kPrepTok;
  const int nt = (int)(n - t0 < kPrepTok ? n - t0 : kPrepTok);
  const int vw = dh + ones_cols;
  const int nch = w / 8;                  // 16B chunks per token row
  // rows -> smem (f32) and -> interleaved bf16 (16B chunks)
  for (int e = threadIdx.x; e < kPrepTok * nch; e += blockDim.x) {
    const int t = e / nch, ch = e % nch;
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (t < nt) raw = *reinterpret_cast<const uint4*>(src + (t0 + t) * ld + ch * 8);
    const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
    for (int j = 0; j < 8; ++j) xt[t * ldt + ch * 8 + j] = __bfloat162float(hv[j]);
    if (t < nt) {
      const int h = (ch * 8) / dh, cc = (ch * 8 - h * dh) / 8;
      const int64_t prow = pad_row[t0 + t];
      *reinterpret_cast<uint4*>(il + (int64_t)h * n_rows_pad * vw + (prow / 8) * (8 * vw) +
                                cc * 64 + (prow % 8) * 8) = raw;
    }
  }
  if (ones_cols) {
    const uint32_t one2 = 0x3F803F80u;  // bf16x2 (1, 1)
    for (int e = threadIdx.x; e < nt * hkv * (ones_cols / 8); e += blockDim.x) {
      const int t = e / (hkv * (ones_cols / 8)), rem = e % (hkv * (ones_cols / 8));
      const int h = rem / (ones_cols / 8), cc = dh / 8 + rem % (ones_cols / 8);
      const int64_t prow = pad_row[t0 + t];
      *reinterpret_cast<uint4*>(il + (int64_t)h * n_rows_pad * vw + (prow / 8) * (8 * vw) +
                                cc * 64 + (prow % 8) * 8) = make_uint4(one2, one2, one2, one2);
    }
  }
  __syncthreads();
  // thread -> (token quad, output quad); w/4 output quads
  const int oq_n = w / 4, tq_n = kPrepTok / 4;
  for (int job = threadIdx.x; job < oq_n * tq_n; job += blockDim.x) {
    const int oq = job % oq_n, tq = job / oq_n;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = b1[oq * 4 + b];
    for (int i = 0; i < w; ++i) {
      const float4 wv = *reinterpret_cast<const float4*>(&W1[i * w + oq * 4]);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float xv = xt[(tq * 4 + a) * ldt + i];
        acc[a][0] = fmaf(xv, wv.x, acc[a][0]);
        acc[a][1] = fmaf(xv, wv.y, acc[a][1]);
        acc[a][2] = fmaf(xv, wv.z, acc[a][2]);
        acc[a][3] = fmaf(xv, wv.w, acc[a][3]);
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float z = acc[a][b];
        ht[(tq * 4 + a) * ldt + oq * 4 + b] = 0.5f * z * (1.f + erff(z * 0.70710678118654752f));
      }
  }
  __syncthreads();
  for (int job = threadIdx.x; job < oq_n * tq_n; job += blockDim.x) {
    const int oq = job % oq_n, tq = job / oq_n;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = b2[oq * 4 + b];
    for (int i = 0; i < w; ++i) {
      const float4 wv = *reinterpret_cast<const float4*>(&W2[i * w + oq * 4]);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float hv = ht[(tq * 4 + a) * ldt + i];
        acc[a][0] = fmaf(hv, wv.x, acc[a][0]);
        acc[a][1] = fmaf(hv, wv.y, acc[a][1]);
        acc[a][2] = fmaf(hv, wv.z, acc[a][2]);
        acc[a][3] = fmaf(hv, wv.w, acc[a][3]);
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int t = tq * 4 + a;
      if (t < nt) {
        float4 o;
        o.x = xt[t * ldt + oq * 4 + 0] + acc[a][0];
        o.y = xt[t * ldt + oq * 4 + 1] + acc[a][1];
        o.z = xt[t * ldt + oq * 4 + 2] + acc[a][2];
        o.w = xt[t * ldt + oq * 4 + 3] + acc[a][3];
        *reinterpret_cast<float4*>(&r_out[(t0 + t) * w + oq * 4]) = o;
      }
    }
  }
}

// Contiguous block mean (rows of block b are [offs[b], offs[b+1]) of r):
// CTA per block, (column, slice) threads, fixed-order slice combine.
__global__ void block_mean_contig_kernel(const float* __restrict__ r, int w,
                                         const int64_t* __restrict__ offs,
                                         float* __restrict__ out) {
  extern __shared__ double partc[];
  const int64_t b = blockIdx.x;
  const int S = blockDim.x / w;
  const int c = threadIdx.x % w, s = threadIdx.x / w;
  const int64_t lo = offs[b], hi = offs[b + 1];
  double acc = 0.0;
  for (int64_t j = lo + s; j < hi; j += S) acc += (double)r[j * w + c];
  partc[s * w + c] = acc;
  __syncthreads();
  if (s == 0) {
    double tot = 0.0;
    for (int k = 0; k < S; ++k) tot += partc[k * w + c];
    out[b * w + c] = (float)(tot / (double)(hi - lo));
  }
}

}  // namespace lsrm

extern "C" int lsrm_kv_prepare(const void* src, int64_t ld, int64_t n, int hkv, int dh,
                               const int32_t* pad_row, int64_t n_rows_pad, void* il,
                               int ones_cols, const float* w1, const float* b1,
                               const float* w2, const float* b2, float* r_out,
                               const int64_t* block_offsets, int64_t n_blocks, float* mean_out,
                               void* stream) {
  using namespace lsrm;
  const int w = hkv * dh;
  LSRM_REQUIRE(w % 8 == 0 && w <= 128 && dh % 8 == 0, "kv_prepare: width must be 8..128");
  LSRM_REQUIRE(ones_cols == 0 || ones_cols == 16, "kv_prepare: ones_cols must be 0 or 16");
  if (n == 0) return LSRM_OK;
  cudaStream_t st = as_stream(stream);
  size_t smem = (2 * (size_t)w * w + 2 * (size_t)kPrepTok * (w + 4)) * sizeof(float);
  if (smem > 48 * 1024)
    LSRM_CUDA(cudaFuncSetAttribute(kv_prepare_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kv_prepare_kernel<<<(unsigned)ceil_div(n, kPrepTok), 256, smem, st>>>(
      (const __nv_bfloat16*)src, ld, n, hkv, dh, pad_row, n_rows_pad, (__nv_bfloat16*)il,
      ones_cols, w1, b1, w2, b2, r_out);
  LSRM_LAUNCHED();
  if (mean_out && n_blocks) {
    const int threads = (1024 / w) * w;
    block_mean_contig_kernel<<<(unsigned)n_blocks, threads, threads * sizeof(double), st>>>(
        r_out, w, block_offsets, mean_out);
    LSRM_LAUNCHED();
  }
  return LSRM_OK;
}
