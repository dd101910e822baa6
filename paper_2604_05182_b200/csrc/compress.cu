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
