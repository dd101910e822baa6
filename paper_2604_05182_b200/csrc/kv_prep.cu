// K/V preparation of the bf16 engine, all (use, K|V) tensors of a layer in ONE
// launch (replaces the per-use interleave + ResBlock + block-mean + compressed
// interleave sequence; lsrm/nsa_attention.py:305-312 with
// lsrm/block_partition.py:141-167 fused in).
//
// Job j = one K or V tensor of one NSA use: token rows [n, w = hkv*dh] bf16
// (a column slice of the fused projection output, block-major order).
// CTA (128-token sub-tile of a block, job j), 8 warps; in the epilogues a
// thread = (token row = TMEM lane, column half):
//   1. rows -> shared memory (UMMA K-major core-matrix layout), and -> the
//      padded 8x8-core-matrix interleaved layout of the tcgen05 attention
//      (plus the 16 ones columns for V);
//   2. ResBlock r = x + W2 gelu(W1 x + b1) + b2 on the 5th-gen tensor cores:
//      tcgen05.mma (M = 128 tokens, N = K = w) into TMEM, x and h from shared
//      memory, W1 / W2 from shared memory (MN-major); the bias + erf-gelu
//      epilogue reads D1 back with tcgen05.ld and writes h (bf16) for the
//      second MMA;
//   3. per-column sums of r over the sub-tile's tokens (fixed order: warp
//      shuffle tree, then the four warps) -> a partial row; the block's
//      last-arriving CTA adds its sub-tiles' partials in sub-tile order
//      (deterministic) -> the block mean (compressed row).
// The compressed row goes to mean_out (f32, for the All-gather-KV shard) and/or
// directly into the interleaved compressed layout cmp_il.
#include "common.cuh"
#include "tcgen05.cuh"

namespace lsrm {

// device copy of lsrm_kv_job (include/lsrm_b200.h)
struct KvJob {
  const __nv_bfloat16* src;
  int64_t ld;
  const int64_t* blk_off;
  const int64_t* pad_off;
  int64_t n_blocks, rows_pad;
  __nv_bfloat16* il;
  int64_t ones_cols;
  const __nv_bfloat16* w1;   // [W][W] bf16 (r = x W1)
  const float* b1;
  const __nv_bfloat16* w2;
  const float* b2;
  float* mean_out;
  __nv_bfloat16* cmp_il;
  int64_t cmp_rows_pad;
  const int32_t* work;   // per CTA: (block << 12) | 64-token sub-tile, ordered by block
  int64_t n_work;
  float* partial;        // [n_work][W] per-sub-tile column sums
  int32_t* arrive;       // [n_blocks] arrival counters (zero between launches)
};
static_assert(sizeof(KvJob) == sizeof(lsrm_kv_job), "KvJob must mirror lsrm_kv_job");

constexpr int kSub = 128;      // tokens per sub-tile = MMA M = TMEM lanes
constexpr int kThreads = 256;  // 8 warps: TMEM lane quarter = warp % 4, column half = warp / 4
constexpr int kSubBits = 12;   // work code = (block << kSubBits) | sub-tile

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// element (row, col) of head h in the interleaved layout [hkv][rows][vw]
__device__ __forceinline__ int64_t il_off(int h, int64_t rows, int vw, int64_t row, int col) {
  return (int64_t)h * rows * vw + (row / 8) * (8 * vw) + (col / 8) * 64 + (row % 8) * 8 + col % 8;
}
// UMMA SWIZZLE_NONE core-matrix layouts of a [rows][W] bf16 tile: 8x8 core
// matrices, (row/8, col/8) at (row/8)*8W + (col/8)*64 elements. As the A
// operand (token rows, K = col) this is K-major (LBO 128 B between K-adjacent
// cores, SBO 16W B between M-adjacent ones); as the B operand with rows = K
// (W1 / W2 are [in][out]) it is MN-major (LBO 16W B, SBO 128 B).
template <int W>
__device__ __forceinline__ int core_off(int row, int col) {
  return (row / 8) * (8 * W) + (col / 8) * 64 + (row % 8) * 8 + col % 8;
}

template <int W>
__global__ void __launch_bounds__(kThreads) kv_prep_kernel(const KvJob* __restrict__ jobs, int dh) {
  extern __shared__ __align__(128) unsigned char kv_smem[];
  __nv_bfloat16* const xs = reinterpret_cast<__nv_bfloat16*>(kv_smem);   // [kSub][W] core
  __nv_bfloat16* const hs = xs + kSub * W;                                // [kSub][W] core
  __nv_bfloat16* const w1s = hs + kSub * W;                               // [W][W] core
  __nv_bfloat16* const w2s = w1s + W * W;                                 // [W][W] core
  float (*csum)[W] = reinterpret_cast<float (*)[W]>(w2s + W * W);       // [kThreads/W][W]
  // [kSub][W] f32 column-sum staging, XOR-swizzled by row (conflict-free);
  // aliases hs / w1s / w2s, which are dead once the second MMA has completed
  float* const red = reinterpret_cast<float*>(hs);
  static_assert(kSub * W * 4 <= (kSub * W + 2 * W * W) * 2, "red must fit hs + w1s + w2s");
  __shared__ uint64_t s_bar;
  __shared__ __align__(16) float s_b1[W], s_b2[W];
  __shared__ uint32_t s_tmem;
  __shared__ int s_last;
  const KvJob& J = jobs[blockIdx.y];
  const int64_t wi = blockIdx.x;
  if (wi >= J.n_work) return;
  const int code = J.work[wi];
  const int64_t b = code >> kSubBits, sub = code & ((1 << kSubBits) - 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hkv = W / dh, vw = dh + (int)J.ones_cols;
  const int64_t lo = J.blk_off[b], occ = J.blk_off[b + 1] - lo, prow0 = J.pad_off[b];
  const int64_t n_sub = (occ + kSub - 1) / kSub;
  if (warp == 0) tc::tmem_alloc(&s_tmem, 2 * W);   // D1 = x W1, D2 = h W2
  if (tid == 0) {
    tc::mbar_init(&s_bar, 1);
    tc::fence_mbar_init();
  }
  // weights and the sub-tile's rows -> smem core layouts, all as async copies
  // in flight together (rows past the block zero-filled)
  for (int i = tid; i < W * W / 8; i += kThreads) {
    const int r = i / (W / 8), c8 = (i % (W / 8)) * 8;
    tc::cp_async16(&w1s[core_off<W>(r, c8)], J.w1 + r * W + c8, 16u);
    tc::cp_async16(&w2s[core_off<W>(r, c8)], J.w2 + r * W + c8, 16u);
  }
  for (int i = tid; i < W; i += kThreads) {
    s_b1[i] = J.b1[i];
    s_b2[i] = J.b2[i];
  }
  const int64_t s0 = sub * kSub;
  const int nt_valid = (int)(occ - s0 < kSub ? occ - s0 : kSub);
  for (int e = tid; e < kSub * (W / 8); e += kThreads) {
    const int r = e / (W / 8), ch = e % (W / 8);
    const bool v = r < nt_valid;
    tc::cp_async16(&xs[core_off<W>(r, ch * 8)], J.src + (v ? (lo + s0 + r) * J.ld + ch * 8 : 0),
                   v ? 16u : 0u);
  }
  tc::cp_async_wait_all();
  tc::fence_async_smem();   // smem writes -> visible to the tensor core
  tc::tc_before_sync();
  __syncthreads();
  tc::tc_after_sync();
  const uint32_t tmem = s_tmem;
  const uint32_t d1 = tmem, d2 = tmem + W;
  const uint32_t idesc = tc::idesc_bf16(kSub, W, 1);   // A K-major, B MN-major
  // 2a. D1 = x W1 (K = W in steps of 16)
  if (warp == 0 && tc::elect_one_sync()) {
    const uint64_t a = tc::sdesc(tc::smem_u32(xs), 128, 16 * W);
    const uint64_t bw = tc::sdesc(tc::smem_u32(w1s), 16 * W, 128);
#pragma unroll
    for (int kk = 0; kk < W / 16; ++kk)
      tc::mma_bf16(d1, a + (uint64_t)(kk * 16), bw + (uint64_t)(kk * 2 * W), idesc, kk > 0);
    tc::mma_commit(&s_bar);
  }
  __syncwarp();
  // 1. (while the MMA runs) rows -> the padded interleaved layout of the
  //    attention (plus the ones columns of [V | ones])
  for (int e = tid; e < nt_valid * (W / 8); e += kThreads) {
    const int r = e / (W / 8), ch = e % (W / 8);
    const int col = ch * 8, h = col / dh;
    *reinterpret_cast<uint4*>(J.il + il_off(h, J.rows_pad, vw, prow0 + s0 + r, col - h * dh)) =
        *reinterpret_cast<const uint4*>(&xs[core_off<W>(r, col)]);
  }
  if (J.ones_cols) {   // [V | ones]: 1 for a real key
    const uint32_t one2 = 0x3F803F80u;
    const int per = (int)J.ones_cols / 8;
    for (int e = tid; e < nt_valid * hkv * per; e += kThreads) {
      const int r = e / (hkv * per), rem = e % (hkv * per), h = rem / per, cc = rem % per;
      *reinterpret_cast<uint4*>(J.il + il_off(h, J.rows_pad, vw, prow0 + s0 + r, dh + cc * 8)) =
          make_uint4(one2, one2, one2, one2);
    }
  }
  tc::mbar_wait(&s_bar, 0);
  tc::tc_after_sync();
  // 2b. h = gelu(D1 + b1) -> smem (this thread's row, core layout); warps whose
  //     rows are all past the block skip it (their D2 rows are never read)
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;                   // TMEM lane = token row
  const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
  constexpr int kHalf = W / 2;                           // columns of this thread
  if (quarter * 32 < nt_valid) {
#pragma unroll
    for (int c0 = half * kHalf; c0 < (half + 1) * kHalf; c0 += 32) {
      uint32_t r[32];
      tc::tmem_ld32(d1 + lane_base + c0, r);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        const float4 ba = *reinterpret_cast<const float4*>(&s_b1[c0 + j]);
        const float4 bb = *reinterpret_cast<const float4*>(&s_b1[c0 + j + 4]);
        const float bv[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const float z0 = __uint_as_float(r[j + e]) + bv[e];
          const float z1 = __uint_as_float(r[j + e + 1]) + bv[e + 1];
          w[e / 2] = pack2(0.5f * z0 * (1.f + erff(z0 * 0.70710678118654752f)),
                           0.5f * z1 * (1.f + erff(z1 * 0.70710678118654752f)));
        }
        *reinterpret_cast<uint4*>(&hs[core_off<W>(row, c0 + j)]) =
            make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  tc::fence_async_smem();
  tc::tc_before_sync();
  __syncthreads();
  tc::tc_after_sync();
  // 2c. D2 = h W2
  if (warp == 0 && tc::elect_one_sync()) {
    const uint64_t a = tc::sdesc(tc::smem_u32(hs), 128, 16 * W);
    const uint64_t bw = tc::sdesc(tc::smem_u32(w2s), 16 * W, 128);
#pragma unroll
    for (int kk = 0; kk < W / 16; ++kk)
      tc::mma_bf16(d2, a + (uint64_t)(kk * 16), bw + (uint64_t)(kk * 2 * W), idesc, kk > 0);
    tc::mma_commit(&s_bar);
  }
  __syncwarp();
  tc::mbar_wait(&s_bar, 1);
  tc::tc_after_sync();
  // 3. r = x + D2 + b2 on valid rows -> red[row][col] (f32); then fixed-order
  //    column sums over the 128 rows (thread = column x row slice)
  const bool ok = row < nt_valid;
  if (quarter * 32 < nt_valid) {
#pragma unroll
    for (int c0 = half * kHalf; c0 < (half + 1) * kHalf; c0 += 32) {
      uint32_t r[32];
      tc::tmem_ld32(d2 + lane_base + c0, r);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        const uint4 xv = *reinterpret_cast<const uint4*>(&xs[core_off<W>(row, c0 + j)]);
        const __nv_bfloat16* xh = reinterpret_cast<const __nv_bfloat16*>(&xv);
        const float4 ba = *reinterpret_cast<const float4*>(&s_b2[c0 + j]);
        const float4 bb = *reinterpret_cast<const float4*>(&s_b2[c0 + j + 4]);
        const float bv[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int e = 0; e < 8; ++e)
          red[row * W + ((c0 + j + e) ^ (row & 31))] =
              ok ? __bfloat162float(xh[e]) + __uint_as_float(r[j + e]) + bv[e] : 0.f;
      }
    }
  } else {
    for (int c = half * kHalf; c < (half + 1) * kHalf; ++c) red[row * W + c] = 0.f;
  }
  tc::tc_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::tc_after_sync();
    tc::tmem_dealloc(tmem, 2 * W);
  }
  {
    constexpr int kSlices = kThreads / W;       // row slices per column (4 for W = 64)
    constexpr int kRows = kSub / kSlices;
    const int col = tid % W, sl = tid / W;
    float acc = 0.f;
    for (int i = 0; i < kRows; ++i) {
      const int rr = sl * kRows + i;
      acc += red[rr * W + (col ^ (rr & 31))];
    }
    csum[sl][col] = acc;
  }
  __syncthreads();
  for (int col = tid; col < W; col += kThreads) {
    float tot = csum[0][col];
    for (int sl = 1; sl < kThreads / W; ++sl) tot += csum[sl][col];
    J.partial[wi * W + col] = tot;
  }
  // 4. the block's last-arriving CTA finishes it
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&J.arrive[b], 1) == (int)n_sub - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t w0 = wi - sub;   // partial row of the block's sub-tile 0
  // K padding rows of the block segment repeat its first key (a duplicate key
  // cannot raise a row max; the matching V rows stay zero): no padding masks
  // in the attention kernel
  if (!J.ones_cols) {
    const int64_t plen = J.pad_off[b + 1] - prow0;
    for (int e = tid; e < (plen - occ) * (W / 8); e += kThreads) {
      const int64_t r = occ + e / (W / 8);
      const int col = (e % (W / 8)) * 8, h = col / dh;
      const uint4 v = *reinterpret_cast<const uint4*>(J.src + lo * J.ld + col);
      *reinterpret_cast<uint4*>(J.il + il_off(h, J.rows_pad, vw, prow0 + r, col - h * dh)) = v;
    }
  }
  const float inv = 1.f / (float)occ;
  for (int col = tid; col < W; col += kThreads) {
    float tot = 0.f;
    for (int64_t k = 0; k < n_sub; ++k) tot += __ldcg(J.partial + (w0 + k) * W + col);
    const float mean = tot * inv;
    if (J.mean_out) J.mean_out[b * W + col] = mean;
    if (J.cmp_il) {
      const int h = col / dh;
      J.cmp_il[il_off(h, J.cmp_rows_pad, vw, b, col - h * dh)] = __float2bfloat16_rn(mean);
      if (b == 0 && !J.ones_cols)   // compressed K padding rows repeat row 0
        for (int64_t r = J.n_blocks; r < J.cmp_rows_pad; ++r)
          J.cmp_il[il_off(h, J.cmp_rows_pad, vw, r, col - h * dh)] = __float2bfloat16_rn(mean);
    }
  }
  if (tid == 0) J.arrive[b] = 0;   // ready for the next launch
  if (J.cmp_il && J.ones_cols)
    for (int e = tid; e < hkv * (int)J.ones_cols; e += kThreads) {
      const int h = e / (int)J.ones_cols, cc = e % (int)J.ones_cols;
      J.cmp_il[il_off(h, J.cmp_rows_pad, vw, b, dh + cc)] = __float2bfloat16_rn(1.f);
    }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" int lsrm_kv_prepare_jobs(const lsrm_kv_job* jobs, int n_jobs, int64_t max_work,
                                    int hkv, int dh, void* stream) {
  const int w = hkv * dh;
  LSRM_REQUIRE(w == 64 || w == 128, "kv_prepare_jobs: width hkv*dh must be 64 or 128, got %d", w);
  LSRM_REQUIRE(dh % 8 == 0, "kv_prepare_jobs: head_dim must be a multiple of 8");
  if (n_jobs == 0 || max_work == 0) return LSRM_OK;
  cudaStream_t st = as_stream(stream);
  const dim3 grid((unsigned)max_work, (unsigned)n_jobs);
  const size_t smem = (size_t)(2 * kSub + 2 * w) * w * 2 + (size_t)kThreads * sizeof(float);
  if (w == 64) {
    LSRM_CUDA(cudaFuncSetAttribute(kv_prep_kernel<64>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kv_prep_kernel<64><<<grid, kThreads, smem, st>>>(reinterpret_cast<const KvJob*>(jobs), dh);
  } else {
    LSRM_CUDA(cudaFuncSetAttribute(kv_prep_kernel<128>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kv_prep_kernel<128><<<grid, kThreads, smem, st>>>(reinterpret_cast<const KvJob*>(jobs), dh);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}
