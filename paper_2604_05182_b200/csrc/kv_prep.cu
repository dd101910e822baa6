// K/V preparation of the bf16 engine, all (use, K|V) tensors of a layer in ONE
// launch (replaces the per-use interleave + ResBlock + block-mean + compressed
// interleave sequence; lsrm/nsa_attention.py:305-312 with
// lsrm/block_partition.py:141-167 fused in).
//
// Job j = one K or V tensor of one NSA use: token rows [n, w = hkv*dh] bf16
// (a column slice of the fused projection output, block-major order).
// CTA (64-token sub-tile of a block, job j), 4 warps:
//   1. rows -> shared memory, and -> the padded 8x8-core-matrix interleaved
//      layout of the tcgen05 attention (plus the 16 ones columns for V);
//   2. ResBlock r = x + W2 gelu(W1 x + b1) + b2 on the tensor cores
//      (mma.sync m16n8k16 bf16, fp32 accumulation; warp = 16 tokens);
//   3. per-column sums of r over the sub-tile's tokens (fixed order) -> a
//      partial row; the block's last-arriving CTA adds its sub-tiles' partials
//      in sub-tile order (deterministic) -> the block mean (compressed row).
// The compressed row goes to mean_out (f32, for the All-gather-KV shard) and/or
// directly into the interleaved compressed layout cmp_il.
#include "common.cuh"

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

constexpr int kSub = 64;   // tokens per sub-tile (4 warps x 16 rows)
constexpr int kSubBits = 12;   // work code = (block << kSubBits) | sub-tile

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2,
                                        uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& b0, uint32_t& b1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(b0), "=r"(b1)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// element (row, col) of head h in the interleaved layout [hkv][rows][vw]
__device__ __forceinline__ int64_t il_off(int h, int64_t rows, int vw, int64_t row, int col) {
  return (int64_t)h * rows * vw + (row / 8) * (8 * vw) + (col / 8) * 64 + (row % 8) * 8 + col % 8;
}

template <int W>
__global__ void __launch_bounds__(128) kv_prep_kernel(const KvJob* __restrict__ jobs, int dh) {
  constexpr int LDS = W + 8;   // padded smem row (bf16): conflict-free ldmatrix
  constexpr int NT = W / 8;    // mma n-tiles
  extern __shared__ __align__(16) unsigned char kv_smem[];
  __nv_bfloat16* const xs = reinterpret_cast<__nv_bfloat16*>(kv_smem);   // [kSub][LDS]
  __nv_bfloat16* const hs = xs + kSub * LDS;                              // [kSub][LDS]
  __nv_bfloat16* const w1s = hs + kSub * LDS;                             // [W][LDS]
  __nv_bfloat16* const w2s = w1s + W * LDS;                               // [W][LDS]
  float (*csum)[W] = reinterpret_cast<float (*)[W]>(w2s + W * LDS);       // [4][W]
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
  // bf16 weights -> smem (16-byte chunks; W1, W2 are [in][out]: r = x W)
  for (int i = tid; i < W * W / 8; i += 128) {
    const int r = i / (W / 8), c8 = (i % (W / 8)) * 8;
    *reinterpret_cast<uint4*>(&w1s[r * LDS + c8]) = *reinterpret_cast<const uint4*>(J.w1 + r * W + c8);
    *reinterpret_cast<uint4*>(&w2s[r * LDS + c8]) = *reinterpret_cast<const uint4*>(J.w2 + r * W + c8);
  }
  // this thread's accumulator columns: n-tile nt, cols 8nt + 2(lane%4) + {0,1}
  const int g = lane >> 2, t4 = lane & 3;
  float cs[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) cs[nt][0] = cs[nt][1] = 0.f;
  {
    const int64_t s0 = sub * kSub;
    const int nt_valid = (int)(occ - s0 < kSub ? occ - s0 : kSub);
    __syncthreads();   // weights staged
    // 1. rows -> smem + interleaved layout
    for (int e = tid; e < kSub * (W / 8); e += 128) {
      const int r = e / (W / 8), ch = e % (W / 8);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < nt_valid) {
        v = *reinterpret_cast<const uint4*>(J.src + (lo + s0 + r) * J.ld + ch * 8);
        const int col = ch * 8, h = col / dh;
        *reinterpret_cast<uint4*>(J.il + il_off(h, J.rows_pad, vw, prow0 + s0 + r, col - h * dh)) = v;
      }
      *reinterpret_cast<uint4*>(&xs[r * LDS + ch * 8]) = v;
    }
    if (J.ones_cols) {   // [V | ones]: 1 for a real key
      const uint32_t one2 = 0x3F803F80u;
      const int per = (int)J.ones_cols / 8;
      for (int e = tid; e < nt_valid * hkv * per; e += 128) {
        const int r = e / (hkv * per), rem = e % (hkv * per), h = rem / per, cc = rem % per;
        *reinterpret_cast<uint4*>(J.il + il_off(h, J.rows_pad, vw, prow0 + s0 + r, dh + cc * 8)) =
            make_uint4(one2, one2, one2, one2);
      }
    }
    __syncthreads();
    // 2. layer 1: h = gelu(x W1 + b1), rows 16*warp .. +16
    const int r0 = 16 * warp;
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
    for (int k0 = 0; k0 < W; k0 += 16) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(smem_addr(&xs[(r0 + (lane & 15)) * LDS + k0 + (lane >> 4) * 8]), a0, a1, a2, a3);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t b0, b1;
        ldsm_x2_t(smem_addr(&w1s[(k0 + (lane & 15)) * LDS + nt * 8]), b0, b1);
        mma16816(acc[nt], a0, a1, a2, a3, b0, b1);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float z = acc[nt][e] + __ldg(J.b1 + 8 * nt + 2 * t4 + (e & 1));
        v[e] = 0.5f * z * (1.f + erff(z * 0.70710678118654752f));
      }
      *reinterpret_cast<uint32_t*>(&hs[(r0 + g) * LDS + nt * 8 + 2 * t4]) = pack2(v[0], v[1]);
      *reinterpret_cast<uint32_t*>(&hs[(r0 + g + 8) * LDS + nt * 8 + 2 * t4]) = pack2(v[2], v[3]);
    }
    __syncwarp();
    // 3. layer 2 + residual: r = x + h W2 + b2; column sums of valid rows
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
    for (int k0 = 0; k0 < W; k0 += 16) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(smem_addr(&hs[(r0 + (lane & 15)) * LDS + k0 + (lane >> 4) * 8]), a0, a1, a2, a3);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t b0, b1;
        ldsm_x2_t(smem_addr(&w2s[(k0 + (lane & 15)) * LDS + nt * 8]), b0, b1);
        mma16816(acc[nt], a0, a1, a2, a3, b0, b1);
      }
    }
    const bool ok_lo = r0 + g < nt_valid, ok_hi = r0 + g + 8 < nt_valid;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const __nv_bfloat162 xlo =
          *reinterpret_cast<const __nv_bfloat162*>(&xs[(r0 + g) * LDS + nt * 8 + 2 * t4]);
      const __nv_bfloat162 xhi =
          *reinterpret_cast<const __nv_bfloat162*>(&xs[(r0 + g + 8) * LDS + nt * 8 + 2 * t4]);
      const float x0 = __low2float(xlo), x1 = __high2float(xlo);
      const float x2 = __low2float(xhi), x3 = __high2float(xhi);
      const float c0 = __ldg(J.b2 + 8 * nt + 2 * t4), c1 = __ldg(J.b2 + 8 * nt + 2 * t4 + 1);
      if (ok_lo) {
        cs[nt][0] += x0 + acc[nt][0] + c0;
        cs[nt][1] += x1 + acc[nt][1] + c1;
      }
      if (ok_hi) {
        cs[nt][0] += x2 + acc[nt][2] + c0;
        cs[nt][1] += x3 + acc[nt][3] + c1;
      }
    }
  }
  // 4. fixed-order reduction: lanes with equal t4 (xor 4, 8, 16), then warps
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float v = cs[nt][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (g == 0) csum[warp][8 * nt + 2 * t4 + e] = v;
    }
  __syncthreads();
  for (int col = tid; col < W; col += 128)
    J.partial[wi * W + col] = ((csum[0][col] + csum[1][col]) + csum[2][col]) + csum[3][col];
  // 5. the block's last-arriving CTA finishes it
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
    for (int e = tid; e < (plen - occ) * (W / 8); e += 128) {
      const int64_t r = occ + e / (W / 8);
      const int col = (e % (W / 8)) * 8, h = col / dh;
      const uint4 v = *reinterpret_cast<const uint4*>(J.src + lo * J.ld + col);
      *reinterpret_cast<uint4*>(J.il + il_off(h, J.rows_pad, vw, prow0 + r, col - h * dh)) = v;
    }
  }
  const float inv = 1.f / (float)occ;
  for (int col = tid; col < W; col += 128) {
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
    for (int e = tid; e < hkv * (int)J.ones_cols; e += 128) {
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
  const size_t smem = (size_t)(2 * kSub + 2 * w) * (w + 8) * 2 + 4 * w * sizeof(float);
  if (w == 64) {
    LSRM_CUDA(cudaFuncSetAttribute(kv_prep_kernel<64>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kv_prep_kernel<64><<<grid, 128, smem, st>>>(reinterpret_cast<const KvJob*>(jobs), dh);
  } else {
    LSRM_CUDA(cudaFuncSetAttribute(kv_prep_kernel<128>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kv_prep_kernel<128><<<grid, 128, smem, st>>>(reinterpret_cast<const KvJob*>(jobs), dh);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}
