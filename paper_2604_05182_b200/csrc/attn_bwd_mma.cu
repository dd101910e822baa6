// Tensor-core backward of the three NSA branches (bf16 operands, fp32
// accumulation, mma.sync m16n8k16), the fast counterpart of attn_bwd.cu's
// fp32 CUDA-core passes, same structure and fixed summation orders:
//
//   * dQ pass, warp per (query, kv head): the G = hq/hkv q-heads of one query
//     share its key set, so they are the 16 MMA rows (padded if G < 16).
//     Pass 1 recomputes the row max / sum over the key set, pass 2 forms
//     P = exp(S - lse), dP = dO V^T, dS = P (dP - D) and dQ += dS K.  It
//     writes lse and D = rowsum(dO * O) for the key pass.
//   * dK/dV pass, CTA (4 warps) per 64-key tile of one block row, kv head and
//     query slice: each warp keeps its 16 keys' K, V (A operands) and dK, dV
//     accumulators in registers, and the CTA streams the matched queries'
//     16 head rows of Q and dO through shared memory:
//     S^T = K Q^T, P^T, dP^T = V dO^T, dV += P^T dO, dK += dS^T Q.
//
// Fragment layouts follow the PTX m16n8k16 bf16 shapes: A row-major 16x16,
// B "col" 16x8, C 16x8 f32 (rows lane/4 and lane/4 + 8, columns 2(lane%4)).
#include <cuda_bf16.h>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

// minimum resident CTAs per SM the register allocation targets (occupancy
// of these latency-bound per-warp passes); unset = the compiler's choice.
// Same-box A/B (tools/ab_train.sh): 6 -> 80 registers with spills, backward
// 13.74 -> 15.1 ms at C3.
#ifdef LSRM_BWD_MINBLOCKS
#define LSRM_BWD_BOUNDS(t) __launch_bounds__(t, LSRM_BWD_MINBLOCKS)
#else
#define LSRM_BWD_BOUNDS(t) __launch_bounds__(t)
#endif

namespace lsrm {
namespace bwdmma {

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// A fragments of a 16 x DH bf16 tile stored row-major in shared memory with a
// row stride of DH + 8 elements (conflict-free ldmatrix): DH/16 k-steps.
template <int DH>
__device__ __forceinline__ void load_a(const __nv_bfloat16* tile, int lane, uint32_t (*a)[4]) {
  constexpr int LD = DH + 8;
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    const int j = lane >> 3, r = lane & 7;
    const int row = r + 8 * (j & 1), col = kk * 16 + 8 * (j >> 1);
    ldsm_x4(s_u32(tile + row * LD + col), a[kk]);
  }
}
// B fragments (k = DH dims, n = 16 rows of the stored tile) for X . T^T where
// T is 16 x DH row-major (rows = n): per k-step, {b0, b1} of n-tile 0 and 1.
template <int DH>
__device__ __forceinline__ void load_b_nt(const __nv_bfloat16* tile, int lane,
                                          uint32_t (*b)[4]) {
  constexpr int LD = DH + 8;
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    // matrices: (n 0-7, k 0-7), (n 0-7, k 8-15), (n 8-15, k 0-7), (n 8-15, k 8-15)
    const int j = lane >> 3, r = lane & 7;
    const int row = r + 8 * (j >> 1), col = kk * 16 + 8 * (j & 1);
    ldsm_x4(s_u32(tile + row * LD + col), b[kk]);   // b[kk] = {n0:b0, n0:b1, n1:b0, n1:b1}
  }
}
// B fragments (k = 16 rows of the stored tile, n = DH dims) for X . T where T
// is 16 x DH row-major (rows = k): per n-pair (16 dims), {b0,b1} x 2 n-tiles.
template <int DH>
__device__ __forceinline__ void load_b_nn(const __nv_bfloat16* tile, int lane,
                                          uint32_t (*b)[4]) {
  constexpr int LD = DH + 8;
#pragma unroll
  for (int np = 0; np < DH / 16; ++np) {
    // matrices (transposed loads): (k 0-7, n 0-7), (k 8-15, n 0-7), (k 0-7, n 8-15), (k 8-15, n 8-15)
    const int j = lane >> 3, r = lane & 7;
    const int row = r + 8 * (j & 1), col = np * 16 + 8 * (j >> 1);
    ldsm_x4_t(s_u32(tile + row * LD + col), b[np]);
  }
}

// key set of query i for a mode (ranges of rows in the branch's key tensor)
struct KeySet {
  int mode;
  int64_t nk;
  const int64_t* offs;
  const int32_t* rows;
  const int32_t* count;
  int kmax;
  const int32_t* own_row;
  __device__ int n_ranges(int64_t i) const {
    return mode == 0 ? 1 : (mode == 1 ? count[i] : 1);
  }
  __device__ void range(int64_t i, int s, int64_t& lo, int64_t& hi) const {
    if (mode == 0) {
      lo = 0;
      hi = nk;
    } else {
      const int r = mode == 1 ? rows[i * kmax + s] : own_row[i];
      lo = offs[r];
      hi = offs[r + 1];
    }
  }
};

constexpr int kDqWarps = 4;

// Walks the 16-key tiles of query i's key set (one warp, warp-private smem
// tiles sK / sV): the next tile's K / V rows are loaded into registers while
// body(k0, hi) computes on the current one.
template <int DH, class Body>
__device__ __forceinline__ void walk_tiles(const KeySet& ks, int64_t i,
                                           const __nv_bfloat16* __restrict__ k,
                                           const __nv_bfloat16* __restrict__ v, int64_t kstride,
                                           int g, int lane, __nv_bfloat16* sK,
                                           __nv_bfloat16* sV, Body&& body) {
  constexpr int LD = DH + 8, PER = 16 * (DH / 8) / 32;
  const int nr = ks.n_ranges(i);
  int sidx = -1;
  int64_t k0 = 0, hi = 0;
  auto advance = [&]() -> bool {
    k0 += 16;
    while (k0 >= hi) {
      if (++sidx >= nr) return false;
      int64_t lo;
      ks.range(i, sidx, lo, hi);
      k0 = lo;
    }
    return true;
  };
  uint4 rk[PER], rv[PER];
  auto fetch = [&]() {
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = lane + 32 * p, r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
      rk[p] = rv[p] = make_uint4(0, 0, 0, 0);
      if (k0 + r < hi) {
        const int64_t base = (k0 + r) * kstride + (int64_t)g * DH + c8;
        rk[p] = *reinterpret_cast<const uint4*>(k + base);
        rv[p] = *reinterpret_cast<const uint4*>(v + base);
      }
    }
  };
  bool have = advance();
  if (have) fetch();
  while (have) {
    const int64_t ck0 = k0, chi = hi;
    __syncwarp();
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = lane + 32 * p, r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
      *reinterpret_cast<uint4*>(sK + r * LD + c8) = rk[p];
      *reinterpret_cast<uint4*>(sV + r * LD + c8) = rv[p];
    }
    __syncwarp();
    have = advance();
    if (have) fetch();   // in flight while the current tile is computed
    body(ck0, chi);
  }
}
constexpr int kCmpKeys = 64;   // CMP: keys per CTA-shared K/V tile

// CMP: the CTA's warps share 64-key K / V tiles of all compressed rows; each
// thread prefetches its share of the next tile into registers while the
// current one is computed.  sub(k0, tk, tv) runs per 16-key sub-tile (valid
// warps only; every thread joins the barriers).
template <int DH, class Sub>
__device__ __forceinline__ void walk_cmp_tiles(int64_t nk, const __nv_bfloat16* __restrict__ k,
                                               const __nv_bfloat16* __restrict__ v,
                                               int64_t kstride, int g, bool valid,
                                               __nv_bfloat16* shK, __nv_bfloat16* shV,
                                               Sub&& sub) {
  constexpr int LD = DH + 8, PER = kCmpKeys * (DH / 8) / (32 * kDqWarps);
  uint4 rk[PER], rv[PER];
  auto fetch = [&](int64_t kb) {
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = threadIdx.x + 32 * kDqWarps * p, r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
      rk[p] = rv[p] = make_uint4(0, 0, 0, 0);
      if (kb + r < nk) {
        const int64_t base = (kb + r) * kstride + (int64_t)g * DH + c8;
        rk[p] = *reinterpret_cast<const uint4*>(k + base);
        rv[p] = *reinterpret_cast<const uint4*>(v + base);
      }
    }
  };
  if (nk > 0) fetch(0);
  for (int64_t kb = 0; kb < nk; kb += kCmpKeys) {
    __syncthreads();   // the previous tile is no longer read
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = threadIdx.x + 32 * kDqWarps * p, r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
      *reinterpret_cast<uint4*>(shK + r * LD + c8) = rk[p];
      *reinterpret_cast<uint4*>(shV + r * LD + c8) = rv[p];
    }
    __syncthreads();
    if (kb + kCmpKeys < nk) fetch(kb + kCmpKeys);   // in flight during the compute
    if (valid)
      for (int t = 0; t < kCmpKeys / 16 && kb + 16 * t < nk; ++t)
        sub(kb + 16 * t, shK + t * 16 * LD, shV + t * 16 * LD);
  }
}

// dQ pass: warp per (query, kv head).
template <int DH, bool CMP>
__global__ void LSRM_BWD_BOUNDS(32 * kDqWarps)
dq_mma_kernel(KeySet ks, const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ dob,
              const float* __restrict__ dO, const float* __restrict__ O,
              const float* __restrict__ lse_in, int64_t nq, int hq,
              int hkv, const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
              float* __restrict__ dq, float* __restrict__ lse_out, float* __restrict__ dsum_out) {
  constexpr int LD = DH + 8;
  __shared__ __align__(16) __nv_bfloat16 sm[kDqWarps][CMP ? 2 : 4][16 * LD];   // Q, dO (, K, V)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CMP: the CTA's warps take kDqWarps queries of one kv head, which share
  // every key (the compressed rows), so K/V tiles are loaded once per CTA
  int64_t i;
  int g;
  bool valid = true;
  if constexpr (CMP) {
    i = (int64_t)(blockIdx.x / hkv) * kDqWarps + warp;
    g = (int)(blockIdx.x % hkv);
    valid = i < nq;
  } else {
    const int64_t wid = (int64_t)blockIdx.x * kDqWarps + warp;
    if (wid >= nq * hkv) return;
    i = wid / hkv;
    g = (int)(wid % hkv);
  }
  const int G = hq / hkv;
  __shared__ __align__(16) __nv_bfloat16 shK[CMP ? kCmpKeys * LD : 8];
  __shared__ __align__(16) __nv_bfloat16 shV[CMP ? kCmpKeys * LD : 8];
  __nv_bfloat16* sQ = sm[warp][0];
  __nv_bfloat16* sO = sm[warp][1];
  __nv_bfloat16* sK = sm[warp][CMP ? 0 : 2];   // private K / V tiles (unused with CMP)
  __nv_bfloat16* sV = sm[warp][CMP ? 1 : 3];
  const int gq = lane >> 2, cq = lane & 3;
  // Q and dO rows of the G heads (rows >= G zero)
  for (int e = lane; e < 16 * (DH / 8); e += 32) {
    const int r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
    uint4 vq = make_uint4(0, 0, 0, 0), vo = make_uint4(0, 0, 0, 0);
    if (valid && r < G) {
      const int64_t base = ((i * hq) + (int64_t)g * G + r) * DH + c8;
      vq = *reinterpret_cast<const uint4*>(q + base);
      vo = *reinterpret_cast<const uint4*>(dob + base);
    }
    *reinterpret_cast<uint4*>(sQ + r * LD + c8) = vq;
    *reinterpret_cast<uint4*>(sO + r * LD + c8) = vo;
  }
  // D = rowsum(dO * O) in fp32 for this thread's two rows (gq, gq + 8)
  float dsum[2] = {0.f, 0.f};
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int r = gq + 8 * hr;
    if (valid && r < G) {
      const int64_t base = ((i * hq) + (int64_t)g * G + r) * DH;
      for (int c = cq; c < DH; c += 4) dsum[hr] = fmaf(dO[base + c], O[base + c], dsum[hr]);
    }
    dsum[hr] += __shfl_xor_sync(0xffffffffu, dsum[hr], 1);
    dsum[hr] += __shfl_xor_sync(0xffffffffu, dsum[hr], 2);
  }
  __syncwarp();
  uint32_t aq[DH / 16][4], ao[DH / 16][4];
  load_a<DH>(sQ, lane, aq);
  load_a<DH>(sO, lane, ao);
  const float scale = 1.0f / sqrtf((float)DH);
  const int64_t kstride = (int64_t)hkv * DH;
  const __nv_bfloat16* tK = sK;   // current 16-key K / V tile
  const __nv_bfloat16* tV = sV;
  auto for_tiles = [&](auto&& body) {
    if constexpr (CMP) {
      walk_cmp_tiles<DH>(ks.nk, k, v, kstride, g, valid, shK, shV,
                         [&](int64_t k0, const __nv_bfloat16* tk, const __nv_bfloat16* tv) {
                           tK = tk;
                           tV = tv;
                           body(k0, ks.nk);
                         });
    } else {
      walk_tiles<DH>(ks, i, k, v, kstride, g, lane, sK, sV, body);
    }
  };
  // S tile (16 rows x 16 keys) = Q K^T, keys past hi masked to -inf
  auto s_tile = [&](int64_t k0, int64_t hi, float (*s)[4]) {
    uint32_t bk[DH / 16][4];
    load_b_nt<DH>(tK, lane, bk);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) mma(s[nt], aq[kk], bk[kk][2 * nt], bk[kk][2 * nt + 1]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t key = k0 + nt * 8 + 2 * cq + (e & 1);
        s[nt][e] = key < hi ? s[nt][e] * scale : -__builtin_huge_valf();
      }
    }
  };
  // pass 1: row max and sum (rows gq, gq + 8), unless the forward saved lse
  float m[2] = {-__builtin_huge_valf(), -__builtin_huge_valf()}, l[2] = {0.f, 0.f};
  if (!lse_in) for_tiles([&](int64_t k0, int64_t hi) {
      float s[2][4];
      s_tile(k0, hi, s);
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        float mx = fmaxf(fmaxf(s[0][2 * hr], s[0][2 * hr + 1]), fmaxf(s[1][2 * hr], s[1][2 * hr + 1]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mn = fmaxf(m[hr], mx);
        float add = __expf(s[0][2 * hr] - mn) + __expf(s[0][2 * hr + 1] - mn) +
                    __expf(s[1][2 * hr] - mn) + __expf(s[1][2 * hr + 1] - mn);
        add += __shfl_xor_sync(0xffffffffu, add, 1);
        add += __shfl_xor_sync(0xffffffffu, add, 2);
        l[hr] = l[hr] * __expf(m[hr] - mn) + add;
        m[hr] = mn;
      }
  });
  float lse[2];
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int r = gq + 8 * hr;
    if (lse_in)
      lse[hr] = (valid && r < G) ? lse_in[i * hq + (int64_t)g * G + r] : 0.f;
    else
      lse[hr] = m[hr] + __logf(l[hr]);
  }
  // pass 2: dQ
  float acc[DH / 8][4];
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
  for_tiles([&](int64_t k0, int64_t hi) {
      float s[2][4], dp[2][4];
      s_tile(k0, hi, s);
      uint32_t bv[DH / 16][4];
      load_b_nt<DH>(tV, lane, bv);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) dp[nt][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) mma(dp[nt], ao[kk], bv[kk][2 * nt], bv[kk][2 * nt + 1]);
      }
      // dS = P (dP - D) * scale as the A operand (16 rows x 16 keys)
      uint32_t ads[4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        float d4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int hr = e >> 1;
          const float p = __expf(s[nt][e] - lse[hr]);
          d4[e] = p * (dp[nt][e] - dsum[hr]) * scale;
        }
        ads[2 * nt] = pk(d4[0], d4[1]);
        ads[2 * nt + 1] = pk(d4[2], d4[3]);
      }
      // dQ += dS K  (B(k = key, n = dim) from the K tile rows, transposed loads)
      uint32_t bk[DH / 16][4];
      load_b_nn<DH>(tK, lane, bk);
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        mma(acc[2 * np], ads, bk[np][0], bk[np][1]);
        mma(acc[2 * np + 1], ads, bk[np][2], bk[np][3]);
      }
  });
  // write dq rows (< G), lse, D
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int r = gq + 8 * hr;
    if (valid && r < G) {
      const int64_t t = i * hq + (int64_t)g * G + r;
#pragma unroll
      for (int nt = 0; nt < DH / 8; ++nt) {
        float* o = dq + t * DH + nt * 8 + 2 * cq;
        o[0] += acc[nt][2 * hr];
        o[1] += acc[nt][2 * hr + 1];
      }
      if (cq == 0) {
        lse_out[t] = lse[hr];
        dsum_out[t] = dsum[hr];
      }
    }
  }
}

// Forward of one branch for training: warp per (query, kv head), online
// softmax over the key set in 16-key tiles; writes the branch output (fp32)
// and lse per (query, head) for the backward.
template <int DH, bool CMP>
__global__ void LSRM_BWD_BOUNDS(32 * kDqWarps)
fwd_mma_kernel(KeySet ks, const __nv_bfloat16* __restrict__ q, int64_t nq, int hq, int hkv,
               const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
               float* __restrict__ out, float* __restrict__ lse_out) {
  constexpr int LD = DH + 8;
  __shared__ __align__(16) __nv_bfloat16 sm[kDqWarps][CMP ? 1 : 3][16 * LD];   // Q (, K, V)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CMP: the CTA's warps take kDqWarps queries of one kv head, which share
  // every key (the compressed rows), so K/V tiles are loaded once per CTA
  int64_t i;
  int g;
  bool valid = true;
  if constexpr (CMP) {
    i = (int64_t)(blockIdx.x / hkv) * kDqWarps + warp;
    g = (int)(blockIdx.x % hkv);
    valid = i < nq;
  } else {
    const int64_t wid = (int64_t)blockIdx.x * kDqWarps + warp;
    if (wid >= nq * hkv) return;
    i = wid / hkv;
    g = (int)(wid % hkv);
  }
  const int G = hq / hkv;
  __shared__ __align__(16) __nv_bfloat16 shK[CMP ? kCmpKeys * LD : 8];
  __shared__ __align__(16) __nv_bfloat16 shV[CMP ? kCmpKeys * LD : 8];
  __nv_bfloat16* sQ = sm[warp][0];
  __nv_bfloat16* sK = sm[warp][CMP ? 0 : 1];   // private K / V tiles (unused with CMP)
  __nv_bfloat16* sV = sm[warp][CMP ? 0 : 2];
  const int gq = lane >> 2, cq = lane & 3;
  for (int e = lane; e < 16 * (DH / 8); e += 32) {
    const int r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
    uint4 vq = make_uint4(0, 0, 0, 0);
    if (valid && r < G)
      vq = *reinterpret_cast<const uint4*>(q + ((i * hq) + (int64_t)g * G + r) * DH + c8);
    *reinterpret_cast<uint4*>(sQ + r * LD + c8) = vq;
  }
  __syncwarp();
  uint32_t aq[DH / 16][4];
  load_a<DH>(sQ, lane, aq);
  const float scale = 1.0f / sqrtf((float)DH);
  const int64_t kstride = (int64_t)hkv * DH;
  float m[2] = {-__builtin_huge_valf(), -__builtin_huge_valf()}, l[2] = {0.f, 0.f};
  float acc[DH / 8][4];
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
  const __nv_bfloat16* tK = sK;   // current 16-key K / V tile
  const __nv_bfloat16* tV = sV;
  auto body = [&](int64_t k0, int64_t hi) {
      uint32_t bk[DH / 16][4];
      load_b_nt<DH>(tK, lane, bk);
      float s[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) mma(s[nt], aq[kk], bk[kk][2 * nt], bk[kk][2 * nt + 1]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t key = k0 + nt * 8 + 2 * cq + (e & 1);
          s[nt][e] = key < hi ? s[nt][e] * scale : -__builtin_huge_valf();
        }
      }
      uint32_t ap[4];
      float p4[2][4];
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        float mx = fmaxf(fmaxf(s[0][2 * hr], s[0][2 * hr + 1]), fmaxf(s[1][2 * hr], s[1][2 * hr + 1]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mn = fmaxf(m[hr], mx);
        const float corr = __expf(m[hr] - mn);
        float add = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float p = __expf(s[nt][2 * hr + e] - mn);
            p4[nt][2 * hr + e] = p;
            add += p;
          }
        add += __shfl_xor_sync(0xffffffffu, add, 1);
        add += __shfl_xor_sync(0xffffffffu, add, 2);
        l[hr] = l[hr] * corr + add;
        m[hr] = mn;
#pragma unroll
        for (int nt = 0; nt < DH / 8; ++nt) {
          acc[nt][2 * hr] *= corr;
          acc[nt][2 * hr + 1] *= corr;
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        ap[2 * nt] = pk(p4[nt][0], p4[nt][1]);
        ap[2 * nt + 1] = pk(p4[nt][2], p4[nt][3]);
      }
      uint32_t bv[DH / 16][4];
      load_b_nn<DH>(tV, lane, bv);
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        mma(acc[2 * np], ap, bv[np][0], bv[np][1]);
        mma(acc[2 * np + 1], ap, bv[np][2], bv[np][3]);
      }
  };
  if constexpr (CMP) {
    walk_cmp_tiles<DH>(ks.nk, k, v, kstride, g, valid, shK, shV,
                       [&](int64_t k0, const __nv_bfloat16* tk, const __nv_bfloat16* tv) {
                         tK = tk;
                         tV = tv;
                         body(k0, ks.nk);
                       });
  } else {
    walk_tiles<DH>(ks, i, k, v, kstride, g, lane, sK, sV, body);
  }
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int r = gq + 8 * hr;
    if (valid && r < G) {
      const int64_t t = i * hq + (int64_t)g * G + r;
      const float inv = 1.f / l[hr];
#pragma unroll
      for (int nt = 0; nt < DH / 8; ++nt) {
        float* o = out + t * DH + nt * 8 + 2 * cq;
        o[0] = acc[nt][2 * hr] * inv;
        o[1] = acc[nt][2 * hr + 1] * inv;
      }
      if (cq == 0) lse_out[t] = m[hr] + __logf(l[hr]);
    }
  }
}

// dK/dV pass: CTA of 4 warps per (64-key tile, kv head, query slice).
constexpr int kKvKeys = 64;
#ifndef LSRM_BWD_QB
#define LSRM_BWD_QB 4
#endif
constexpr int kQB = LSRM_BWD_QB;   // matched queries staged per shared-memory round

template <int DH>
__global__ void LSRM_BWD_BOUNDS(128)
dkdv_mma_kernel(KeySet ks, const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ dob,
                const float* __restrict__ lse, const float* __restrict__ dsum, int64_t nq, int hq,
                int hkv, const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                int n_rows, int tiles_per_row, int n_slices,
                const int64_t* __restrict__ t_offs, const int32_t* __restrict__ t_q,
                float* __restrict__ part_dk, float* __restrict__ part_dv) {
  constexpr int LD = DH + 8;
  constexpr int QB = DH <= 32 ? kQB : 4;   // staging rounds fit the 48 KB static limit
  __shared__ __align__(16) __nv_bfloat16 sKV[2][kKvKeys * LD];
  __shared__ __align__(16) __nv_bfloat16 sQ[QB][16 * LD];   // QB matched queries per round
  __shared__ __align__(16) __nv_bfloat16 sO[QB][16 * LD];
  __shared__ float sL[QB][16], sD[QB][16];
  __shared__ int qlist[128];
  __shared__ int wsum[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mode = ks.mode;
  const int row = mode == 0 ? -1 : (int)(blockIdx.x / tiles_per_row);
  const int tile = mode == 0 ? (int)blockIdx.x : (int)(blockIdx.x % tiles_per_row);
  const int g = blockIdx.y, slice = blockIdx.z;
  const int64_t r_lo = mode == 0 ? 0 : ks.offs[row];
  const int64_t r_hi = mode == 0 ? ks.nk : ks.offs[row + 1];
  const int64_t key0 = r_lo + (int64_t)tile * kKvKeys;
  if (key0 >= r_hi) return;
  const int G = hq / hkv;
  const float scale = 1.0f / sqrtf((float)DH);
  const int64_t kstride = (int64_t)hkv * DH;
  const int gq = lane >> 2, cq = lane & 3;
  // K, V of the tile (rows past the row end zero)
  for (int e = tid; e < kKvKeys * (DH / 8); e += 128) {
    const int r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
    uint4 vk = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
    if (key0 + r < r_hi) {
      const int64_t base = (key0 + r) * kstride + (int64_t)g * DH + c8;
      vk = *reinterpret_cast<const uint4*>(k + base);
      vv = *reinterpret_cast<const uint4*>(v + base);
    }
    *reinterpret_cast<uint4*>(&sKV[0][r * LD + c8]) = vk;
    *reinterpret_cast<uint4*>(&sKV[1][r * LD + c8]) = vv;
  }
  __syncthreads();
  uint32_t ak[DH / 16][4], av[DH / 16][4];
  load_a<DH>(&sKV[0][warp * 16 * LD], lane, ak);
  load_a<DH>(&sKV[1][warp * 16 * LD], lane, av);
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[nt][e] = dv[nt][e] = 0.f;
  // queries that see this row: with a transposed index (t_offs / t_q: per
  // row, its queries in ascending order) this slice's share of the row's
  // list; otherwise scan the slice of all queries and test membership
  const bool listed = t_offs != nullptr && mode != 0;
  int64_t q_lo, q_hi;
  if (listed) {
    const int64_t l0 = t_offs[row], len = t_offs[row + 1] - l0;
    q_lo = l0 + len * slice / n_slices;
    q_hi = l0 + len * (slice + 1) / n_slices;
  } else {
    q_lo = nq * slice / n_slices;
    q_hi = nq * (slice + 1) / n_slices;
  }
  for (int64_t base = q_lo; base < q_hi; base += 128) {
    const int64_t i = listed ? (base + tid < q_hi ? (int64_t)t_q[base + tid] : 0) : base + tid;
    bool match = false;
    if (listed) {
      match = base + tid < q_hi;
    } else if (i < q_hi) {
      if (mode == 0) {
        match = true;
      } else if (mode == 1) {
        const int cnt = ks.count[i];
        for (int s = 0; s < cnt; ++s) match |= ks.rows[i * ks.kmax + s] == row;
      } else {
        match = ks.own_row[i] == row;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, match);
    __syncthreads();   // qlist / wsum of the previous batch fully consumed
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = __popc(bal & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) before += wsum[w];
    const int n_match = wsum[0] + wsum[1] + wsum[2] + wsum[3];
    if (match) qlist[before] = (int)i;   // absolute query index
    __syncthreads();
    // Q / dO rows of the G heads of QB queries (rows >= G zero; lse = +inf ->
    // P = 0), staged through registers: round mb+QB is fetched while round mb
    // is computed
    constexpr int PERQ = QB * 2 * 16 * (DH / 8) / 128;
    static_assert(PERQ * 128 == QB * 2 * 16 * (DH / 8) && QB * 16 <= 128, "staging shape");
    uint4 rq[PERQ];
    float rl = __builtin_huge_valf(), rd = 0.f;
    auto fetch = [&](int mb) {
      const int nb = min(QB, n_match - mb);
#pragma unroll
      for (int p = 0; p < PERQ; ++p) {
        const int e2 = tid + 128 * p;
        const int qb = e2 / (2 * 16 * (DH / 8)), rem = e2 % (2 * 16 * (DH / 8));
        const int which = rem / (16 * (DH / 8)), e = rem % (16 * (DH / 8));
        const int r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
        rq[p] = make_uint4(0, 0, 0, 0);
        if (qb < nb && r < G) {
          const int64_t src = (((int64_t)qlist[mb + qb] * hq) + (int64_t)g * G + r) * DH + c8;
          rq[p] = *reinterpret_cast<const uint4*>((which ? dob : q) + src);
        }
      }
      if (tid < QB * 16) {
        const int qb = tid / 16, h = tid % 16;
        const bool ok = qb < nb && h < G;
        const int64_t t = ok ? (int64_t)qlist[mb + qb] * hq + (int64_t)g * G + h : 0;
        rl = ok ? lse[t] : __builtin_huge_valf();
        rd = ok ? dsum[t] : 0.f;
      }
    };
    if (n_match > 0) fetch(0);
    for (int mb = 0; mb < n_match; mb += QB) {
      const int nb = min(QB, n_match - mb);
#pragma unroll
      for (int p = 0; p < PERQ; ++p) {
        const int e2 = tid + 128 * p;
        const int qb = e2 / (2 * 16 * (DH / 8)), rem = e2 % (2 * 16 * (DH / 8));
        const int which = rem / (16 * (DH / 8)), e = rem % (16 * (DH / 8));
        const int r = e / (DH / 8), c8 = (e % (DH / 8)) * 8;
        *reinterpret_cast<uint4*>((which ? sO[qb] : sQ[qb]) + r * LD + c8) = rq[p];
      }
      if (tid < QB * 16) {
        sL[tid / 16][tid % 16] = rl;
        sD[tid / 16][tid % 16] = rd;
      }
      __syncthreads();
      if (mb + QB < n_match) fetch(mb + QB);   // in flight during this round
      for (int qb = 0; qb < nb; ++qb) {
        uint32_t bq[DH / 16][4], bo[DH / 16][4];
        load_b_nt<DH>(sQ[qb], lane, bq);
        load_b_nt<DH>(sO[qb], lane, bo);
        // S^T, dP^T: 16 keys x 16 heads (two n-tiles of 8 heads)
        float st[2][4], dpt[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) st[nt][e] = dpt[nt][e] = 0.f;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            mma(st[nt], ak[kk], bq[kk][2 * nt], bq[kk][2 * nt + 1]);
            mma(dpt[nt], av[kk], bo[kk][2 * nt], bo[kk][2 * nt + 1]);
          }
        }
        uint32_t ap[4], ads[4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          float p4[4], d4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int h = nt * 8 + 2 * cq + (e & 1);
            const float p = __expf(st[nt][e] * scale - sL[qb][h]);
            p4[e] = p;
            d4[e] = p * (dpt[nt][e] - sD[qb][h]) * scale;
          }
          ap[2 * nt] = pk(p4[0], p4[1]);
          ap[2 * nt + 1] = pk(p4[2], p4[3]);
          ads[2 * nt] = pk(d4[0], d4[1]);
          ads[2 * nt + 1] = pk(d4[2], d4[3]);
        }
        // dV += P^T dO, dK += dS^T Q  (B(k = head, n = dim): transposed loads)
        uint32_t bo2[DH / 16][4], bq2[DH / 16][4];
        load_b_nn<DH>(sO[qb], lane, bo2);
        load_b_nn<DH>(sQ[qb], lane, bq2);
#pragma unroll
        for (int np = 0; np < DH / 16; ++np) {
          mma(dv[2 * np], ap, bo2[np][0], bo2[np][1]);
          mma(dv[2 * np + 1], ap, bo2[np][2], bo2[np][3]);
          mma(dk[2 * np], ads, bq2[np][0], bq2[np][1]);
          mma(dk[2 * np + 1], ads, bq2[np][2], bq2[np][3]);
        }
      }
      __syncthreads();   // staging reused by the next round
    }
  }
  // partials of this warp's 16 keys
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int64_t key = key0 + warp * 16 + gq + 8 * hr;
    if (key < r_hi) {
      const int64_t o = ((int64_t)slice * ks.nk * hkv + key * hkv + g) * DH;
#pragma unroll
      for (int nt = 0; nt < DH / 8; ++nt) {
        const int c = nt * 8 + 2 * cq;
        part_dk[o + c] = dk[nt][2 * hr];
        part_dk[o + c + 1] = dk[nt][2 * hr + 1];
        part_dv[o + c] = dv[nt][2 * hr];
        part_dv[o + c + 1] = dv[nt][2 * hr + 1];
      }
    }
  }
}

__global__ void reduce_kernel(const float* __restrict__ pk_, const float* __restrict__ pv_,
                              int n_slices, int64_t n, float* __restrict__ dk,
                              float* __restrict__ dv) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int s = 0; s < n_slices; ++s) {
      a += pk_[(int64_t)s * n + e];
      b += pv_[(int64_t)s * n + e];
    }
    dk[e] += a;
    dv[e] += b;
  }
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

__global__ void transpose_keys_kernel(const int32_t* __restrict__ rows,
                                      const int32_t* __restrict__ count, int64_t nq, int kmax,
                                      uint64_t* __restrict__ keys) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nq * kmax) return;
  const int64_t i = e / kmax;
  const int s = (int)(e % kmax);
  const uint64_t r = s < count[i] ? (uint64_t)(uint32_t)rows[e] : 0xffffffffull;
  keys[e] = (r << 32) | (uint64_t)i;
}

// offs[r] = first sorted position with row >= r (binary search)
__global__ void transpose_offsets_kernel(const uint64_t* __restrict__ sorted, int64_t n,
                                         int n_rows, int64_t* __restrict__ offs) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > n_rows) return;
  const uint64_t key = (uint64_t)(uint32_t)r << 32;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < key) lo = mid + 1; else hi = mid;
  }
  offs[r] = lo;
}

__global__ void transpose_fill_kernel(const uint64_t* __restrict__ sorted, int64_t n,
                                      int32_t* __restrict__ q_out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) q_out[e] = (int32_t)(sorted[e] & 0xffffffffull);
}

}  // namespace bwdmma
}  // namespace lsrm

using namespace lsrm;
using namespace lsrm::bwdmma;

extern "C" {

// Same contract as lsrm_attention_bwd_f32 (workspace: lsrm_attention_bwd_workspace)
// with bf16 copies of q, dO [nq, hq, dh] and k, v [nk, hkv, dh] for the MMAs;
// dO and O in f32 give D = rowsum(dO * O).  head_dim in {16, 32, 64},
// hq / hkv <= 16.
int lsrm_attention_bwd_mma(int mode, const void* q_bf16, const void* dO_bf16, const float* dO,
                           const float* O, const float* lse_in, int64_t nq, int hq, int hkv, int dh,
                           const void* k_bf16, const void* v_bf16, int64_t nk,
                           const int64_t* block_offsets, int n_rows, int max_row_keys,
                           const int32_t* rows, const int32_t* count, int kmax_rows,
                           const int32_t* own_row, int n_slices, const int64_t* t_offs,
                           const int32_t* t_q, float* dq, float* dk, float* dv,
                           void* workspace, size_t ws_bytes, void* stream) {
  LSRM_REQUIRE(mode >= 0 && mode <= 2, "attention_bwd: mode must be 0 (cmp), 1 (sel), 2 (win)");
  LSRM_REQUIRE(hq % hkv == 0 && hq / hkv <= 16, "attention_bwd_mma: group size must be <= 16");
  LSRM_REQUIRE((t_offs == nullptr) == (t_q == nullptr), "attention_bwd_mma: t_offs and t_q go together");
  LSRM_REQUIRE(n_slices >= 1 && n_slices <= 65535, "attention_bwd: n_slices out of range");
  LSRM_REQUIRE(mode == 0 || (block_offsets && n_rows >= 1 && max_row_keys >= 1),
               "attention_bwd: sel/win need block offsets");
  const size_t need = 2 * align256((size_t)nq * hq * sizeof(float)) +
                      2 * align256((size_t)n_slices * nk * hkv * dh * sizeof(float));
  LSRM_REQUIRE(ws_bytes >= need, "attention_bwd: workspace too small");
  if (nq == 0 || nk == 0) return LSRM_OK;
  char* ws = (char*)workspace;
  float* lse = (float*)ws;
  float* dsum = (float*)(ws + align256((size_t)nq * hq * sizeof(float)));
  float* pk_ = (float*)(ws + 2 * align256((size_t)nq * hq * sizeof(float)));
  float* pv_ = (float*)((char*)pk_ + align256((size_t)n_slices * nk * hkv * dh * sizeof(float)));
  cudaStream_t st = as_stream(stream);
  KeySet ks{mode, nk, block_offsets, rows, count, kmax_rows, own_row};
  const unsigned g1 = mode == 0 ? (unsigned)(ceil_div(nq, kDqWarps) * hkv)
                                : (unsigned)ceil_div(nq * hkv, kDqWarps);
  const int tiles_per_row = mode == 0 ? 0 : (int)ceil_div(max_row_keys, kKvKeys);
  const dim3 g2(mode == 0 ? (unsigned)ceil_div(nk, kKvKeys) : (unsigned)(n_rows * tiles_per_row),
                (unsigned)hkv, (unsigned)n_slices);
  LSRM_CUDA(cudaMemsetAsync(pk_, 0, (size_t)n_slices * nk * hkv * dh * sizeof(float), st));
  LSRM_CUDA(cudaMemsetAsync(pv_, 0, (size_t)n_slices * nk * hkv * dh * sizeof(float), st));
  const __nv_bfloat16 *qb = (const __nv_bfloat16*)q_bf16, *ob = (const __nv_bfloat16*)dO_bf16,
                      *kb = (const __nv_bfloat16*)k_bf16, *vb = (const __nv_bfloat16*)v_bf16;
#define LSRM_BWD_MMA_CASE(D)                                                                   \
  case D:                                                                                      \
    if (mode == 0)                                                                             \
      dq_mma_kernel<D, true><<<g1, 32 * kDqWarps, 0, st>>>(ks, qb, ob, dO, O, lse_in, nq, hq,  \
                                                           hkv, kb, vb, dq, lse, dsum);        \
    else                                                                                       \
      dq_mma_kernel<D, false><<<g1, 32 * kDqWarps, 0, st>>>(ks, qb, ob, dO, O, lse_in, nq, hq, \
                                                            hkv, kb, vb, dq, lse, dsum);       \
    dkdv_mma_kernel<D><<<g2, 128, 0, st>>>(ks, qb, ob, lse, dsum, nq, hq, hkv, kb, vb, n_rows,  \
                                           tiles_per_row, n_slices, t_offs, t_q, pk_, pv_);     \
    break;
  switch (dh) {
    LSRM_BWD_MMA_CASE(16)
    LSRM_BWD_MMA_CASE(32)
    LSRM_BWD_MMA_CASE(64)
    default:
      return set_error(LSRM_E_CONFIG, "attention_bwd_mma: head_dim %d not in {16,32,64}", dh);
  }
#undef LSRM_BWD_MMA_CASE
  LSRM_LAUNCHED();
  const int64_t n = nk * hkv * dh;
  const unsigned g3 = (unsigned)(ceil_div(n, 256) < 148 * 8 ? ceil_div(n, 256) : 148 * 8);
  reduce_kernel<<<g3, 256, 0, st>>>(pk_, pv_, n_slices, n, dk, dv);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

// Transposed routing index: for every kv row, the queries whose resolved
// selection holds it, in ascending query order (deterministic: one stable
// radix sort of (row, query) keys).  offs [n_rows + 1], q [sum(count)].
size_t lsrm_transpose_rows_workspace(int64_t nq, int kmax) {
  size_t tmp = 0;
  const int64_t n = nq * kmax;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                 (int)n);
  return 2 * align256((size_t)n * sizeof(uint64_t)) + align256(sizeof(int)) + align256(tmp);
}

int lsrm_transpose_rows(const int32_t* rows, const int32_t* count, int64_t nq, int kmax,
                        int n_rows, int64_t* offs, int32_t* q_out, void* workspace,
                        size_t ws_bytes, void* stream) {
  LSRM_REQUIRE(ws_bytes >= lsrm_transpose_rows_workspace(nq, kmax),
               "transpose_rows: workspace too small");
  LSRM_REQUIRE(nq * (int64_t)kmax < (1ll << 31), "transpose_rows: too many entries");
  cudaStream_t st = as_stream(stream);
  const int64_t n = nq * kmax;
  char* ws = (char*)workspace;
  uint64_t* keys = (uint64_t*)ws;
  uint64_t* sorted = (uint64_t*)(ws + align256((size_t)n * sizeof(uint64_t)));
  void* tmp = ws + 2 * align256((size_t)n * sizeof(uint64_t)) + align256(sizeof(int));
  size_t tmp_bytes = ws_bytes - (2 * align256((size_t)n * sizeof(uint64_t)) + align256(sizeof(int)));
  // entry (i, s): key = row << 32 | i; unused slots sort last (row = all ones)
  transpose_keys_kernel<<<(unsigned)ceil_div(n > 0 ? n : 1, 256), 256, 0, st>>>(rows, count, nq,
                                                                               kmax, keys);
  LSRM_LAUNCHED();
  if (n > 0 &&
      cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, (int)n, 0, 64, st) !=
          cudaSuccess)
    return set_error(LSRM_E_CUDA, "transpose_rows: radix sort failed");
  transpose_offsets_kernel<<<(unsigned)ceil_div(n_rows + 1, 256), 256, 0, st>>>(sorted, n, n_rows,
                                                                              offs);
  transpose_fill_kernel<<<(unsigned)ceil_div(n > 0 ? n : 1, 256), 256, 0, st>>>(sorted, n, q_out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

// Forward of one branch (mode 0 cmp, 1 sel, 2 win) for training: bf16 q
// [nq, hq, dh], k / v [nk, hkv, dh]; writes out f32 [nq, hq, dh] and lse
// [nq, hq] (natural log).  head_dim in {16, 32, 64}, hq / hkv <= 16.
int lsrm_attention_fwd_mma(int mode, const void* q_bf16, int64_t nq, int hq, int hkv, int dh,
                           const void* k_bf16, const void* v_bf16, int64_t nk,
                           const int64_t* block_offsets, const int32_t* rows,
                           const int32_t* count, int kmax_rows, const int32_t* own_row,
                           float* out, float* lse, void* stream) {
  LSRM_REQUIRE(mode >= 0 && mode <= 2, "attention_fwd_mma: mode must be 0, 1 or 2");
  LSRM_REQUIRE(hq % hkv == 0 && hq / hkv <= 16, "attention_fwd_mma: group size must be <= 16");
  LSRM_REQUIRE(mode == 0 || block_offsets, "attention_fwd_mma: sel/win need block offsets");
  if (nq == 0) return LSRM_OK;
  LSRM_REQUIRE(nk > 0, "attention over an empty key set");
  KeySet ks{mode, nk, block_offsets, rows, count, kmax_rows, own_row};
  const unsigned g1 = mode == 0 ? (unsigned)(ceil_div(nq, kDqWarps) * hkv)
                                : (unsigned)ceil_div(nq * hkv, kDqWarps);
  cudaStream_t st = as_stream(stream);
  const __nv_bfloat16 *qb = (const __nv_bfloat16*)q_bf16, *kb = (const __nv_bfloat16*)k_bf16,
                      *vb = (const __nv_bfloat16*)v_bf16;
#define LSRM_FWD_MMA(D)                                                                      \
  if (mode == 0)                                                                             \
    fwd_mma_kernel<D, true><<<g1, 32 * kDqWarps, 0, st>>>(ks, qb, nq, hq, hkv, kb, vb, out,  \
                                                          lse);                              \
  else                                                                                       \
    fwd_mma_kernel<D, false><<<g1, 32 * kDqWarps, 0, st>>>(ks, qb, nq, hq, hkv, kb, vb, out, \
                                                           lse);
  switch (dh) {
    case 16: LSRM_FWD_MMA(16) break;
    case 32: LSRM_FWD_MMA(32) break;
    case 64: LSRM_FWD_MMA(64) break;
    default:
      return set_error(LSRM_E_CONFIG, "attention_fwd_mma: head_dim %d not in {16,32,64}", dh);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
