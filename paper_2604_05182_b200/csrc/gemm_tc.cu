// Grouped bf16 GEMM on the 5th-gen tensor cores: TMA-staged operands
// (cp.async.bulk.tensor, SWIZZLE_128B), tcgen05.mma with the accumulator in
// TMEM, fused epilogue (bias, exact-erf gelu, residual, bf16 or f32 out).
//
// Replaces the library GEMMs of the layer's hot path: the per-stream fused
// projection (q | gate logits + bias | k | v of every use that reads the
// stream; reference lsrm/nsa_attention.py:303-307 q/k/v `affine`, :266-273
// gate GEMM, built on lsrm/tensor_core.py:100-116), the W_o projection of
// each use (nsa_attention.py:284) and the Stage-2 FFN
// (lsrm/recon_pipeline.py:497-512).
//
// Problem g:  C_g[m,n] = epi(A_g[m,k] . Wt_g[n,k]^T)
//   A   bf16 [m,k] row-major (K contiguous, row stride lda)
//   Wt  bf16 [n,k] (the weight TRANSPOSED, K contiguous, row stride ldb):
//       both K-major, the canonical UMMA layout; or, per problem, either
//       operand MN-major (A^T [k,m] / W [k,n] as stored, flags A_MN / B_MN):
//       TMA boxes of 64 (MN) x 64 (K) with SWIZZLE_128B, UMMA descriptors
//       with LBO = 8 KB between 64-wide MN atoms and SBO = 1 KB between
//       8-row K groups, the instruction descriptor's transpose bits set
//   epi(acc) = act(acc + bias[n]) (+ res[m,n])  -> bf16 or f32
//
// One persistent launch runs every problem of the group: 148 CTAs (one per
// SM) walk a static tile sequence (tiles of 128 x 256, N fastest inside a
// problem so neighbouring CTAs share the A tile in L2).  Warp roles:
//   warp 0  TMA producer (one lane): A {64,128} and B {64,256} boxes into a
//           4-stage ring (48 KB per stage), full/empty mbarriers
//   warp 1  MMA issuer (one lane): 4 x tcgen05.mma 128x256x16 per stage,
//           tcgen05.commit frees the stage; accumulators double-buffered in
//           TMEM (2 x 256 columns) so the epilogue of tile i overlaps the
//           main loop of tile i+1
//   warp 2  TMEM allocator
//   warps 4-11 epilogue: thread = TMEM lane = one output row, two warps per
//           lane quadrant (column halves); 32-column tcgen05.ld pieces, bias /
//           gelu / residual in fp32, 16-byte stores
// Deterministic: fixed K order per output element, no atomics.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tcgen05.cuh"

namespace lsrm {
namespace gemm {

using namespace lsrm::tc;

constexpr int BM = 128, BN = 256, BK = 64, kAccStages = 2;
constexpr int kABytes = BM * BK * 2;
constexpr int kEpiWarps = 8;                 // two per TMEM lane quadrant
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kMaxProblems = 32;   // ~15 KB of kernel parameters (limit 32 KB)

struct Prob {
  int64_t m, n, k;
  void* c;
  int64_t ldc;
  const void* bias;
  const void* res;
  int64_t ldr;
  int flags;
  int tiles_n;
  int64_t tile_begin;
};

struct __align__(64) Params {
  CUtensorMap ta[kMaxProblems];
  CUtensorMap tb[kMaxProblems];
  CUtensorMap tc[kMaxProblems];   // C, TMA-store boxes of 64 B x 32 rows (SWIZZLE_64B)
  Prob p[kMaxProblems];
  int n_prob;
  int64_t total_tiles;
};

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}

// MN-major SW128 operand: 64-element MN atoms 8 KB apart (one TMA box each),
// 8-row K groups 1 KB apart; a 16-element K step advances 2 KB
__device__ __forceinline__ uint64_t sdesc_sw128_mn(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(8192 >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void locate(const Params& P, int64_t t, int& g, int64_t& mt, int& nt) {
  g = 0;
  while (g + 1 < P.n_prob && t >= P.p[g + 1].tile_begin) ++g;
  const int64_t r = t - P.p[g].tile_begin;
  mt = r / P.p[g].tiles_n;
  nt = (int)(r % P.p[g].tiles_n);
}

// 32 accumulator columns of one row (thread = row = row0 + lane) -> bias /
// gelu / residual in fp32 -> TMA store of the warp's 32 x 32 piece.
__device__ __forceinline__ void store_piece(const Prob& pb, const void* tmap_c, int64_t row0,
                                            int lane, int64_t col0, const uint32_t* r,
                                            uint8_t* stage, int& sub) {
  const int64_t row = row0 + lane;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  const int ncols = (int)lmin(32, pb.n - col0);
  if (pb.bias) {
    if (pb.flags & LSRM_GEMM_BIAS_F32) {
      const float4* b4 = reinterpret_cast<const float4*>((const float*)pb.bias + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j * 4 < ncols) {
          float4 b = __ldg(b4 + j);
          v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
        }
      }
    } else {
      const uint4* b8 = reinterpret_cast<const uint4*>((const __nv_bfloat16*)pb.bias + col0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j * 8 < ncols) {
          uint4 b = __ldg(b8 + j);
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 f = __bfloat1622float2(h[e]);
            v[8 * j + 2 * e] += f.x;
            v[8 * j + 2 * e + 1] += f.y;
          }
        }
      }
    }
  }
  if (pb.flags & LSRM_GEMM_GELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
  }
  if (pb.res && row < pb.m) {
    if (pb.flags & LSRM_GEMM_RES_F32) {
      const float4* r4 = reinterpret_cast<const float4*>((const float*)pb.res + row * pb.ldr + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j * 4 < ncols) {
          float4 b = r4[j];
          v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
        }
      }
    } else {
      const uint4* r8 =
          reinterpret_cast<const uint4*>((const __nv_bfloat16*)pb.res + row * pb.ldr + col0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j * 8 < ncols) {
          uint4 b = r8[j];
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 f = __bfloat1622float2(h[e]);
            v[8 * j + 2 * e] += f.x;
            v[8 * j + 2 * e + 1] += f.y;
          }
        }
      }
    }
  }
  // stage the piece in this warp's shared buffers (64-byte rows, 16-byte
  // chunks XOR-swizzled like CU_TENSOR_MAP_SWIZZLE_64B) and TMA-store it:
  // bf16 = one 32 x 32 box, f32 = two 32 x 16 boxes.  A buffer is rewritten
  // only after the bulk store issued from it two sub-pieces ago has read it.
  const bool f32 = pb.flags & LSRM_GEMM_OUT_F32;
  const int n_sub = f32 ? 2 : 1;
  for (int h = 0; h < n_sub; ++h) {
    uint32_t w[16];
    if (f32) {
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j] = __float_as_uint(v[16 * h + j]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
    }
    uint8_t* buf = stage + (sub & 1) * 2048;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    const int sw = (lane >> 1) & 3;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<uint4*>(buf + lane * 64 + ((c ^ sw) << 4)) =
          make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap_c),
          "r"((int32_t)(col0 + 16 * h)), "r"((int32_t)row0), "r"(smem_u32(buf))
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    ++sub;
  }
}

// CG = 1: one CTA per 128 x 256 tile.  CG = 2: a CTA pair (cluster of 2 on
// one TPC) per 256 x 256 tile with tcgen05.mma.cta_group::2: each CTA stages
// its 128 rows of A and its half (128 rows) of Bt, the leader CTA issues the
// M = 256 MMAs that read both CTAs' shared memory and write both CTAs' TMEM
// (rows 0-127 in the leader's, 128-255 in the peer's).  Both CTAs' TMA
// complete on the leader's full barrier; the MMA commits multicast to both
// CTAs' empty / acc_full barriers; both CTAs' epilogues release the
// leader's acc_empty barrier.
template <int CG>
struct Cfg {
  static constexpr int kBRows = BN / CG;                 // Bt rows staged per CTA
  static constexpr int kStageBytes = kABytes + kBRows * BK * 2;
  static constexpr int kStages = CG == 1 ? 4 : 6;
  static constexpr int kStagingBytes = kEpiWarps * 2 * 2048;   // epilogue TMA-store buffers
  static constexpr int kSmem = kStages * kStageBytes + kStagingBytes + 1024 + 256;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
// shared::cluster address of the same object in the pair's leader CTA
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  return smem_u32(p) & 0xFEFFFFFFu;
}

template <int CG>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(const __grid_constant__ Params P) {
  using C = Cfg<CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + C::kStagingBytes);
  uint64_t* full = bars;                               // [kStages]
  uint64_t* empty = bars + C::kStages;                 // [kStages]
  uint64_t* acc_full = bars + 2 * C::kStages;          // [kAccStages]
  uint64_t* acc_empty = bars + 2 * C::kStages + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 2 * kAccStages);
  auto stage_a = [&](int s) { return smem + s * C::kStageBytes; };
  auto stage_b = [&](int s) { return smem + s * C::kStageBytes + kABytes; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const int64_t unit0 = blockIdx.x / CG, n_units = gridDim.x / CG;
  if (warp == 0 && lane == 0) {
    for (int g = 0; g < P.n_prob; ++g) {
      prefetch_tmap(&P.ta[g]);
      prefetch_tmap(&P.tb[g]);
      prefetch_tmap(&P.tc[g]);
    }
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kAccStages; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kEpiWarps * CG);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      tmem_alloc(tmem_slot, BN * kAccStages);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(BN * kAccStages)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_before_sync();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (each CTA: its A rows, its half of Bt) ----------------
    if (elect_one_sync()) {
      uint32_t stage = 0, phase = 0;
      for (int64_t t = unit0; t < P.total_tiles; t += n_units) {
        int g, nt;
        int64_t mt;
        locate(P, t, g, mt, nt);
        const int kb_n = (int)((P.p[g].k + BK - 1) / BK);
        const int32_t arow = (int32_t)(mt * BM * CG + rank * BM);
        const int32_t brow = (int32_t)(nt * BN + rank * C::kBRows);
        const bool a_mn = P.p[g].flags & LSRM_GEMM_A_MN, b_mn = P.p[g].flags & LSRM_GEMM_B_MN;
        // one box: K-major {BK, rows} at (k, row); MN-major {64, BK} at (row, k)
        auto load = [&](uint8_t* dst, const CUtensorMap* map, int32_t x, int32_t y,
                        uint64_t* bar_local, uint32_t bar_cluster) {
          if constexpr (CG == 1) {
            tma_load_2d(dst, map, x, y, bar_local);
          } else {
            asm volatile(
                "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
                "l"(map), "r"(x), "r"(y), "r"(bar_cluster)
                : "memory");
          }
        };
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (CG == 1) {
            mbar_expect_tx(&full[stage], C::kStageBytes);
          } else {
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * C::kStageBytes);
          }
          const uint32_t fb = CG == 1 ? 0u : leader_addr(&full[stage]);
          if (a_mn) {
#pragma unroll
            for (int h = 0; h < BM / 64; ++h)
              load(stage_a(stage) + h * 8192, &P.ta[g], arow + 64 * h, kb * BK, &full[stage], fb);
          } else {
            load(stage_a(stage), &P.ta[g], kb * BK, arow, &full[stage], fb);
          }
          if (b_mn) {
#pragma unroll
            for (int h = 0; h < C::kBRows / 64; ++h)
              load(stage_b(stage) + h * 8192, &P.tb[g], brow + 64 * h, kb * BK, &full[stage], fb);
          } else {
            load(stage_b(stage), &P.tb[g], kb * BK, brow, &full[stage], fb);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (leader CTA) ----------------
    const uint32_t idesc0 = idesc_bf16(BM * CG, BN, 0);
    uint32_t stage = 0, phase = 0;
    int it = 0;
    for (int64_t t = unit0; t < P.total_tiles; t += n_units, ++it) {
      int g, nt;
      int64_t mt;
      locate(P, t, g, mt, nt);
      const int kb_n = (int)((P.p[g].k + BK - 1) / BK);
      const bool a_mn = P.p[g].flags & LSRM_GEMM_A_MN, b_mn = P.p[g].flags & LSRM_GEMM_B_MN;
      // transpose bits of the instruction descriptor: 15 = A, 16 = B MN-major
      const uint32_t idesc = idesc0 | (a_mn ? 1u << 15 : 0u) | (b_mn ? 1u << 16 : 0u);
      // per 16-element K step, in 16-byte descriptor units: K-major +32 B, MN-major +2 KB
      const uint64_t ka = a_mn ? 128 : 2, kbs = b_mn ? 128 : 2;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      tc_after_sync();
      const uint32_t d_tmem = tmem + acc * BN;
      for (int kb = 0; kb < kb_n; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_after_sync();
        if (elect_one_sync()) {
          const uint64_t da = a_mn ? sdesc_sw128_mn(smem_u32(stage_a(stage)))
                                   : sdesc_sw128(smem_u32(stage_a(stage)));
          const uint64_t db = b_mn ? sdesc_sw128_mn(smem_u32(stage_b(stage)))
                                   : sdesc_sw128(smem_u32(stage_b(stage)));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {   // +32 bytes per 16-element K step
            if constexpr (CG == 1) {
              mma_bf16(d_tmem, da + ka * k, db + kbs * k, idesc, (kb | k) != 0);
            } else {
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
                  "l"(da + ka * k), "l"(db + kbs * k), "r"(idesc), "r"((uint32_t)((kb | k) != 0)));
            }
          }
          if constexpr (CG == 1) {
            mma_commit(&empty[stage]);
            if (kb == kb_n - 1) mma_commit(&acc_full[acc]);
          } else {
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                " [%0], %1;" ::"r"(smem_u32(&empty[stage])), "h"((uint16_t)3)
                : "memory");
            if (kb == kb_n - 1)
              asm volatile(
                  "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                  " [%0], %1;" ::"r"(smem_u32(&acc_full[acc])), "h"((uint16_t)3)
                  : "memory");
          }
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (each CTA: its 128 rows of the tile) ----------------
    const int wq = warp & 3;                       // TMEM lane quadrant
    const int half = (warp - 4) >> 2;              // column half of the tile
    constexpr int kPieces = BN / 32 / (kEpiWarps / 4);
    uint8_t* my_stage = staging + (warp - 4) * 2 * 2048;
    int sub = 0;
    int it = 0;
    for (int64_t t = unit0; t < P.total_tiles; t += n_units, ++it) {
      int g, nt;
      int64_t mt;
      locate(P, t, g, mt, nt);
      const Prob& pb = P.p[g];
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&acc_full[acc], acc_phase);
      tc_after_sync();
      const int64_t row0 = mt * BM * CG + rank * BM + wq * 32;
      const int64_t col_base = (int64_t)nt * BN + half * kPieces * 32;
      const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + acc * BN + half * kPieces * 32;
      const int n_pieces = (int)lmax(0, lmin(kPieces, (pb.n - col_base + 31) / 32));
      uint32_t r[32];
      if (n_pieces == 0) {            // this half lies beyond n: nothing to read
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1)
            mbar_arrive(&acc_empty[acc]);
          else
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                             leader_addr(&acc_empty[acc]))
                         : "memory");
        }
      }
      for (int pc = 0; pc < n_pieces; ++pc) {
        tmem_ld32(taddr + pc * 32, r);
        tmem_wait_ld();
        if (pc == n_pieces - 1) {     // accumulator drained: hand it back to the MMA warp
          tc_before_sync();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1)
              mbar_arrive(&acc_empty[acc]);
            else
              asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                               leader_addr(&acc_empty[acc]))
                           : "memory");
          }
        }
        store_piece(pb, &P.tc[g], row0, lane, col_base + pc * 32, r, my_stage, sub);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_before_sync();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  if (warp == 2) {
    if constexpr (CG == 1)
      tmem_dealloc(tmem, BN * kAccStages);
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(BN * kAccStages)
                   : "memory");
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int make_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize,
                    int64_t inner, int64_t outer, int64_t ld, int box_inner, int box_outer,
                    CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return set_error(LSRM_E_CUDA, "gemm_tc: cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esize)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(LSRM_E_CUDA, "gemm_tc: tensor map encode failed (%d)", (int)r);
  return LSRM_OK;
}

}  // namespace gemm
}  // namespace lsrm

using namespace lsrm;
using namespace lsrm::gemm;

template <int CG>
static int launch(const Params& p, int64_t units, void* stream) {
  int dev = 0, sms = 0;
  LSRM_CUDA(cudaGetDevice(&dev));
  LSRM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  LSRM_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg<CG>::kSmem));
  const int64_t max_units = sms / CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((units < max_units ? units : max_units) * CG));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg<CG>::kSmem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LSRM_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<CG>, p));
  LSRM_LAUNCHED();
  return LSRM_OK;
}

// CTA-pair tiles (cta_group::2) by default; LSRM_GEMM_CG=1 selects one CTA
// per 128 x 256 tile.
static int gemm_cg() {
  static int cg = [] {
    const char* e = getenv("LSRM_GEMM_CG");
    return (e && e[0] == '1') ? 1 : 2;
  }();
  return cg;
}

extern "C" int lsrm_gemm_tc(const lsrm_gemm_problem* probs, int n_problems, void* stream) {
  const int cg = gemm_cg();
  LSRM_REQUIRE(n_problems >= 0 && n_problems <= kMaxProblems,
               "gemm_tc: 0..%d problems per launch (got %d)", kMaxProblems, n_problems);
  Params p;                   // built per call on the host, passed by value
  memset(&p, 0, sizeof(p));
  int64_t tiles = 0;
  int n = 0;
  for (int i = 0; i < n_problems; ++i) {
    const lsrm_gemm_problem& q = probs[i];
    LSRM_REQUIRE(q.m >= 0 && q.n >= 0 && q.k >= 0, "gemm_tc: negative size");
    if (q.m == 0 || q.n == 0) continue;
    LSRM_REQUIRE(q.k > 0, "gemm_tc: k must be positive");
    const bool a_mn = q.flags & LSRM_GEMM_A_MN, b_mn = q.flags & LSRM_GEMM_B_MN;
    LSRM_REQUIRE(((a_mn && b_mn) || q.k % 8 == 0) && q.n % 8 == 0 && q.lda % 8 == 0 &&
                     q.ldb % 8 == 0 && q.ldc % 8 == 0 && (q.res == nullptr || q.ldr % 8 == 0),
                 "gemm_tc: k, n and every row stride must be multiples of 8 elements");
    LSRM_REQUIRE(q.lda >= (a_mn ? q.m : q.k) && q.ldb >= (b_mn ? q.n : q.k) && q.ldc >= q.n,
                 "gemm_tc: row stride smaller than the row");
    const uintptr_t al = (uintptr_t)q.a | (uintptr_t)q.bt | (uintptr_t)q.c |
                         (uintptr_t)q.bias | (uintptr_t)q.res;
    LSRM_REQUIRE((al & 15) == 0, "gemm_tc: pointers must be 16-byte aligned");
    const bool c32 = q.flags & LSRM_GEMM_OUT_F32;
    int rc = a_mn ? make_map(&p.ta[n], q.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q.m, q.k, q.lda,
                             64, BK, CU_TENSOR_MAP_SWIZZLE_128B)
                  : make_map(&p.ta[n], q.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q.k, q.m, q.lda,
                             BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!rc)
      rc = b_mn ? make_map(&p.tb[n], q.bt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q.n, q.k, q.ldb,
                           64, BK, CU_TENSOR_MAP_SWIZZLE_128B)
                : make_map(&p.tb[n], q.bt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q.k, q.n, q.ldb,
                           BK, BN / cg, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!rc)
      rc = make_map(&p.tc[n], q.c, c32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                    c32 ? 4 : 2, q.n, q.m, q.ldc, c32 ? 16 : 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
    Prob& pb = p.p[n];
    pb.m = q.m; pb.n = q.n; pb.k = q.k;
    pb.c = q.c; pb.ldc = q.ldc;
    pb.bias = q.bias; pb.res = q.res; pb.ldr = q.ldr;
    pb.flags = q.flags;
    pb.tiles_n = (int)ceil_div(q.n, BN);
    pb.tile_begin = tiles;
    tiles += ceil_div(q.m, BM * cg) * pb.tiles_n;
    ++n;
  }
  if (!tiles) return LSRM_OK;
  p.n_prob = n;
  p.total_tiles = tiles;
  return cg == 1 ? launch<1>(p, tiles, stream) : launch<2>(p, tiles, stream);
}
