// Fused bf16 three-branch NSA attention on the 5th-gen tensor cores
// (tcgen05.mma + TMEM accumulators + bulk-async (TMA engine) K/V staging),
// with the sigmoid-gated branch merge in the epilogue.
//
// Replaces, fused: cmp_attention / sel_attention / win_attention and the
// gated sum of combine_nsa_branches (lsrm/nsa_attention.py:84-112,157-207,
// 266-284).  The W_o projection stays a plain GEMM.
//
// Work item = (query tile, kv head).  A query tile is up to T = 128/G
// consecutive tokens of ONE query block (block-major order), and its MMA
// M-dimension is the 128 rows (token, q-head-in-group) sharing kv head h.
// Every branch streams key chunks of <= 128 keys:
//   cmp : all compressed rows (one per occupied KV block),
//   sel : the sorted union of the tile tokens' selected blocks; a row only
//         sees the blocks ITS token selected (others masked to -inf),
//   win : the tile's own block (self uses).
// Per chunk: bulk-async copy K,V (each KV block is one contiguous 16-row
// padded segment in the interleaved layout) -> S = Q K^T (TMEM) -> masked
// online softmax, one thread per TMEM lane/row -> P (bf16, smem) -> O_part =
// P V (TMEM) -> rescale-accumulate in registers.  The branch outputs are
// normalised, gated by sigmoid(gate logits) and summed in registers; one
// bf16 row of the merged [nq, hq*dh] tensor is written per thread.
//
// SMEM operand layout (all operands): 8x8 "core matrices" of 128 contiguous
// bytes, SWIZZLE_NONE canonical layouts (cute mma_sm100_desc.hpp):
//   K-major  Q, K, P : element (row, k) at (row/8)*RS + (k/8)*64 + (row%8)*8 + k%8
//   MN-major V       : the same storage read with N = head dim, K = keys.
#include "common.cuh"

namespace lsrm {
namespace tc {

constexpr int kM = 128;        // MMA rows per tile
constexpr int kNK = 128;       // keys per chunk (= TMEM S columns)
constexpr int kThreads = 128;
constexpr int kTmemCols = 256;
constexpr int kMaxEnt = 256;   // tile tokens * selected rows
constexpr int kMaxPieces = kNK / 16;

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, Blackwell version bit.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32.
__device__ __forceinline__ uint32_t idesc_bf16(int m, int n, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 16 consecutive f32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

struct Params {
  const __nv_bfloat16* q;
  int64_t ld_q;
  int64_t nq;
  int hq, hkv;
  const __nv_bfloat16* k_il;
  const __nv_bfloat16* v_il;
  const int64_t* pad_off;   // [B+1] padded row offsets (multiples of 16)
  const int64_t* kv_off;    // [B+1] real token offsets
  int64_t n_rows_pad;
  const __nv_bfloat16* kc_il;
  const __nv_bfloat16* vc_il;
  int64_t n_blocks;
  const int32_t* tiles;
  int64_t n_tiles;
  const int32_t* rows;
  const int32_t* count;
  int kmax;
  const __nv_bfloat16* gl;
  int64_t ld_gl, gcol0;
  const float* gbias;
  int n_gates;
  __nv_bfloat16* out;
};

struct Piece {
  int seg;        // segment index (union slot for sel, 0 otherwise)
  int col;        // first chunk column
  int ncols;      // multiple of 16
  int nvalid;     // valid keys at the start of the piece
  int64_t src;    // first padded source row
};

template <int DH>
struct Smem {
  __nv_bfloat16 q[kM * DH];
  __nv_bfloat16 k[kNK * DH];
  __nv_bfloat16 v[kNK * DH];
  __nv_bfloat16 p[kM * kNK];
  int32_t ent[kMaxEnt];     // selected rows of the tile tokens, [t][kmax]
  int32_t uni[kMaxEnt];     // sorted union of selected rows
  uint8_t uniq[kMaxEnt];
  Piece pieces[kMaxPieces];
  int8_t grp_piece[kNK / 16];
  int n_pieces, n_cols, n_uni, cur_seg;
  int64_t cur_off;
  uint64_t bar_kv, bar_mma;
  uint32_t tmem_base;
};

template <int DH>
__global__ void __launch_bounds__(kThreads, 1) nsa_fused_kernel(Params P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem<DH>& S = *reinterpret_cast<Smem<DH>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int G = P.hq / P.hkv, T = kM / G;
  const int64_t item = blockIdx.x;
  const int tile = (int)(item / P.hkv), h = (int)(item % P.hkv);
  const int q_first = P.tiles[4 * tile], q_cnt = P.tiles[4 * tile + 1],
            own = P.tiles[4 * tile + 2];
  const int t = tid / G, g = tid % G;
  const bool row_ok = t < q_cnt;
  const int64_t tok = (int64_t)q_first + t;
  const int d_model = P.hq * DH;
  const int head = h * G + g;

  if (tid == 0) {
    mbar_init(&S.bar_kv, 1);
    mbar_init(&S.bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Q tile -> smem (K-major core-matrix layout), zero rows past the tile.
  for (int i = tid; i < kM * (DH / 8); i += kThreads) {
    int m = i / (DH / 8), cc = i % (DH / 8);
    int tt = m / G, gg = m % G;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (tt < q_cnt)
      v = *reinterpret_cast<const uint4*>(P.q + (int64_t)(q_first + tt) * P.ld_q + (h * G + gg) * DH +
                                          cc * 8);
    *reinterpret_cast<uint4*>(&S.q[(m / 8) * (8 * DH) + cc * 64 + (m % 8) * 8]) = v;
  }
  // selected rows of the tile tokens and their sorted union
  const int n_ent = T * P.kmax;
  for (int i = tid; i < n_ent; i += kThreads) {
    int tt = i / P.kmax, s = i % P.kmax;
    int r = -1;
    if (tt < q_cnt && s < P.count[q_first + tt]) r = P.rows[(int64_t)(q_first + tt) * P.kmax + s];
    S.ent[i] = r;
  }
  __syncthreads();
  for (int i = tid; i < n_ent; i += kThreads) {
    int r = S.ent[i];
    bool u = r >= 0;
    for (int j = 0; j < i && u; ++j) u = S.ent[j] != r;
    S.uniq[i] = u;
  }
  __syncthreads();
  for (int i = tid; i < n_ent; i += kThreads) {
    if (!S.uniq[i]) continue;
    int r = S.ent[i], rank = 0;
    for (int j = 0; j < n_ent; ++j) rank += S.uniq[j] && S.ent[j] < r;
    S.uni[rank] = r;
  }
  if (tid == 0) {
    int nu = 0;
    for (int j = 0; j < n_ent; ++j) nu += S.uniq[j];
    S.n_uni = nu;
  }
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = S.tmem_base;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  const uint32_t row_bytes_kv = DH * 2;
  uint32_t ph_kv = 0, ph_mma = 0;

  float merged[DH];
#pragma unroll
  for (int c = 0; c < DH; ++c) merged[c] = 0.f;

  for (int br = 0; br < P.n_gates; ++br) {
    // segments of this branch
    int n_seg;
    const __nv_bfloat16 *kb, *vb;
    int64_t head_rows;
    if (br == 0) {
      n_seg = 1;
      head_rows = (P.n_blocks + 15) / 16 * 16;
      kb = P.kc_il + (int64_t)h * head_rows * DH;
      vb = P.vc_il + (int64_t)h * head_rows * DH;
    } else {
      n_seg = br == 1 ? S.n_uni : 1;
      head_rows = P.n_rows_pad;
      kb = P.k_il + (int64_t)h * head_rows * DH;
      vb = P.v_il + (int64_t)h * head_rows * DH;
    }
    float m_run = -__builtin_huge_valf(), l_run = 0.f, o[DH];
#pragma unroll
    for (int c = 0; c < DH; ++c) o[c] = 0.f;
    if (tid == 0) {
      S.cur_seg = 0;
      S.cur_off = 0;
    }
    __syncthreads();
    while (S.cur_seg < n_seg) {
      // ---- build the chunk (thread 0) and launch its K/V bulk copies
      if (tid == 0) {
        int seg = S.cur_seg;
        int64_t seg_off = S.cur_off;
        int np = 0, ncol = 0;
        uint32_t bytes = 0;
        while (seg < n_seg && ncol < kNK) {
          int64_t lo, plen, occ;
          if (br == 0) {
            lo = 0;
            plen = head_rows;
            occ = P.n_blocks;
          } else {
            int r = br == 1 ? S.uni[seg] : own;
            lo = P.pad_off[r];
            plen = P.pad_off[r + 1] - lo;
            occ = P.kv_off[r + 1] - P.kv_off[r];
          }
          int take = (int)lmin(plen - seg_off, (int64_t)(kNK - ncol));
          Piece pc;
          pc.seg = seg;
          pc.col = ncol;
          pc.ncols = take;
          pc.nvalid = (int)lmax(0, lmin(occ - seg_off, (int64_t)take));
          pc.src = lo + seg_off;
          S.pieces[np] = pc;
          for (int gi = ncol / 16; gi < (ncol + take) / 16; ++gi) S.grp_piece[gi] = (int8_t)np;
          ++np;
          ncol += take;
          bytes += 2u * take * row_bytes_kv;
          seg_off += take;
          if (seg_off >= plen) {
            ++seg;
            seg_off = 0;
          }
        }
        S.n_pieces = np;
        S.n_cols = ncol;
        S.cur_seg = seg;
        S.cur_off = seg_off;
        mbar_expect_tx(&S.bar_kv, bytes);
        for (int i = 0; i < np; ++i) {
          const Piece& pc = S.pieces[i];
          bulk_g2s(&S.k[pc.col * DH], kb + pc.src * DH, pc.ncols * row_bytes_kv, &S.bar_kv);
          bulk_g2s(&S.v[pc.col * DH], vb + pc.src * DH, pc.ncols * row_bytes_kv, &S.bar_kv);
        }
      }
      __syncthreads();
      const int ncol = S.n_cols;
      mbar_wait(&S.bar_kv, ph_kv);
      ph_kv ^= 1;
      // ---- S = Q K^T  (M=128, N=ncol, K=DH)
      if (tid == 0) {
        tc_after_sync();
        uint32_t id = idesc_bf16(kM, ncol, 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          uint64_t a = sdesc(smem_u32(S.q) + kk * 256, 128, 16 * DH);
          uint64_t b = sdesc(smem_u32(S.k) + kk * 256, 128, 16 * DH);
          mma_bf16(tmem, a, b, id, kk > 0);
        }
        mma_commit(&S.bar_mma);
      }
      mbar_wait(&S.bar_mma, ph_mma);
      ph_mma ^= 1;
      tc_after_sync();
      // ---- masked online softmax on this thread's row
      const int n_grp = ncol / 16;
      float cmax = -__builtin_huge_valf();
      for (int gi = 0; gi < n_grp; ++gi) {
        const Piece& pc = S.pieces[S.grp_piece[gi]];
        int nv = min(16, pc.nvalid - (gi * 16 - pc.col));
        bool sel_ok = row_ok;
        if (br == 1 && sel_ok) {
          int r = S.uni[pc.seg];
          bool f = false;
          for (int s = 0; s < P.kmax; ++s) f |= S.ent[t * P.kmax + s] == r;
          sel_ok = f;
        }
        float sv[16];
        tmem_ld16(tmem + lane_base + gi * 16, sv);   // warp-uniform: every lane loads
        if (sel_ok)
          for (int j = 0; j < nv; ++j) cmax = fmaxf(cmax, sv[j]);
      }
      float m_new = fmaxf(m_run, cmax * scale_log2);
      float alpha = (m_new == -__builtin_huge_valf()) ? 1.f : ex2(m_run - m_new);
      float psum = 0.f;
      for (int gi = 0; gi < n_grp; ++gi) {
        const Piece& pc = S.pieces[S.grp_piece[gi]];
        int nv = min(16, pc.nvalid - (gi * 16 - pc.col));
        bool sel_ok = row_ok;
        if (br == 1 && sel_ok) {
          int r = S.uni[pc.seg];
          bool f = false;
          for (int s = 0; s < P.kmax; ++s) f |= S.ent[t * P.kmax + s] == r;
          sel_ok = f;
        }
        float sv[16];
        tmem_ld16(tmem + lane_base + gi * 16, sv);
        float pv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float p = (sel_ok && j < nv) ? ex2(sv[j] * scale_log2 - m_new) : 0.f;
          pv[j] = p;
        }
        uint4 w0, w1;
        w0.x = pack_bf16(pv[0], pv[1]);
        w0.y = pack_bf16(pv[2], pv[3]);
        w0.z = pack_bf16(pv[4], pv[5]);
        w0.w = pack_bf16(pv[6], pv[7]);
        w1.x = pack_bf16(pv[8], pv[9]);
        w1.y = pack_bf16(pv[10], pv[11]);
        w1.z = pack_bf16(pv[12], pv[13]);
        w1.w = pack_bf16(pv[14], pv[15]);
        // row sum of the bf16-rounded probabilities: consistent with P V
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t wv = j < 4 ? (&w0.x)[j] : (&w1.x)[j - 4];
          __nv_bfloat162 hb = *reinterpret_cast<__nv_bfloat162*>(&wv);
          float2 f2 = __bfloat1622float2(hb);
          psum += f2.x + f2.y;
        }
        const int m = tid;
        unsigned char* base = reinterpret_cast<unsigned char*>(S.p) + (m / 8) * (8 * kNK * 2) +
                              (m % 8) * 16;
        *reinterpret_cast<uint4*>(base + (gi * 2) * 128) = w0;
        *reinterpret_cast<uint4*>(base + (gi * 2 + 1) * 128) = w1;
      }
      l_run = l_run * alpha + psum;
      m_run = m_new;
      fence_async_smem();
      tc_before_sync();
      __syncthreads();
      // ---- O_part = P V  (M=128, N=DH, K=ncol), V read MN-major
      if (tid == 0) {
        tc_after_sync();
        uint32_t id = idesc_bf16(kM, DH, 1);
        for (int kk = 0; kk < ncol / 16; ++kk) {
          uint64_t a = sdesc(smem_u32(S.p) + kk * 256, 128, 8 * kNK * 2);
          uint64_t b = sdesc(smem_u32(S.v) + kk * 2 * (16 * DH), 16 * DH, 128);
          mma_bf16(tmem + kNK, a, b, id, kk > 0);
        }
        mma_commit(&S.bar_mma);
      }
      mbar_wait(&S.bar_mma, ph_mma);
      ph_mma ^= 1;
      tc_after_sync();
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 16) {
        float ov[16];
        tmem_ld16(tmem + lane_base + kNK + c0, ov);
#pragma unroll
        for (int j = 0; j < 16; ++j) o[c0 + j] = o[c0 + j] * alpha + ov[j];
      }
      tc_before_sync();
      __syncthreads();
    }
    // ---- branch epilogue: normalise, gate, accumulate
    if (row_ok) {
      float inv = 1.f / l_run;
      const __nv_bfloat16* gp = P.gl + tok * P.ld_gl + P.gcol0 + (int64_t)br * d_model + head * DH;
      const float* bp = P.gbias ? P.gbias + (int64_t)br * d_model + head * DH : nullptr;
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 8) {
        uint4 raw = *reinterpret_cast<const uint4*>(gp + c0);
        const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float z = __bfloat162float(hv[j]) + (bp ? bp[c0 + j] : 0.f);
          float gate = 1.f / (1.f + __expf(-z));
          merged[c0 + j] += gate * (o[c0 + j] * inv);
        }
      }
    }
  }
  if (row_ok) {
    __nv_bfloat16* op = P.out + tok * d_model + head * DH;
#pragma unroll
    for (int c0 = 0; c0 < DH; c0 += 8) {
      uint4 w;
      w.x = pack_bf16(merged[c0], merged[c0 + 1]);
      w.y = pack_bf16(merged[c0 + 2], merged[c0 + 3]);
      w.z = pack_bf16(merged[c0 + 4], merged[c0 + 5]);
      w.w = pack_bf16(merged[c0 + 6], merged[c0 + 7]);
      *reinterpret_cast<uint4*>(op + c0) = w;
    }
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// K/V (token order, f32 or bf16, row stride ld) -> padded interleaved bf16.
// One CTA per block (or one CTA per 128 rows of an un-partitioned row set).
__global__ void kv_interleave_kernel(int src_bf16, const void* __restrict__ src, int64_t ld,
                                     int hkv, int dh, const int64_t* __restrict__ tok,
                                     const int64_t* __restrict__ offs,
                                     const int64_t* __restrict__ pad_off, int64_t n_rows_pad,
                                     int64_t n_plain, __nv_bfloat16* __restrict__ dst) {
  int64_t r = blockIdx.x;
  int64_t lo, plen, occ, base;
  if (tok) {
    lo = offs[r];
    occ = offs[r + 1] - lo;
    base = pad_off[r];
    plen = pad_off[r + 1] - base;
  } else {  // identity rows [0, n_plain) padded to n_rows_pad, 128 rows per CTA
    lo = r * 128;
    base = lo;
    plen = lmin(128, n_rows_pad - lo);
    occ = lmax(0, lmin(128, n_plain - lo));
  }
  const int nchunk = dh / 8;
  int64_t total = (int64_t)hkv * plen * nchunk;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    int cc = (int)(e % nchunk);
    int64_t rr = (e / nchunk) % plen;
    int h = (int)(e / (nchunk * plen));
    __align__(16) __nv_bfloat16 vals[8];
    if (rr < occ) {
      int64_t row = tok ? tok[lo + rr] : lo + rr;
      if (src_bf16) {
        *reinterpret_cast<uint4*>(vals) = *reinterpret_cast<const uint4*>(
            (const __nv_bfloat16*)src + row * ld + h * dh + cc * 8);
      } else {
        const float* s = (const float*)src + row * ld + h * dh + cc * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) vals[j] = __float2bfloat16_rn(s[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) vals[j] = __float2bfloat16_rn(0.f);
    }
    int64_t prow = base + rr;
    int64_t off = (int64_t)h * n_rows_pad * dh + (prow / 8) * (8 * dh) + cc * 64 + (prow % 8) * 8;
    *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<uint4*>(vals);
  }
}

}  // namespace tc
}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_nsa_attention_tc(const void* q, int64_t ld_q, int64_t nq, int hq, int hkv, int dh,
                          const void* k_il, const void* v_il, const int64_t* pad_offsets,
                          const int64_t* kv_offsets, int64_t n_kv_rows_pad, const void* kcmp_il,
                          const void* vcmp_il, int64_t n_blocks, const int32_t* tiles,
                          int64_t n_tiles, const int32_t* rows, const int32_t* count,
                          int kmax_rows, const void* gate_logits, int64_t ld_gl,
                          int64_t gate_col0, const float* gate_bias, int n_gates,
                          void* merged, void* stream) {
  LSRM_REQUIRE(hq % hkv == 0, "n_q_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  int G = hq / hkv;
  LSRM_REQUIRE(G <= tc::kM && tc::kM % G == 0, "tcgen05 path needs (hq/hkv) | 128, got %d", G);
  LSRM_REQUIRE(n_gates == 2 || n_gates == 3, "n_gates must be 2 or 3");
  LSRM_REQUIRE((tc::kM / G) * kmax_rows <= tc::kMaxEnt,
               "tile tokens x selected rows = %d exceeds %d", (tc::kM / G) * kmax_rows,
               tc::kMaxEnt);
  if (n_blocks == 0) return set_error(LSRM_E_EMPTY_CONTEXT, "no occupied KV blocks");
  if (n_tiles == 0) return LSRM_OK;
  tc::Params p;
  p.q = (const __nv_bfloat16*)q;
  p.ld_q = ld_q;
  p.nq = nq;
  p.hq = hq;
  p.hkv = hkv;
  p.k_il = (const __nv_bfloat16*)k_il;
  p.v_il = (const __nv_bfloat16*)v_il;
  p.pad_off = pad_offsets;
  p.kv_off = kv_offsets;
  p.n_rows_pad = n_kv_rows_pad;
  p.kc_il = (const __nv_bfloat16*)kcmp_il;
  p.vc_il = (const __nv_bfloat16*)vcmp_il;
  p.n_blocks = n_blocks;
  p.tiles = tiles;
  p.n_tiles = n_tiles;
  p.rows = rows;
  p.count = count;
  p.kmax = kmax_rows;
  p.gl = (const __nv_bfloat16*)gate_logits;
  p.ld_gl = ld_gl;
  p.gcol0 = gate_col0;
  p.gbias = gate_bias;
  p.n_gates = n_gates;
  p.out = (__nv_bfloat16*)merged;
  cudaStream_t st = as_stream(stream);
  unsigned grid = (unsigned)(n_tiles * hkv);
#define LSRM_TC_CASE(D)                                                                     \
  case D: {                                                                                 \
    size_t smem = sizeof(tc::Smem<D>) + 1024;                                               \
    if (smem < 100 * 1024) smem = 100 * 1024; /* TMEM: at most 2 CTAs (2x256 cols) per SM */ \
    LSRM_CUDA(cudaFuncSetAttribute(tc::nsa_fused_kernel<D>,                                 \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    tc::nsa_fused_kernel<D><<<grid, tc::kThreads, smem, st>>>(p);                           \
    break;                                                                                  \
  }
  switch (dh) {
    LSRM_TC_CASE(16)
    LSRM_TC_CASE(32)
    LSRM_TC_CASE(64)
    default:
      return set_error(LSRM_E_CONFIG, "tcgen05 path: head_dim %d not in {16,32,64}", dh);
  }
#undef LSRM_TC_CASE
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_kv_interleave(int src_is_bf16, const void* src, int64_t ld_src, int64_t n, int hkv,
                       int dh, const int64_t* block_token_ids, const int64_t* block_offsets,
                       int64_t n_blocks, const int64_t* pad_offsets, int64_t n_rows_pad,
                       void* dst, void* stream) {
  LSRM_REQUIRE(dh % 8 == 0, "kv_interleave: head_dim must be a multiple of 8");
  LSRM_REQUIRE(n_rows_pad % 16 == 0, "kv_interleave: padded rows must be a multiple of 16");
  cudaStream_t st = as_stream(stream);
  if (block_token_ids) {
    if (n_blocks == 0) return LSRM_OK;
    tc::kv_interleave_kernel<<<(unsigned)n_blocks, 256, 0, st>>>(
        src_is_bf16, src, ld_src, hkv, dh, block_token_ids, block_offsets, pad_offsets,
        n_rows_pad, 0, (__nv_bfloat16*)dst);
  } else {
    if (n_rows_pad == 0) return LSRM_OK;
    tc::kv_interleave_kernel<<<(unsigned)ceil_div(n_rows_pad, 128), 256, 0, st>>>(
        src_is_bf16, src, ld_src, hkv, dh, nullptr, nullptr, nullptr, n_rows_pad, n,
        (__nv_bfloat16*)dst);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
