// Fused bf16 three-branch NSA attention on the 5th-gen tensor cores
// (tcgen05.mma + TMEM accumulators + bulk-async (TMA engine) K/V staging),
// with the sigmoid-gated branch merge in the epilogue.
//
// Replaces, fused: cmp_attention / sel_attention / win_attention and the
// gated sum of combine_nsa_branches (lsrm/nsa_attention.py:84-112,157-207,
// 266-284).  The W_o projection stays a plain GEMM.
//
// Work item = (query tile, kv head).  A query tile is up to T = 128/G
// consecutive tokens of ONE query block (block-major order); the MMA
// M-dimension is the 128 rows (token, q-head-in-group) sharing kv head h.
// Each item streams key chunks of <= 128 keys, branch after branch:
//   cmp : all compressed rows (one per occupied KV block),
//   sel : the sorted union of the tile tokens' selected blocks; a row only
//         sees the blocks ITS token selected (others masked out),
//   win : the tile's own block (self uses).
//
// Persistent, warp-specialised CTA (one per SM, 192 threads):
//   warps 0-3  softmax/epilogue: thread = TMEM lane = one row; masked online
//              softmax (exp2), bf16 P to smem, rescale-accumulate O in
//              registers, gate + merge at branch ends;
//   warp 4     producer: union of the tile's selections, chunk plans, and
//              cp.async.bulk K/V copies (each KV block is one contiguous
//              16-row-padded segment of the interleaved layout) into a
//              2-stage ring;
//   warp 5     MMA issuer: S = Q K^T into a double-buffered TMEM S, and
//              O_part = P V into TMEM, in the order QK(j+1), PV(j) so the
//              tensor core runs one chunk ahead of the softmax warps.
// mbarriers: kv_full/kv_empty (ring), s_full (S ready), p_full (P written,
// S slot free), o_full/o_empty (PV partial).  Phases follow a chunk counter
// that all roles advance identically.
//
// SMEM operand layout: 8x8 "core matrices" of 128 contiguous bytes,
// SWIZZLE_NONE canonical layouts (cute mma_sm100_desc.hpp):
//   K-major  Q, K, P : element (row, k) at (row/8)*RS + (k/8)*64 + (row%8)*8 + k%8
//   MN-major V       : the same storage read with N = head dim, K = keys.
#include "common.cuh"

namespace lsrm {
namespace tc {

constexpr int kM = 128;          // MMA rows per tile
constexpr int kNK = 128;         // keys per chunk
constexpr int kGroups = kNK / 16;
constexpr int kParts = 4;                    // softmax warps per TMEM lane quadrant
constexpr int kSoftThreads = 128 * kParts;   // softmax warps 0 .. 4*kParts-1
constexpr int kProducerWarp = 4 * kParts, kMmaWarp = 4 * kParts + 1;
constexpr int kThreads = kSoftThreads + 64;
constexpr int kTmemCols = 512;   // S0 [0,128) S1 [128,256) O [256, 256+DH)
constexpr int kMaxEnt = 256;     // tile tokens * selected rows
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
// kind::f16 instruction descriptor: bf16 x bf16 -> f32, A K-major.
__device__ __forceinline__ uint32_t idesc_bf16(int m, int n, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// D[tmem] (+)= A[tmem] . B[smem]: A (P) read from TMEM, 16 bf16 per lane in 8
// packed 32-bit columns per K=16 step.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t elect_one_sync() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 %%rx;\n\t.reg .pred %%px;\n\t"
      "elect.sync %%rx|%%px, %1;\n\t@%%px mov.s32 %0, 1;\n\t}"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred;
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// 16 consecutive f32 columns of this thread's TMEM lane (no wait).
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// N (1, 8, 16) consecutive f32 columns of this thread's TMEM lane (no wait).
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
  if constexpr (N == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
  } else if constexpr (N == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  } else {
    static_assert(N % 16 == 0, "tmem_ld_cols: N must be 1, 8 or a multiple of 16");
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 16) tmem_ld16_nowait(taddr + c0, r + c0);
  }
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
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

// Optional event trace (debug): CTA 0 stamps clock64() per chunk and event.
__device__ long long* g_trace = nullptr;
constexpr int kTraceEv = 8, kTraceChunks = 1024;
__device__ __forceinline__ void trace(long long* tr, uint32_t c, int ev) {
  if (tr && c < (uint32_t)kTraceChunks) tr[c * kTraceEv + ev] = clock64();
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

constexpr int kStages = 6;       // K/V ring depth
constexpr int kOnesCols = 16;    // extra V columns holding 1 (valid key) / 0 (padding)
constexpr int kBitmapWords = 512;  // union bitmap: up to 16384 occupied KV blocks

__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// One chunk of <= 128 keys as the softmax and MMA warps see it.  The
// producer resolves visibility per 16-key group: gnv = valid keys in the
// group, gmask = tile tokens allowed to see it.
struct ChunkDesc {
  uint32_t gmask[kGroups];
  int32_t gnv[kGroups];
  int ncols, branch;
  int first_in_branch, last_in_branch, first_in_item, last_in_item, last_overall;
  int q_first, q_cnt, h, qb, item_seq;
};

template <int DH>
struct Smem {
  __nv_bfloat16 q[2][kM * DH];
  __nv_bfloat16 k[kStages][kNK * DH];
  __nv_bfloat16 v[kStages][kNK * (DH + kOnesCols)];   // [V | ones] rows
  float merged[kM][DH + 1];
  float xmax[2][kParts][kM];    // per-part partial row maxima (chunk parity)
  int32_t ent[kMaxEnt];         // selected rows of the tile tokens, [t][kmax]
  uint32_t bitmap[kBitmapWords]; // selected-row bitmap of the current item
  int32_t wpre[kBitmapWords];    // rank of the first set bit of each word
  int32_t uni_row[kMaxEnt];      // sorted union of selected rows
  uint32_t uni_mask[kMaxEnt];   // per union slot: tokens that selected it
  int64_t seg_lo[kMaxEnt + 1];  // per union slot (+1: own block) padded first row
  int32_t seg_plen[kMaxEnt + 1];
  int32_t seg_occ[kMaxEnt + 1];
  int32_t seg_cum[kMaxEnt];
  ChunkDesc desc[kStages];
  uint64_t kv_full[kStages], kv_empty[kStages], s_full[2], p_full[2], o_full[2], o_empty[2],
      q_full[2], q_empty[2];
  uint32_t tmem_base;
};

template <int DH>
__global__ void __launch_bounds__(kThreads, 1) nsa_fused_kernel(Params P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem<DH>& S = *reinterpret_cast<Smem<DH>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = P.hq / P.hkv, T = kM / G;
  const int d_model = P.hq * DH;
  const int64_t n_items = P.n_tiles * P.hkv;
  if ((int64_t)blockIdx.x >= n_items) return;
  // TMEM columns: S slots [0,128) [128,256); O/L double-buffered per chunk parity
  // P(c) (bf16x2 packed, 64 columns) aliases the upper half of S slot c&1:
  // every part has loaded its S values before the max-exchange barrier, and
  // QK(c+2) is issued after PV(c) in the in-order tensor pipe.
  constexpr int VW = DH + kOnesCols;   // V row width incl. the ones columns
  constexpr uint32_t kColO = 2 * kNK, kColP = kNK / 2;   // O|L slots: kColO + parity * VW

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&S.kv_full[i], 1);
      mbar_init(&S.kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.s_full[i], 1);
      mbar_init(&S.p_full[i], kSoftThreads);
      mbar_init(&S.q_full[i], 1);
      mbar_init(&S.q_empty[i], 1);
      mbar_init(&S.o_full[i], 1);
      mbar_init(&S.o_empty[i], kSoftThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp < 4)
    for (int c = 0; c < DH; ++c) S.merged[tid][c] = 0.f;  // warps 0-3 cover all rows
  for (int i = tid; i < kBitmapWords; i += kThreads) S.bitmap[i] = 0u;
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = S.tmem_base;
  const uint32_t row_bytes_kv = DH * 2;
  long long* const trp = blockIdx.x == 0 ? g_trace : nullptr;  // debug event trace

  if (warp == kProducerWarp) {
    // ===================== producer: Q tiles, unions, chunk plans, K/V copies
    uint32_t c = 0;
    int it = 0;
    const uint32_t all_tok = T >= 32 ? 0xffffffffu : ((1u << T) - 1u);
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int tile = (int)(item / P.hkv), h = (int)(item % P.hkv);
      const int q_first = P.tiles[4 * tile], q_cnt = P.tiles[4 * tile + 1],
                own = P.tiles[4 * tile + 2];
      const bool last_item = item + gridDim.x >= n_items;
      const int qb = it & 1;
      // ---- selected rows of the tile tokens (resolved rows are -1 padded,
      //      so no dependent load of `count`) -> bitmap; they overlap Q
      const int n_ent = T * P.kmax, n_valid_ent = q_cnt * P.kmax;
      const int32_t* rows_t = P.rows + (int64_t)q_first * P.kmax;
      for (int i = lane; i < n_ent; i += 32) {
        const int r = i < n_valid_ent ? rows_t[i] : -1;
        S.ent[i] = r;
        if (r >= 0) atomicOr(&S.bitmap[r >> 5], 1u << (r & 31));
      }
      // ---- Q tile -> sQ[qb] (cp.async, zero-filled past the tile), once the
      //      MMAs of item it-2 are done with the buffer
      if (it >= 2) mbar_wait(&S.q_empty[qb], ((it >> 1) - 1) & 1);
#pragma unroll
      for (int i = lane; i < kM * (DH / 8); i += 32) {
        const int m = i / (DH / 8), cc = i % (DH / 8);
        const int tt = m / G, gg = m % G;
        const bool ok = tt < q_cnt;
        const __nv_bfloat16* src =
            P.q + (ok ? (int64_t)(q_first + tt) * P.ld_q + (h * G + gg) * DH + cc * 8 : 0);
        cp_async16(&S.q[qb][(m / 8) * (8 * DH) + cc * 64 + (m % 8) * 8], src, ok ? 16u : 0u);
      }
      cp_async_wait_all();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.q_full[qb]);
      // ---- sorted union = set bits of the bitmap in order; lane l owns a
      //      contiguous run of words, ranks by a warp prefix of popcounts
      const int n_words = (int)((P.n_blocks + 31) / 32);
      const int per_w = (n_words + 31) / 32;
      int cnt_w = 0;
      for (int k = 0; k < per_w; ++k) {
        const int w = lane * per_w + k;
        if (w < n_words) cnt_w += __popc(S.bitmap[w]);
      }
      int incl_w = cnt_w;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl_w, o);
        if (lane >= o) incl_w += v;
      }
      const int nu = __shfl_sync(0xffffffffu, incl_w, 31);
      {
        int rank = incl_w - cnt_w;
        for (int k = 0; k < per_w; ++k) {
          const int w = lane * per_w + k;
          if (w >= n_words) break;
          uint32_t bits = S.bitmap[w];
          S.wpre[w] = rank;
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            S.uni_row[rank] = w * 32 + b;
            S.uni_mask[rank] = 0u;
            ++rank;
          }
        }
      }
      __syncwarp();
      // token masks: entry i belongs to token i / kmax
      for (int i = lane; i < n_ent; i += 32) {
        const int r = S.ent[i];
        if (r >= 0) {
          const int w = r >> 5;
          const int rank = S.wpre[w] + __popc(S.bitmap[w] & ((1u << (r & 31)) - 1u));
          atomicOr(&S.uni_mask[rank], 1u << (i / P.kmax));
        }
      }
      // segment geometry of every union slot (independent loads, all lanes)
      for (int u = lane; u < nu; u += 32) {
        const int r = S.uni_row[u];
        const int64_t a0 = P.pad_off[r], a1 = P.pad_off[r + 1];
        const int64_t b0 = P.kv_off[r], b1 = P.kv_off[r + 1];
        S.seg_lo[u] = a0;
        S.seg_plen[u] = (int)(a1 - a0);
        S.seg_occ[u] = (int)(b1 - b0);
      }
      if (lane == 0 && own >= 0) {
        const int64_t a0 = P.pad_off[own], a1 = P.pad_off[own + 1];
        const int64_t b0 = P.kv_off[own], b1 = P.kv_off[own + 1];
        S.seg_lo[kMaxEnt] = a0;
        S.seg_plen[kMaxEnt] = (int)(a1 - a0);
        S.seg_occ[kMaxEnt] = (int)(b1 - b0);
      }
      __syncwarp();
      for (int k = 0; k < per_w; ++k) {  // clear the bitmap for the next item
        const int w = lane * per_w + k;
        if (w < n_words) S.bitmap[w] = 0u;
      }
      __syncwarp();
      // exclusive prefix of the union segments' padded lengths (sel branch)
      int total_sel;
      {
        const int per = (nu + 31) / 32;
        int local = 0;
        for (int k = 0; k < per; ++k) {
          int u = lane * per + k;
          if (u < nu) local += S.seg_plen[u];
        }
        int incl = local;
        for (int o = 1; o < 32; o <<= 1) {
          int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        int run = incl - local;
        for (int k = 0; k < per; ++k) {
          int u = lane * per + k;
          if (u < nu) {
            S.seg_cum[u] = run;
            run += S.seg_plen[u];
          }
        }
        total_sel = __shfl_sync(0xffffffffu, incl, 31);
      }
      __syncwarp();
      // ---- chunk j of a branch = keys [128j, 128j+128) of the concatenation
      //      of its 16-row-padded segments; lane i turns the i-th overlapping
      //      segment into a piece, fills its groups' visibility and issues the
      //      piece's K and V bulk copies
      const int64_t cmp_rows = (P.n_blocks + 15) / 16 * 16;
      for (int br = 0; br < P.n_gates; ++br) {
        const int n_seg = br == 1 ? nu : 1;
        const int64_t total = br == 0 ? cmp_rows : (br == 1 ? total_sel : S.seg_plen[kMaxEnt]);
        const int64_t head_rows = br == 0 ? cmp_rows : P.n_rows_pad;
        const __nv_bfloat16* kb = (br == 0 ? P.kc_il : P.k_il) + (int64_t)h * head_rows * DH;
        const __nv_bfloat16* vb = (br == 0 ? P.vc_il : P.v_il) + (int64_t)h * head_rows * VW;
        int cur = 0;
        for (int64_t start = 0; start < total; start += kNK) {
          const int64_t end = lmin(start + kNK, total);
          const int st = c % kStages;
          if (c >= kStages) mbar_wait(&S.kv_empty[st], ((c / kStages) - 1) & 1);
          if (lane == 0) trace(trp, c, 0);
          ChunkDesc& D = S.desc[st];
          const int s = cur + lane;
          bool ov = false, done = false;
          int col = 0, ncols = 0, nvalid = 0;
          uint32_t tm = all_tok;
          int64_t src = 0;
          if (s < n_seg) {
            int64_t lo, plen, occ, cs;
            if (br == 0) {
              lo = 0; plen = cmp_rows; occ = P.n_blocks; cs = 0;
            } else if (br == 1) {
              lo = S.seg_lo[s]; plen = S.seg_plen[s]; occ = S.seg_occ[s]; cs = S.seg_cum[s];
              tm = S.uni_mask[s];
            } else {
              lo = S.seg_lo[kMaxEnt]; plen = S.seg_plen[kMaxEnt]; occ = S.seg_occ[kMaxEnt];
              cs = 0;
            }
            const int64_t a = lmax(cs, start), b = lmin(cs + plen, end);
            if (a < b) {
              ov = true;
              done = cs + plen <= end;
              col = (int)(a - start);
              ncols = (int)(b - a);
              nvalid = (int)lmax(0, lmin(occ - (a - cs), b - a));
              src = lo + (a - cs);
            }
          }
          if (ov) {
            for (int gi = col / 16; gi < (col + ncols) / 16; ++gi) {
              const int nv = nvalid - (gi * 16 - col);
              D.gnv[gi] = nv < 0 ? 0 : (nv > 16 ? 16 : nv);
              D.gmask[gi] = tm;
            }
          }
          if (lane == 0) {
            D.ncols = (int)(end - start);
            D.branch = br;
            D.first_in_branch = start == 0;
            D.last_in_branch = end == total;
            D.first_in_item = br == 0 && start == 0;
            D.last_in_item = end == total && br == P.n_gates - 1;
            D.last_overall = D.last_in_item && last_item;
            D.q_first = q_first;
            D.q_cnt = q_cnt;
            D.h = h;
            D.qb = qb;
            D.item_seq = it;
          }
          __syncwarp();
          if (lane == 0)
            mbar_expect_tx(&S.kv_full[st], (uint32_t)(end - start) * (row_bytes_kv + 2u * VW));
          __syncwarp();
          if (ov) {
            bulk_g2s(&S.k[st][col * DH], kb + src * DH, ncols * row_bytes_kv, &S.kv_full[st]);
            bulk_g2s(&S.v[st][col * VW], vb + src * VW, ncols * 2u * VW, &S.kv_full[st]);
          }
          cur += __popc(__ballot_sync(0xffffffffu, done));
          ++c;
        }
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (warp converged; one elected lane issues)
    {
      const uint32_t id_pv = idesc_bf16(kM, VW, 1);   // O | rowsum = P . [V | ones]
      // S = Q K^T for chunk cc into TMEM S slot cc&1
      auto issue_qk = [&](uint32_t cc) {
        const int st = cc % kStages;
        mbar_wait(&S.kv_full[st], (cc / kStages) & 1);
        if (lane == 0) trace(trp, cc, 1);
        const ChunkDesc& D = S.desc[st];
        if (D.first_in_item) mbar_wait(&S.q_full[D.qb], (D.item_seq >> 1) & 1);
        tc_after_sync();
        const uint32_t id = idesc_bf16(kM, D.ncols, 0);
        const uint64_t a0 = sdesc(smem_u32(S.q[D.qb]), 128, 16 * DH);
        const uint64_t b0 = sdesc(smem_u32(S.k[st]), 128, 16 * DH);
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            mma_bf16(tmem + (cc & 1) * kNK, a0 + (uint64_t)(kk * 16), b0 + (uint64_t)(kk * 16),
                     id, kk > 0);
          mma_commit(&S.s_full[cc & 1]);
        }
        __syncwarp();
        if (lane == 0) trace(trp, cc, 2);
      };
      // QK runs two chunks ahead: QK(c+2) reuses S slot c&1 once the softmax
      // of chunk c has released it; it is issued right after PV(c)
      uint32_t c = 0;
      issue_qk(0);
      bool ahead = !S.desc[0].last_overall;  // is there a chunk 1?
      if (ahead) issue_qk(1);
      uint32_t next_qk = ahead ? 2 : 1;
      bool more = ahead && !S.desc[1 % kStages].last_overall;
      for (;;) {
        const int st = c % kStages;
        const ChunkDesc& D = S.desc[st];
        const bool last = D.last_overall;
        const int nk = D.ncols / 16;
        const bool last_in_item = D.last_in_item;
        const int qb = D.qb;
        mbar_wait(&S.p_full[c & 1], (c >> 1) & 1);
        if (lane == 0) trace(trp, c, 5);
        // [O | rowsum](c) = P V' into the O slot of parity c&1 (absorbed two
        // chunks ago: no wait on the previous chunk's absorb)
        if (c >= 2) mbar_wait(&S.o_empty[c & 1], ((c >> 1) - 1) & 1);
        tc_after_sync();
        const uint32_t pa = tmem + (c & 1) * kNK + kColP;   // P(c): packed bf16 in TMEM
        const uint64_t vb = sdesc(smem_u32(S.v[st]), 16 * VW, 128);
        const uint32_t to = tmem + kColO + (c & 1) * VW;
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < kGroups; ++kk)
            if (kk < nk) mma_bf16_ts(to, pa + kk * 8, vb + (uint64_t)(kk * 2 * VW), id_pv, kk > 0);
          mma_commit(&S.o_full[c & 1]);
          if (last_in_item) mma_commit(&S.q_empty[qb]);
          mma_commit(&S.kv_empty[st]);
        }
        __syncwarp();
        if (lane == 0) trace(trp, c, 6);
        if (more) {
          issue_qk(next_qk);
          more = !S.desc[next_qk % kStages].last_overall;
          ++next_qk;
        }
        ++c;
        if (last) break;
      }
    }
    __syncwarp();
  } else {
    // ===================== softmax / epilogue (warps 0 .. 4*kParts-1)
    // kParts warps per TMEM lane quadrant: warps q, q+4, q+8, ... share rows
    // 32q..32q+31; part p takes key groups [p*HG, (p+1)*HG) and O columns
    // [p*HD, (p+1)*HD).  Row maxima are exchanged through smem (named barrier
    // per quadrant); row sums come from the tensor core (P . ones).
    constexpr int HG = kGroups / kParts, HD = DH / kParts;
    const int q4 = warp & 3, half = warp >> 2;   // half == part index
    const int m = q4 * 32 + lane;
    const int t = m / G, g_in = m % G;
    const int bar_id = 1 + q4;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const float sl2 = 1.4426950408889634f / sqrtf((float)DH);
    float m_run = -__builtin_huge_valf(), l_acc = 0.f;
    // state of the chunk whose PV partial is still in flight
    float alpha_pend = 1.f;
    int br_pend = 0, lastbr_pend = 0, lastit_pend = 0;
    int64_t tok_pend = 0;
    bool rowok_pend = false;
    int head_pend = 0;
    uint4 gate_cur[HD / 8], gate_pend[HD / 8];   // gate logits, prefetched at branch start
    float o[HD];
#pragma unroll
    for (int j = 0; j < HD; ++j) o[j] = 0.f;
    uint32_t c = 0;
    bool have_pend = false;
    // O_part / L_part of the previous chunk: o = o * alpha + O_part, same for l
    auto absorb_pv = [&]() {
      mbar_wait(&S.o_full[(c - 1) & 1], ((c - 1) >> 1) & 1);
      if (tid == 0) trace(trp, c - 1, 7);
      const uint32_t ps = (c - 1) & 1;  // O/L slot of the absorbed chunk
      tc_after_sync();
      uint32_t r[HD], rl[1];
      tmem_ld_cols<HD>(tmem + lane_base + kColO + ps * VW + half * HD, r);
      tmem_ld_cols<1>(tmem + lane_base + kColO + ps * VW + DH, rl);
      tmem_wait_ld();
      tc_before_sync();
      mbar_arrive(&S.o_empty[ps]);
#pragma unroll
      for (int j = 0; j < HD; ++j) o[j] = o[j] * alpha_pend + __uint_as_float(r[j]);
      l_acc = l_acc * alpha_pend + __uint_as_float(rl[0]);
      if (lastbr_pend) {
        if (rowok_pend) {
          // gate + merge the finished branch (nsa_attention.py:266-284)
          const float inv = 1.f / l_acc;
          const int64_t col0 = (int64_t)br_pend * d_model + head_pend * DH + half * HD;
          const __nv_bfloat16* gp = P.gl + tok_pend * P.ld_gl + P.gcol0 + col0;
          const float* bp = P.gbias ? P.gbias + col0 : nullptr;
          (void)gp;
#pragma unroll
          for (int c0 = 0; c0 < HD; c0 += 8) {
            uint4 raw = gate_pend[c0 / 8];
            const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float z = __bfloat162float(hv[j]) + (bp ? bp[c0 + j] : 0.f);
              float gate = 1.f / (1.f + __expf(-z));
              S.merged[m][half * HD + c0 + j] += gate * (o[c0 + j] * inv);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < HD; ++j) o[j] = 0.f;
        l_acc = 0.f;
        if (lastit_pend) {
          if (rowok_pend) {
            __nv_bfloat16* op = P.out + tok_pend * d_model + head_pend * DH + half * HD;
#pragma unroll
            for (int c0 = 0; c0 < HD; c0 += 8) {
              const float* mr = &S.merged[m][half * HD + c0];
              uint4 w;
              w.x = pack_bf16(mr[0], mr[1]);
              w.y = pack_bf16(mr[2], mr[3]);
              w.z = pack_bf16(mr[4], mr[5]);
              w.w = pack_bf16(mr[6], mr[7]);
              *reinterpret_cast<uint4*>(op + c0) = w;
            }
          }
#pragma unroll
          for (int j = 0; j < HD; ++j) S.merged[m][half * HD + j] = 0.f;
        }
      }
    };
    for (;;) {
      mbar_wait(&S.s_full[c & 1], (c >> 1) & 1);
      if (tid == 0) trace(trp, c, 3);
      tc_after_sync();
      const ChunkDesc& D = S.desc[c % kStages];
      const int n_grp = D.ncols / 16;
      const int br = D.branch;
      const bool first_br = D.first_in_branch, last_br = D.last_in_branch,
                 last_it = D.last_in_item, last_all = D.last_overall;
      const bool row_ok = t < D.q_cnt;
      const int64_t tok = (int64_t)D.q_first + t;
      const int head = D.h * G + g_in;
      if (first_br) {
        m_run = -__builtin_huge_valf();
        if (row_ok) {  // prefetch this branch's gate logits (used at its end)
          const __nv_bfloat16* gp = P.gl + tok * P.ld_gl + P.gcol0 +
                                    (int64_t)br * d_model + head * DH + half * HD;
#pragma unroll
          for (int c0 = 0; c0 < HD; c0 += 8) gate_cur[c0 / 8] = *reinterpret_cast<const uint4*>(gp + c0);
        }
      }
      // this half's S groups -> registers (all in flight, one wait)
      uint32_t sr[HG * 16];
#pragma unroll
      for (int k = 0; k < HG; ++k)
        if (half * HG + k < n_grp)
          tmem_ld16_nowait(tmem + lane_base + (c & 1) * kNK + (half * HG + k) * 16, sr + k * 16);
      // group visibility (producer-resolved) while the loads are in flight
      int nv_grp[HG];
#pragma unroll
      for (int k = 0; k < HG; ++k) {
        const int gi = half * HG + k;
        nv_grp[k] = (gi < n_grp && row_ok && ((D.gmask[gi] >> t) & 1u)) ? D.gnv[gi] : 0;
      }
      tmem_wait_ld();
      // masked group maxima (log-depth trees)
      float gmax[HG];
#pragma unroll
      for (int k = 0; k < HG; ++k) {
        gmax[k] = -__builtin_huge_valf();
        if (nv_grp[k] == 16) {
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            v[j] = fmaxf(__uint_as_float(sr[k * 16 + j]), __uint_as_float(sr[k * 16 + j + 8]));
#pragma unroll
          for (int w = 4; w; w >>= 1)
#pragma unroll
            for (int j = 0; j < w; ++j) v[j] = fmaxf(v[j], v[j + w]);
          gmax[k] = v[0];
        } else if (nv_grp[k] > 0) {
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            v[j] = j < nv_grp[k] ? __uint_as_float(sr[k * 16 + j]) : -__builtin_huge_valf();
#pragma unroll
          for (int w = 8; w; w >>= 1)
#pragma unroll
            for (int j = 0; j < w; ++j) v[j] = fmaxf(v[j], v[j + w]);
          gmax[k] = v[0];
        }
      }
#pragma unroll
      for (int w = HG / 2; w; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) gmax[j] = fmaxf(gmax[j], gmax[j + w]);
      // row max across the two halves
      S.xmax[c & 1][half][m] = gmax[0];
      named_sync(bar_id, 32 * kParts);
      float cmax = gmax[0];
#pragma unroll
      for (int p2 = 0; p2 < kParts; ++p2) cmax = fmaxf(cmax, S.xmax[c & 1][p2][m]);
      const float m_new = fmaxf(m_run, cmax * sl2);
      const float alpha = (m_new == -__builtin_huge_valf()) ? 1.f : ex2(m_run - m_new);
      const uint32_t pbase = tmem + lane_base + (c & 1) * kNK + kColP;
#pragma unroll
      for (int k = 0; k < HG; ++k) {
        const int gi = half * HG + k;
        if (gi < n_grp) {
          uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          const int nv = nv_grp[k];
          if (nv > 0) {
            float pv[16];
            if (nv == 16) {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                pv[j] = ex2(fmaf(__uint_as_float(sr[k * 16 + j]), sl2, -m_new));
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                pv[j] = j < nv ? ex2(fmaf(__uint_as_float(sr[k * 16 + j]), sl2, -m_new)) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) w[j] = pack_bf16(pv[2 * j], pv[2 * j + 1]);
          }
          tmem_st8(pbase + gi * 8, w);
        }
      }
      tmem_wait_st();
      tc_before_sync();
      mbar_arrive(&S.p_full[c & 1]);
      if (tid == 0) trace(trp, c, 4);
      // previous chunk's PV partial (its rescale factor is alpha_pend)
      if (have_pend) absorb_pv();
      m_run = m_new;
      alpha_pend = alpha;
      br_pend = br;
      lastbr_pend = last_br;
      lastit_pend = last_it;
      tok_pend = tok;
      rowok_pend = row_ok;
      if (last_br) {
#pragma unroll
        for (int j = 0; j < HD / 8; ++j) gate_pend[j] = gate_cur[j];
      }
      head_pend = head;
      have_pend = true;
      ++c;
      if (last_all) break;
    }
    absorb_pv();
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
                                     int hkv, int dh, int ones_cols,
                                     const int64_t* __restrict__ tok,
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
  const int nchunk = (dh + ones_cols) / 8, w = dh + ones_cols;
  int64_t total = (int64_t)hkv * plen * nchunk;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    int cc = (int)(e % nchunk);
    int64_t rr = (e / nchunk) % plen;
    int h = (int)(e / (nchunk * plen));
    __align__(16) __nv_bfloat16 vals[8];
    if (cc * 8 >= dh) {  // ones columns: 1 for a real key, 0 for padding
#pragma unroll
      for (int j = 0; j < 8; ++j) vals[j] = __float2bfloat16_rn(rr < occ ? 1.f : 0.f);
    } else if (rr < occ) {
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
    int64_t off = (int64_t)h * n_rows_pad * w + (prow / 8) * (8 * w) + cc * 64 + (prow % 8) * 8;
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
  LSRM_REQUIRE(G >= 4 && G <= tc::kM && tc::kM % G == 0,
               "tcgen05 path needs 4 <= hq/hkv, (hq/hkv) | 128, got %d", G);
  LSRM_REQUIRE(n_gates == 2 || n_gates == 3, "n_gates must be 2 or 3");
  LSRM_REQUIRE((tc::kM / G) * kmax_rows <= tc::kMaxEnt,
               "tile tokens x selected rows = %d exceeds %d", (tc::kM / G) * kmax_rows,
               tc::kMaxEnt);
  LSRM_REQUIRE(ld_q % 8 == 0 && ld_gl % 8 == 0 && gate_col0 % 8 == 0,
               "tcgen05 path: row strides must be multiples of 8 elements");
  if (n_blocks == 0) return set_error(LSRM_E_EMPTY_CONTEXT, "no occupied KV blocks");
  LSRM_REQUIRE(n_blocks <= (int64_t)tc::kBitmapWords * 32,
               "tcgen05 path: %lld occupied KV blocks exceed %d", (long long)n_blocks,
               tc::kBitmapWords * 32);
  LSRM_REQUIRE(tc::kM / G <= 32, "tcgen05 path: at most 32 tokens per tile");
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
  int dev = 0, n_sm = 148;
  LSRM_CUDA(cudaGetDevice(&dev));
  LSRM_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  int64_t n_items = n_tiles * hkv;
  unsigned grid = (unsigned)(n_items < n_sm ? n_items : n_sm);
#define LSRM_TC_CASE(D)                                                                     \
  case D: {                                                                                 \
    size_t smem = sizeof(tc::Smem<D>) + 1024;                                               \
    LSRM_CUDA(cudaFuncSetAttribute(tc::nsa_fused_kernel<D>,                                 \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    tc::nsa_fused_kernel<D><<<grid, tc::kThreads, smem, st>>>(p);                           \
    break;                                                                                  \
  }
  switch (dh) {
    LSRM_TC_CASE(32)
    LSRM_TC_CASE(64)
    default:
      return set_error(LSRM_E_CONFIG, "tcgen05 path: head_dim %d not in {32,64}", dh);
  }
#undef LSRM_TC_CASE
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_debug_set_trace(void* buf) {
  LSRM_CUDA(cudaMemcpyToSymbol(tc::g_trace, &buf, sizeof(buf)));
  return LSRM_OK;
}

int lsrm_kv_interleave(int src_is_bf16, const void* src, int64_t ld_src, int64_t n, int hkv,
                       int dh, int ones_cols, const int64_t* block_token_ids, const int64_t* block_offsets,
                       int64_t n_blocks, const int64_t* pad_offsets, int64_t n_rows_pad,
                       void* dst, void* stream) {
  LSRM_REQUIRE(dh % 8 == 0, "kv_interleave: head_dim must be a multiple of 8");
  LSRM_REQUIRE(n_rows_pad % 16 == 0, "kv_interleave: padded rows must be a multiple of 16");
  LSRM_REQUIRE(ones_cols == 0 || ones_cols == 16, "kv_interleave: ones_cols must be 0 or 16");
  cudaStream_t st = as_stream(stream);
  if (block_token_ids) {
    if (n_blocks == 0) return LSRM_OK;
    tc::kv_interleave_kernel<<<(unsigned)n_blocks, 256, 0, st>>>(
        src_is_bf16, src, ld_src, hkv, dh, ones_cols, block_token_ids, block_offsets, pad_offsets,
        n_rows_pad, 0, (__nv_bfloat16*)dst);
  } else {
    if (n_rows_pad == 0) return LSRM_OK;
    tc::kv_interleave_kernel<<<(unsigned)ceil_div(n_rows_pad, 128), 256, 0, st>>>(
        src_is_bf16, src, ld_src, hkv, dh, ones_cols, nullptr, nullptr, nullptr, n_rows_pad, n,
        (__nv_bfloat16*)dst);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
