// Fused bf16 three-branch NSA attention on the 5th-gen tensor cores
// (tcgen05.mma + TMEM accumulators + cp.async.bulk K/V staging), with the
// sigmoid-gated branch merge in the epilogue.
//
// Replaces, fused: cmp_attention / sel_attention / win_attention and the
// gated sum of combine_nsa_branches (lsrm/nsa_attention.py:84-112,157-207,
// 266-284).  The W_o projection stays a plain GEMM.
//
// One persistent launch runs the four uses of a layer
// (lsrm_nsa_attention_tc_multi): work items (use, query tile, kv head) are
// claimed from a heaviest-first queue with an atomic counter.  A query tile
// is T = 128/G tokens (G = hq/hkv) in a per-use permuted order: signature-
// sorted within each query block, or across blocks for cross uses; the MMA
// M dimension is its 128 (token, q-head-in-group) rows.  Each item streams
// key chunks of <= 128 keys, branch after branch:
//   cmp : all compressed rows (one per occupied KV block),
//   sel : the sorted union of the tile tokens' selected blocks; a row sees
//         only the 16-key groups of blocks ITS token selected,
//   win : the own block (self uses), or each token's own block (own_rows).
// Block padding needs no masks: padding K rows repeat the block's first key
// and padding V rows (with their ones column) are zero.
//
// CTA = NP = 2 independent pipelines (d_h = 32), each: 4 softmax warps
// (thread = TMEM lane = one row, all keys of a chunk: two-pass max / exp2 in
// 32-key pieces, running max with 2^8 headroom, bf16 P stored to TMEM, gate +
// merge at branch ends into an f16 TMEM accumulator), 1 producer warp (tile
// unions, chunk plans, bulk copies into a 3-stage K/V ring), 1 MMA warp
// (S(c+1) = Q K^T once S(c) is in registers; [O | rowsum] += P.[V | ones] in
// TS mode once P(c) is written).  The two pipelines' phases interleave on
// each SMSP.  TMEM per pipeline: S 128 + P 64 + [O|rowsum] 48 + merge 16.
// mbarriers: kv_full/kv_empty (ring), s_full/s_free, p_full, o_full,
// q_full/q_empty; phases follow a chunk counter all roles advance alike.
//
// Build switches (-D...): LSRM_POLY_PER16 (exponentials on the FMA pipe),
// LSRM_STAGES, LSRM_NK / LSRM_NP, LSRM_HEADPAIR; LSRM_TRACE for
// tools/attn_trace.py.  The variants measured slower over the two rounds
// (split rows, double-buffered S, held S pieces, ping-pong, per-group skips,
// split epilogue, one-pass streaming, early S release, FMA sigmoid, ...) are
// recorded in DESIGN.md §4 with their numbers and removed from the code.
//
// SMEM operand layout: 8x8 "core matrices" of 128 contiguous bytes,
// SWIZZLE_NONE canonical layouts (cute mma_sm100_desc.hpp):
//   K-major  Q, K : element (row, k) at (row/8)*RS + (k/8)*64 + (row%8)*8 + k%8
//   MN-major V    : the same storage read with N = head dim, K = keys.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "tcgen05.cuh"

namespace lsrm {
namespace tc {

constexpr int kM = 128;          // MMA rows per head-tile
// LSRM_NK: keys per chunk of the default layout (128).  LSRM_NK = 64 with
// LSRM_NP = 2 measured 1.13 -> 1.35 ms (chunk overhead); three pipelines
// (which 64-key chunks would let TMEM hold: 3 x 160 columns) do not launch:
// 18 warps put 5 on some SMSP, capping registers at 96 (spills).
#ifndef LSRM_NK
#define LSRM_NK 128
#endif
#ifndef LSRM_NP
#define LSRM_NP 2
#endif
static_assert(LSRM_NP == 1 || LSRM_NP == 2, "LSRM_NP: 1 or 2 pipelines per CTA");
constexpr int kNK = LSRM_NK;
constexpr int kGroups = kNK / 16;
constexpr int kMaxEnt = 256;     // tile tokens * selected rows


// Optional event trace (debug): CTA 0 stamps clock64() per chunk and event.
__device__ long long* g_trace = nullptr;
constexpr int kTraceEv = 32, kTraceChunks = 256;
__device__ __forceinline__ void trace(long long* tr, uint32_t c, int ev) {
#ifdef LSRM_TRACE
  if (tr && c < (uint32_t)kTraceChunks) tr[c * kTraceEv + ev] = clock64();
#endif
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
  const int32_t* perm;   // optional: tile position -> query row (rows[] are in tile order)
  const int32_t* count;
  int kmax;
  const __nv_bfloat16* gl;
  int64_t ld_gl, gcol0;
  const float* gbias;
  int n_gates;
  __nv_bfloat16* out;
  int br_first;   // first branch this use's items run (2: window only)
  int accum;      // add the gated merge to `out` instead of storing it
  const int32_t* own_rows;   // optional [nq] (tile order): each token's own kv row;
                             // the window branch then spans the tile's distinct own blocks
  int q_tma;                 // 1: Q tiles by TMA through tmq (G % 8 == 0)
  // optional (training forward): each branch's normalized output, f32
  // [n_gates][nq][hq*DH], and its log-sum-exp of the scaled logits (natural
  // log), f32 [n_gates][nq][hq]
  float* o_br;
  float* lse_br;
  // Q as a 5-D tensor map {d%8, g%8, d/8, g/8, row} (strides 1, DH, 8, 8 DH,
  // ld_q elements): the box of one token and 8k q-heads lands in shared
  // memory directly in the UMMA K-major core-matrix layout
  alignas(64) CUtensorMap tmq;
};

// One launch: up to kMaxUses NSA uses (same head geometry).  order == nullptr:
// static round-robin over use 0's items.  Otherwise a work queue: order[i] =
// (use << 28) | item, heaviest first (LPT); pipeline p takes item p, then
// n_pipes + atomicAdd(counter, 1), ... (counter zeroed before the launch).
constexpr int kMaxUses = 4;
struct Launch {
  Params use[kMaxUses];
  int n_uses;
  const int32_t* order;
  int64_t n_order;
  int* counter;
};

// Build-time variants (measured against each other on the GPU; the variants
// that lost were removed and are listed in DESIGN.md §4): the K/V ring depth.
#ifndef LSRM_STAGES
#define LSRM_STAGES 3
#endif
constexpr int kStages = LSRM_STAGES;   // K/V ring depth (each stage holds every head of the item)
// gate biases staged in shared memory as [n_gates * hq][DH + 1] (padded rows:
// the 16 heads of a warp hit 16 banks) when they fit, else read from global
constexpr int kBiasMax = LSRM_STAGES <= 3 ? 3328 : 4;
constexpr int kOnesCols = 16;    // extra V columns holding 1 (valid key) / 0 (padding)
constexpr int kBitmapWords = 512;  // union bitmap: up to 16384 occupied KV blocks


__device__ __forceinline__ float max16(const uint32_t* s) {
  const float* x = reinterpret_cast<const float*>(s);
  float a = fmaxf(fmaxf(x[0], x[1]), x[2]), b = fmaxf(fmaxf(x[3], x[4]), x[5]);
  float d = fmaxf(fmaxf(x[6], x[7]), x[8]), e = fmaxf(fmaxf(x[9], x[10]), x[11]);
  float f = fmaxf(fmaxf(x[12], x[13]), x[14]);
  a = fmaxf(fmaxf(a, b), d);
  e = fmaxf(fmaxf(e, f), x[15]);
  return fmaxf(a, e);
}
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// exp2 on the FMA pipe: x = j + f (j = round(x), |f| <= 1/2), 2^f by a
// degree-3 polynomial (rel. error < 7e-4, a sixth of a bf16 ulp), 2^j added to
// the exponent bits.  x is clamped to >= -125 (masked -inf -> ~2e-38, which
// contributes nothing measurable); x <= 8 by the softmax headroom.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;   // 1.5 * 2^23: round to integer in the mantissa
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.0555041086648216f, 0.2402264923172690f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// Of every 16 exponentials, kPolyPer16 go to the FMA pipe (ex2_poly) and the
// rest to the MUFU, whose issue rate (16/clk/SM) bounds the kernel.
// same-box A/B (round 2, profiles/r2/ab_poly1_vs_default.txt): 1 of 16 on
// the FMA pipe, attention 1.149 -> 1.132 ms, layer 1.557 -> 1.544 ms; 2/16
// and 3/16 lose again (C3 sweep).  The exp phase is MUFU-bound while both
// pipelines' warps are in it.
#ifndef LSRM_POLY_PER16
#define LSRM_POLY_PER16 1
#endif
constexpr int kPolyPer16 = LSRM_POLY_PER16;
__device__ __forceinline__ float ex2_mixed(float x, int j) {
  return j >= 16 - kPolyPer16 ? ex2_poly(x) : ex2(x);
}
// Gate sigmoid of the branch epilogue: 0.5 + 0.5 tanh(z / 2), one MUFU op
// (an FMA-pipe version measured slower: the epilogue is on the softmax
// warps' critical path).
__device__ __forceinline__ float sigmoid_gate(float z) {
  return fmaf(0.5f, tanh_approx(0.5f * z), 0.5f);
}

// 16 logits -> 8 words of packed bf16 exp2(s * sl2 + nb)
__device__ __forceinline__ void exp16(const uint32_t* s, float sl2, float nb, uint32_t* w) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    w[j] = pack_bf16(ex2_mixed(fmaf(__uint_as_float(s[2 * j]), sl2, nb), 2 * j),
                     ex2_mixed(fmaf(__uint_as_float(s[2 * j + 1]), sl2, nb), 2 * j + 1));
}
__device__ __forceinline__ void zero8(uint32_t* w) {
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = 0u;
}

// One chunk of <= 128 keys as the softmax and MMA warps see it.  The
// producer resolves visibility per 16-key group: gnv = valid keys in the
// group, gmask = tile tokens allowed to see it.
struct __align__(16) ChunkDesc {
  int ncols, branch, flags, q_first;   // flags: kF* bits | NSA use << 16
  int q_cnt, h, qb, item_seq;
  uint32_t gmask[kGroups];             // producer scratch: tokens allowed per group
  int32_t gnv[kGroups];                // valid keys per group (tail groups: < 16)
  uint8_t tokvis[32];                  // per tile token: groups it sees (bit g)
  int32_t tok[32];                     // per tile token: its query row (output / gates)
};
constexpr int kFFirstBranch = 1, kFLastBranch = 2, kFFirstItem = 4, kFLastItem = 8,
              kFLastOverall = 16;

// TMEM columns of one head-tile: S (f32 logits), P (bf16 packed), the branch
// accumulator [O | rowsum] of P.[V | ones], and the gated merge (f16 packed).
template <int DH>
struct HeadCols {
  static constexpr int VW = DH + kOnesCols;
  static constexpr uint32_t kS = 0, kP = kNK, kO = kNK + kNK / 2, kMerged = kO + VW;
  static constexpr int kTotal = kNK + kNK / 2 + VW + DH / 2;
};
template <int DH, int HP, int NP>
constexpr int tmem_alloc_cols() {
  int n = NP * HP * HeadCols<DH>::kTotal, a = 32;
  while (a < n) a *= 2;
  return a;
}

// Shared memory of one pipeline (producer + MMA warp(s) + softmax warps that
// stream their own items).
template <int DH, int HP>
struct alignas(128) Pipe {   // 128-byte aligned: q is a TMA destination
  __nv_bfloat16 q[2][HP][kM * DH];
  __nv_bfloat16 k[kStages][HP][kNK * DH];
  __nv_bfloat16 v[kStages][HP][kNK * (DH + kOnesCols)];   // [V | ones] rows
  __nv_bfloat16 gate[HP][kM * DH];  // per row: gate logits of the branch that just ended
  int32_t ent[kMaxEnt];          // selected rows of the tile tokens, [t][kmax]
  uint32_t bitmap[kBitmapWords]; // selected-row bitmap of the current item
  int32_t wpre[kBitmapWords];    // rank of the first set bit of each word
  int32_t uni_row[kMaxEnt];      // sorted union of selected rows
  uint32_t uni_mask[kMaxEnt];    // per union slot: tokens that selected it
  int64_t seg_lo[kMaxEnt + 1];   // per union slot (+1: own block) padded first row
  int32_t seg_plen[kMaxEnt + 1];
  int32_t seg_occ[kMaxEnt + 1];
  int32_t seg_cum[kMaxEnt];
  int64_t wseg_lo[32];            // window segments: the tile tokens' distinct own blocks
  int32_t wseg_plen[32], wseg_occ[32], wseg_cum[32];
  uint32_t wseg_mask[32];
  ChunkDesc desc[kStages];
  uint64_t kv_full[kStages], kv_empty[kStages], s_full[2 * HP], s_free[HP], p_full[2 * HP],
      o_full[HP],
      q_full[2], q_empty[2];
};

template <int DH, int HP, int NP>
struct Smem {
  Pipe<DH, HP> pipe[NP];
  float bias[kBiasMax];             // gate biases, padded rows (if they fit)
  uint32_t tmem_base;
};

// per pipeline: 4 softmax warps per head-tile, 1 producer, 1 MMA warp per head-tile
template <int HP, int NP>
constexpr int threads_of() { return 32 * NP * (4 * HP + HP + 1); }

// Work item = (query tile, group of HP kv heads).  The HP head-tiles share the
// chunk plan (same tokens, same union of selected blocks) but not K/V, so
// their softmax warpgroups run out of phase: while one computes
// exponentials, the tensor core serves the other (ping-pong).
//
// Warps: 4*HP softmax (warpgroup hh = head-tile hh; thread = TMEM lane = one
// row, all 128 keys of a chunk, so no cross-warp max exchange), 1 producer,
// 1 MMA issuer.
//
// NP independent pipelines per CTA (own items, producer, ring, MMA warp(s),
// softmax warps, TMEM columns): their warps share each SMSP but not a chunk
// plan, so one pipeline's loads / maxima / epilogue overlap the other's
// exponentials instead of running in lockstep.  Odd pipelines walk their item
// list backwards so the two of a CTA start on different tiles.
template <int DH, int HP, int NP>
__global__ void __launch_bounds__(threads_of<HP, NP>(), 1) nsa_fused_kernel(const __grid_constant__ Launch L) {
  const Params& P = L.use[0];   // head geometry (shared by all uses); static mode's use
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem<DH, HP, NP>& SM = *reinterpret_cast<Smem<DH, HP, NP>*>(smem_raw);
  using HCols = HeadCols<DH>;
  constexpr int VW = HCols::VW, HC = HCols::kTotal;
  constexpr int kSoftPerPipe = 4 * HP;
  constexpr int kSoftWarps = kSoftPerPipe * NP, kProducerWarp = kSoftWarps;
  constexpr int kAlloc = tmem_alloc_cols<DH, HP, NP>();
  static_assert(kAlloc <= 512, "TMEM budget");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = P.hq / P.hkv, T = kM / G;
  const int d_model = P.hq * DH;
  const int n_hgroups = P.hkv / HP;
  const bool dyn = L.order != nullptr;
  const int64_t n_items = dyn ? L.n_order : P.n_tiles * n_hgroups;
  // role -> pipeline: softmax warps [0, 4*HP*NP), producers, then MMA warps
  const int pipe_id = warp < kSoftWarps ? warp / kSoftPerPipe
                      : (warp < kSoftWarps + NP ? warp - kSoftWarps
                                                : (warp - kSoftWarps - NP) / HP);
  Pipe<DH, HP>& S = SM.pipe[pipe_id];
  const int64_t n_pipes = (int64_t)gridDim.x * NP;
  const int64_t gp = (int64_t)blockIdx.x * NP + pipe_id;
  // items of this pipeline (static mode); in queue mode only "any" matters:
  // every pipeline's first item is its own index gp
  const int64_t m_items = gp < n_items ? (dyn ? 1 : (n_items - gp + n_pipes - 1) / n_pipes) : 0;
  auto item_of = [&](int64_t k) -> int64_t {
    return (pipe_id & 1) ? gp + (m_items - 1 - k) * n_pipes : gp + k * n_pipes;
  };

  if (tid == 0) {
    for (int pp = 0; pp < NP; ++pp) {
    Pipe<DH, HP>& S = SM.pipe[pp];
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&S.kv_full[i], 1);
      mbar_init(&S.kv_empty[i], HP);   // one commit per head-tile's MMA warp
    }
    for (int hh = 0; hh < HP; ++hh) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&S.s_full[2 * hh + b], 1);
        mbar_init(&S.p_full[2 * hh + b], 128);
      }
      mbar_init(&S.s_free[hh], 128);
      mbar_init(&S.o_full[hh], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.q_full[i], 1);
      mbar_init(&S.q_empty[i], HP);
    }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&SM.tmem_base)),
                 "r"(kAlloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < NP * kBitmapWords; i += blockDim.x)
    SM.pipe[i / kBitmapWords].bitmap[i % kBitmapWords] = 0u;
  const bool bias_smem = !dyn && P.gbias && P.n_gates * P.hq * (DH + 1) <= kBiasMax;
  if (bias_smem)
    for (int i = tid; i < P.n_gates * d_model; i += blockDim.x)
      SM.bias[(i / DH) * (DH + 1) + i % DH] = P.gbias[i];
  const float* const bias_all = bias_smem ? SM.bias : P.gbias;
  const int bias_ld = bias_smem ? DH + 1 : DH;   // floats per (branch, head) row
  fence_async_smem();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = SM.tmem_base + (uint32_t)(pipe_id * HP * HC);   // this pipeline's columns
  long long* const trp = (blockIdx.x == 0 && pipe_id == 0) ? g_trace : nullptr;  // debug trace
#ifdef LSRM_TRACE
  // per-pipeline start / end (globaltimer ns) after the chunk trace: the
  // tail of the LPT queue (tools/attn_trace.py)
  auto gtime = []() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (g_trace && (tid & 31) == 0 && warp % kSoftPerPipe == 0 && gp < 1024)
    g_trace[kTraceChunks * kTraceEv + 2 * gp] = gtime();
#endif

  if (m_items == 0) {
    // this pipeline has no work (small launches)
  } else if (warp >= kProducerWarp && warp < kProducerWarp + NP) {
    // ===================== producer: Q tiles, unions, chunk plans, K/V copies
    uint32_t c = 0;
    int it = 0;
    const uint32_t all_tok = T >= 32 ? 0xffffffffu : ((1u << T) - 1u);
    int64_t cur = dyn ? gp : 0;   // queue mode: global queue position; static: k
    for (;;) {
      if (!dyn && cur >= m_items) break;
      if (dyn && cur >= n_items) break;
      int64_t nxt = cur + 1;
      if (dyn) {   // claim the next queue entry now, so the last item is known
        if (lane == 0) nxt = n_pipes + (int64_t)atomicAdd(L.counter, 1);
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
      }
      const bool last_item = dyn ? nxt >= n_items : nxt >= m_items;
      int use = 0;
      int64_t item;
      if (dyn) {
        const int32_t code = L.order[cur];
        use = code >> 28;
        item = code & 0x0FFFFFFF;
      } else {
        item = item_of(cur);
      }
      const Params& P = L.use[use];
      const int tile = (int)(item / n_hgroups), h0 = (int)(item % n_hgroups) * HP;
      const int q_first = P.tiles[4 * tile], q_cnt = P.tiles[4 * tile + 1],
                own = P.tiles[4 * tile + 2];
      const int qb = it & 1;
      // query row of tile token `lane` (constant over the item's chunks)
      const int64_t my_tok =
          lane < q_cnt ? (P.perm ? (int64_t)P.perm[q_first + lane] : (int64_t)(q_first + lane)) : 0;
      // ---- selected rows of the tile tokens (resolved rows are -1 padded)
      // (window-only items need no union of selected blocks)
      const int n_ent = P.br_first <= 1 ? T * P.kmax : 0, n_valid_ent = q_cnt * P.kmax;
      const int32_t* rows_t = P.rows + (int64_t)q_first * P.kmax;
      for (int i = lane; i < n_ent; i += 32) {
        const int r = i < n_valid_ent ? rows_t[i] : -1;
        S.ent[i] = r;
        if (r >= 0) atomicOr(&S.bitmap[r >> 5], 1u << (r & 31));
      }
      // ---- Q tiles of the HP heads -> sQ[qb], once the MMAs of item it-2 are
      //      done with the buffer: TMA boxes (one per token and head-tile,
      //      rows past the tile read out of bounds -> zeros), else cp.async
      if (it >= 2) mbar_wait(&S.q_empty[qb], ((it >> 1) - 1) & 1);
      if (P.q_tma) {
        if (lane == 0) mbar_expect_tx(&S.q_full[qb], (uint32_t)(HP * kM * DH * 2));
        __syncwarp();
        if (lane < T) {
          const int32_t row = lane < q_cnt ? (int32_t)my_tok : (int32_t)P.nq;
#pragma unroll
          for (int hh = 0; hh < HP; ++hh)
            tma_load_5d(&S.q[qb][hh][lane * G * DH], &P.tmq, 0, 0, 0, ((h0 + hh) * G) / 8, row,
                        &S.q_full[qb]);
        }
      } else {
        constexpr int kQChunks = kM * (DH / 8);
#pragma unroll 4
        for (int i = lane; i < HP * kQChunks; i += 32) {
          const int hh = i / kQChunks, rem = i % kQChunks;
          const int m = rem / (DH / 8), cc = rem % (DH / 8);
          const int tt = m / G, gg = m % G;
          const bool ok = tt < q_cnt;
          const int64_t qrow = __shfl_sync(0xffffffffu, my_tok, tt & 31);
          const __nv_bfloat16* src =
              P.q + (ok ? qrow * P.ld_q + ((h0 + hh) * G + gg) * DH + cc * 8 : 0);
          cp_async16(&S.q[qb][hh][(m / 8) * (8 * DH) + cc * 64 + (m % 8) * 8], src,
                     ok ? 16u : 0u);
        }
        cp_async_wait_all();
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.q_full[qb]);
      }
      // ---- sorted union = set bits of the bitmap in order
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
      for (int i = lane; i < n_ent; i += 32) {   // token masks: entry i is token i / kmax
        const int r = S.ent[i];
        if (r >= 0) {
          const int w = r >> 5;
          const int rank = S.wpre[w] + __popc(S.bitmap[w] & ((1u << (r & 31)) - 1u));
          atomicOr(&S.uni_mask[rank], 1u << (i / P.kmax));
        }
      }
      for (int u = lane; u < nu; u += 32) {   // segment geometry of every union slot
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
      // per-token own rows: one window segment per distinct own block of the
      // tile (in token order), each seen by the tokens that own it
      int n_wseg = 1;
      int64_t total_win = 0;
      if (P.own_rows && P.n_gates == 3) {
        const bool tv = lane < q_cnt;
        const int r = tv ? P.own_rows[q_first + lane] : -1;
        const uint32_t vmask = __ballot_sync(0xffffffffu, tv);
        const uint32_t same = __match_any_sync(0xffffffffu, r) & vmask;
        const bool leader = tv && (__ffs(same) - 1) == lane;
        const uint32_t leaders = __ballot_sync(0xffffffffu, leader);
        n_wseg = __popc(leaders);
        const int idx = __popc(leaders & ((1u << lane) - 1u));
        int plen = 0;
        if (leader) {
          const int64_t a0 = P.pad_off[r], a1 = P.pad_off[r + 1];
          S.wseg_lo[idx] = a0;
          plen = (int)(a1 - a0);
          S.wseg_plen[idx] = plen;
          S.wseg_occ[idx] = (int)(P.kv_off[r + 1] - P.kv_off[r]);
          S.wseg_mask[idx] = same;
        }
        // segment starts: exclusive prefix over the leaders in token order
        int incl = plen;
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (leader) S.wseg_cum[idx] = incl - plen;
        total_win = __shfl_sync(0xffffffffu, incl, 31);
      }
      __syncwarp();
      for (int k = 0; k < per_w; ++k) {  // clear the bitmap for the next item
        const int w = lane * per_w + k;
        if (w < n_words) S.bitmap[w] = 0u;
      }
      __syncwarp();
      int total_sel;   // exclusive prefix of the union segments' padded lengths
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
      //      piece's K and V bulk copies for every head of the item
      const int64_t cmp_rows = (P.n_blocks + 15) / 16 * 16;
      for (int br = P.br_first; br < P.n_gates; ++br) {
        const bool win_tok = br == 2 && P.own_rows != nullptr;
        const int n_seg = br == 1 ? nu : (win_tok ? n_wseg : 1);
        const int64_t total = br == 0 ? cmp_rows
                              : (br == 1 ? total_sel : (win_tok ? total_win : S.seg_plen[kMaxEnt]));
        const int64_t head_rows = br == 0 ? cmp_rows : P.n_rows_pad;
        const __nv_bfloat16* kb = (br == 0 ? P.kc_il : P.k_il) + (int64_t)h0 * head_rows * DH;
        const __nv_bfloat16* vb = (br == 0 ? P.vc_il : P.v_il) + (int64_t)h0 * head_rows * VW;
        int cur_seg = 0;   // first segment not yet consumed by earlier chunks
        for (int64_t start = 0; start < total; start += kNK) {
          const int64_t end = lmin(start + kNK, total);
          const int st = c % kStages;
          if (c >= kStages) mbar_wait(&S.kv_empty[st], ((c / kStages) - 1) & 1);
          if (lane == 0) trace(trp, c, 0);
          ChunkDesc& D = S.desc[st];
          const int s = cur_seg + lane;
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
            } else if (win_tok) {
              lo = S.wseg_lo[s]; plen = S.wseg_plen[s]; occ = S.wseg_occ[s]; cs = S.wseg_cum[s];
              tm = S.wseg_mask[s];
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
          __syncwarp();
          const int n_grp = (int)(end - start) / 16;
          if (lane == 0) {
            const bool li = end == total && br == P.n_gates - 1;
            D.ncols = (int)(end - start);
            D.branch = br;
            D.flags = (start == 0 ? kFFirstBranch : 0) | (end == total ? kFLastBranch : 0) |
                      (br == P.br_first && start == 0 ? kFFirstItem : 0) |
                      (li ? kFLastItem : 0) |
                      (li && last_item ? kFLastOverall : 0) | (use << 16);
            D.q_first = q_first;
            D.q_cnt = q_cnt;
            D.h = h0;
            D.qb = qb;
            D.item_seq = it;
          }
          {   // per token: the groups it sees (padding rows of the tile see none);
              // the chunk's group table read with four 16-byte loads
            static_assert(kGroups % 4 == 0 && kGroups <= 8, "tokvis: 4 or 8 groups per chunk");
            uint32_t gm[kGroups];
            int gn[kGroups];
#pragma unroll
            for (int q = 0; q < kGroups / 4; ++q) {
              const uint4 mq = *reinterpret_cast<const uint4*>(&D.gmask[4 * q]);
              const int4 nq = *reinterpret_cast<const int4*>(&D.gnv[4 * q]);
              gm[4 * q] = mq.x; gm[4 * q + 1] = mq.y; gm[4 * q + 2] = mq.z; gm[4 * q + 3] = mq.w;
              gn[4 * q] = nq.x; gn[4 * q + 1] = nq.y; gn[4 * q + 2] = nq.z; gn[4 * q + 3] = nq.w;
            }
            uint32_t v = 0;
#pragma unroll
            for (int gi = 0; gi < kGroups; ++gi)
              v |= (gi < n_grp && gn[gi] > 0 ? (gm[gi] >> (lane & 31)) & 1u : 0u) << gi;
            D.tokvis[lane] = (uint8_t)(lane < q_cnt ? v : 0u);
            D.tok[lane] = (int32_t)my_tok;
          }
          __syncwarp();
          if (lane == 0)
            mbar_expect_tx(&S.kv_full[st],
                           (uint32_t)(end - start) * HP * (uint32_t)(2 * DH + 2 * VW));
          __syncwarp();
          if (ov) {
#pragma unroll
            for (int hh = 0; hh < HP; ++hh) {
              bulk_g2s(&S.k[st][hh][col * DH], kb + ((int64_t)hh * head_rows + src) * DH,
                       ncols * DH * 2u, &S.kv_full[st]);
              bulk_g2s(&S.v[st][hh][col * VW], vb + ((int64_t)hh * head_rows + src) * VW,
                       ncols * VW * 2u, &S.kv_full[st]);
            }
          }
          cur_seg += __popc(__ballot_sync(0xffffffffu, done));
          ++c;
        }
      }
      __syncwarp();
      cur = nxt;
      ++it;
    }
  } else if (warp >= kProducerWarp + NP) {
    // ===================== MMA issuer of head-tile hh (one warp per head-tile,
    // so neither head-tile's MMAs wait behind the other's barriers)
    const int hh = (warp - kProducerWarp - NP) % HP;
    const uint32_t id_pv = idesc_bf16(kM, VW, 1);   // [O | rowsum] += P . [V | ones]
    const uint32_t t_s = tmem + hh * HC + HCols::kS, t_p = tmem + hh * HC + HCols::kP,
                   t_o = tmem + hh * HC + HCols::kO;
    // S = Q K^T for chunk cc into this head-tile's S columns
    auto issue_qk = [&](uint32_t cc) {
      const int st = cc % kStages;
      const ChunkDesc& D = S.desc[st];
      mbar_wait(&S.kv_full[st], (cc / kStages) & 1);
#ifndef LSRM_TRACE_LD
      if (lane == 0 && hh == 0) trace(trp, cc, 1);
#endif
      if (D.flags & kFFirstItem) mbar_wait(&S.q_full[D.qb], (D.item_seq >> 1) & 1);
      tc_after_sync();
      const uint32_t id = idesc_bf16(kM, D.ncols, 0);
      const uint64_t a0 = sdesc(smem_u32(S.q[D.qb][hh]), 128, 16 * DH);
      const uint64_t b0 = sdesc(smem_u32(S.k[st][hh]), 128, 16 * DH);
      if (elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          mma_bf16(t_s, a0 + (uint64_t)(kk * 16), b0 + (uint64_t)(kk * 16), id, kk > 0);
        mma_commit(&S.s_full[2 * hh]);
      }
      __syncwarp();
      if (lane == 0 && hh == 0) trace(trp, cc, 2);
    };
    issue_qk(0);
    // per chunk: S(c+1) = Q K^T as soon as the softmax has S(c) in registers
    // (s_free), then PV(c) accumulates P(c).[V|ones] into the branch's O as
    // soon as P(c) is written (p_full)
    uint32_t c = 0;
    for (;;) {
      const int st = c % kStages;
      const ChunkDesc& D = S.desc[st];
      const int fl = D.flags;
      const bool last = fl & kFLastOverall, last_in_item = fl & kFLastItem;
      const uint32_t acc0 = (fl & kFFirstBranch) ? 0u : 1u;
      const int nk = D.ncols / 16;
      const int qb = D.qb;
      if (!last) {
        mbar_wait(&S.s_free[hh], c & 1);
        issue_qk(c + 1);
      }
      mbar_wait(&S.p_full[2 * hh], c & 1);
      if (lane == 0 && hh == 0) trace(trp, c, 5);
      tc_after_sync();
      const uint64_t vdesc = sdesc(smem_u32(S.v[st][hh]), 16 * VW, 128);
      if (elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < kGroups; ++kk)
          if (kk < nk)
            mma_bf16_ts(t_o, t_p + kk * 8, vdesc + (uint64_t)(kk * 2 * VW), id_pv,
                        kk > 0 ? 1u : acc0);
        mma_commit(&S.o_full[hh]);
        if (last_in_item) mma_commit(&S.q_empty[qb]);
        mma_commit(&S.kv_empty[st]);
      }
      __syncwarp();
      if (lane == 0 && hh == 0) trace(trp, c, 6);
      ++c;
      if (last) break;
    }
    __syncwarp();
  } else {
    // ===================== softmax / epilogue (warpgroup hh = head-tile hh)
    const int hh = (warp % kSoftPerPipe) / 4, q4 = warp & 3;
    const int m = q4 * 32 + lane;
    const int t = m / G, g_in = m % G;
    const uint32_t tS = tmem + ((uint32_t)(q4 * 32) << 16) + hh * HC;
    const uint32_t tP = tS + HCols::kP, tO = tS + HCols::kO, tM = tS + HCols::kMerged;
    const float sl2 = 1.4426950408889634f / sqrtf((float)DH);
    const float kNegInf = -__builtin_huge_valf();
    // O accumulates in TMEM over a branch relative to the running max m_run;
    // m_run only moves (and O is rescaled) when the chunk max exceeds it by
    // more than 2^kHeadroom, so P <= 2^kHeadroom and rescales are rare.
#ifndef LSRM_HEADROOM   // 16 measured identical (rescales are rare either way)
#define LSRM_HEADROOM 8
#endif
    constexpr float kHeadroom = (float)LSRM_HEADROOM;
    float m_run = kNegInf;
    // finished-branch state: its epilogue runs in the next chunk, before that
    // chunk's PV overwrites O
    int br_pend = 0, head_pend = 0, use_pend = 0;
    float m_pend = 0.f;   // the finished branch's running max (for its lse)
    // the item's first branch (items may start at the window branch); a
    // branch that is its item's first starts the merge instead of adding
    int item_br0 = 0;
    bool firstbr_pend = true;
    bool lastit_pend = false, rowok_pend = false, epi_pend = false;
    int64_t tok_pend = 0;
    __nv_bfloat16* const gate_s = &S.gate[hh][m * DH];   // this row's staged gate logits
    uint32_t c = 0;

    // gate + merge of a finished branch (nsa_attention.py:266-284); the
    // running merge is f16 in TMEM; at an item end the merged row is stored.
    // epi_load reads the branch's O and row sum (this must precede PV(c),
    // which overwrites O); epi_finish does the gate, the merge and the stores.
    auto epi_load = [&](uint32_t pc, uint32_t* eo) {
      mbar_wait(&S.o_full[hh], pc & 1);   // PV(pc) complete
      if (tid == 0) trace(trp, pc, 7);
      tc_after_sync();
      tmem_ld_cols<1>(tO + DH, eo + DH);
#pragma unroll
      for (int cq = 0; cq < DH; cq += 16) tmem_ld16_nowait(tO + cq, eo + cq);
      tmem_wait_ld();
    };
    auto epi_finish = [&](const uint32_t* eo) {
      cp_async_wait_all();                // gate logits staged by this thread
      const float inv = rowok_pend ? 1.f / __uint_as_float(eo[DH]) : 0.f;
      const float* bp =
          bias_all ? bias_all + ((int64_t)br_pend * P.hq + head_pend) * bias_ld : nullptr;
      const Params& PB = L.use[use_pend];
      if (PB.o_br && rowok_pend) {   // training forward: the branch's own output and lse
        const int64_t brow = (int64_t)br_pend * PB.nq + tok_pend;
        float4* ob = reinterpret_cast<float4*>(PB.o_br + brow * d_model + head_pend * DH);
#pragma unroll
        for (int j = 0; j < DH / 4; ++j)
          ob[j] = make_float4(__uint_as_float(eo[4 * j]) * inv, __uint_as_float(eo[4 * j + 1]) * inv,
                              __uint_as_float(eo[4 * j + 2]) * inv,
                              __uint_as_float(eo[4 * j + 3]) * inv);
        PB.lse_br[brow * P.hq + head_pend] =
            (m_pend + __log2f(__uint_as_float(eo[DH]))) * 0.6931471805599453f;
      }
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 16) {   // 16 columns at a time (registers)
        uint32_t r[16], mr[8];
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = eo[c0 + j];
        if (!firstbr_pend) {
          tmem_ld_cols<8>(tM + c0 / 2, mr);
          tmem_wait_ld();
        }
#pragma unroll
        for (int k8 = 0; k8 < 2; ++k8) {
          const uint4 raw = *reinterpret_cast<const uint4*>(gate_s + c0 + 8 * k8);
          const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int cj = 8 * k8 + j;
            const float z = __bfloat162float(hv[j]) + (bp ? bp[c0 + cj] : 0.f);
            float v = rowok_pend ? __uint_as_float(r[cj]) * inv * sigmoid_gate(z) : 0.f;
            if (!firstbr_pend) {
              const __half2 hm = *reinterpret_cast<const __half2*>(&mr[cj / 2]);
              v += (cj & 1) ? __high2float(hm) : __low2float(hm);
            }
            r[cj] = __float_as_uint(v);
          }
        }
        if (lastit_pend) {
          if (rowok_pend) {
            __nv_bfloat16* op = L.use[use_pend].out + tok_pend * d_model + head_pend * DH + c0;
#pragma unroll
            for (int k8 = 0; k8 < 2; ++k8) {
              float* v = reinterpret_cast<float*>(r + 8 * k8);
              if (L.use[use_pend].accum) {   // second launch: add to the first's merge
                const uint4 old = *reinterpret_cast<const uint4*>(op + 8 * k8);
                const __nv_bfloat16* ov = reinterpret_cast<const __nv_bfloat16*>(&old);
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] += __bfloat162float(ov[j]);
              }
              uint4 w;
              w.x = pack_bf16(v[0], v[1]);
              w.y = pack_bf16(v[2], v[3]);
              w.z = pack_bf16(v[4], v[5]);
              w.w = pack_bf16(v[6], v[7]);
              *reinterpret_cast<uint4*>(op + 8 * k8) = w;
            }
          }
        } else {
          uint32_t w[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const __half2 h2 = __floats2half2_rn(__uint_as_float(r[2 * j]),
                                                 __uint_as_float(r[2 * j + 1]));
            w[j] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          tmem_st8(tM + c0 / 2, w);
        }
      }
      if (!lastit_pend) tmem_wait_st();
    };
    auto epilogue = [&](uint32_t pc) {
      uint32_t eo[DH + 1];
      epi_load(pc, eo);
      epi_finish(eo);
    };

    for (;;) {
      mbar_wait(&S.s_full[2 * hh], c & 1);
      if (tid == 0) trace(trp, c, 3);
      tc_after_sync();
      // chunk plan (a few wide shared loads) and S pieces 0,1 in flight together
      const ChunkDesc& D = S.desc[c % kStages];
      const int4 hdr0 = *reinterpret_cast<const int4*>(&D.ncols);
      const int4 hdr1 = *reinterpret_cast<const int4*>(&D.q_cnt);
      const uint32_t visb = D.tokvis[t];
      const int ncols = hdr0.x;
      uint32_t sa[32], sb[32];
      tmem_ld32(tS + HCols::kS, sa);
      if (ncols > 32) tmem_ld32(tS + HCols::kS + 32, sb);
#ifdef LSRM_TRACE_LD
      tmem_wait_ld();
      if (tid == 0) trace(trp, c, 1);
#endif
      const int br = hdr0.y, fl = hdr0.z, use_c = fl >> 16;
      const bool first_br = fl & kFFirstBranch, last_br = fl & kFLastBranch,
                 last_it = fl & kFLastItem, last_all = fl & kFLastOverall;
      if (fl & kFFirstItem) item_br0 = br;
      const bool row_ok = t < hdr1.x;
      const int64_t tok = D.tok[t];
      const int head = (hdr1.y + hh) * G + g_in;
      // `live` groups are seen by some row of this warp (others are skipped,
      // P = 0); a row sees a group if its token selected it (visb).  Block
      // padding needs no mask: padding K rows repeat a real key of the block
      // (no effect on the max) and padding V rows are zero.
      const uint32_t live = __reduce_or_sync(0xffffffffu, visb);
      if (first_br) m_run = kNegInf;
      float mx = kNegInf;
      tmem_wait_ld();
      if (tid == 0) trace(trp, c, 8);
      // pass 1: straight-line group maxima; groups this row does not see are
      // not selected
#define LSRM_MAX(arr, off, gi)                                  \
  {                                                             \
    const float g_ = max16(arr + (off));                        \
    mx = ((visb >> (gi)) & 1u) ? fmaxf(mx, g_) : mx;            \
  }
      LSRM_MAX(sa, 0, 0)
      LSRM_MAX(sa, 16, 1)
      if (ncols > 32) {
        LSRM_MAX(sb, 0, 2)
        LSRM_MAX(sb, 16, 3)
      }
      const bool hi = ncols > 64;   // pieces 2,3 end up in registers
      if (tid == 0) trace(trp, c, 9);
      if (hi) {
        tmem_ld32(tS + HCols::kS + 64, sa);
        if (ncols > 96) tmem_ld32(tS + HCols::kS + 96, sb);
        tmem_wait_ld();
        LSRM_MAX(sa, 0, 4)
        LSRM_MAX(sa, 16, 5)
        if (ncols > 96) {
          LSRM_MAX(sb, 0, 6)
          LSRM_MAX(sb, 16, 7)
        }
      } else {
        tc_before_sync();
        mbar_arrive(&S.s_free[hh]);   // S(c) fully in registers: QK(c+1) may overwrite it
      }
#undef LSRM_MAX
      if (tid == 0) trace(trp, c, 10);
      // running max with headroom; rescale O (and its row sum) if it moves
      const float m_cand = fmaxf(m_run, mx * sl2);
      float m_use = m_run, scale = 1.f;
      bool need = false;
      if (m_run == kNegInf) {
        m_use = m_cand;
      } else if (m_cand > m_run + kHeadroom) {
        m_use = m_cand;
        scale = ex2(m_run - m_cand);
        need = true;
      }
      // PV(c-1) must be complete before P(c) overwrites P(c-1) and before O is
      // rescaled or read: waited for lazily, right before the first of those
      bool pv_done = c == 0;
      auto wait_pv = [&]() {
        if (!pv_done) {
          mbar_wait(&S.o_full[hh], (c - 1) & 1);
          tc_after_sync();
          pv_done = true;
        }
      };
      if (__any_sync(0xffffffffu, need)) {
        wait_pv();
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 16) {
          uint32_t r[16];
          tmem_ld16_nowait(tO + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * scale);
          tmem_st16(tO + c0, r);
        }
        uint32_t rl[1];
        tmem_ld_cols<1>(tO + DH, rl);
        tmem_wait_ld();
        rl[0] = __float_as_uint(__uint_as_float(rl[0]) * scale);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tO + DH),
                     "r"(rl[0])
                     : "memory");
      }
      m_run = m_use;
      if (tid == 0) trace(trp, c, 11);
      // pass 2: P = exp2(S * scale - m) as packed bf16; rows that do not see a
      // group get a -inf bias (P = 0); fully masked rows so far use m = 0;
      // 32-key pieces no row of the warp sees are zero
      const float nbv = m_use == kNegInf ? 0.f : -m_use;
      auto exp_piece = [&](const uint32_t* arr, int pc) {
        uint32_t w[16];
        if ((live >> (2 * pc)) & 3u) {
          exp16(arr, sl2, ((visb >> (2 * pc)) & 1u) ? nbv : kNegInf, w);
          exp16(arr + 16, sl2, ((visb >> (2 * pc + 1)) & 1u) ? nbv : kNegInf, w + 8);
        } else {
          zero8(w);
          zero8(w + 8);
        }
        wait_pv();
        tmem_st16(tP + 16 * pc, w);
      };
      if (hi) {
        exp_piece(sa, 2);
        if (ncols > 96) exp_piece(sb, 3);
        tmem_ld32(tS + HCols::kS, sa);   // pieces 0,1 again (both full: ncols > 64)
        tmem_ld32(tS + HCols::kS + 32, sb);
        tmem_wait_ld();
        tc_before_sync();
        mbar_arrive(&S.s_free[hh]);
        if (tid == 0) trace(trp, c, 12);
      }
      exp_piece(sa, 0);
      if (ncols > 32) exp_piece(sb, 1);
      if (tid == 0) trace(trp, c, 13);
      tmem_wait_st();
      if (tid == 0) trace(trp, c, 14);
      if (epi_pend) {   // the previous branch's O must be read before PV(c) overwrites it
        epilogue(c - 1);
        epi_pend = false;
      }
      if (tid == 0) trace(trp, c, 15);
      tc_before_sync();
      mbar_arrive(&S.p_full[2 * hh]);
      if (tid == 0) trace(trp, c, 4);
      if (last_br) {
        if (row_ok) {   // stage this branch's gate logits for its epilogue
          const Params& PU = L.use[use_c];
          const __nv_bfloat16* gp = PU.gl + tok * PU.ld_gl + PU.gcol0 + (int64_t)br * d_model +
                                    head * DH;
#pragma unroll
          for (int cq = 0; cq < DH; cq += 8) cp_async16(gate_s + cq, gp + cq, 16u);
        }
        br_pend = br;
        m_pend = m_run;
        firstbr_pend = br == item_br0;
        use_pend = use_c;
        head_pend = head;
        tok_pend = tok;
        rowok_pend = row_ok;
        lastit_pend = last_it;
        epi_pend = true;
      }
      ++c;
      if (last_all) break;
    }
    epilogue(c - 1);
#ifdef LSRM_TRACE
    if (g_trace && (tid & 31) == 0 && warp % kSoftPerPipe == 0 && gp < 1024)
      g_trace[kTraceChunks * kTraceEv + 2 * gp + 1] = gtime();
#endif
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kAlloc));
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
    } else if (ones_cols == 0 && (tok ? occ > 0 : n_plain > 0)) {
      // K padding rows repeat the set's first key: a duplicate key cannot
      // raise a row max, and its value row (V padding) is zero, so padding
      // needs no masking in the attention kernel
      int64_t row = tok ? tok[lo] : 0;
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

namespace lsrm {
namespace tc {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}
// Q tensor map of one use (see Params::tmq); G % 8 != 0 keeps the cp.async path.
static int make_q_map(Params& p, int G, int dh) {
  p.q_tma = 0;
  if (G % 8 != 0 || p.nq == 0) return LSRM_OK;
  auto fn = encode_fn();
  if (!fn) return set_error(LSRM_E_CUDA, "tcgen05 attention: cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[5] = {8, 8, (cuuint64_t)(dh / 8), (cuuint64_t)(p.hq / 8), (cuuint64_t)p.nq};
  cuuint64_t strides[4] = {(cuuint64_t)dh * 2, 16, (cuuint64_t)dh * 16, (cuuint64_t)p.ld_q * 2};
  cuuint32_t box[5] = {8, 8, (cuuint32_t)(dh / 8), (cuuint32_t)(G / 8), 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(&p.tmq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<__nv_bfloat16*>(p.q),
                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(LSRM_E_CUDA, "tcgen05 attention: Q tensor map encode failed (%d)", (int)r);
  p.q_tma = 1;
  return LSRM_OK;
}
// Picks the variant and grid: d_h = 32 runs two independent single-head
// pipelines per CTA (or, with -DLSRM_HEADPAIR in static mode, one pipeline
// whose items are kv-head pairs); d_h = 64 one pipeline (TMEM budget).
static int launch(const Launch& L, int dh, int hkv, int64_t n_tiles_static, void* stream) {
  cudaStream_t st = as_stream(stream);
  int dev = 0, n_sm = 148;
  LSRM_CUDA(cudaGetDevice(&dev));
  LSRM_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const bool dyn = L.order != nullptr;
#ifdef LSRM_HEADPAIR
  const int hp = (!dyn && dh == 32 && hkv % 2 == 0) ? 2 : 1, np_ = hp == 2 ? 1 : (dh == 32 ? 2 : 1);
#else
  const int hp = 1, np_ = dh == 32 ? LSRM_NP : 1;
#endif
  const int64_t n_items = dyn ? L.n_order : n_tiles_static * (hkv / hp);
  if (n_items == 0) return LSRM_OK;
  if (dyn) LSRM_CUDA(cudaMemsetAsync(L.counter, 0, sizeof(int), st));
  const int64_t want = (n_items + np_ - 1) / np_;
  const unsigned grid = (unsigned)(want < n_sm ? want : n_sm);
#define LSRM_TC_CASE(D, HP, NP)                                                             \
  if (dh == D && hp == HP && np_ == NP) {                                                   \
    size_t smem = sizeof(Smem<D, HP, NP>) + 1024;                                           \
    LSRM_CUDA(cudaFuncSetAttribute(nsa_fused_kernel<D, HP, NP>,                             \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    nsa_fused_kernel<D, HP, NP><<<grid, threads_of<HP, NP>(), smem, st>>>(L);               \
  } else
  LSRM_TC_CASE(32, 1, LSRM_NP)
  LSRM_TC_CASE(32, 2, 1)
  LSRM_TC_CASE(32, 1, 1)
  LSRM_TC_CASE(64, 1, 1)
  return set_error(LSRM_E_CONFIG, "tcgen05 path: head_dim %d not in {32,64}", dh);
#undef LSRM_TC_CASE
  LSRM_LAUNCHED();
  return LSRM_OK;
}
}  // namespace tc
}  // namespace lsrm

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
  p.perm = nullptr;
  p.kmax = kmax_rows;
  p.gl = (const __nv_bfloat16*)gate_logits;
  p.ld_gl = ld_gl;
  p.gcol0 = gate_col0;
  p.gbias = gate_bias;
  p.n_gates = n_gates;
  p.out = (__nv_bfloat16*)merged;
  p.br_first = 0;
  p.accum = 0;
  p.own_rows = nullptr;
  p.o_br = nullptr;
  p.lse_br = nullptr;
  if (int rc = tc::make_q_map(p, G, dh)) return rc;
  tc::Launch L{};
  L.use[0] = p;
  L.n_uses = 1;
  return tc::launch(L, dh, hkv, n_tiles, stream);
}

int lsrm_nsa_attention_tc_multi(const lsrm_nsa_use* uses, int n_uses, int hq, int hkv, int dh,
                                const int32_t* order, int64_t n_order, int32_t* counter,
                                void* stream) {
  LSRM_REQUIRE(n_uses >= 1 && n_uses <= tc::kMaxUses, "tc_multi: 1..%d uses, got %d",
               tc::kMaxUses, n_uses);
  LSRM_REQUIRE(order && counter, "tc_multi: needs the item order and a counter");
  LSRM_REQUIRE(hq % hkv == 0, "n_q_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  const int G = hq / hkv;
  LSRM_REQUIRE(G >= 4 && G <= tc::kM && tc::kM % G == 0 && tc::kM / G <= 32,
               "tcgen05 path needs 4 <= hq/hkv, (hq/hkv) | 128, got %d", G);
  tc::Launch L{};
  for (int u = 0; u < n_uses; ++u) {
    const lsrm_nsa_use& U = uses[u];
    LSRM_REQUIRE(U.n_gates == 2 || U.n_gates == 3, "use %d: n_gates must be 2 or 3", u);
    LSRM_REQUIRE((tc::kM / G) * U.kmax_rows <= tc::kMaxEnt,
                 "use %d: tile tokens x selected rows exceeds %d", u, tc::kMaxEnt);
    LSRM_REQUIRE(U.ld_q % 8 == 0 && U.ld_gl % 8 == 0 && U.gate_col0 % 8 == 0,
                 "use %d: row strides must be multiples of 8 elements", u);
    if (U.n_blocks == 0) return set_error(LSRM_E_EMPTY_CONTEXT, "use %d: no occupied KV blocks", u);
    LSRM_REQUIRE(U.n_blocks <= (int64_t)tc::kBitmapWords * 32,
                 "use %d: %lld occupied KV blocks exceed %d", u, (long long)U.n_blocks,
                 tc::kBitmapWords * 32);
    tc::Params& p = L.use[u];
    p.q = (const __nv_bfloat16*)U.q;
    p.ld_q = U.ld_q;
    p.nq = U.nq;
    p.hq = hq;
    p.hkv = hkv;
    p.k_il = (const __nv_bfloat16*)U.k_il;
    p.v_il = (const __nv_bfloat16*)U.v_il;
    p.pad_off = U.pad_offsets;
    p.kv_off = U.kv_offsets;
    p.n_rows_pad = U.n_kv_rows_pad;
    p.kc_il = (const __nv_bfloat16*)U.kcmp_il;
    p.vc_il = (const __nv_bfloat16*)U.vcmp_il;
    p.n_blocks = U.n_blocks;
    p.tiles = U.tiles;
    p.n_tiles = U.n_tiles;
    p.rows = U.rows;
    p.count = U.count;
    p.perm = U.perm;
    p.kmax = (int)U.kmax_rows;
    p.gl = (const __nv_bfloat16*)U.gate_logits;
    p.ld_gl = U.ld_gl;
    p.gcol0 = U.gate_col0;
    p.gbias = nullptr;   // folded into the gate logits by the caller
    p.n_gates = (int)U.n_gates;
    p.out = (__nv_bfloat16*)U.merged;
    p.br_first = (int)U.branch_first;
    p.accum = (int)U.accumulate;
    p.own_rows = U.own_rows;
    p.o_br = (float*)U.branch_out;
    p.lse_br = (float*)U.branch_lse;
    LSRM_REQUIRE((U.branch_out == nullptr) == (U.branch_lse == nullptr) &&
                     ((uintptr_t)U.branch_out % 16) == 0,
                 "use %d: branch_out and branch_lse go together (16-byte aligned)", u);
    if (int rc = tc::make_q_map(p, G, dh)) return rc;
  }
  L.n_uses = n_uses;
  L.order = order;
  L.n_order = n_order;
  L.counter = counter;
  return tc::launch(L, dh, hkv, 0, stream);
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
