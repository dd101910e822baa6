/*
 * lsrm_b200.h — C ABI of the B200-native LSRM sparse-attention hot path.
 *
 * Every entry point takes plain pointers to caller-owned DEVICE memory
 * (unless a parameter says "host"), sizes as int64_t, and the CUDA stream to
 * run on (cudaStream_t passed as void*).  Nothing allocates device memory
 * behind the caller's back except the per-thread cuBLAS handle of the fp32
 * library GEMM (lsrm_gemm / lsrm_gemm_f32_ex).
 * Calls are reentrant: no shared scratch, per-call stream, per-thread error
 * buffer.  Outputs are deterministic (fixed reduction orders, no float
 * atomics on outputs).
 *
 * Each function cites the reference interface it replaces
 * (/root/reference/pkg/src/lsrm/<file>:<line>); INTEGRATION.md shows the
 * ctypes binding the reference-side `lsrm` package would add.
 *
 * Status codes map 1:1 onto the reference exception classes
 * (lsrm/errors.py:8-59); lsrm_last_error() returns the message of the
 * calling thread's last failure.
 */
#ifndef LSRM_B200_H
#define LSRM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum lsrm_status {
  LSRM_OK = 0,
  LSRM_E_CONFIG = 1,          /* ConfigurationError  (errors.py:14-17) */
  LSRM_E_EMPTY_CONTEXT = 2,   /* EmptyContextError   (errors.py:30-31) */
  LSRM_E_EMPTY_ROW = 3,       /* EmptyAttentionRowError (errors.py:26-27) */
  LSRM_E_PROTOCOL = 4,        /* ProtocolError       (errors.py:42-43) */
  LSRM_E_CUDA = 5,            /* LsrmError (internal, exit code 4) */
  LSRM_E_OUT_OF_DOMAIN = 6    /* OutOfDomainError    (errors.py:34-35) */
};

/* ---- runtime ------------------------------------------------------------ */
int lsrm_abi_version(void);
const char* lsrm_last_error(void);
/* Number of kernels this library launched on the calling thread since the
 * last reset (evidence for bench.py's gpu_launches). */
int64_t lsrm_launch_count(void);
void lsrm_reset_launch_count(void);

/* ---- K11 spatial block partition  (block_partition.py:54-105) ----------
 * modality 0 = volume (coords (i,j,k), grid g0=g1=g2=S),
 *          1 = image  (coords (view,u,v), g0 = views, g1 = g2 = S_img).
 * Outputs sized for the worst case (n_blocks_total rows); *n_occupied (host)
 * receives B.  centers: [B,3] (volume, object units) or [B,2] (image, patch
 * units); block_views [B] (image only, may be NULL for volume).
 * workspace >= lsrm_partition_workspace(n, n_blocks_total) bytes. */
size_t lsrm_partition_workspace(int64_t n, int64_t n_blocks_total);
int lsrm_partition(int modality, const int64_t* coords, int64_t n, int g0,
                   int g1, int g2, int block_size, int64_t* block_of_token,
                   int64_t* block_token_ids, int64_t* occupied_ids,
                   int64_t* block_offsets, int64_t* occupancy,
                   double* centers, int64_t* block_views,
                   int64_t* n_occupied, void* workspace, size_t ws_bytes,
                   void* stream);

/* ---- K6 per-block KV compression  (block_partition.py:141-167) ---------
 * x: [N, width] in token order, row stride ld_x.  src_bf16 flags: bit 0 =
 * bf16 source (else f32); bit 1 = fp32 ResBlock arithmetic (bf16 engine).
 * Default (bit 1 clear):
 * ResBlock x + W2 gelu(W1 x + b1) + b2 in f64 with the reference's f32
 * roundings, then the in-block mean in ascending token order with an f64
 * running sum.  out: [B, width] f32; scratch: [N, width] f32. */
int lsrm_compress_block(int src_bf16, const void* x, int64_t ld_x, int64_t n,
                        int width, const float* w1, const float* b1,
                        const float* w2, const float* b2,
                        const int64_t* block_token_ids,
                        const int64_t* block_offsets, int64_t n_blocks,
                        float* out, float* scratch, void* stream);

/* ---- K7 volume router  (block_routing.py:115-143) ----------------------
 * points [nq,3] f64; centers [B,3] f64.  out_rows [nq, budget] int32
 * occupied-row indices (-1 padded), out_count [nq].  f64, no FMA:
 * bit-exact with the reference including tie order. */
int lsrm_route_volume(const double* points, int64_t nq, const double* centers,
                      int64_t n_blocks, int budget, int32_t* out_rows,
                      int32_t* out_count, void* stream);

/* ---- K8 image router  (block_routing.py:150-230) -----------------------
 * cams: [n_views, 21] f64 rows = K(9) R(9) t(3), row-major.
 * view_row_start [n_views+1]: occupied-row range of each view.
 * block_centers [B,2] (patch units); token_points_bm [3, Ni] f64 (x, y, z
 * rows, SoA) in block-major order; block_offsets [B+1]; max_view_rows = the largest
 * occupied-row count of any view (sizes the per-warp shared scratch). */
int lsrm_route_image(const double* points, int64_t nq, const double* cams,
                     int n_views, const int64_t* view_row_start,
                     const double* block_centers, int64_t n_blocks,
                     const double* token_points_bm, const double* block_bounds,
                     const int64_t* block_offsets, int b_i, int budget,
                     int max_view_rows, int32_t* out_rows, int32_t* out_count,
                     void* stream);
/* Bounding box of every block's token points: token_points_soa [3, n_points]
 * block-major, bounds [n_blocks, 6] = (min xyz, max xyz).  The image router
 * prunes candidates with it (exact: the box distance is a lower bound of the
 * rounded point distances). */
int lsrm_block_bounds(const double* token_points_soa, int64_t n_points,
                      const int64_t* block_offsets, int64_t n_blocks, double* bounds,
                      void* stream);

/* ---- SDF fields  (camera_geometry.py:151-205, runner.py:301-306) -------
 * kind 0 analytic: prims = n_prims rows of 8 f64 (as lsrm_voxel_mask);
 * kind 1 decoded: the coarse dense feature grid [side^3, d_f] f32 through the
 *   decoder's SDF head (w1 [d_f, hidden], b1 [hidden], gelu, w2 [hidden, 1],
 *   b2 [1]) plus |p - c| - radius, with the reference's f32 rounding points
 *   and NumPy's einsum reduction order (decode_points(...)[1] of
 *   recon_pipeline.py:349-365 on FeatureVolume(grid));
 * kind 2 values: s of each sample precomputed (an opaque callable evaluated
 *   by the host at the points lsrm_voxel_sample_points /
 *   lsrm_ray_sample_points produce), indexed by sample id. */
typedef struct lsrm_sdf_field {
  int32_t kind;
  int32_t n_prims;
  const double* prims;
  const float* grid;
  int32_t side;
  int32_t d_f;
  int32_t hidden;
  int32_t pad_;
  const float* w1;
  const float* b1;
  const float* w2;
  const float* b2;
  double radius;
  const double* values;
} lsrm_sdf_field;

/* LSRM_OK if the descriptor is usable, else LSRM_E_CONFIG with a message. */
int lsrm_check_field(const lsrm_sdf_field* field);

/* ---- router input producer  (block_routing.py:73-108,
 *      camera_geometry.py:236-302) ------------------------------------------
 * Surface point of every image token's patch-center ray: 128-sample Laplace
 * opacity march through [0,1]^3 of the analytic scene (sdf rows as in
 * lsrm_voxel_mask), peak of transmittance x alpha, cube-entry / closest-
 * approach fallbacks with miss flags.  coords [n,3] int64 (view, u, v);
 * cams [n_views,21] K R t; image_wh [n_views,2] pixels; rows_f = patch grid
 * side.  points [n,3] f64 clipped to [0,1]; miss [n].  f64, no FMA; exp and
 * the reference's BLAS rotation are not bit-identical, so points match the
 * reference to a stated tolerance. */
int lsrm_image_token_points(const int64_t* coords, int64_t n, const double* cams,
                            const int32_t* image_wh, int n_views, int rows_f,
                            const double* sdf, int n_prims, double beta,
                            double* points, uint8_t* miss, void* stream);

/* The same for any field (analytic, decoded, or values with sample id
 * ray * 128 + k). */
int lsrm_image_token_points_field(const int64_t* coords, int64_t n, const double* cams,
                                  const int32_t* image_wh, int n_views, int rows_f,
                                  const lsrm_sdf_field* field, double beta, double* points,
                                  uint8_t* miss, void* stream);
/* The 128 march sample points of every ray, points [n, 128, 3] f64, for an
 * opaque field the host evaluates; has_span [n] = 0 for rays missing the cube
 * (their samples are placeholders the march never reads). */
int lsrm_ray_sample_points(const int64_t* coords, int64_t n, const double* cams,
                           const int32_t* image_wh, int n_views, int rows_f, double* points,
                           uint8_t* has_span, void* stream);

/* Plücker rays (camera_geometry.py:91-107): [n_views, gh, gw, 6] float32
 * rows (unit direction d, moment t x d) through the centers of a gw x gh grid
 * over each view's image. */
int lsrm_pluecker_rays(const double* cams, const int32_t* image_wh, int n_views, int gw,
                       int gh, float* out, void* stream);
/* Silhouettes (camera_geometry.py:308-350): alpha [n_views, max_h, max_w]
 * float32, 1 where the pixel ray (float32 Plücker direction, as the
 * reference) hits the analytic scene (sdf rows as in lsrm_voxel_mask). */
int lsrm_silhouette_alpha(const double* cams, const int32_t* image_wh, int n_views,
                          int max_w, int max_h, const double* sdf, int n_prims,
                          float* alpha, void* stream);

/* ---- gather table  (nsa_attention.py:123-154) -------------------------
 * Resolves routed rows (fallback: own block row, else row 0) into padded
 * token-id rows.  own_row may be NULL.  With fallback = 0 an empty row stays
 * empty (resolved_count 0, length 0); the host raises EmptyAttentionRowError.
 * resolved_rows/resolved_count receive the fallback-applied rows (the
 * attention kernels' input).  ids/valid may be NULL (lengths only). */
int lsrm_build_gather_table(const int32_t* rows, const int32_t* count,
                            int64_t nq, int kmax_rows, const int32_t* own_row,
                            int fallback, const int64_t* block_offsets,
                            const int64_t* block_token_ids, int64_t width,
                            int32_t* resolved_rows, int32_t* resolved_count,
                            int64_t* ids, uint8_t* valid, int64_t* lengths,
                            void* stream);

/* ---- K9 foreground patch mask  (tokenizer.py:200-208) ------------------ */
int lsrm_foreground_mask(const float* alpha, int n_views, int h, int w,
                         int patch, uint8_t* mask, void* stream);

/* ---- K10 informative voxel mask  (tokenizer.py:211-239) ---------------
 * sdf: n_prims rows of 8 f64 = kind(0 sphere, 1 box), cx, cy, cz,
 * radius | hx, hy, hz, unused.  The field is the union (min) of all
 * primitives (camera_geometry.py:190-205). */
int lsrm_voxel_mask(const double* sdf, int n_prims, int s_vol, double tau,
                    int t_side, uint8_t* mask, void* stream);

/* Eq. 11 for any field over the voxels of x-slabs [i0, i1) (mask is the full
 * [s_vol^3] array; other slabs untouched).  For kind 2 the values cover
 * exactly those slabs in the layout of lsrm_voxel_sample_points. */
int lsrm_voxel_mask_field(const lsrm_sdf_field* field, int s_vol, double tau, int t_side,
                          int i0, int i1, uint8_t* mask, void* stream);
/* Cell-center sample points of x-slabs [i0, i1), the reference's layout
 * (tokenizer.py:227-235): points [(i1-i0) * t * (t s)^2, 3] f64. */
int lsrm_voxel_sample_points(int s_vol, int t_side, int i0, int i1, double* points,
                             void* stream);

/* ---- compaction  (tokenizer.py:255-313) -------------------------------
 * Stream-compacts mask-true cells in flat order and gathers parent feature +
 * factorized fine pos-embed with the reference's two f64 roundings.
 * volume: mask [S^3], parent grid S/factor; image: mask [V,S,S] (view, row,
 * col), coords written as (view, u=col, v=row).  *n_out (host) = count.
 * Call with features == NULL to only count (coords may be NULL too). */
size_t lsrm_compact_workspace(int64_t n_cells);
int lsrm_compact_volume(const uint8_t* mask, int s_fine, int factor,
                        const float* x_d, int d, const float* pe0,
                        const float* pe1, const float* pe2, int64_t* coords,
                        float* features, int64_t max_out, int64_t* n_out,
                        void* workspace, size_t ws_bytes, void* stream);
int lsrm_compact_image(const uint8_t* mask, int n_views, int s_fine,
                       int factor, const float* y_d, int d, const float* pe_u,
                       const float* pe_v, int64_t* coords, float* features,
                       int64_t max_out, int64_t* n_out, void* workspace,
                       size_t ws_bytes, void* stream);
/* Second half of a two-call compaction: after lsrm_compact_volume /
 * lsrm_compact_image ran with coords = features = NULL (mask scan, cell list
 * left in `workspace`, count in *n_out), write the n_out tokens' coords and
 * features from that cell list without rescanning the mask (no host sync).
 * modality 0 = volume (pe0..pe2 the three axis tables), 1 = image (pe0 = u
 * table, pe1 = v table, pe2 unused); n_cells = the mask's cell count. */
int lsrm_compact_rows(int modality, const void* workspace, int64_t n_cells, int64_t n_out,
                      int n_views, int s_fine, int factor, const float* parents, int d,
                      const float* pe0, const float* pe1, const float* pe2, int64_t* coords,
                      float* features, void* stream);

/* ---- fp32 attention branches on CUDA cores  (nsa_attention.py:84-207) --
 * q [nq, hq, dh]; keys/values [nk, hkv, dh] f32 in BLOCK-MAJOR order of the
 * KV partition (row r = block_offsets[r]..block_offsets[r+1]).
 * mode 0 = cmp (all nk rows are keys), 1 = sel (rows[i, :count[i]] are
 * occupied rows, resolved), 2 = win (own_row[i]), 3 = explicit gather table
 * (ids [nq, width] token ids into kv_token_order arrays, lengths[i]).
 * out [nq, hq, dh]. */
int lsrm_attention_f32(int mode, const float* q, int64_t nq, int hq, int hkv,
                       int dh, const float* k, const float* v, int64_t nk,
                       const int64_t* block_offsets, const int32_t* rows,
                       const int32_t* count, int kmax_rows,
                       const int32_t* own_row, const int64_t* ids,
                       const int64_t* lengths, int64_t width, float* out,
                       void* stream);

/* ---- gated merge, fp32 path  (nsa_attention.py:266-284) ---------------
 * merged[i,:] = f32( sum_b f64(sigmoid(gl[i, b*d:(b+1)*d] + gb)) * f64(o_b) )
 * gl: gate logits [n, n_gates*d] (row stride ld_gl); o_b: [n, d] each. */
int lsrm_gated_merge_f32(const float* gate_logits, int64_t ld_gl,
                         const float* gate_bias, int n_gates,
                         const float* o0, const float* o1, const float* o2,
                         int64_t n, int d, float* merged, void* stream);

/* out[n, cols] = f32(sigmoid_f64(f32(logits + bias)))  (tensor_core.py:89-94) */
int lsrm_sigmoid_f32(const float* logits, int64_t ld, const float* bias,
                     int64_t n, int cols, float* out, void* stream);

/* ---- vanilla score top-k  (nsa_attention.py:210-232) ------------------
 * score[i,b] = sum_h sum_d q[i,h,:] . k_cmp[b, h/group, :] in f64 (unscaled);
 * out_rows [nq, b_sel] = stable descending top-min(b_sel, B) columns. */
int lsrm_score_topk(const float* q, int64_t nq, int hq, int hkv, int dh,
                    const float* k_cmp, int64_t n_blocks, int b_sel,
                    int32_t* out_rows, int32_t* out_count, void* stream);

/* ---- GEMM (plain library GEMM, cuBLAS; fp32 reference-API path) --------
 * C[m,n] = A[m,k] @ B[k,n] (+ bias[n]), row-major, lda/ldb/ldc in elements.
 * dtype 0 = fp32 (FFMA, no TF32), 1 = bf16 in / fp32 accumulate / bf16 out,
 * 2 = bf16 in / fp32 out. */
int lsrm_gemm(int dtype, int64_t m, int64_t n, int64_t k, const void* a,
              int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc,
              void* stream);

/* ---- grouped bf16 GEMM on tcgen05 (hand-written; TMA + TMEM) ----------
 * Replaces the library GEMMs of the layer's hot path: the per-stream fused
 * projection (q/k/v `affine` + gate GEMM, nsa_attention.py:266-273,303-307
 * over tensor_core.py:100-116), W_o (nsa_attention.py:284) and the Stage-2
 * FFN (recon_pipeline.py:497-512).  For every problem:
 *   C[m,n] = act(A[m,k] . Bt[n,k]^T + bias[n]) + res[m,n]
 * A bf16 [m,k] and Bt bf16 [n,k] (the weight stored TRANSPOSED) both with K
 * contiguous; fp32 accumulation in TMEM; bias/res/C dtypes per flags.
 * k, n and every row stride must be multiples of 8 elements and pointers
 * 16-byte aligned.  One persistent launch runs all problems (<= 32). */
#define LSRM_GEMM_OUT_F32  1   /* C is f32 (else bf16) */
#define LSRM_GEMM_BIAS_F32 2   /* bias is f32 (else bf16) */
#define LSRM_GEMM_RES_F32  4   /* res is f32 (else bf16) */
#define LSRM_GEMM_GELU     8   /* act = exact-erf gelu, applied before res */
/* MN-major operands (no transposed copy needed; e.g. weight gradients
 * X^T . dY take X [k,m] and dY [k,n] as stored):
 *   A_MN: `a` is A^T stored row-major, [k, m] with row stride lda >= m;
 *   B_MN: `bt` is B stored row-major, [k, n] with row stride ldb >= n.
 * Rows of an MN-major operand past k read as zeros. */
#define LSRM_GEMM_A_MN    16
#define LSRM_GEMM_B_MN    32
typedef struct lsrm_gemm_problem {
  int64_t m, n, k;
  const void* a;  int64_t lda;
  const void* bt; int64_t ldb;
  void* c;        int64_t ldc;
  const void* bias;             /* [n] or NULL */
  const void* res; int64_t ldr; /* [m,n] or NULL; may alias c */
  int32_t flags;
  int32_t reserved;
} lsrm_gemm_problem;
/* problems: HOST array of n_problems descriptors.  With A_MN / B_MN the
 * K-major rules above apply to the remaining K-major operand only (k % 8 == 0
 * when one is K-major). */
int lsrm_gemm_tc(const lsrm_gemm_problem* problems, int n_problems, void* stream);

/* ---- fused bf16 three-branch NSA attention, tcgen05/TMEM  -------------
 * (nsa_attention.py:84-112,157-207,266-284 fused)
 * q: [nq, hq, dh] bf16 in query BLOCK-MAJOR order; kv_il: K and V in the
 * padded interleaved layout written by lsrm_kv_interleave; kcmp_il/vcmp_il
 * likewise for the compressed rows.  tiles: [n_tiles, 4] int32 = (first
 * query, count, own kv row (or -1), unused).  rows/count: resolved selected
 * rows per query.  gate_logits bf16 [nq, ld_gl] with the n_gates width-d
 * slices at column gate_col0.  merged bf16 [nq, hq*dh]. */
int lsrm_nsa_attention_tc(const void* q, int64_t ld_q, int64_t nq, int hq, int hkv, int dh,
                          const void* k_il, const void* v_il,
                          const int64_t* pad_offsets, const int64_t* kv_offsets,
                          int64_t n_kv_rows_pad,
                          const void* kcmp_il, const void* vcmp_il,
                          int64_t n_blocks, const int32_t* tiles,
                          int64_t n_tiles, const int32_t* rows,
                          const int32_t* count, int kmax_rows,
                          const void* gate_logits, int64_t ld_gl,
                          int64_t gate_col0, const float* gate_bias,
                          int n_gates, void* merged, void* stream);

/* All NSA uses of a layer (same head geometry) in ONE persistent launch, with
 * a heaviest-first work queue.  Each use is described like the arguments of
 * lsrm_nsa_attention_tc (uses is a HOST array); gate biases must already be
 * folded into the gate logits.  A use may regroup its query tiles through
 * `perm` (e.g. tokens of a block sorted by selection signature, so a tile's
 * union of selected blocks shrinks).  order [n_order]: (use << 28) | item, item =
 * tile * hkv + kv head, sorted by estimated cost, descending; counter: one
 * int32 of device memory (zeroed by this call on `stream`). */
typedef struct lsrm_nsa_use {
  const void* q;
  int64_t ld_q;
  int64_t nq;
  const void* k_il;
  const void* v_il;
  const int64_t* pad_offsets;
  const int64_t* kv_offsets;
  int64_t n_kv_rows_pad;
  const void* kcmp_il;
  const void* vcmp_il;
  int64_t n_blocks;
  const int32_t* tiles;
  int64_t n_tiles;
  const int32_t* rows;
  const int32_t* count;
  int64_t kmax_rows;
  const void* gate_logits;
  int64_t ld_gl;
  int64_t gate_col0;
  int64_t n_gates;
  void* merged;
  const int32_t* perm;   /* optional [nq]: tile position -> query row; tiles,
                            rows and count are then in permuted (tile) order,
                            q / gate_logits / merged stay in query-row order */
  int64_t branch_first;  /* first branch the items run: 0, or 2 for window-only
                            items (self uses split over two launches) */
  int64_t accumulate;    /* 1: add the gated result to `merged` (second launch) */
  const int32_t* own_rows; /* optional [nq] (tile order): each token's own kv row;
                              the window branch then spans the tile's distinct own
                              blocks, so self-use tiles may cross query blocks */
  void* branch_out;      /* optional f32 [n_gates][nq][hq*dh]: each branch's own
                            normalized output (training forward; query-row order) */
  void* branch_lse;      /* optional f32 [n_gates][nq][hq]: each branch's
                            log-sum-exp of the scaled logits (natural log);
                            set with branch_out or not at all */
} lsrm_nsa_use;
int lsrm_nsa_attention_tc_multi(const lsrm_nsa_use* uses, int n_uses, int hq, int hkv, int dh,
                                const int32_t* order, int64_t n_order, int32_t* counter,
                                void* stream);

/* Re-layout K or V ([n, hkv, dh] f32 or bf16, token order) into the padded,
 * 8x8-core-matrix interleaved bf16 layout the tcgen05 kernel consumes:
 * per kv head, per block, rows padded to a multiple of 16.  ones_cols = 16
 * appends 16 columns holding 1 (real key) / 0 (padding): the V operand then
 * yields the softmax row sums in the same P.V MMA.  Padding rows of V are
 * zero; padding rows of K (ones_cols = 0) repeat the block's first key, so
 * they can neither raise a row max nor contribute (the attention kernel
 * needs no padding masks). */
int lsrm_kv_interleave(int src_is_bf16, const void* src, int64_t ld_src,
                       int64_t n, int hkv, int dh, int ones_cols,
                       const int64_t* block_token_ids,
                       const int64_t* block_offsets, int64_t n_blocks,
                       const int64_t* pad_offsets, int64_t n_rows_pad,
                       void* dst, void* stream);

/* Debug: device buffer of 256 x 32 int64 that CTA 0 of the fused attention
 * kernel fills with clock64() stamps per chunk/event (NULL disables). */
int lsrm_debug_set_trace(void* buf);

/* K/V preparation of the bf16 engine, every (use, K|V) tensor of a layer in
 * ONE launch (nsa_attention.py:305-312 with block_partition.py:141-167 fused
 * in).  One job per tensor: token rows src [n, hkv*dh] bf16 (row stride ld) in
 * block-major order; blk_off [n_blocks+1] token offsets and pad_off
 * [n_blocks+1] 16-row-padded offsets into il.  Writes the interleaved layout
 * il [hkv][rows_pad][dh+ones_cols] (ones_cols = 16 for V: row-sum columns), the
 * ResBlock block means (tensor-core bf16 MLP, fp32 accumulation, fixed-order
 * sums; one CTA per 64-token sub-tile, the block's last-arriving CTA adds
 * the sub-tiles' partials in order) to mean_out [n_blocks][hkv*dh] f32 and/or, interleaved, to cmp_il
 * [hkv][cmp_rows_pad][dh+ones_cols] (either may be NULL).  jobs points to
 * DEVICE memory; hkv*dh must be 64 or 128. */
typedef struct lsrm_kv_job {
  const void* src;
  int64_t ld;
  const int64_t* blk_off;
  const int64_t* pad_off;
  int64_t n_blocks;
  int64_t rows_pad;
  void* il;
  int64_t ones_cols;
  const void* w1;        /* [w][w] bf16, r = x W1 (w = hkv*dh) */
  const float* b1;
  const void* w2;        /* [w][w] bf16 */
  const float* b2;
  float* mean_out;
  void* cmp_il;
  int64_t cmp_rows_pad;
  const int32_t* work;   /* [n_work]: (block << 12) | 64-token sub-tile, by block;
                            one CTA each */
  int64_t n_work;
  float* partial;        /* [n_work][hkv*dh] scratch: per-sub-tile column sums */
  int32_t* arrive;       /* [n_blocks] counters, zero between launches (the
                            block's last-arriving CTA resets its entry) */
} lsrm_kv_job;
int lsrm_kv_prepare_jobs(const lsrm_kv_job* jobs, int n_jobs, int64_t max_work, int hkv,
                         int dh, void* stream);

/* Byte-segment copy: segs [n_segs, 3] int64 = (src offset, dst offset,
 * bytes), all multiples of 16.  Places all-gathered per-rank KV shards into
 * the canonical block-major layout (seq_parallel.py All-gather-KV). */
int lsrm_copy_segments(const void* src, void* dst, const int64_t* segs,
                       int64_t n_segs, void* stream);

/* Row permutation helpers (block-major <-> token order). */
int lsrm_gather_rows(int elem_bytes, const void* src, int64_t ld_src,
                     const int64_t* index, int64_t n, int64_t row_elems,
                     void* dst, int64_t ld_dst, void* stream);
int lsrm_scatter_rows(int elem_bytes, const void* src, int64_t ld_src,
                      const int64_t* index, int64_t n, int64_t row_elems,
                      void* dst, int64_t ld_dst, void* stream);
/* Host rows -> device rows for the reference API's NumPy inputs
 * (nsa_attention.py:287 `nsa_cross_attention(x, kv_feats, ...)` takes host
 * arrays).  src is HOST f32 (pageable is fine), [*, ld_src]; row i of dst
 * (device, [n_rows, ld_dst]) is src row row_index[i] (row_index is a HOST
 * int64 array, NULL = identity), converted to bf16 (round-to-nearest-even,
 * bit-identical to lsrm_cast) when to_bf16, else copied as f32.  Host
 * threads convert into pinned staging chunks that are copied on `stream`
 * while the next chunk is converted; returns once src has been read (the
 * copies complete in stream order).  lsrm_host_threads(): the pool size. */
int lsrm_host_threads(void);
int lsrm_h2d_rows(int to_bf16, const float* src, int64_t ld_src, const int64_t* row_index,
                  int64_t n_rows, int64_t row_elems, void* dst, int64_t ld_dst, void* stream);
/* f32 <-> bf16 conversion, LayerNorm (tensor_core.py:139-146). */
int lsrm_cast(int to_bf16, const void* src, void* dst, int64_t n, void* stream);
int lsrm_layer_norm(int in_bf16, const void* x, int64_t n, int d,
                    const float* gamma, const float* beta, float eps,
                    int out_bf16, void* y, void* stream);

/* ---- Stage-2 sparse block around the NSA uses (recon_pipeline.py:461-497) --
 * exact = 1: the reference's f32 storage with f64 arithmetic (reference API);
 * exact = 0: fp32 arithmetic (bf16 engine).  Row kernels run a warp per row
 * with f64 LayerNorm statistics (tensor_core.py:139-146).
 * add_layer_norm: sum_out = f32(a + b) (b may be NULL), y = LN(sum_out);
 * exact = 0 keeps the row in registers with fp32 statistics (d = 1024). */
int lsrm_add_layer_norm(int exact, const float* a, const void* b, int b_bf16, int64_t n, int d,
                        const float* gamma, const float* beta, float eps,
                        float* sum_out, int out_bf16, void* y, void* stream);
/* x1 = f32(xe + sigmoid(gl[:, :d] + gb[:d]) * o_self
 *           + sigmoid(gl[:, d:2d] + gb[d:]) * o_cross),  h = LN(x1). */
int lsrm_gate_mix_layer_norm(int exact, const float* xe, const void* gate_logits,
                             int64_t ld_gl, int gl_bf16, const float* gate_b,
                             const void* o_self, const void* o_cross, int o_bf16,
                             int64_t n, int d, float* x1, const float* gamma,
                             const float* beta, float eps, int out_bf16, void* h,
                             void* stream);
/* out = f32(act(f32(h + bias))) (+ residual f32 [n, cols]); act 0 = identity,
 * 1 = exact-erf gelu (tensor_core.py:82-86). */
int lsrm_bias_act(int exact, const void* h, int h_bf16, int64_t ld, const float* bias,
                  int64_t n, int cols, int act, const float* residual, void* out,
                  int out_bf16, int64_t ld_out, void* stream);

/* ---- backward of one gated NSA use (training) -----
 * fp32, recompute-based, deterministic (fixed summation orders, no float
 * atomics); the reference has no backward (oracle: oracle/torch_nsa.py, f64
 * autograd).
 * attention_bwd: key sets as lsrm_attention_f32 (mode 0 cmp over all nk
 * rows, 1 sel over the resolved rows, 2 win over own_row), q/dO/O
 * [nq, hq, dh] and k/v [nk, hkv, dh] (block-major for sel/win).  n_rows and
 * max_row_keys describe block_offsets (sel/win).  The key pass splits the
 * queries into n_slices ranges (more CTAs for few keys); workspace holds the
 * per-slice partials.  Accumulates: dq += ..., dk += ..., dv += .... */
size_t lsrm_attention_bwd_workspace(int64_t nq, int hq, int64_t nk, int hkv, int dh,
                                    int n_slices);
int lsrm_attention_bwd_f32(int mode, const float* q, const float* dO, const float* O,
                           int64_t nq, int hq, int hkv, int dh, const float* k,
                           const float* v, int64_t nk, const int64_t* block_offsets,
                           int n_rows, int max_row_keys, const int32_t* rows,
                           const int32_t* count, int kmax_rows, const int32_t* own_row,
                           int n_slices, float* dq, float* dk, float* dv, void* workspace,
                           size_t ws_bytes, void* stream);
/* Tensor-core variant (mma.sync bf16, fp32 accumulation), same contract and
 * workspace: bf16 copies of q, dO and k, v feed the MMAs; dO and O in f32
 * give D = rowsum(dO * O); lse_in (optional, from lsrm_attention_fwd_mma)
 * skips the statistics pass.  head_dim in {16, 32, 64}, hq / hkv <= 16. */
int lsrm_attention_bwd_mma(int mode, const void* q_bf16, const void* dO_bf16, const float* dO,
                           const float* O, const float* lse_in, int64_t nq, int hq, int hkv, int dh,
                           const void* k_bf16, const void* v_bf16, int64_t nk,
                           const int64_t* block_offsets, int n_rows, int max_row_keys,
                           const int32_t* rows, const int32_t* count, int kmax_rows,
                           const int32_t* own_row, int n_slices, const int64_t* t_offs,
                           const int32_t* t_q, float* dq, float* dk, float* dv,
                           void* workspace, size_t ws_bytes, void* stream);
/* Transposed routing index for the key-major pass: offs [n_rows + 1] and
 * q [nq * kmax] (the first offs[n_rows] used): per kv row, the queries whose
 * resolved selection holds it, ascending (stable radix sort of (row, query)
 * keys).  The backward takes it as t_offs / t_q (sel), or the query
 * partition's block offsets / token ids (win). */
size_t lsrm_transpose_rows_workspace(int64_t nq, int kmax);
int lsrm_transpose_rows(const int32_t* rows, const int32_t* count, int64_t nq, int kmax,
                        int n_rows, int64_t* offs, int32_t* q_out, void* workspace,
                        size_t ws_bytes, void* stream);
/* merged = sum_b sigmoid(gl[:, b*d:(b+1)*d] + gb[b*d:]) * o_b:
 * do_b = dM g_b,  dz[:, b*d + c] = dM o_b g_b (1 - g_b)   (dz [n, n_gates*d]). */
int lsrm_gate_merge_bwd_f32(const float* gate_logits, int64_t ld_gl, const float* gate_bias,
                            int n_gates, const float* o0, const float* o1, const float* o2,
                            const float* dmerged, int64_t n, int d, int fast, float* do0,
                            float* do1, float* do2, float* dz, void* stream);
/* Training forward of the gated merge in fp32 (fp32 sigmoid and sum; the
 * reference-API lsrm_gated_merge_f32 keeps f64): merged = sum_b g_b * o_b. */
int lsrm_gated_merge_fast_f32(const float* gate_logits, int64_t ld_gl, const float* gate_bias,
                              int n_gates, const float* o0, const float* o1, const float* o2,
                              int64_t n, int d, float* merged, void* stream);
/* Compression ResBlock under the block mean (block_partition.py:141-158):
 * dr_t = dcmp[row(t)] / occupancy[row(t)];  dx_t += dr_t + (dr_t W2^T * gelu'(z1_t)) W1^T;
 * writes dr, dz1, h = gelu(z1) rows [n, width] for the weight-gradient GEMMs. */
int lsrm_res_block_bwd_f32(const float* x, int64_t n, int width, const float* w1,
                           const float* b1, const float* w2, const float* dcmp,
                           const int32_t* row_of_token, const int64_t* occupancy, float* dx,
                           float* dr_out, float* dz1_out, float* h_out, void* stream);
/* Row-major fp32 C[m,n] = alpha op(A) op(B) + beta C (op = transpose if
 * trans_*); tf32 = 1 allows TF32 tensor cores (the fast training mode). */
int lsrm_gemm_f32_ex(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, float alpha,
                     const float* a, int64_t lda, const float* b, int64_t ldb, float beta,
                     float* c, int64_t ldc, int tf32, void* stream);
/* Training forward of one branch on tensor cores (mma.sync bf16): out f32
 * [nq, hq, dh] and lse [nq, hq] (natural log) for the backward.  Key-set
 * arguments as lsrm_attention_f32. */
int lsrm_attention_fwd_mma(int mode, const void* q_bf16, int64_t nq, int hq, int hkv, int dh,
                           const void* k_bf16, const void* v_bf16, int64_t nk,
                           const int64_t* block_offsets, const int32_t* rows,
                           const int32_t* count, int kmax_rows, const int32_t* own_row,
                           float* out, float* lse, void* stream);

/* ---- feature decode around the sparse stage (recon_pipeline.py:209-348) --
 * f64 arithmetic, the reference's f32 rounding points, NumPy operation order.
 * decode_scatter: vec [side^3, t^3*d_f] (token-major, slice [dz,dy,dx,c]) ->
 * grid [(t*side)^3, d_f]. */
/* y[n, dout] (row stride ldy) = f32(act(f32(x W + bias))): the reference's
 * affine (tensor_core.py:100-116: f64 accumulation in np.einsum's order) and
 * activation (act 0 identity, 1 erf-gelu, 2 sigmoid; tensor_core.py:82-94).
 * x [n, din] f32 (row stride ldx), W [din, dout] f32, bias [dout] or NULL. */
int lsrm_affine_exact(const float* x, int64_t ldx, int64_t n, int din, const float* w,
                      const float* bias, int dout, int act, float* y, int64_t ldy,
                      void* stream);
int lsrm_decode_scatter(const float* vec, int side, int t, int d_f, float* grid, void* stream);
/* sparse fine features: rows [n*t^3, d_f] and index [s_f^3] int64 (-1 absent). */
int lsrm_sparse_features(const float* vec, const int64_t* coords, int64_t n, int t, int d_f,
                         int64_t s_f, int64_t* index, float* rows, void* stream);
/* Blended field query (sparse_index NULL: dense trilinear only) at f64 points
 * [n,3] in [0,1]^3, then the z (gelu, sigmoid) and s (gelu, identity) heads
 * + the bounding-sphere offset.  head_w: host array of 8 device pointers
 * (z w1 b1 w2 b2, s w1 b1 w2 b2) or NULL for the field only; field_out
 * [n, d_f] optional. */
int lsrm_decode_points(const float* grid, int s_df, const int64_t* sparse_index,
                       const float* sparse_rows, int s_f, int d_f, const double* points,
                       int64_t n, const float* const* head_w, int hidden, int z_channels,
                       float* z_out, float* s_out, float* field_out, void* stream);


/* ---- sequence-parallel exchanges over NCCL (csrc/comm.cu) -----------------
 * Replace the reference's simulated collectives `all_gather_kv`
 * (lsrm/seq_parallel.py:181-218) and `all_to_all` (:146-178) with real
 * NVLink transfers. NCCL is bound at run time (libnccl.so.2, the process's
 * copy if one is loaded); every call is enqueued on `stream`. */

/* 128-byte NCCL unique id, created on one rank and shared by the host. */
int lsrm_comm_unique_id(uint8_t* id_out);
/* Communicator of `world` ranks (one per GPU); *comm_out is opaque. */
int lsrm_comm_init(const uint8_t* id, int world, int rank, void** comm_out);
int lsrm_comm_destroy(void* comm);

/* All-gather-KV of one NSA use: every rank's packed shard (`shard_bytes`,
 * [k_il | v_il | k_cmp | v_cmp]) lands in `stage` at stage_off[r] (host
 * array [world+1]); then for each of the n_dst canonical buffers dst[i]
 * the placement segments segs[i] (device [n_segs[i], 3] int64, see
 * lsrm_copy_segments) are applied. Grouped ncclSend/ncclRecv (all-gather-v). */
int lsrm_allgather_kv(void* comm, int rank, int world, const void* shard,
                      int64_t shard_bytes, void* stage, const int64_t* stage_off,
                      const int64_t* const* segs, const int64_t* n_segs,
                      void* const* dst, int n_dst, void* stream);

/* all-to-all-v of bytes: send_bytes[p] (host) from `send` (consecutive per
 * peer) to peer p, recv_bytes[p] from peer p into `recv` (consecutive per
 * peer). Token dispatch / return of the sharded stage. */
int lsrm_all_to_all_v(void* comm, int rank, int world, const void* send,
                      const int64_t* send_bytes, void* recv, const int64_t* recv_bytes,
                      void* stream);


/* ---- backward of the Stage-2 block around the NSA uses (csrc/train_block.cu;
 * training; forward lsrm/recon_pipeline.py:461-497).
 * fp32, deterministic (fixed-order partial sums, no float atomics).
 * colsum_parts(n): rows of partial sums a reduction over n rows needs
 * (workspace `part` = 2 * parts * d + 2 * n floats for layer_norm_bwd: the
 * partials and the rows' mean / rstd; parts * d for colsum). */
int64_t lsrm_colsum_parts(int64_t n);
/* out[i] (+)= sum over s of parts[s * n + i], slices in order (split-K partial
 * products of the training GEMMs; deterministic).  n % 4 == 0. */
int lsrm_sum_slices_f32(const float* parts, int n_slices, int64_t n, float* out, int accumulate,
                        void* stream);
/* dx (+)= dLN(x)/dx . dy; dgamma = sum_rows dy x_hat; dbeta = sum_rows dy. */
int lsrm_layer_norm_bwd_f32(const float* x, int64_t ld_x, int64_t n, int d, const float* gamma,
                            float eps, const float* dy, int64_t ld_dy, float* dx, int64_t ld_dx,
                            int accumulate, float* part, float* dgamma, float* dbeta,
                            void* stream);
/* out[c] = sum_rows x[r, c] (bias gradients). */
int lsrm_colsum_f32(const float* x, int64_t ld, int64_t n, int d, float* part, float* out,
                    void* stream);
/* gated mixture x1 = xe + s(l_s) o_s + s(l_c) o_c (l = logits + bias [2d]):
 * do_s, do_c [n, d] and dlogits [n, 2d] from dx1. */
int lsrm_gate_mix_bwd_f32(const float* logits, int64_t ld_l, const float* bias, const float* o_s,
                          const float* o_c, const float* dx1, int64_t n, int d, float* do_s,
                          float* do_c, float* dlogits, void* stream);
/* dst [cols][rows_pad] bf16 = src[rows][cols]^T (f32, row stride ld), rows
 * past `rows` zero: the K-major operands of the training GEMMs. */
int lsrm_transpose_cast_bf16(const float* src, int64_t ld, int64_t rows, int64_t cols,
                             void* dst, int64_t rows_pad, void* stream);
/* dt = du * gelu'(z + bias) (exact erf gelu). */
int lsrm_gelu_bwd_f32(const float* z, const float* bias, const float* du, int64_t n, int d,
                      float* dt, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LSRM_B200_H */
