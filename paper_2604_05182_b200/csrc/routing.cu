// K7/K8 3D-aware spatial router (lsrm/block_routing.py:115-230) and the
// gather-table resolution (lsrm/nsa_attention.py:123-154).
//
// One warp per query.  All distance arithmetic is f64 with explicit
// round-to-nearest primitives (no FMA contraction) in NumPy's operation
// order, and every top-k is an exact lexicographic (distance, row) selection
// == np.argsort(kind="stable"), so lists match the reference bit for bit,
// ties included.
#include "common.cuh"

namespace lsrm {

constexpr double kInf = __builtin_huge_val();

// Warp-wide lexicographic min of (val, idx); returns the winner in all lanes.
__device__ __forceinline__ void warp_lexmin(double& val, int& idx) {
  for (int o = 16; o; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, val, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (lex_less(ov, oi, val, idx)) { val = ov; idx = oi; }
  }
}

__global__ void route_volume_kernel(const double* __restrict__ points, int64_t nq,
                                    const double* __restrict__ centers, int nb,
                                    int budget, int32_t* __restrict__ out_rows,
                                    int32_t* __restrict__ out_count) {
  int64_t q = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (q >= nq) return;
  double px = points[3 * q], py = points[3 * q + 1], pz = points[3 * q + 2];
  int take = min(budget, nb);
  double last_v = -kInf;
  int last_i = -1;
  for (int s = 0; s < take; ++s) {
    double best = kInf;
    int bi = 0x7fffffff;
    for (int r = lane; r < nb; r += 32) {
      double d2 = dist2(px, py, pz, centers[3 * r], centers[3 * r + 1], centers[3 * r + 2]);
      if (lex_less(last_v, last_i, d2, r) && lex_less(d2, r, best, bi)) { best = d2; bi = r; }
    }
    warp_lexmin(best, bi);
    if (lane == 0) out_rows[q * budget + s] = bi;
    last_v = best;
    last_i = bi;
  }
  if (lane == 0) {
    for (int s = take; s < budget; ++s) out_rows[q * budget + s] = -1;
    out_count[q] = take;
  }
}

__global__ void route_image_kernel(const double* __restrict__ points, int64_t nq,
                                   const double* __restrict__ cams, int n_views,
                                   const int64_t* __restrict__ view_row_start,
                                   const double* __restrict__ bc,
                                   const double* __restrict__ tp,
                                   const int64_t* __restrict__ offs, int b_i,
                                   int budget, int32_t* __restrict__ out_rows,
                                   int32_t* __restrict__ out_count) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int cap = n_views * b_i;
  int* cand_row = (int*)smem_raw + warp * cap;
  double* cand_d2 = (double*)((int*)smem_raw + (blockDim.x / 32) * cap +
                              ((blockDim.x / 32) * cap & 1)) + warp * cap;
  int64_t q = blockIdx.x * (int64_t)(blockDim.x / 32) + warp;
  if (q >= nq) return;
  const double px = points[3 * q], py = points[3 * q + 1], pz = points[3 * q + 2];
  int ncand = 0;
  for (int v = 0; v < n_views; ++v) {
    int r0 = (int)view_row_start[v], r1 = (int)view_row_start[v + 1];
    if (r1 <= r0) continue;
    const double* K = cams + 21 * v;
    const double* R = K + 9;
    const double* t = K + 18;
    // camera-space coordinates via R^T, reference order (camera_geometry.py:52-74)
    double dx = dsub(px, t[0]), dy = dsub(py, t[1]), dz = dsub(pz, t[2]);
    double xc = dadd(dadd(dmul(R[0], dx), dmul(R[3], dy)), dmul(R[6], dz));
    double yc = dadd(dadd(dmul(R[1], dx), dmul(R[4], dy)), dmul(R[7], dz));
    double zc = dadd(dadd(dmul(R[2], dx), dmul(R[5], dy)), dmul(R[8], dz));
    if (!(zc > 0.0)) continue;
    double u = dadd(dmul(K[0], ddiv(xc, zc)), K[2]);
    double w = dadd(dmul(K[4], ddiv(yc, zc)), K[5]);
    double uu = ddiv(u, 8.0), vv = ddiv(w, 8.0);
    int take = min(b_i, r1 - r0);
    double last_v = -kInf;
    int last_i = -1;
    for (int s = 0; s < take; ++s) {
      double best = kInf;
      int bi = 0x7fffffff;
      for (int r = r0 + lane; r < r1; r += 32) {
        double du = dsub(uu, bc[2 * r]), dv = dsub(vv, bc[2 * r + 1]);
        double d2 = dadd(dmul(du, du), dmul(dv, dv));
        if (lex_less(last_v, last_i, d2, r) && lex_less(d2, r, best, bi)) { best = d2; bi = r; }
      }
      warp_lexmin(best, bi);
      if (lane == 0) cand_row[ncand + s] = bi;
      last_v = best;
      last_i = bi;
    }
    ncand += take;
  }
  __syncwarp();
  // min 3D squared distance from the query to each candidate block's points
  for (int c = 0; c < ncand; ++c) {
    int r = cand_row[c];
    double best = kInf;
    for (int64_t j = offs[r] + lane; j < offs[r + 1]; j += 32) {
      double d2 = dist2(px, py, pz, tp[3 * j], tp[3 * j + 1], tp[3 * j + 2]);
      best = fmin(best, d2);
    }
    for (int o = 16; o; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) cand_d2[c] = best;
  }
  __syncwarp();
  int take = min(budget, ncand);
  double last_v = -kInf;
  int last_i = -1;
  for (int s = 0; s < take; ++s) {
    double best = kInf;
    int bi = 0x7fffffff;
    for (int c = lane; c < ncand; c += 32) {
      double d2 = cand_d2[c];
      int r = cand_row[c];
      if (lex_less(last_v, last_i, d2, r) && lex_less(d2, r, best, bi)) { best = d2; bi = r; }
    }
    warp_lexmin(best, bi);
    if (lane == 0) out_rows[q * budget + s] = bi;
    last_v = best;
    last_i = bi;
  }
  if (lane == 0) {
    for (int s = take; s < budget; ++s) out_rows[q * budget + s] = -1;
    out_count[q] = take;
  }
}

// Fallback resolution + token-id expansion, one thread per query.
__global__ void gather_table_kernel(const int32_t* __restrict__ rows,
                                    const int32_t* __restrict__ count, int64_t nq,
                                    int kmax, const int32_t* __restrict__ own_row,
                                    int fallback, const int64_t* __restrict__ offs,
                                    const int64_t* __restrict__ tok, int64_t width,
                                    int32_t* __restrict__ res_rows,
                                    int32_t* __restrict__ res_count,
                                    int64_t* __restrict__ ids, uint8_t* __restrict__ valid,
                                    int64_t* __restrict__ lengths) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = count[i];
    int32_t buf0 = -1;
    const int32_t* lst = rows + i * kmax;
    if (c == 0 && fallback) {
      buf0 = own_row ? own_row[i] : 0;
      lst = &buf0;
      c = 1;
    }
    int64_t len = 0;
    for (int s = 0; s < c; ++s) {
      int r = lst[s];
      if (res_rows) res_rows[i * kmax + s] = r;
      int64_t lo = offs[r], hi = offs[r + 1];
      if (ids)
        for (int64_t j = lo; j < hi; ++j) {
          ids[i * width + len + (j - lo)] = tok[j];
          valid[i * width + len + (j - lo)] = 1;
        }
      len += hi - lo;
    }
    if (res_rows)
      for (int s = c; s < kmax; ++s) res_rows[i * kmax + s] = -1;
    if (res_count) res_count[i] = c;
    if (ids)
      for (int64_t j = len; j < width; ++j) {
        ids[i * width + j] = 0;
        valid[i * width + j] = 0;
      }
    if (lengths) lengths[i] = len;
  }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_route_volume(const double* points, int64_t nq, const double* centers,
                      int64_t n_blocks, int budget, int32_t* out_rows,
                      int32_t* out_count, void* stream) {
  LSRM_REQUIRE(budget >= 0, "route_volume: negative budget");
  if (nq == 0) return LSRM_OK;
  unsigned blocks = (unsigned)ceil_div(nq, 8);
  route_volume_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      points, nq, centers, (int)n_blocks, budget, out_rows, out_count);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_route_image(const double* points, int64_t nq, const double* cams,
                     int n_views, const int64_t* view_row_start,
                     const double* block_centers, int64_t n_blocks,
                     const double* token_points_bm, const int64_t* block_offsets,
                     int b_i, int budget, int32_t* out_rows, int32_t* out_count,
                     void* stream) {
  LSRM_REQUIRE(budget >= 0 && b_i >= 0, "route_image: negative budget");
  if (nq == 0) return LSRM_OK;
  (void)n_blocks;
  const int warps = 8;
  size_t cap = (size_t)n_views * b_i;
  size_t smem = warps * cap * sizeof(int) + ((warps * cap) & 1) * sizeof(int) +
                warps * cap * sizeof(double);
  LSRM_REQUIRE(smem <= 200 * 1024, "route_image: n_views*b_i too large");
  if (smem > 48 * 1024)
    LSRM_CUDA(cudaFuncSetAttribute(route_image_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned blocks = (unsigned)ceil_div(nq, warps);
  route_image_kernel<<<blocks, warps * 32, smem, as_stream(stream)>>>(
      points, nq, cams, n_views, view_row_start, block_centers, token_points_bm,
      block_offsets, b_i, budget, out_rows, out_count);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_build_gather_table(const int32_t* rows, const int32_t* count, int64_t nq,
                            int kmax_rows, const int32_t* own_row, int fallback,
                            const int64_t* block_offsets,
                            const int64_t* block_token_ids, int64_t width,
                            int32_t* resolved_rows, int32_t* resolved_count,
                            int64_t* ids, uint8_t* valid, int64_t* lengths,
                            void* stream) {
  LSRM_REQUIRE(kmax_rows >= 1, "gather_table: kmax_rows must be >= 1");
  LSRM_REQUIRE(!ids || valid, "gather_table: ids requires valid");
  if (nq == 0) return LSRM_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(nq, 128), 148 * 8);
  gather_table_kernel<<<blocks, 128, 0, as_stream(stream)>>>(
      rows, count, nq, kmax_rows, own_row, fallback, block_offsets, block_token_ids,
      width, resolved_rows, resolved_count, ids, valid, lengths);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
