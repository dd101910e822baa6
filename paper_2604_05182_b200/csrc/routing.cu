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

// Two-stage image rule, one warp per query:
//  1. per view, the projected query's 2D squared distance to every block
//     center of the view (lanes over rows, staged in the warp's shared
//     scratch); a row is a candidate iff fewer than b_i rows of the view
//     precede it in (d2, row) order: the set np.argsort(kind="stable")[:b_i]
//     selects.  Rank counting over the staged values needs no cross-lane
//     selection passes; candidates are appended with a ballot prefix.
//  2. per candidate block (eight lanes per candidate), the minimum 3D
//     squared distance from the query to the block's token points.
//  3. the budget smallest candidates in (min d2, row) order.
// f64 with explicit round-to-nearest operations in the reference's order, so
// lists are bit-exact including ties.
__global__ void route_image_kernel(const double* __restrict__ points, int64_t nq,
                                   const double* __restrict__ cams, int n_views,
                                   const int64_t* __restrict__ view_row_start,
                                   const double* __restrict__ bc,
                                   const double* __restrict__ tp,
                                   const double* __restrict__ bounds,
                                   const int64_t* __restrict__ offs, int n_blocks, int b_i,
                                   int budget, int max_view_rows,
                                   int32_t* __restrict__ out_rows,
                                   int32_t* __restrict__ out_count) {
  extern __shared__ double smem_d[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x / 32;
  const int cap = n_views * b_i;
  double* vd2 = smem_d + (size_t)warp * max_view_rows;                 // [max_view_rows]
  double* cand_d2 = smem_d + (size_t)nwarps * max_view_rows + (size_t)warp * cap;
  int* cand_row = reinterpret_cast<int*>(smem_d + (size_t)nwarps * (max_view_rows + cap)) +
                  (size_t)warp * cap;
  int64_t q = blockIdx.x * (int64_t)nwarps + warp;
  if (q >= nq) return;
  const double px = points[3 * q], py = points[3 * q + 1], pz = points[3 * q + 2];
  const int64_t offs_end = offs[n_blocks];
  int ncand = 0;
  for (int v = 0; v < n_views; ++v) {
    const int r0 = (int)view_row_start[v], n = (int)view_row_start[v + 1] - r0;
    if (n <= 0) continue;
    const double* K = cams + 21 * v;
    const double* R = K + 9;
    const double* t = K + 18;
    // camera-space coordinates via R^T, reference order (block_routing.py:149-162)
    const double dx = dsub(px, t[0]), dy = dsub(py, t[1]), dz = dsub(pz, t[2]);
    const double zc = dadd(dadd(dmul(R[2], dx), dmul(R[5], dy)), dmul(R[8], dz));
    if (!(zc > 0.0)) continue;
    const double xc = dadd(dadd(dmul(R[0], dx), dmul(R[3], dy)), dmul(R[6], dz));
    const double yc = dadd(dadd(dmul(R[1], dx), dmul(R[4], dy)), dmul(R[7], dz));
    const double uu = ddiv(dadd(dmul(K[0], ddiv(xc, zc)), K[2]), 8.0);
    const double vv = ddiv(dadd(dmul(K[4], ddiv(yc, zc)), K[5]), 8.0);
    if (n <= b_i) {                         // every row of the view is shortlisted
      for (int i = lane; i < n; i += 32) cand_row[ncand + i] = r0 + i;
      ncand += n;
      continue;
    }
    for (int i = lane; i < n; i += 32) {
      const double du = dsub(uu, bc[2 * (r0 + i)]), dv = dsub(vv, bc[2 * (r0 + i) + 1]);
      vd2[i] = dadd(dmul(du, du), dmul(dv, dv));
    }
    __syncwarp();
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      bool take = false;
      if (i < n) {
        const double di = vd2[i];
        int rank = 0;
        for (int j = 0; j < n && rank < b_i; ++j) rank += lex_less(vd2[j], j, di, i);
        take = rank < b_i;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (take) cand_row[ncand + __popc(bal & ((1u << lane) - 1u))] = r0 + i;
      ncand += __popc(bal);
    }
    __syncwarp();
  }
  __syncwarp();
  // Prune candidates that cannot reach the top `budget`: per candidate a
  // lower bound LB (distance to the block's token-point bounding box, the
  // same rounded operations on clamped coordinates: rounding is monotone, so
  // LB <= every token point's rounded d2) and an upper bound UB (d2 to the
  // block's first token point).  T = the budget-th smallest of the lanes'
  // smallest UBs (distinct candidates), so a candidate with LB > T has at
  // least `budget` candidates strictly closer and is dropped; LB == T is kept
  // (possible tie).
  {
    const int64_t ni = offs_end;
    double ub = kInf;
    for (int c = lane; c < ncand; c += 32) {
      const int r = cand_row[c];
      const double* b = bounds + 6 * (size_t)r;
      const double cx = px < b[0] ? b[0] : (px > b[3] ? b[3] : px);
      const double cy = py < b[1] ? b[1] : (py > b[4] ? b[4] : py);
      const double cz = pz < b[2] ? b[2] : (pz > b[5] ? b[5] : pz);
      cand_d2[c] = dist2(px, py, pz, cx, cy, cz);
      const int64_t j = offs[r];
      ub = fmin(ub, dist2(px, py, pz, tp[j], tp[ni + j], tp[2 * ni + j]));
    }
    double thr = kInf;
    if (budget > 0 && budget <= 32) {
      int rank = 0;                 // lanes with a smaller UB (ties: lower lane)
      for (int o = 0; o < 32; ++o) {
        const double u = __shfl_sync(0xffffffffu, ub, o);
        rank += (u < ub) || (u == ub && o < lane);
      }
      const unsigned hit = __ballot_sync(0xffffffffu, rank == budget - 1 && ub < kInf);
      if (hit) thr = __shfl_sync(0xffffffffu, ub, __ffs(hit) - 1);
    }
    __syncwarp();
    // compact the survivors (order kept)
    int nkeep = 0;
    for (int c0 = 0; c0 < ncand; c0 += 32) {
      const int c = c0 + lane;
      const bool keep = c < ncand && cand_d2[c] <= thr;
      const int r = c < ncand ? cand_row[c] : 0;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) cand_row[nkeep + __popc(bal & ((1u << lane) - 1u))] = r;
      nkeep += __popc(bal);
      __syncwarp();
    }
    ncand = nkeep;
    // exact min 3D squared distance to each surviving block's points: four
    // candidates per pass, eight lanes per candidate striding its points
    // (token points are SoA, so a group's loads are contiguous), then a
    // three-round min over the group
    const int grp = lane >> 3, sub = lane & 7;
    for (int c0 = 0; c0 < ncand; c0 += 4) {
      const int c = c0 + grp;
      double best = kInf;
      if (c < ncand) {
        const int r = cand_row[c];
        for (int64_t j = offs[r] + sub, e = offs[r + 1]; j < e; j += 8)
          best = fmin(best, dist2(px, py, pz, tp[j], tp[ni + j], tp[2 * ni + j]));
      }
      best = fmin(best, __shfl_xor_sync(0xffffffffu, best, 4));
      best = fmin(best, __shfl_xor_sync(0xffffffffu, best, 2));
      best = fmin(best, __shfl_xor_sync(0xffffffffu, best, 1));
      if (sub == 0 && c < ncand) cand_d2[c] = best;
    }
  }
  __syncwarp();
  const int take = min(budget, ncand);
  double last_v = -kInf;
  int last_i = -1;
  for (int s = 0; s < take; ++s) {
    double best = kInf;
    int bi = 0x7fffffff;
    for (int c = lane; c < ncand; c += 32) {
      const double d2 = cand_d2[c];
      const int r = cand_row[c];
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

// Per-block bounding box of the token points (SoA [3, Ni], block-major):
// bounds [B, 6] = (min x, min y, min z, max x, max y, max z); warp per block.
__global__ void block_bounds_kernel(const double* __restrict__ tp, int64_t ni,
                                    const int64_t* __restrict__ offs, int64_t nb,
                                    double* __restrict__ bounds) {
  const int64_t b = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (b >= nb) return;
  double lo[3] = {kInf, kInf, kInf}, hi[3] = {-kInf, -kInf, -kInf};
  for (int64_t j = offs[b] + lane; j < offs[b + 1]; j += 32)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], tp[a * ni + j]);
      hi[a] = fmax(hi[a], tp[a * ni + j]);
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  if (lane < 3) bounds[6 * b + lane] = lo[lane];
  else if (lane < 6) bounds[6 * b + lane] = hi[lane - 3];
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
                     const double* token_points_bm, const double* block_bounds,
                     const int64_t* block_offsets,
                     int b_i, int budget, int max_view_rows, int32_t* out_rows,
                     int32_t* out_count, void* stream) {
  LSRM_REQUIRE(budget >= 0 && b_i >= 0, "route_image: negative budget");
  LSRM_REQUIRE(max_view_rows >= 0 && max_view_rows <= n_blocks,
               "route_image: max_view_rows must be in [0, n_blocks]");
  if (nq == 0) return LSRM_OK;
  int warps = 8;
  const size_t cap = (size_t)n_views * b_i;
  auto bytes = [&](int w) {
    return (size_t)w * ((max_view_rows + cap) * sizeof(double) + cap * sizeof(int));
  };
  while (warps > 1 && bytes(warps) > 200 * 1024) warps /= 2;
  const size_t smem = bytes(warps);
  LSRM_REQUIRE(smem <= 200 * 1024, "route_image: n_views*b_i or rows per view too large");
  if (smem > 48 * 1024)
    LSRM_CUDA(cudaFuncSetAttribute(route_image_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned blocks = (unsigned)ceil_div(nq, warps);
  route_image_kernel<<<blocks, warps * 32, smem, as_stream(stream)>>>(
      points, nq, cams, n_views, view_row_start, block_centers, token_points_bm,
      block_bounds, block_offsets, (int)n_blocks, b_i, budget, max_view_rows, out_rows,
      out_count);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_block_bounds(const double* token_points_soa, int64_t n_points,
                      const int64_t* block_offsets, int64_t n_blocks, double* bounds,
                      void* stream) {
  if (n_blocks == 0) return LSRM_OK;
  block_bounds_kernel<<<(unsigned)ceil_div(n_blocks, 8), 256, 0, as_stream(stream)>>>(
      token_points_soa, n_points, block_offsets, n_blocks, bounds);
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
