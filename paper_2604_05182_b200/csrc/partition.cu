// K11 spatial block partition (lsrm/block_partition.py:54-105).
//
// Global block id per token, stable (block id, token id) order, occupied ids
// ascending, offsets/occupancy/centers.  Integer work, bit-exact:
//   1. block id + histogram (atomics on counts only; order fixed later)
//   2. one-CTA exclusive scans over the n_blocks_total histogram: token
//      starts per block and the occupied-row compaction (+ centers)
//   3. unordered scatter into each block's segment
//   4. per-segment rank sort by token id (CTA per occupied block) -> stable
#include "common.cuh"

namespace lsrm {

__global__ void partition_bid_kernel(int modality, const int64_t* __restrict__ coords,
                                     int64_t n, int g1, int bs,
                                     int64_t* __restrict__ bid_out,
                                     int* __restrict__ counts) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c0 = coords[3 * t], c1 = coords[3 * t + 1], c2 = coords[3 * t + 2];
    int64_t sb = g1 / bs, b;
    if (modality == 0)
      b = ((c0 / bs) * sb + c1 / bs) * sb + c2 / bs;
    else  // (view, u, v): id = view*sb^2 + (v/bs)*sb + u/bs
      b = c0 * sb * sb + (c2 / bs) * sb + c1 / bs;
    bid_out[t] = b;
    atomicAdd(&counts[b], 1);
  }
}

// Block-wide inclusive scan of one int per thread (blockDim = 1024).
__device__ int block_scan_incl(int v, int* smem_warp) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) smem_warp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < (int)(blockDim.x >> 5)) ? smem_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    smem_warp[lane] = w;
  }
  __syncthreads();
  int add = warp ? smem_warp[warp - 1] : 0;
  __syncthreads();
  return v + add;
}

__global__ void __launch_bounds__(1024)
partition_scan_kernel(int modality, int64_t total, int64_t n, int g1, int bs,
                      const int* __restrict__ counts,
                      int64_t* __restrict__ starts, int* __restrict__ cursor,
                      int64_t* __restrict__ occupied_ids,
                      int64_t* __restrict__ offsets, int64_t* __restrict__ occupancy,
                      double* __restrict__ centers, int64_t* __restrict__ views,
                      int64_t* __restrict__ n_occ_out, int* __restrict__ row_of_bid) {
  __shared__ int warp_sums[32];
  __shared__ int64_t carry_tok, carry_occ;
  if (threadIdx.x == 0) { carry_tok = 0; carry_occ = 0; }
  __syncthreads();
  int64_t sb = g1 / bs;
  for (int64_t base = 0; base < total; base += blockDim.x) {
    int64_t b = base + threadIdx.x;
    int cnt = b < total ? counts[b] : 0;
    int occ = cnt > 0 ? 1 : 0;
    int incl_tok = block_scan_incl(cnt, warp_sums);
    int incl_occ = block_scan_incl(occ, warp_sums);
    int64_t start = carry_tok + incl_tok - cnt;
    int64_t row = carry_occ + incl_occ - occ;
    if (b < total) {
      starts[b] = start;
      cursor[b] = 0;
      row_of_bid[b] = occ ? (int)row : -1;
      if (occ) {
        occupied_ids[row] = b;
        offsets[row] = start;
        occupancy[row] = cnt;
        double half = bs / 2.0;
        if (modality == 0) {
          int64_t bi = b / (sb * sb), bj = (b / sb) % sb, bk = b % sb;
          double side = (double)g1;
          centers[3 * row + 0] = ddiv(dadd((double)(bs * bi), half), side);
          centers[3 * row + 1] = ddiv(dadd((double)(bs * bj), half), side);
          centers[3 * row + 2] = ddiv(dadd((double)(bs * bk), half), side);
        } else {
          int64_t rem = b % (sb * sb);
          centers[2 * row + 0] = dadd((double)(bs * (rem % sb)), half);
          centers[2 * row + 1] = dadd((double)(bs * (rem / sb)), half);
          if (views) views[row] = b / (sb * sb);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_tok += incl_tok;
      carry_occ += incl_occ;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    offsets[carry_occ] = n;
    *n_occ_out = carry_occ;
  }
}

__global__ void partition_scatter_kernel(const int64_t* __restrict__ bid, int64_t n,
                                         const int64_t* __restrict__ starts,
                                         int* __restrict__ cursor,
                                         int64_t* __restrict__ token_ids) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = bid[t];
    int slot = atomicAdd(&cursor[b], 1);
    token_ids[starts[b] + slot] = t;
  }
}

// Rank sort of each occupied block's segment by token id (ids are unique).
__global__ void partition_segsort_kernel(const int64_t* __restrict__ offsets,
                                         const int64_t* __restrict__ n_occ,
                                         int64_t* __restrict__ token_ids) {
  extern __shared__ int64_t seg[];
  int64_t row = blockIdx.x;
  if (row >= *n_occ) return;
  int64_t lo = offsets[row], len = offsets[row + 1] - lo;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) seg[i] = token_ids[lo + i];
  __syncthreads();
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
    int64_t v = seg[i];
    int64_t rank = 0;
    for (int64_t j = 0; j < len; ++j) rank += seg[j] < v;
    token_ids[lo + rank] = v;
  }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

size_t lsrm_partition_workspace(int64_t n, int64_t n_blocks_total) {
  (void)n;
  // counts(int) cursor(int) row_of_bid(int) starts(int64) n_occ(int64)
  return (size_t)n_blocks_total * (3 * sizeof(int) + sizeof(int64_t)) + 64;
}

int lsrm_partition(int modality, const int64_t* coords, int64_t n, int g0,
                   int g1, int g2, int block_size, int64_t* block_of_token,
                   int64_t* block_token_ids, int64_t* occupied_ids,
                   int64_t* block_offsets, int64_t* occupancy, double* centers,
                   int64_t* block_views, int64_t* n_occupied, void* workspace,
                   size_t ws_bytes, void* stream) {
  LSRM_REQUIRE(modality == 0 || modality == 1, "partition: bad modality %d", modality);
  LSRM_REQUIRE(block_size >= 1, "partition: block_size must be positive");
  LSRM_REQUIRE(g1 % block_size == 0,
               "grid side %d not divisible by block %d", g1, block_size);
  LSRM_REQUIRE(modality == 1 || g0 % block_size == 0,
               "grid side %d not divisible by block %d", g0, block_size);
  (void)g2;
  int64_t sb = g1 / block_size;
  int64_t total = modality == 0 ? sb * sb * sb : (int64_t)g0 * sb * sb;
  LSRM_REQUIRE(ws_bytes >= lsrm_partition_workspace(n, total),
               "partition: workspace too small");
  cudaStream_t st = as_stream(stream);
  char* ws = (char*)workspace;
  int64_t* starts = (int64_t*)ws;
  int64_t* n_occ_dev = starts + total;
  int* counts = (int*)(n_occ_dev + 1);
  int* cursor = counts + total;
  int* row_of_bid = cursor + total;
  LSRM_CUDA(cudaMemsetAsync(counts, 0, total * sizeof(int), st));
  if (n > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
    partition_bid_kernel<<<blocks, 256, 0, st>>>(modality, coords, n, g1, block_size,
                                                 block_of_token, counts);
    LSRM_LAUNCHED();
  }
  partition_scan_kernel<<<1, 1024, 0, st>>>(modality, total, n, g1, block_size, counts,
                                            starts, cursor, occupied_ids, block_offsets,
                                            occupancy, centers, block_views, n_occ_dev,
                                            row_of_bid);
  LSRM_LAUNCHED();
  LSRM_CUDA(cudaMemcpyAsync(n_occupied, n_occ_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (n > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
    partition_scatter_kernel<<<blocks, 256, 0, st>>>(block_of_token, n, starts, cursor,
                                                     block_token_ids);
    LSRM_LAUNCHED();
  }
  LSRM_CUDA(cudaStreamSynchronize(st));
  int64_t B = *n_occupied;
  if (B > 0) {
    int64_t max_seg = modality == 0 ? (int64_t)block_size * block_size * block_size
                                    : (int64_t)block_size * block_size;
    size_t smem = max_seg * sizeof(int64_t);
    LSRM_REQUIRE(smem <= 200 * 1024, "partition: block of %lld tokens too large",
                 (long long)max_seg);
    if (smem > 48 * 1024)
      LSRM_CUDA(cudaFuncSetAttribute(partition_segsort_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    partition_segsort_kernel<<<(unsigned)B, 256, smem, st>>>(block_offsets, n_occ_dev,
                                                             block_token_ids);
    LSRM_LAUNCHED();
  }
  return LSRM_OK;
}

}  // extern "C"
