// K9/K10 foreground pruning + informative-voxel mask and the fine-token
// compaction (lsrm/tokenizer.py:180-313).  Bit-exact: masks are exact f64
// compares on correctly rounded SDF values; compaction keeps flat (argwhere)
// order via a two-level scan; features reproduce the reference's two f64
// roundings f32(f64(parent) + f64(f32(sum of pos-embed rows in f64))).
#include "field.cuh"

namespace lsrm {

constexpr int kScanChunk = 4096;   // cells per CTA in the compaction scan

__global__ void fg_mask_kernel(const float* __restrict__ alpha, int n_views, int h,
                               int w, int patch, uint8_t* __restrict__ mask) {
  int ph = h / patch, pw = w / patch;
  int64_t total = (int64_t)n_views * ph * pw;
  int lane = threadIdx.x & 31;
  for (int64_t cell = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
       cell < total; cell += (int64_t)gridDim.x * (blockDim.x / 32)) {
    int64_t view = cell / (ph * pw);
    int r = (int)((cell / pw) % ph), c = (int)(cell % pw);
    const float* base = alpha + (view * h + (int64_t)r * patch) * w + (int64_t)c * patch;
    bool any = false;
    for (int e = lane; e < patch * patch; e += 32)
      any |= base[(e / patch) * (int64_t)w + (e % patch)] > 0.5f;
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) mask[cell] = any ? 1 : 0;
  }
}

// Float4 fast path: patch == 8, one thread per (patch row) reads 2 float4.
__global__ void fg_mask8_kernel(const float4* __restrict__ alpha, int n_views, int h,
                                int w, uint8_t* __restrict__ mask) {
  int ph = h / 8, pw = w / 8;
  int64_t total = (int64_t)n_views * ph * pw;
  // 8 threads per patch (one per pixel row), 4 patches per warp
  int sub = threadIdx.x & 7, lane = threadIdx.x & 31;
  int64_t warp_g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp_g * 4; base < total; base += n_warps * 4) {  // warp-uniform
    int64_t cell = base + (lane >> 3);
    bool hit = false;
    if (cell < total) {
      int64_t view = cell / (ph * pw);
      int r = (int)((cell / pw) % ph), c = (int)(cell % pw);
      int64_t row = view * h + (int64_t)r * 8 + sub;
      const float4* p = alpha + (row * w + (int64_t)c * 8) / 4;
      float4 a = p[0], b = p[1];
      hit = a.x > 0.5f || a.y > 0.5f || a.z > 0.5f || a.w > 0.5f || b.x > 0.5f ||
            b.y > 0.5f || b.z > 0.5f || b.w > 0.5f;
    }
    unsigned ball = __ballot_sync(0xffffffffu, hit);
    if (cell < total && sub == 0) mask[cell] = ((ball >> (lane & 24)) & 0xffu) ? 1 : 0;
  }
}

__global__ void voxel_mask_kernel(const double* __restrict__ prims, int n_prims, int s_vol,
                                  double tau, int t, uint8_t* __restrict__ mask) {
  extern __shared__ double sh_prims[];
  for (int i = threadIdx.x; i < 8 * n_prims; i += blockDim.x) sh_prims[i] = prims[i];
  __syncthreads();
  int64_t total = (int64_t)s_vol * s_vol * s_vol;
  double fine = (double)t * s_vol;
  for (int64_t vox = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vox < total;
       vox += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(vox / ((int64_t)s_vol * s_vol)), j = (int)((vox / s_vol) % s_vol),
        k = (int)(vox % s_vol);
    double smin = __builtin_huge_val(), smax = -__builtin_huge_val(),
           amin = __builtin_huge_val();
    for (int a = 0; a < t; ++a) {
      double x = ddiv(dadd((double)(t * i + a), 0.5), fine);
      for (int b = 0; b < t; ++b) {
        double y = ddiv(dadd((double)(t * j + b), 0.5), fine);
        for (int c = 0; c < t; ++c) {
          double z = ddiv(dadd((double)(t * k + c), 0.5), fine);
          double s = sdf_prims(sh_prims, n_prims, x, y, z);
          smin = fmin(smin, s);
          smax = fmax(smax, s);
          amin = fmin(amin, fabs(s));
        }
      }
    }
    mask[vox] = (amin <= tau) || (dmul(smin, smax) <= 0.0);
  }
}

// Eq. 11 for a general field (decoded coarse volume, or values of an opaque
// callable), one warp per voxel: the lanes evaluate the t^3 samples, exact
// f64 min / max / min|s| by shuffles.  Voxels of x-slabs [i0, i1).  For the
// values kind, sample ids follow the reference's slab layout
// (tokenizer.py:227-235): ((i - i0) * t + a) * fine^2 + (t j + b) * fine + t k + c.
__global__ void voxel_mask_field_kernel(FieldDev F, int s_vol, double tau, int t, int i0,
                                        int i1, uint8_t* __restrict__ mask) {
  const int lane = threadIdx.x & 31;
  const int64_t plane = (int64_t)s_vol * s_vol;
  const int64_t total = (int64_t)(i1 - i0) * plane;
  const int fine = t * s_vol;
  const double finef = (double)fine;
  const int t3 = t * t * t;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < total;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int i = i0 + (int)(v / plane), j = (int)((v / s_vol) % s_vol), k = (int)(v % s_vol);
    double smin = __builtin_huge_val(), smax = -__builtin_huge_val(),
           amin = __builtin_huge_val();
    for (int e = lane; e < t3; e += 32) {
      const int a = e / (t * t), b = (e / t) % t, c = e % t;
      const int xa = t * i + a, yb = t * j + b, zc = t * k + c;
      const double x = ddiv(dadd((double)xa, 0.5), finef);
      const double y = ddiv(dadd((double)yb, 0.5), finef);
      const double z = ddiv(dadd((double)zc, 0.5), finef);
      const int64_t id = ((int64_t)(i - i0) * t + a) * fine * (int64_t)fine +
                         (int64_t)yb * fine + zc;
      const double s = field_sdf(F, id, x, y, z);
      smin = fmin(smin, s);
      smax = fmax(smax, s);
      amin = fmin(amin, fabs(s));
    }
    for (int o = 16; o; o >>= 1) {
      smin = fmin(smin, __shfl_xor_sync(0xffffffffu, smin, o));
      smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
      amin = fmin(amin, __shfl_xor_sync(0xffffffffu, amin, o));
    }
    if (lane == 0) mask[(int64_t)i * plane + (int64_t)j * s_vol + k] =
        (amin <= tau) || (dmul(smin, smax) <= 0.0);
  }
}

// sample points of x-slabs [i0, i1) in the reference's layout (for an opaque
// field evaluated on the host): pts [(i1-i0) * t * fine^2, 3]
__global__ void voxel_samples_kernel(int s_vol, int t, int i0, int i1,
                                     double* __restrict__ pts) {
  const int fine = t * s_vol;
  const int64_t per_slab = (int64_t)t * fine * fine;
  const int64_t total = (int64_t)(i1 - i0) * per_slab;
  const double finef = (double)fine;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int sl = (int)(e / per_slab);
    const int a = (int)((e / ((int64_t)fine * fine)) % t);
    const int yb = (int)((e / fine) % fine), zc = (int)(e % fine);
    pts[3 * e] = ddiv(dadd((double)(t * (i0 + sl) + a), 0.5), finef);
    pts[3 * e + 1] = ddiv(dadd((double)yb, 0.5), finef);
    pts[3 * e + 2] = ddiv(dadd((double)zc, 0.5), finef);
  }
}

__device__ int block_incl_scan(int v, int* warp_sums) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) warp_sums[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    warp_sums[lane] = w;
  }
  __syncthreads();
  int r = v + (warp ? warp_sums[warp - 1] : 0);
  __syncthreads();
  return r;
}

// Pass 1: count set flags per chunk.
__global__ void __launch_bounds__(1024)
chunk_count_kernel(const uint8_t* __restrict__ flags, int64_t n, int* __restrict__ counts) {
  __shared__ int warp_sums[32];
  int64_t base = (int64_t)blockIdx.x * kScanChunk;
  int c = 0;
  for (int e = threadIdx.x; e < kScanChunk; e += blockDim.x)
    c += (base + e < n && flags[base + e]) ? 1 : 0;
  int tot = block_incl_scan(c, warp_sums);
  if (threadIdx.x == blockDim.x - 1) counts[blockIdx.x] = tot;
}

// Pass 2: exclusive scan of chunk counts (single CTA) + total.
__global__ void __launch_bounds__(1024)
chunk_scan_kernel(int* __restrict__ counts, int64_t n_chunks, int64_t* __restrict__ total) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < n_chunks; b += blockDim.x) {
    int64_t i = b + threadIdx.x;
    int v = i < n_chunks ? counts[i] : 0;
    int incl = block_incl_scan(v, warp_sums);
    if (i < n_chunks) counts[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Pass 3: write the flat cell index of every set flag at its output position.
__global__ void __launch_bounds__(1024)
chunk_emit_kernel(const uint8_t* __restrict__ flags, int64_t n,
                  const int* __restrict__ starts, int32_t* __restrict__ out_cells) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = starts[blockIdx.x];
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kScanChunk;
  for (int e0 = 0; e0 < kScanChunk; e0 += blockDim.x) {
    int64_t cell = base + e0 + threadIdx.x;
    int f = (cell < n && flags[cell]) ? 1 : 0;
    int incl = block_incl_scan(f, warp_sums);
    if (f) out_cells[carry + incl - 1] = (int32_t)cell;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += incl;
    __syncthreads();
  }
}

// One warp per output token: coords + f32(f64(parent) + f64(pe)).
__global__ void compact_volume_rows(const int32_t* __restrict__ cells, int64_t n_out,
                                    int s, int f, const float* __restrict__ x_d, int d,
                                    const float* __restrict__ pe0, const float* __restrict__ pe1,
                                    const float* __restrict__ pe2, int64_t* __restrict__ coords,
                                    float* __restrict__ feats) {
  int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (row >= n_out) return;
  int64_t cell = cells[row];
  int i = (int)(cell / ((int64_t)s * s)), j = (int)((cell / s) % s), k = (int)(cell % s);
  if (lane == 0 && coords) {
    coords[3 * row] = i;
    coords[3 * row + 1] = j;
    coords[3 * row + 2] = k;
  }
  if (!feats) return;
  int sc = s / f;
  int64_t parent = ((int64_t)(i / f) * sc + j / f) * sc + k / f;
  for (int c = lane; c < d; c += 32) {
    double pe = dadd(dadd(dadd(0.0, (double)pe0[(int64_t)i * d + c]), (double)pe1[(int64_t)j * d + c]),
                     (double)pe2[(int64_t)k * d + c]);
    float pe32 = (float)pe;
    feats[row * d + c] = (float)dadd((double)x_d[parent * d + c], (double)pe32);
  }
}

__global__ void compact_image_rows(const int32_t* __restrict__ cells, int64_t n_out,
                                   int s, int f, const float* __restrict__ y_d, int d,
                                   const float* __restrict__ pe_u, const float* __restrict__ pe_v,
                                   int64_t* __restrict__ coords, float* __restrict__ feats) {
  int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (row >= n_out) return;
  int64_t cell = cells[row];
  int64_t view = cell / ((int64_t)s * s);
  int r = (int)((cell / s) % s), col = (int)(cell % s);
  if (lane == 0 && coords) {
    coords[3 * row] = view;
    coords[3 * row + 1] = col;   // u
    coords[3 * row + 2] = r;     // v
  }
  if (!feats) return;
  int sc = s / f;
  int64_t parent = (view * sc + r / f) * sc + col / f;
  for (int c = lane; c < d; c += 32) {
    double pe = dadd(dadd(0.0, (double)pe_u[(int64_t)col * d + c]), (double)pe_v[(int64_t)r * d + c]);
    float pe32 = (float)pe;
    feats[row * d + c] = (float)dadd((double)y_d[parent * d + c], (double)pe32);
  }
}

// Vectorised variant (d % 4 == 0, 16-byte aligned rows): one warp per output
// token, four columns per lane per step (float4 loads and stores), the same
// f64 add order as compact_*_rows.  kind 0 = volume (three tables), 1 = image
// (pe0 = u table, pe1 = v table).
template <int KIND>
__global__ void compact_rows_vec4(const int32_t* __restrict__ cells, int64_t n_out, int s, int f,
                                  const float4* __restrict__ par, int d4,
                                  const float4* __restrict__ pe0, const float4* __restrict__ pe1,
                                  const float4* __restrict__ pe2, int64_t* __restrict__ coords,
                                  float4* __restrict__ feats) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= n_out) return;
  const int64_t cell = cells[row];
  const int sc = s / f;
  int64_t a, b, c, parent;
  if (KIND == 0) {
    a = cell / ((int64_t)s * s); b = (cell / s) % s; c = cell % s;
    parent = ((a / f) * sc + b / f) * sc + c / f;
  } else {
    a = cell / ((int64_t)s * s); b = (cell / s) % s; c = cell % s;   // view, row, col
    parent = (a * sc + b / f) * sc + c / f;
  }
  if (lane == 0 && coords) {
    coords[3 * row] = a;
    coords[3 * row + 1] = KIND == 0 ? b : c;
    coords[3 * row + 2] = KIND == 0 ? c : b;
  }
  if (!feats) return;
  for (int k = lane; k < d4; k += 32) {
    float4 x = __ldg(par + parent * d4 + k);
    float4 o;
    float* op = &o.x;
    const float* xp = &x.x;
    if (KIND == 0) {
      const float4 t0 = __ldg(pe0 + a * d4 + k), t1 = __ldg(pe1 + b * d4 + k),
                   t2 = __ldg(pe2 + c * d4 + k);
      const float *p0 = &t0.x, *p1 = &t1.x, *p2 = &t2.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float pe = (float)dadd(dadd(dadd(0.0, (double)p0[e]), (double)p1[e]), (double)p2[e]);
        op[e] = (float)dadd((double)xp[e], (double)pe);
      }
    } else {
      const float4 tu = __ldg(pe0 + c * d4 + k), tv = __ldg(pe1 + b * d4 + k);
      const float *pu = &tu.x, *pv = &tv.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float pe = (float)dadd(dadd(0.0, (double)pu[e]), (double)pv[e]);
        op[e] = (float)dadd((double)xp[e], (double)pe);
      }
    }
    feats[row * d4 + k] = o;
  }
}

static int compact_cells(const uint8_t* mask, int64_t n_cells, void* workspace,
                         size_t ws_bytes, int32_t** cells_out, int64_t* n_out,
                         cudaStream_t st) {
  int64_t n_chunks = ceil_div(n_cells, kScanChunk);
  LSRM_REQUIRE(ws_bytes >= lsrm_compact_workspace(n_cells), "compact: workspace too small");
  char* ws = (char*)workspace;
  int64_t* total = (int64_t*)ws;
  int* counts = (int*)(ws + 16);
  int32_t* cells = (int32_t*)(ws + 16 + ((n_chunks * sizeof(int) + 15) / 16) * 16);
  chunk_count_kernel<<<(unsigned)n_chunks, 1024, 0, st>>>(mask, n_cells, counts);
  LSRM_LAUNCHED();
  chunk_scan_kernel<<<1, 1024, 0, st>>>(counts, n_chunks, total);
  LSRM_LAUNCHED();
  chunk_emit_kernel<<<(unsigned)n_chunks, 1024, 0, st>>>(mask, n_cells, counts, cells);
  LSRM_LAUNCHED();
  LSRM_CUDA(cudaMemcpyAsync(n_out, total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  LSRM_CUDA(cudaStreamSynchronize(st));
  *cells_out = cells;
  return LSRM_OK;
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_foreground_mask(const float* alpha, int n_views, int h, int w, int patch,
                         uint8_t* mask, void* stream) {
  LSRM_REQUIRE(patch >= 1 && h % patch == 0 && w % patch == 0,
               "alpha %dx%d not divisible by patch %d", h, w, patch);
  int64_t total = (int64_t)n_views * (h / patch) * (w / patch);
  if (total == 0) return LSRM_OK;
  if (patch == 8 && ((uintptr_t)alpha % 16) == 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(total * 8, 256), 148 * 16);
    fg_mask8_kernel<<<blocks, 256, 0, as_stream(stream)>>>((const float4*)alpha, n_views, h, w,
                                                           mask);
  } else {
    int blocks = (int)std::min<int64_t>(ceil_div(total, 8), 148 * 16);
    fg_mask_kernel<<<blocks, 256, 0, as_stream(stream)>>>(alpha, n_views, h, w, patch, mask);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_voxel_mask(const double* sdf, int n_prims, int s_vol, double tau, int t_side,
                    uint8_t* mask, void* stream) {
  LSRM_REQUIRE(s_vol >= 1 && t_side >= 1, "bad mask resolution");
  LSRM_REQUIRE(tau > 0, "tau must be positive");
  LSRM_REQUIRE(n_prims >= 1 && n_prims <= 256, "voxel_mask: 1..256 SDF primitives");
  int64_t total = (int64_t)s_vol * s_vol * s_vol;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 128), 148 * 32);
  voxel_mask_kernel<<<blocks, 128, 8 * n_prims * sizeof(double), as_stream(stream)>>>(
      sdf, n_prims, s_vol, tau, t_side, mask);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_voxel_mask_field(const lsrm_sdf_field* field, int s_vol, double tau, int t_side,
                          int i0, int i1, uint8_t* mask, void* stream) {
  LSRM_REQUIRE(s_vol >= 1 && t_side >= 1, "bad mask resolution");
  LSRM_REQUIRE(tau > 0, "tau must be positive");
  LSRM_REQUIRE(0 <= i0 && i0 <= i1 && i1 <= s_vol, "voxel mask: slab range [%d, %d) out of "
               "[0, %d)", i0, i1, s_vol);
  int rc = lsrm_check_field(field);
  if (rc) return rc;
  if (i0 == i1) return LSRM_OK;
  if (field->kind == kFieldAnalytic && i0 == 0 && i1 == s_vol)
    return lsrm_voxel_mask(field->prims, field->n_prims, s_vol, tau, t_side, mask, stream);
  FieldDev F{};
  F.kind = field->kind;
  F.prims = field->prims;
  F.n_prims = field->n_prims;
  F.grid = field->grid;
  F.side = field->side;
  F.d_f = field->d_f;
  F.hidden = field->hidden;
  F.w1 = field->w1;
  F.b1 = field->b1;
  F.w2 = field->w2;
  F.b2 = field->b2;
  F.radius = field->radius;
  F.values = field->values;
  const int64_t voxels = (int64_t)(i1 - i0) * s_vol * s_vol;
  const int blocks = (int)std::min<int64_t>(ceil_div(voxels, 4), 148 * 64);
  voxel_mask_field_kernel<<<blocks, 128, 0, as_stream(stream)>>>(F, s_vol, tau, t_side, i0, i1,
                                                                 mask);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_voxel_sample_points(int s_vol, int t_side, int i0, int i1, double* points,
                             void* stream) {
  LSRM_REQUIRE(s_vol >= 1 && t_side >= 1, "bad mask resolution");
  LSRM_REQUIRE(0 <= i0 && i0 <= i1 && i1 <= s_vol, "voxel samples: bad slab range");
  const int64_t fine = (int64_t)t_side * s_vol;
  const int64_t total = (int64_t)(i1 - i0) * t_side * fine * fine;
  if (total == 0) return LSRM_OK;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 32);
  voxel_samples_kernel<<<blocks, 256, 0, as_stream(stream)>>>(s_vol, t_side, i0, i1, points);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

size_t lsrm_compact_workspace(int64_t n_cells) {
  int64_t n_chunks = ceil_div(n_cells, kScanChunk);
  return 16 + ((n_chunks * sizeof(int) + 15) / 16) * 16 + n_cells * sizeof(int32_t) + 16;
}

int lsrm_compact_volume(const uint8_t* mask, int s_fine, int factor, const float* x_d,
                        int d, const float* pe0, const float* pe1, const float* pe2,
                        int64_t* coords, float* features, int64_t max_out,
                        int64_t* n_out, void* workspace, size_t ws_bytes, void* stream) {
  LSRM_REQUIRE(factor >= 1 && s_fine % factor == 0, "volume mask not divisible by factor");
  cudaStream_t st = as_stream(stream);
  int32_t* cells = nullptr;
  int rc = compact_cells(mask, (int64_t)s_fine * s_fine * s_fine, workspace, ws_bytes,
                         &cells, n_out, st);
  if (rc) return rc;
  if ((!coords && !features) || *n_out == 0) return LSRM_OK;
  LSRM_REQUIRE(*n_out <= max_out, "compact_volume: %lld tokens exceed max_out %lld",
               (long long)*n_out, (long long)max_out);
  compact_volume_rows<<<(unsigned)ceil_div(*n_out, 8), 256, 0, st>>>(
      cells, *n_out, s_fine, factor, x_d, d, pe0, pe1, pe2, coords, features);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_compact_image(const uint8_t* mask, int n_views, int s_fine, int factor,
                       const float* y_d, int d, const float* pe_u, const float* pe_v,
                       int64_t* coords, float* features, int64_t max_out, int64_t* n_out,
                       void* workspace, size_t ws_bytes, void* stream) {
  LSRM_REQUIRE(factor >= 1 && s_fine % factor == 0, "image mask not divisible by factor");
  cudaStream_t st = as_stream(stream);
  int32_t* cells = nullptr;
  int rc = compact_cells(mask, (int64_t)n_views * s_fine * s_fine, workspace, ws_bytes,
                         &cells, n_out, st);
  if (rc) return rc;
  if ((!coords && !features) || *n_out == 0) return LSRM_OK;
  LSRM_REQUIRE(*n_out <= max_out, "compact_image: %lld tokens exceed max_out %lld",
               (long long)*n_out, (long long)max_out);
  compact_image_rows<<<(unsigned)ceil_div(*n_out, 8), 256, 0, st>>>(
      cells, *n_out, s_fine, factor, y_d, d, pe_u, pe_v, coords, features);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_compact_rows(int modality, const void* workspace, int64_t n_cells, int64_t n_out,
                      int n_views, int s_fine, int factor, const float* parents, int d,
                      const float* pe0, const float* pe1, const float* pe2, int64_t* coords,
                      float* features, void* stream) {
  LSRM_REQUIRE(modality == 0 || modality == 1, "compact_rows: modality must be 0 or 1");
  LSRM_REQUIRE(factor >= 1 && s_fine % factor == 0, "mask not divisible by factor");
  (void)n_views;
  if (n_out == 0) return LSRM_OK;
  const int64_t n_chunks = ceil_div(n_cells, kScanChunk);
  const int32_t* cells = (const int32_t*)((const char*)workspace + 16 +
                                          ((n_chunks * sizeof(int) + 15) / 16) * 16);
  cudaStream_t st = as_stream(stream);
  const uintptr_t al = (uintptr_t)parents | (uintptr_t)pe0 | (uintptr_t)pe1 |
                       (uintptr_t)(modality == 0 ? pe2 : nullptr) | (uintptr_t)features;
  const unsigned blocks = (unsigned)ceil_div(n_out, 8);
  if (d % 4 == 0 && (al & 15) == 0) {
    if (modality == 0)
      compact_rows_vec4<0><<<blocks, 256, 0, st>>>(
          cells, n_out, s_fine, factor, (const float4*)parents, d / 4, (const float4*)pe0,
          (const float4*)pe1, (const float4*)pe2, coords, (float4*)features);
    else
      compact_rows_vec4<1><<<blocks, 256, 0, st>>>(
          cells, n_out, s_fine, factor, (const float4*)parents, d / 4, (const float4*)pe0,
          (const float4*)pe1, nullptr, coords, (float4*)features);
  } else if (modality == 0) {
    compact_volume_rows<<<blocks, 256, 0, st>>>(cells, n_out, s_fine, factor, parents, d, pe0,
                                                pe1, pe2, coords, features);
  } else {
    compact_image_rows<<<blocks, 256, 0, st>>>(cells, n_out, s_fine, factor, parents, d, pe0,
                                               pe1, coords, features);
  }
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
