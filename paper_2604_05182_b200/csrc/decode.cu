// Feature decode around the sparse stage (lsrm/recon_pipeline.py:209-348;
// SURVEY.md §8f rank 4): the dense coarse feature grid, the sparse fine
// feature rows + cell index, and the blended field query feeding the two
// decoder heads.  f64 arithmetic with the reference's f32 rounding points
// and NumPy's unfused operation order (compiled with --fmad=false).
#include "field.cuh"

namespace lsrm {

constexpr int kMaxDf = kFieldMaxDf;
constexpr int kMaxHidden = kFieldMaxHidden;

// grid[(t*side)^3, d_f]: fine cell (t*i+dx, t*j+dy, t*k+dz) takes slice
// [dz, dy, dx] of token (i, j, k)'s vector (recon_pipeline.py:209-220)
__global__ void decode_scatter_kernel(const float* __restrict__ vec, int side, int t, int d_f,
                                      float* __restrict__ grid) {
  const int64_t s = (int64_t)side * t;
  const int64_t total = s * s * s * d_f;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % d_f);
    const int64_t cell = e / d_f;
    const int64_t Z = cell % s, Y = (cell / s) % s, X = cell / (s * s);
    const int64_t tok = ((X / t) * side + Y / t) * side + Z / t;
    const int dx = (int)(X % t), dy = (int)(Y % t), dz = (int)(Z % t);
    grid[e] = vec[tok * (int64_t)t * t * t * d_f + (((int64_t)dz * t + dy) * t + dx) * d_f + c];
  }
}

// rows[n*t^3 + (dx*t+dy)*t+dz] = slice [dz,dy,dx] of token n; index of the
// fine cell (t*x+dx, t*y+dy, t*z+dz) = that row (recon_pipeline.py:234-258)
__global__ void sparse_features_kernel(const float* __restrict__ vec,
                                       const int64_t* __restrict__ coords, int64_t n, int t,
                                       int d_f, int64_t s_f, int64_t* __restrict__ index,
                                       float* __restrict__ rows) {
  const int64_t t3 = (int64_t)t * t * t;
  const int64_t total = n * t3 * d_f;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % d_f);
    const int64_t r = e / d_f;
    const int64_t tok = r / t3;
    const int m = (int)(r % t3);
    const int dx = m / (t * t), dy = (m / t) % t, dz = m % t;
    rows[e] = vec[tok * t3 * d_f + (((int64_t)dz * t + dy) * t + dx) * d_f + c];
    if (c == 0) {
      const int64_t x = coords[3 * tok] * t + dx, y = coords[3 * tok + 1] * t + dy,
                    z = coords[3 * tok + 2] * t + dz;
      index[(x * s_f + y) * s_f + z] = r;
    }
  }
}

struct DecodeHeads {
  const float *zw1, *zb1, *zw2, *zb2, *sw1, *sb1, *sw2, *sb2;
  int hidden, zc;
};

__global__ void decode_points_kernel(const float* __restrict__ grid, int s_df,
                                     const int64_t* __restrict__ index,
                                     const float* __restrict__ rows, int s_f, int d_f,
                                     const double* __restrict__ pts, int64_t n,
                                     DecodeHeads H, float* __restrict__ z_out,
                                     float* __restrict__ s_out, float* __restrict__ f_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  float f[kMaxDf];
  if (index) {
    // query_field (recon_pipeline.py:304-346)
    int64_t i0[3];
    double fr[3];
    tri_prepare(p, s_f, i0, fr);
    double acc[kMaxDf];
    for (int c = 0; c < d_f; ++c) acc[c] = 0.0;
    int active = 0;
    float corner[kMaxDf];
    for (int dx = 0; dx < 2; ++dx) {
      const double wx = dx ? fr[0] : 1.0 - fr[0];
      for (int dy = 0; dy < 2; ++dy) {
        const double wy = dy ? fr[1] : 1.0 - fr[1];
        for (int dz = 0; dz < 2; ++dz) {
          const double wz = dz ? fr[2] : 1.0 - fr[2];
          const int64_t ci[3] = {i0[0] + dx, i0[1] + dy, i0[2] + dz};
          const int64_t row = index[(ci[0] * s_f + ci[1]) * s_f + ci[2]];
          if (row >= 0) {
            ++active;
            for (int c = 0; c < d_f; ++c) corner[c] = rows[row * d_f + c];
          } else {
            const double cc[3] = {((double)ci[0] + 0.5) / s_f, ((double)ci[1] + 0.5) / s_f,
                                  ((double)ci[2] + 0.5) / s_f};
            trilinear_dense(grid, s_df, d_f, cc, corner);
          }
          const double w = dmul(dmul(wx, wy), wz);
          for (int c = 0; c < d_f; ++c) acc[c] = dadd(acc[c], dmul(w, (double)corner[c]));
        }
      }
    }
    const double lam = (double)active / 8.0;
    trilinear_dense(grid, s_df, d_f, p, corner);
    for (int c = 0; c < d_f; ++c)
      f[c] = (float)dadd(dmul(lam, acc[c]), dmul(1.0 - lam, (double)corner[c]));
  } else {
    trilinear_dense(grid, s_df, d_f, p, f);
  }
  if (f_out)
    for (int c = 0; c < d_f; ++c) f_out[i * d_f + c] = f[c];
  if (!H.zw1) return;   // field query only
  float h[kMaxHidden], o[kMaxHidden];
  affine_act_row(f, d_f, H.zw1, H.zb1, H.hidden, 1, h);
  affine_act_row(h, H.hidden, H.zw2, H.zb2, H.zc, 2, o);
  for (int c = 0; c < H.zc; ++c) z_out[i * H.zc + c] = o[c];
  affine_act_row(f, d_f, H.sw1, H.sb1, H.hidden, 1, h);
  affine_act_row(h, H.hidden, H.sw2, H.sb2, 1, 0, o);
  // + bounding-sphere offset |p - c| - r (camera_geometry.py:219-221)
  s_out[i] = s_with_bias(o[0], p, 0.45);
}

// y = f32(act(f32(x W + b))): tensor_core.affine (+ activation) in f64 with
// np.einsum's reduction order (field.cuh), one thread per output element;
// consecutive threads take consecutive output columns (coalesced W reads,
// broadcast x reads).
__global__ void affine_exact_kernel(const float* __restrict__ x, int64_t ldx, int64_t n, int din,
                                    const float* __restrict__ w, const float* __restrict__ b,
                                    int dout, int act, float* __restrict__ y, int64_t ldy) {
  const int64_t total = n * dout;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / dout;
    const int o = (int)(e % dout);
    const float* xr = x + r * ldx;
    double s;
    if (dout == 1) {
      s = einsum_dot(xr, w, 1, din);
    } else {
      s = 0.0;
      for (int i = 0; i < din; ++i) s = dadd(s, dmul((double)xr[i], (double)w[(int64_t)i * dout + o]));
    }
    if (b) s = dadd(s, (double)b[o]);
    float v = (float)s;
    if (act == 1) v = gelu_ref(v);
    else if (act == 2) v = sigmoid_ref_f(v);
    y[r * ldy + o] = v;
  }
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_affine_exact(const float* x, int64_t ldx, int64_t n, int din, const float* w,
                      const float* bias, int dout, int act, float* y, int64_t ldy,
                      void* stream) {
  LSRM_REQUIRE(din >= 1 && dout >= 1, "affine: bad widths %d x %d", din, dout);
  LSRM_REQUIRE(act >= 0 && act <= 2, "affine: activation %d not in {0 identity, 1 gelu, "
               "2 sigmoid}", act);
  if (n == 0) return LSRM_OK;
  const int64_t total = n * dout;
  const unsigned g = (unsigned)(ceil_div(total, 256) < 148 * 64 ? ceil_div(total, 256) : 148 * 64);
  affine_exact_kernel<<<g, 256, 0, as_stream(stream)>>>(x, ldx, n, din, w, bias, dout, act, y, ldy);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_decode_scatter(const float* vec, int side, int t, int d_f, float* grid, void* stream) {
  LSRM_REQUIRE(side >= 1 && t >= 1 && d_f >= 1, "decode_scatter: bad sizes");
  const int64_t total = (int64_t)side * side * side * t * t * t * d_f;
  const unsigned g = (unsigned)(ceil_div(total, 256) < 148 * 32 ? ceil_div(total, 256) : 148 * 32);
  decode_scatter_kernel<<<g, 256, 0, as_stream(stream)>>>(vec, side, t, d_f, grid);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_sparse_features(const float* vec, const int64_t* coords, int64_t n, int t, int d_f,
                         int64_t s_f, int64_t* index, float* rows, void* stream) {
  LSRM_REQUIRE(t >= 1 && d_f >= 1 && s_f >= 1, "sparse_features: bad sizes");
  cudaStream_t st = as_stream(stream);
  LSRM_CUDA(cudaMemsetAsync(index, 0xff, (size_t)s_f * s_f * s_f * sizeof(int64_t), st));
  if (n == 0) return LSRM_OK;
  const int64_t total = n * t * t * t * d_f;
  const unsigned g = (unsigned)(ceil_div(total, 256) < 148 * 32 ? ceil_div(total, 256) : 148 * 32);
  sparse_features_kernel<<<g, 256, 0, st>>>(vec, coords, n, t, d_f, s_f, index, rows);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_decode_points(const float* grid, int s_df, const int64_t* sparse_index,
                       const float* sparse_rows, int s_f, int d_f, const double* points,
                       int64_t n, const float* const* head_w, int hidden, int z_channels,
                       float* z_out, float* s_out, float* field_out, void* stream) {
  LSRM_REQUIRE(d_f >= 1 && d_f <= kMaxDf, "decode_points: d_f %d out of range", d_f);
  LSRM_REQUIRE(hidden >= 1 && hidden <= kMaxHidden && z_channels >= 1 &&
                   z_channels <= kMaxHidden, "decode_points: head width out of range");
  LSRM_REQUIRE(s_df >= 2, "trilinear needs side >= 2");
  if (n == 0) return LSRM_OK;
  LSRM_REQUIRE(head_w || field_out, "decode_points: nothing to compute");
  DecodeHeads H{};
  if (head_w)
    H = DecodeHeads{head_w[0], head_w[1], head_w[2], head_w[3], head_w[4], head_w[5],
                    head_w[6], head_w[7], hidden, z_channels};
  decode_points_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(
      grid, s_df, sparse_index, sparse_rows, s_f, d_f, points, n, H, z_out, s_out, field_out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
