// Router input producer: the 3D surface point of every image token's
// patch-center ray (lsrm/block_routing.py:73-108 with
// lsrm/camera_geometry.py:236-302), one thread per ray, f64.
//
// 128 mid-segment samples between cube entry and exit, SDF of the analytic
// scene (union of spheres / boxes), Laplace density, and the sample with the
// largest transmittance x alpha (first maximum).  Rays that miss the cube or
// whose min SDF stays above 3 beta fall back to the cube-entry point / the
// clamped closest approach to the cube center and are flagged.
//
// Compiled with --fmad=false: the elementwise steps follow NumPy's
// unfused operation order.  exp() and the reference's BLAS-evaluated
// rotation / norm are not bit-identical across libraries, so the points are
// tolerance-matched (tests/test_raymarch.py), not bit-exact.
#include "common.cuh"

namespace lsrm {

constexpr int kMarch = 128;
constexpr double kNoPeakMargin = 3.0;

__device__ __forceinline__ double sdf_union(const double* prims, int n_prims, double x, double y,
                                            double z) {
  double best = 1e300;
  for (int k = 0; k < n_prims; ++k) {
    const double* p = prims + 8 * k;
    double s;
    if (p[0] == 0.0) {   // sphere: |p - c| - r
      const double dx = x - p[1], dy = y - p[2], dz = z - p[3];
      s = sqrt(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz))) - p[4];
    } else {             // box: |max(q, 0)| + min(max(q), 0), q = |p - c| - h
      const double qx = fabs(x - p[1]) - p[4], qy = fabs(y - p[2]) - p[5],
                   qz = fabs(z - p[3]) - p[6];
      const double mx = fmax(qx, 0.0), my = fmax(qy, 0.0), mz = fmax(qz, 0.0);
      const double outside = sqrt(dadd(dadd(dmul(mx, mx), dmul(my, my)), dmul(mz, mz)));
      s = outside + fmin(fmax(fmax(qx, qy), qz), 0.0);
    }
    best = fmin(best, s);
  }
  return best;
}

// slab method against [0,1]^3 (camera_geometry.py:236-252); false = no span
__device__ __forceinline__ bool cube_span(const double* o, const double* d, double& t0o,
                                          double& t1o) {
  double t0 = -INFINITY, t1 = INFINITY;
  for (int ax = 0; ax < 3; ++ax) {
    if (fabs(d[ax]) < 1e-12) {
      if (o[ax] < 0.0 || o[ax] > 1.0) return false;
      continue;
    }
    const double a = (0.0 - o[ax]) / d[ax], b = (1.0 - o[ax]) / d[ax];
    t0 = fmax(t0, fmin(a, b));
    t1 = fmin(t1, fmax(a, b));
  }
  if (t1 <= t0 || t1 <= 0.0) return false;
  t0o = fmax(t0, 0.0);
  t1o = t1;
  return true;
}

__global__ void image_points_kernel(const int64_t* __restrict__ coords, int64_t n,
                                    const double* __restrict__ cams,
                                    const int32_t* __restrict__ wh, int rows_f,
                                    const double* __restrict__ prims, int n_prims, double beta,
                                    double* __restrict__ out, uint8_t* __restrict__ miss) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int view = (int)coords[3 * i];
  const double u = (double)coords[3 * i + 1], v = (double)coords[3 * i + 2];
  const double* K = cams + 21 * view;
  const double* R = K + 9;
  const double* T = K + 18;
  const double W = (double)wh[2 * view], H = (double)wh[2 * view + 1];
  const double px = dmul(u + 0.5, W / rows_f), py = dmul(v + 0.5, H / rows_f);
  const double dc[3] = {(px - K[2]) / K[0], (py - K[5]) / K[4], 1.0};
  double d[3];
  for (int r = 0; r < 3; ++r)
    d[r] = dadd(dadd(dmul(R[3 * r], dc[0]), dmul(R[3 * r + 1], dc[1])), dmul(R[3 * r + 2], dc[2]));
  for (int pass = 0; pass < 2; ++pass) {   // normalised twice, as the reference does
    const double nrm = sqrt(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
    d[0] /= nrm;
    d[1] /= nrm;
    d[2] /= nrm;
  }
  const double o[3] = {T[0], T[1], T[2]};
  double t0, t1, p[3];
  bool peak = false;
  if (cube_span(o, d, t0, t1)) {
    const double step = (t1 - t0) / kMarch;
    double trans = 1.0, best_w = -1.0, s_min = INFINITY;
    int best = 0;
    for (int k = 0; k < kMarch; ++k) {
      const double t = dadd(t0, dmul(k + 0.5, step));
      const double x = dadd(o[0], dmul(t, d[0])), y = dadd(o[1], dmul(t, d[1])),
                   z = dadd(o[2], dmul(t, d[2]));
      const double s = sdf_union(prims, n_prims, x, y, z);
      s_min = fmin(s_min, s);
      const double psi = s >= 0.0 ? 0.5 * exp(-s / beta) : 1.0 - 0.5 * exp(s / beta);
      const double alpha = 1.0 - exp(-dmul(psi / beta, step));
      const double w = dmul(trans, alpha);
      if (w > best_w) {   // first maximum (np.argmax)
        best_w = w;
        best = k;
      }
      trans = dmul(trans, 1.0 - alpha);
    }
    if (!(s_min > kNoPeakMargin * beta)) {
      peak = true;
      const double t = dadd(t0, dmul(best + 0.5, step));
      p[0] = dadd(o[0], dmul(t, d[0]));
      p[1] = dadd(o[1], dmul(t, d[1]));
      p[2] = dadd(o[2], dmul(t, d[2]));
    } else {
      p[0] = dadd(o[0], dmul(t0, d[0]));
      p[1] = dadd(o[1], dmul(t0, d[1]));
      p[2] = dadd(o[2], dmul(t0, d[2]));
    }
  } else {   // closest approach to the cube center, clamped to t >= 0
    const double tn = dadd(dadd(dmul(0.5 - o[0], d[0]), dmul(0.5 - o[1], d[1])),
                           dmul(0.5 - o[2], d[2]));
    const double t = fmax(tn, 0.0);
    p[0] = dadd(o[0], dmul(t, d[0]));
    p[1] = dadd(o[1], dmul(t, d[1]));
    p[2] = dadd(o[2], dmul(t, d[2]));
  }
  for (int c = 0; c < 3; ++c) out[3 * i + c] = fmin(fmax(p[c], 0.0), 1.0);
  miss[i] = peak ? 0 : 1;
}

}  // namespace lsrm

using namespace lsrm;

extern "C" int lsrm_image_token_points(const int64_t* coords, int64_t n, const double* cams,
                                       const int32_t* image_wh, int n_views, int rows_f,
                                       const double* sdf, int n_prims, double beta,
                                       double* points, uint8_t* miss, void* stream) {
  LSRM_REQUIRE(n_views >= 1 && rows_f >= 1, "image points: bad view count / grid");
  LSRM_REQUIRE(n_prims >= 1, "image points: empty SDF");
  LSRM_REQUIRE(beta > 0.0, "beta must be positive");
  if (n == 0) return LSRM_OK;
  image_points_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(
      coords, n, cams, image_wh, rows_f, sdf, n_prims, beta, points, miss);
  LSRM_LAUNCHED();
  return LSRM_OK;
}
