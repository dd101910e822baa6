// Per-pixel / per-patch camera rays (lsrm/camera_geometry.py:91-107) and the
// analytic-scene silhouettes that feed the foreground patch mask
// (camera_geometry.py:308-350), f64 with NumPy's unfused operation order
// (compiled with --fmad=false).
#include "common.cuh"

namespace lsrm {

// unit world-space direction of the ray through grid cell (x, y) of view cam
__device__ __forceinline__ void ray_dir(const double* K, const double* R, double W, double H,
                                        int gw, int gh, int x, int y, double* d) {
  const double u = dmul(x + 0.5, W / gw), v = dmul(y + 0.5, H / gh);
  const double dc[3] = {(u - K[2]) / K[0], (v - K[5]) / K[4], 1.0};
  for (int r = 0; r < 3; ++r)   // d_cam @ R^T
    d[r] = dadd(dadd(dmul(dc[0], R[3 * r]), dmul(dc[1], R[3 * r + 1])), dmul(dc[2], R[3 * r + 2]));
  const double nrm = sqrt(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
  d[0] /= nrm;
  d[1] /= nrm;
  d[2] /= nrm;
}

__global__ void pluecker_kernel(const double* __restrict__ cams, const int32_t* __restrict__ wh,
                                int n_views, int gw, int gh, float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)gw * gh;
  if (i >= per * n_views) return;
  const int view = (int)(i / per), y = (int)((i % per) / gw), x = (int)(i % gw);
  const double* K = cams + 21 * view;
  double d[3];
  ray_dir(K, K + 9, (double)wh[2 * view], (double)wh[2 * view + 1], gw, gh, x, y, d);
  const double* t = K + 18;
  const double m[3] = {dsub(dmul(t[1], d[2]), dmul(t[2], d[1])),
                       dsub(dmul(t[2], d[0]), dmul(t[0], d[2])),
                       dsub(dmul(t[0], d[1]), dmul(t[1], d[0]))};
  float* o = out + 6 * i;
  for (int c = 0; c < 3; ++c) {
    o[c] = (float)d[c];
    o[3 + c] = (float)m[c];
  }
}

// forward hit of a ray (o, unit d) against one primitive (camera_geometry.py:308-336)
__device__ __forceinline__ bool prim_hit(const double* p, const double* o, const double* d) {
  if (p[0] == 0.0) {   // sphere
    const double b[3] = {p[1] - o[0], p[2] - o[1], p[3] - o[2]};
    const double tca = dadd(dadd(dmul(d[0], b[0]), dmul(d[1], b[1])), dmul(d[2], b[2]));
    const double bb = dadd(dadd(dmul(b[0], b[0]), dmul(b[1], b[1])), dmul(b[2], b[2]));
    const double perp2 = bb - dmul(tca, tca);
    return perp2 <= dmul(p[4], p[4]) && tca >= -p[4];
  }
  // box: slab test with NumPy's NaN semantics (minimum/maximum propagate,
  // nanmax/nanmin skip)
  double t0 = NAN, t1 = NAN;
  bool ok = true;
  for (int ax = 0; ax < 3; ++ax) {
    const double lo = p[1 + ax] - p[4 + ax], hi = p[1 + ax] + p[4 + ax];
    const double ta = (lo - o[ax]) / d[ax], tb = (hi - o[ax]) / d[ax];
    const bool nan_ab = isnan(ta) || isnan(tb);
    const double mn = nan_ab ? NAN : fmin(ta, tb), mx = nan_ab ? NAN : fmax(ta, tb);
    if (!isnan(mn)) t0 = isnan(t0) ? mn : fmax(t0, mn);
    if (!isnan(mx)) t1 = isnan(t1) ? mx : fmin(t1, mx);
    const bool par = fabs(d[ax]) < 1e-12, inside = o[ax] >= lo && o[ax] <= hi;
    if (par && !inside) ok = false;
  }
  const double t0c = isnan(t0) ? NAN : fmax(t0, 0.0);
  return ok && (t1 >= t0c);   // NaN compares false
}

__global__ void silhouette_kernel(const double* __restrict__ cams, const int32_t* __restrict__ wh,
                                  int n_views, int max_w, int max_h,
                                  const double* __restrict__ prims, int n_prims,
                                  float* __restrict__ alpha) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)max_w * max_h;
  if (i >= per * n_views) return;
  const int view = (int)(i / per), y = (int)((i % per) / max_w), x = (int)(i % max_w);
  const int W = wh[2 * view], H = wh[2 * view + 1];
  if (x >= W || y >= H) return;
  const double* K = cams + 21 * view;
  double d[3];
  ray_dir(K, K + 9, (double)W, (double)H, W, H, x, y, d);
  for (int c = 0; c < 3; ++c) d[c] = (double)(float)d[c];   // pluecker_rays is float32
  const double* o = K + 18;
  bool hit = false;
  for (int k = 0; k < n_prims; ++k) hit = hit || prim_hit(prims + 8 * k, o, d);
  alpha[(int64_t)view * per + (int64_t)y * max_w + x] = hit ? 1.f : 0.f;
}

}  // namespace lsrm

using namespace lsrm;

extern "C" {

int lsrm_pluecker_rays(const double* cams, const int32_t* image_wh, int n_views, int gw, int gh,
                       float* out, void* stream) {
  LSRM_REQUIRE(gw >= 1 && gh >= 1 && n_views >= 1, "ray grid must be at least 1x1");
  const int64_t n = (int64_t)gw * gh * n_views;
  pluecker_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(cams, image_wh,
                                                                             n_views, gw, gh, out);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_silhouette_alpha(const double* cams, const int32_t* image_wh, int n_views, int max_w,
                          int max_h, const double* sdf, int n_prims, float* alpha,
                          void* stream) {
  LSRM_REQUIRE(n_views >= 1 && max_w >= 1 && max_h >= 1, "silhouette: bad image size");
  LSRM_REQUIRE(n_prims >= 1, "silhouette: empty SDF");
  const int64_t n = (int64_t)max_w * max_h * n_views;
  silhouette_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(
      cams, image_wh, n_views, max_w, max_h, sdf, n_prims, alpha);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
