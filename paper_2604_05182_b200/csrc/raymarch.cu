// Router input producer: the 3D surface point of every image token's
// patch-center ray (lsrm/block_routing.py:73-108 with
// lsrm/camera_geometry.py:236-302), one warp per ray, f64.
//
// 128 mid-segment samples between cube entry and exit, the field's SDF at
// each (analytic scene, decoded coarse volume, or values an opaque host
// callable produced; field.cuh), Laplace density, and the sample with the
// largest transmittance x alpha (first maximum).  The lanes evaluate the
// SDF samples in parallel; lane 0 then runs the sequential transmittance
// product in sample order, as np.cumprod does.  Rays that miss the cube or
// whose min SDF stays above 3 beta fall back to the cube-entry point / the
// clamped closest approach to the cube center and are flagged.
//
// Compiled with --fmad=false: the elementwise steps follow NumPy's
// unfused operation order.  exp() and the reference's BLAS-evaluated
// rotation / norm are not bit-identical across libraries, so the points are
// tolerance-matched (tests/test_raymarch.py), not bit-exact.
#include "field.cuh"

namespace lsrm {

constexpr int kMarch = 128;
constexpr double kNoPeakMargin = 3.0;
constexpr int kRayWarps = 4;   // rays per CTA

struct Ray {
  double o[3], d[3], t0, t1;
  bool span;
};

// slab method against [0,1]^3 (camera_geometry.py:236-252); false = no span
__device__ __forceinline__ bool cube_span(const double* o, const double* d, double& t0o,
                                          double& t1o) {
  double t0 = -INFINITY, t1 = INFINITY;
  for (int ax = 0; ax < 3; ++ax) {
    if (fabs(d[ax]) < 1e-12) {
      if (o[ax] < 0.0 || o[ax] > 1.0) return false;
      continue;
    }
    const double a = ddiv(dsub(0.0, o[ax]), d[ax]), b = ddiv(dsub(1.0, o[ax]), d[ax]);
    t0 = fmax(t0, fmin(a, b));
    t1 = fmin(t1, fmax(a, b));
  }
  if (t1 <= t0 || t1 <= 0.0) return false;
  t0o = fmax(t0, 0.0);
  t1o = t1;
  return true;
}

// patch-center ray of image token i (block_routing.py:88-97)
__device__ __forceinline__ Ray token_ray(const int64_t* __restrict__ coords, int64_t i,
                                         const double* __restrict__ cams,
                                         const int32_t* __restrict__ wh, int rows_f) {
  Ray r;
  const int view = (int)coords[3 * i];
  const double u = (double)coords[3 * i + 1], v = (double)coords[3 * i + 2];
  const double* K = cams + 21 * view;
  const double* R = K + 9;
  const double* T = K + 18;
  const double W = (double)wh[2 * view], H = (double)wh[2 * view + 1];
  const double px = dmul(dadd(u, 0.5), ddiv(W, (double)rows_f));
  const double py = dmul(dadd(v, 0.5), ddiv(H, (double)rows_f));
  const double dc[3] = {ddiv(dsub(px, K[2]), K[0]), ddiv(dsub(py, K[5]), K[4]), 1.0};
  for (int a = 0; a < 3; ++a)
    r.d[a] = dadd(dadd(dmul(R[3 * a], dc[0]), dmul(R[3 * a + 1], dc[1])),
                  dmul(R[3 * a + 2], dc[2]));
  for (int pass = 0; pass < 2; ++pass) {   // normalised twice, as the reference does
    const double nrm =
        __dsqrt_rn(dadd(dadd(dmul(r.d[0], r.d[0]), dmul(r.d[1], r.d[1])), dmul(r.d[2], r.d[2])));
    for (int a = 0; a < 3; ++a) r.d[a] = ddiv(r.d[a], nrm);
  }
  for (int a = 0; a < 3; ++a) r.o[a] = T[a];
  r.span = cube_span(r.o, r.d, r.t0, r.t1);
  return r;
}

__device__ __forceinline__ void sample_point(const Ray& r, int k, double step, double* p) {
  const double t = dadd(r.t0, dmul((double)k + 0.5, step));
  for (int a = 0; a < 3; ++a) p[a] = dadd(r.o[a], dmul(t, r.d[a]));
}

__global__ void __launch_bounds__(32 * kRayWarps)
image_points_kernel(const int64_t* __restrict__ coords, int64_t n,
                    const double* __restrict__ cams, const int32_t* __restrict__ wh, int rows_f,
                    FieldDev F, double beta, double* __restrict__ out,
                    uint8_t* __restrict__ miss) {
  __shared__ double s_buf[kRayWarps][kMarch];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = blockIdx.x * (int64_t)kRayWarps + warp;
  if (i >= n) return;
  const Ray r = token_ray(coords, i, cams, wh, rows_f);
  double p[3];
  bool peak = false;
  if (r.span) {
    const double step = ddiv(dsub(r.t1, r.t0), (double)kMarch);
    for (int k = lane; k < kMarch; k += 32) {
      double q[3];
      sample_point(r, k, step, q);
      s_buf[warp][k] = field_sdf(F, i * kMarch + k, q[0], q[1], q[2]);
    }
    __syncwarp();
    if (lane == 0) {
      double trans = 1.0, best_w = -1.0, s_min = INFINITY;
      int best = 0;
      for (int k = 0; k < kMarch; ++k) {
        const double s = s_buf[warp][k];
        s_min = fmin(s_min, s);
        // laplace_density (camera_geometry.py:255-261), alpha = 1 - exp(-density step)
        const double psi = s >= 0.0 ? dmul(0.5, exp(ddiv(-s, beta)))
                                    : dsub(1.0, dmul(0.5, exp(ddiv(s, beta))));
        const double alpha = dsub(1.0, exp(-dmul(ddiv(psi, beta), step)));
        const double w = dmul(trans, alpha);
        if (w > best_w) {   // first maximum (np.argmax)
          best_w = w;
          best = k;
        }
        trans = dmul(trans, dsub(1.0, alpha));
      }
      if (!(s_min > dmul(kNoPeakMargin, beta))) {
        peak = true;
        sample_point(r, best, step, p);
      } else {
        for (int a = 0; a < 3; ++a) p[a] = dadd(r.o[a], dmul(r.t0, r.d[a]));
      }
    }
  } else if (lane == 0) {   // closest approach to the cube center, clamped to t >= 0
    const double tn = dadd(dadd(dmul(dsub(0.5, r.o[0]), r.d[0]), dmul(dsub(0.5, r.o[1]), r.d[1])),
                           dmul(dsub(0.5, r.o[2]), r.d[2]));
    const double t = fmax(tn, 0.0);
    for (int a = 0; a < 3; ++a) p[a] = dadd(r.o[a], dmul(t, r.d[a]));
  }
  if (lane == 0) {
    for (int c = 0; c < 3; ++c) out[3 * i + c] = fmin(fmax(p[c], 0.0), 1.0);
    miss[i] = peak ? 0 : 1;
  }
}

// sample points of every ray (for an opaque field evaluated on the host):
// pts [n, 128, 3]; has_span [n] (rays missing the cube sample nothing)
__global__ void ray_samples_kernel(const int64_t* __restrict__ coords, int64_t n,
                                   const double* __restrict__ cams,
                                   const int32_t* __restrict__ wh, int rows_f,
                                   double* __restrict__ pts, uint8_t* __restrict__ has_span) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * kMarch) return;
  const int64_t i = e / kMarch;
  const int k = (int)(e % kMarch);
  const Ray r = token_ray(coords, i, cams, wh, rows_f);
  double p[3] = {0.5, 0.5, 0.5};
  if (r.span) sample_point(r, k, ddiv(dsub(r.t1, r.t0), (double)kMarch), p);
  for (int a = 0; a < 3; ++a) pts[3 * e + a] = p[a];
  if (k == 0) has_span[i] = r.span ? 1 : 0;
}

}  // namespace lsrm

using namespace lsrm;

namespace {
FieldDev field_of(const lsrm_sdf_field* f) {
  FieldDev F{};
  F.kind = f->kind;
  F.prims = f->prims;
  F.n_prims = f->n_prims;
  F.grid = f->grid;
  F.side = f->side;
  F.d_f = f->d_f;
  F.hidden = f->hidden;
  F.w1 = f->w1;
  F.b1 = f->b1;
  F.w2 = f->w2;
  F.b2 = f->b2;
  F.radius = f->radius;
  F.values = f->values;
  return F;
}
}  // namespace

extern "C" {

int lsrm_check_field(const lsrm_sdf_field* f) {
  LSRM_REQUIRE(f != nullptr, "sdf field: NULL descriptor");
  if (f->kind == kFieldAnalytic) {
    LSRM_REQUIRE(f->prims && f->n_prims >= 1 && f->n_prims <= 256,
                 "sdf field: 1..256 analytic primitives");
  } else if (f->kind == kFieldDecoded) {
    LSRM_REQUIRE(f->grid && f->w1 && f->b1 && f->w2 && f->b2, "sdf field: decoded weights missing");
    LSRM_REQUIRE(f->side >= 2, "trilinear needs side >= 2");
    LSRM_REQUIRE(f->d_f >= 1 && f->d_f <= kFieldMaxDf, "sdf field: d_f %d out of 1..%d", f->d_f,
                 kFieldMaxDf);
    LSRM_REQUIRE(f->hidden >= 1 && f->hidden <= kFieldMaxHidden,
                 "sdf field: head width %d out of 1..%d", f->hidden, kFieldMaxHidden);
  } else if (f->kind == kFieldValues) {
    LSRM_REQUIRE(f->values != nullptr, "sdf field: values missing");
  } else {
    return set_error(LSRM_E_CONFIG, "sdf field: unknown kind %d", f->kind);
  }
  return LSRM_OK;
}

int lsrm_image_token_points_field(const int64_t* coords, int64_t n, const double* cams,
                                  const int32_t* image_wh, int n_views, int rows_f,
                                  const lsrm_sdf_field* field, double beta, double* points,
                                  uint8_t* miss, void* stream) {
  LSRM_REQUIRE(n_views >= 1 && rows_f >= 1, "image points: bad view count / grid");
  LSRM_REQUIRE(beta > 0.0, "beta must be positive");
  int rc = lsrm_check_field(field);
  if (rc) return rc;
  if (n == 0) return LSRM_OK;
  image_points_kernel<<<(unsigned)ceil_div(n, kRayWarps), 32 * kRayWarps, 0,
                        as_stream(stream)>>>(coords, n, cams, image_wh, rows_f, field_of(field),
                                             beta, points, miss);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

int lsrm_image_token_points(const int64_t* coords, int64_t n, const double* cams,
                            const int32_t* image_wh, int n_views, int rows_f, const double* sdf,
                            int n_prims, double beta, double* points, uint8_t* miss,
                            void* stream) {
  lsrm_sdf_field f{};
  f.kind = kFieldAnalytic;
  f.prims = sdf;
  f.n_prims = n_prims;
  return lsrm_image_token_points_field(coords, n, cams, image_wh, n_views, rows_f, &f, beta,
                                       points, miss, stream);
}

int lsrm_ray_sample_points(const int64_t* coords, int64_t n, const double* cams,
                           const int32_t* image_wh, int n_views, int rows_f, double* points,
                           uint8_t* has_span, void* stream) {
  LSRM_REQUIRE(n_views >= 1 && rows_f >= 1, "ray samples: bad view count / grid");
  if (n == 0) return LSRM_OK;
  ray_samples_kernel<<<(unsigned)ceil_div(n * kMarch, 256), 256, 0, as_stream(stream)>>>(
      coords, n, cams, image_wh, rows_f, points, has_span);
  LSRM_LAUNCHED();
  return LSRM_OK;
}

}  // extern "C"
