// SDF fields evaluated on the device, bit-faithful to the reference's NumPy
// arithmetic (compile with --fmad=false):
//
//  * analytic: union (min) of spheres / boxes (camera_geometry.py:151-205);
//  * decoded: the coarse dense feature grid through the decoder's SDF head
//    plus the bounding-sphere offset -- the field the reference's
//    coarse-to-fine path builds with
//    callable_field(lambda p: decode_points(FeatureVolume(grid), heads, p)[1])
//    (runner.py:301-306, recon_pipeline.py:349-365);
//  * values: samples already evaluated elsewhere (an opaque host callable),
//    indexed by sample id.
//
// Rounding points follow the reference: trilinear in f64 -> f32
// (tensor_core.py:228-247); affine = np.einsum("...d,do->...o") in f64 -> f32
// (tensor_core.py:100-116); gelu f64 erf form -> f32 (tensor_core.py:82-86);
// s = f32(f64(f32 head) + |p - c| - r).
//
// einsum's reduction order (NumPy's baseline-SIMD sum-of-products, x86-64
// SSE2, no FMA): with d_out > 1 the reduction index is an outer loop and
// every output accumulates sequentially, acc = acc + x[d] w[d, o];
// with d_out == 1 the operands are contiguous and einsum runs its dot
// kernel: two f64 lanes, groups of 8 elements added as (6+l, 4+l, 2+l, l)
// per lane l, the tail pair by pair, then lane 0 + lane 1.
#pragma once
#include "common.cuh"

namespace lsrm {

constexpr int kFieldMaxDf = 64;
constexpr int kFieldMaxHidden = 128;

enum FieldKind { kFieldAnalytic = 0, kFieldDecoded = 1, kFieldValues = 2 };

struct FieldDev {
  int kind;
  // analytic
  const double* prims;
  int n_prims;
  // decoded: dense grid [side^3, d_f] + s head (w1 [d_f, hidden], b1, w2 [hidden, 1], b2)
  const float* grid;
  int side, d_f, hidden;
  const float *w1, *b1, *w2, *b2;
  double radius;        // bounding-sphere radius of the s offset (camera_geometry.py:21)
  // values: s of sample id
  const double* values;
};

__device__ __forceinline__ double sdf_prims(const double* __restrict__ prims, int n, double x,
                                            double y, double z) {
  double s = 0.0;
  for (int p = 0; p < n; ++p) {
    const double* P = prims + 8 * p;
    double v;
    if (P[0] == 0.0) {  // sphere: |p - c| - r
      v = dsub(__dsqrt_rn(dist2(x, y, z, P[1], P[2], P[3])), P[4]);
    } else {            // box: |max(q,0)| + min(max(q), 0), q = |p - c| - h
      double qx = dsub(fabs(dsub(x, P[1])), P[4]);
      double qy = dsub(fabs(dsub(y, P[2])), P[5]);
      double qz = dsub(fabs(dsub(z, P[3])), P[6]);
      double ox = fmax(qx, 0.0), oy = fmax(qy, 0.0), oz = fmax(qz, 0.0);
      double out = __dsqrt_rn(dadd(dadd(dmul(ox, ox), dmul(oy, oy)), dmul(oz, oz)));
      double in = fmin(fmax(fmax(qx, qy), qz), 0.0);
      v = dadd(out, in);
    }
    s = p == 0 ? v : fmin(s, v);
  }
  return s;
}

// einsum dot kernel order (see the header comment): sum_i a[i] * b[i*stride]
__device__ __forceinline__ double einsum_dot(const float* a, const float* __restrict__ b,
                                             int stride, int n) {
  double v0 = 0.0, v1 = 0.0;
  int i = 0;
  for (; n - i >= 8; i += 8) {
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      v0 = dadd(dmul((double)a[i + 2 * j], (double)b[(i + 2 * j) * stride]), v0);
      v1 = dadd(dmul((double)a[i + 2 * j + 1], (double)b[(i + 2 * j + 1) * stride]), v1);
    }
  }
  for (; i < n; i += 2) {
    v0 = dadd(dmul((double)a[i], (double)b[i * stride]), v0);
    if (i + 1 < n) v1 = dadd(dmul((double)a[i + 1], (double)b[(i + 1) * stride]), v1);
  }
  return dadd(0.0, dadd(v0, v1));
}

__device__ __forceinline__ float gelu_ref(float v) {
  const double z = (double)v;
  return (float)dmul(dmul(0.5, z), dadd(1.0, erf(ddiv(z, 1.4142135623730951))));
}

__device__ __forceinline__ float sigmoid_ref_f(float v) {
  const double z = (double)v;
  return (float)(z >= 0.0 ? ddiv(1.0, dadd(1.0, exp(-z))) : ddiv(exp(z), dadd(1.0, exp(z))));
}

// y[o] = f32(act(f32(x W + b))) for one row (tensor_core.py:100-136); act 0
// identity, 1 gelu, 2 sigmoid
__device__ __forceinline__ void affine_act_row(const float* x, int din,
                                               const float* __restrict__ w,
                                               const float* __restrict__ b, int dout, int act,
                                               float* y) {
  for (int o = 0; o < dout; ++o) {
    double s;
    if (dout == 1) {
      s = einsum_dot(x, w, 1, din);
    } else {
      s = 0.0;
      for (int i = 0; i < din; ++i) s = dadd(s, dmul((double)x[i], (double)w[i * dout + o]));
    }
    if (b) s = dadd(s, (double)b[o]);
    float v = (float)s;
    if (act == 1) v = gelu_ref(v);
    else if (act == 2) v = sigmoid_ref_f(v);
    y[o] = v;
  }
}

// _trilinear_prepare (tensor_core.py:212-225)
__device__ __forceinline__ void tri_prepare(const double* p, int side, int64_t* i0,
                                            double* frac) {
  for (int a = 0; a < 3; ++a) {
    const double t = dsub(dmul(p[a], (double)side), 0.5);
    double f = floor(t);
    f = f < 0.0 ? 0.0 : (f > (double)(side - 2) ? (double)(side - 2) : f);
    i0[a] = (int64_t)f;
    frac[a] = dsub(t, (double)i0[a]);
  }
}

// trilinear_interpolate_many (tensor_core.py:228-247): f64 accumulation in
// (dx, dy, dz) corner order, weight ((wx*wy)*wz), result rounded to f32.
__device__ __forceinline__ void trilinear_dense(const float* __restrict__ grid, int side,
                                                int d_f, const double* p, float* out) {
  int64_t i0[3];
  double fr[3];
  tri_prepare(p, side, i0, fr);
  double acc[kFieldMaxDf];
  for (int c = 0; c < d_f; ++c) acc[c] = 0.0;
  for (int dx = 0; dx < 2; ++dx) {
    const double wx = dx ? fr[0] : dsub(1.0, fr[0]);
    for (int dy = 0; dy < 2; ++dy) {
      const double wy = dy ? fr[1] : dsub(1.0, fr[1]);
      for (int dz = 0; dz < 2; ++dz) {
        const double wz = dz ? fr[2] : dsub(1.0, fr[2]);
        const double w = dmul(dmul(wx, wy), wz);
        const float* cr =
            grid + (((i0[0] + dx) * side + (i0[1] + dy)) * side + (i0[2] + dz)) * d_f;
        for (int c = 0; c < d_f; ++c) acc[c] = dadd(acc[c], dmul(w, (double)cr[c]));
      }
    }
  }
  for (int c = 0; c < d_f; ++c) out[c] = (float)acc[c];
}

// s = f32(f64(s head) + (|p - c| - r)): decode_points' s (recon_pipeline.py:
// 362-364) with camera_geometry.s_bias_many (:219-221)
__device__ __forceinline__ float s_with_bias(float head, const double* p, double radius) {
  const double dx = dsub(p[0], 0.5), dy = dsub(p[1], 0.5), dz = dsub(p[2], 0.5);
  const double nrm = __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
  return (float)dadd((double)head, dsub(nrm, radius));
}

__device__ __forceinline__ double decoded_sdf(const FieldDev& F, double x, double y, double z) {
  const double p[3] = {x, y, z};
  float f[kFieldMaxDf], h[kFieldMaxHidden], o;
  trilinear_dense(F.grid, F.side, F.d_f, p, f);
  affine_act_row(f, F.d_f, F.w1, F.b1, F.hidden, 1, h);
  affine_act_row(h, F.hidden, F.w2, F.b2, 1, 0, &o);
  return (double)s_with_bias(o, p, F.radius);
}

// s at sample `id` (values kind) or at (x, y, z)
__device__ __forceinline__ double field_sdf(const FieldDev& F, int64_t id, double x, double y,
                                            double z) {
  if (F.kind == kFieldValues) return F.values[id];
  if (F.kind == kFieldDecoded) return decoded_sdf(F, x, y, z);
  return sdf_prims(F.prims, F.n_prims, x, y, z);
}

}  // namespace lsrm
