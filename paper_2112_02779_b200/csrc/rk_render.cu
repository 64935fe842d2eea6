// rk_render.cu -- analytic plane/sphere/box ray caster along the exact sensor
// rays (synth.py:108-134), used to synthesise benchmark inputs on the device
// (SURVEY §8f N4).  One thread per (pose, pixel); float64 throughout, in
// numpy's rounding order (BLAS FMA chains for the matrix products, sequential
// sums for np.sum over 3 terms), so images equal render_scene's bit for bit
// (tests/test_gpu_parity.py::test_render_matches_reference_render_scene).
#include "rk_common.cuh"

using namespace rk;

namespace {

constexpr double kMinHit = 1e-9;  // synth.py:19

// numpy (N,3) @ (3,) goes through OpenBLAS dgemv; its SkylakeX kernel rounds
// fma(a2,n2, fma(a0,n0, a1*n1)) (probed on 10^4 rows of several lengths)
__device__ __forceinline__ double gemv3(const double a[3], const double* n) {
  return __fma_rn(a[2], n[2], __fma_rn(a[0], n[0], __dmul_rn(a[1], n[1])));
}

// (N,3) @ (3,3) column a through dgemm: fma(p2,M2a, fma(p1,M1a, p0*M0a))
//
__device__ __forceinline__ double gemm3(double p0, double p1, double p2, const double* M, int a) {
  return __fma_rn(p2, M[2 * 3 + a], __fma_rn(p1, M[1 * 3 + a], __dmul_rn(p0, M[0 * 3 + a])));
}

__device__ double hit_plane(const double* q, const double o[3], const double d[3]) {
  double den = gemv3(d, q + 1);
  double t = (q[4] - gemv3(o, q + 1)) / den;
  if (fabs(den) < 1e-15 || !(t > kMinHit)) return INFINITY;
  return t;
}

__device__ double hit_sphere(const double* q, const double o[3], const double d[3]) {
  double oc[3] = {o[0] - q[1], o[1] - q[2], o[2] - q[3]};
  double b = oc[0] * d[0] + oc[1] * d[1] + oc[2] * d[2];
  double c = oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2] - q[4] * q[4];
  double disc = b * b - c;
  if (!(disc >= 0.0)) return INFINITY;
  double s = sqrt(disc);
  double t = (-b - s > kMinHit) ? -b - s : -b + s;
  return t > kMinHit ? t : INFINITY;
}

__device__ double hit_box(const double* q, const double o[3], const double d[3]) {
  const double* R = q + 7;  // rotation, row-major; local = (x - c) @ R
  double lo_t = -INFINITY, hi_t = INFINITY;
  for (int a = 0; a < 3; ++a) {
    double ol = gemm3(o[0] - q[1], o[1] - q[2], o[2] - q[3], R, a);
    double dl = gemm3(d[0], d[1], d[2], R, a);
    double half = 0.5 * q[4 + a];
    if (fabs(dl) < 1e-15) {
      if (!(fabs(ol) <= half)) return INFINITY;
      continue;
    }
    double inv = 1.0 / dl;
    double ta = (-half - ol) * inv, tb = (half - ol) * inv;
    lo_t = fmax(lo_t, fmin(ta, tb));
    hi_t = fmin(hi_t, fmax(ta, tb));
  }
  double t = lo_t > kMinHit ? lo_t : hi_t;
  if (lo_t > hi_t || !(t > kMinHit)) return INFINITY;
  return t;
}

__global__ void k_render(SensorDev s, const double* __restrict__ prims, int n_prims,
                         const double* __restrict__ poses, int64_t total, float* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t HW = (int64_t)s.H * s.W;
  const int64_t b = i / HW;
  const int p = (int)(i - b * HW);
  const int u = p % s.W;
  const double* P = poses + 12 * b;
  double dd[3] = {s.dirs[3 * p], s.dirs[3 * p + 1], s.dirs[3 * p + 2]};
  double oo[3] = {s.origins[3 * u], s.origins[3 * u + 1], s.origins[3 * u + 2]};
  double d[3], o[3];
  xform_rows(P, nullptr, dd[0], dd[1], dd[2], d);
  xform_rows(P, P + 9, oo[0], oo[1], oo[2], o);
  double best = INFINITY;
  for (int k = 0; k < n_prims; ++k) {
    const double* q = prims + 16 * k;
    int type = (int)q[0];
    double t = type == 0 ? hit_plane(q, o, d) : (type == 1 ? hit_sphere(q, o, d) : hit_box(q, o, d));
    best = fmin(best, t);
  }
  out[i] = isinf(best) ? 0.0f : (float)best;
}

}  // namespace

extern "C" int rk_render(const rk_sensor* s, const double* prims, int32_t n_prims,
                         const double* poses12, int32_t batch, float* out, void* stream) {
  int64_t total = (int64_t)batch * s->dev.H * s->dev.W;
  if (total <= 0) return RK_OK;
  k_render<<<(unsigned)((total + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      s->dev, prims, n_prims, poses12, total, out);
  RK_LAUNCHED("k_render");
  return RK_OK;
}
