// rk_icp.cu -- the per-call registration API around K3 (the batched
// multi-scale kernel itself lives in rk_register.cu):
//  * projective_correspondences(single=True) for an explicit float64 cloud
//    (registration.py:117-187), bit-exact float32 association;
//  * the float64 path's association given rk_project_f64 output (single=False);
//  * float64 robust normal equations, point-to-plane residuals and centroid
//    translation (registration.py:96-102, 190-234) with fixed-order block
//    partials -- deterministic, no float atomics;
//  * surfel maps from an explicit NormalImage.
#include "rk_common.cuh"
#include "rk_linalg.cuh"

using namespace rk;

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

namespace {

constexpr int kNumAcc = 29;  // 21 H (upper) + 6 b + cost + sumsq

// projective_correspondences(single=True) for an explicit float64 cloud
template <int MATH>
__global__ void k_correspondences(SensorDev s, const double* __restrict__ pts, int64_t n,
                                  const float4* __restrict__ surf, const double* __restrict__ pose12,
                                  float gate2, int stride, float inv_s, uint8_t* keep, float* target,
                                  float* normal) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double pose[12];
  for (int k = 0; k < 12; ++k) pose[k] = pose12[k];
  double m[3];
  xform_rows(pose, pose + 9, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], m, n == 1);
  const float mx = (float)m[0], my = (float)m[1], mz = (float)m[2];
  Proj32 pr = project_f32<MATH>(s, mx, my, mz);
  bool ok = pr.status == PROJ_OK;
  int col = (int)__fadd_rn(__fmul_rn(pr.u, inv_s), 0.5f) * stride;
  if (col >= s.W) col = 0;
  int row = (int)__fadd_rn(__fmul_rn((float)pr.v, inv_s), 0.5f) * stride;
  ok = ok && row < s.H;
  float4 nv = make_float4(0.f, 0.f, 0.f, 0.f);
  float qx = 0.f, qy = 0.f, qz = 0.f;
  if (ok) {
    const int flat = row * s.W + col;
    nv = surf[flat];
    ok = nv.w > 0.0f;
    float4 d = s.dirs32[flat];
    float4 o = s.origins32[col];
    qx = __fadd_rn(__fmul_rn(nv.w, d.x), o.x);
    qy = __fadd_rn(__fmul_rn(nv.w, d.y), o.y);
    qz = __fadd_rn(__fmul_rn(nv.w, d.z), o.z);
    float dx = __fsub_rn(mx, qx), dy = __fsub_rn(my, qy), dz = __fsub_rn(mz, qz);
    float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
    ok = ok && d2 <= gate2;
  }
  keep[i] = ok ? 1 : 0;
  if (target) { target[3 * i] = qx; target[3 * i + 1] = qy; target[3 * i + 2] = qz; }
  if (normal) { normal[3 * i] = nv.x; normal[3 * i + 1] = nv.y; normal[3 * i + 2] = nv.z; }
}

}  // namespace

extern "C" int rk_correspondences_f32(const rk_sensor* s, const double* src_pts, int64_t n,
                                      const float* dst_range, const float* dst_surfel,
                                      const double* pose12, double max_dist, int32_t stride,
                                      int math, uint8_t* keep, float* target, float* normal,
                                      void* stream) {
  (void)dst_range;  // the surfel map carries the stored range of valid pixels
  if (n <= 0) return RK_OK;
  if (stride < 1) { rk_set_error("stride must be >= 1"); return RK_EGENERIC; }
  const float g = (float)max_dist;
  const float gate2 = g * g;  // float32 product (numpy weak scalars)
  const float inv_s = (float)(1.0 / stride);
  unsigned blocks = (unsigned)((n + 255) / 256);
  const float4* surf = reinterpret_cast<const float4*>(dst_surfel);
  if (math == MATH_CR)
    k_correspondences<MATH_CR><<<blocks, 256, 0, S(stream)>>>(s->dev, src_pts, n, surf, pose12, gate2,
                                                              stride, inv_s, keep, target, normal);
  else if (math == MATH_NP)
    k_correspondences<MATH_NP><<<blocks, 256, 0, S(stream)>>>(s->dev, src_pts, n, surf, pose12, gate2,
                                                              stride, inv_s, keep, target, normal);
  else
    k_correspondences<MATH_FAST><<<blocks, 256, 0, S(stream)>>>(s->dev, src_pts, n, surf, pose12, gate2,
                                                                stride, inv_s, keep, target, normal);
  RK_LAUNCHED("k_correspondences");
  return RK_OK;
}


// surfel map from an arbitrary NormalImage (vectors, valid) + range
__global__ void k_make_surfel(const float* __restrict__ range, const float* __restrict__ nrm,
                              const uint8_t* __restrict__ valid, int64_t n, float4* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float r = range[i];
  bool ok = valid[i] != 0 && r > 0.0f;
  out[i] = make_float4(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2], ok ? r : 0.0f);
}

extern "C" int rk_make_surfel(const float* range, const float* normals, const uint8_t* valid,
                              int64_t n, float* surfel, void* stream) {
  if (n <= 0) return RK_OK;
  k_make_surfel<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(range, normals, valid, n,
                                                                    reinterpret_cast<float4*>(surfel));
  RK_LAUNCHED("k_make_surfel");
  return RK_OK;
}

// ------------------------------------------------------------------ float64 helpers
// RigidTransform.apply / `pts @ R.T + t` for an arbitrary cloud (se3.py:76-79)
__global__ void k_transform(const double* __restrict__ pose12, const double* __restrict__ pts,
                            int64_t n, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double pose[12];
  for (int k = 0; k < 12; ++k) pose[k] = pose12[k];
  double m[3];
  xform_rows(pose, pose + 9, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], m, n == 1);
  out[3 * i] = m[0];
  out[3 * i + 1] = m[1];
  out[3 * i + 2] = m[2];
}

extern "C" int rk_transform_points(const double* pose12, const double* pts, int64_t n, double* out,
                                   void* stream) {
  if (n <= 0) return RK_OK;
  k_transform<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(pose12, pts, n, out);
  RK_LAUNCHED("k_transform");
  return RK_OK;
}

// association of the float64 path (registration.py:151-187, single=False) given
// moved points and their float64 projections
__global__ void k_associate_f64(SensorDev s, const double* __restrict__ moved, const double* __restrict__ u,
                                const int32_t* __restrict__ v, const int8_t* __restrict__ st, int64_t n,
                                const float4* __restrict__ surf, double max_dist, int stride,
                                uint8_t* keep, double* target, double* normal) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double inv_s = 1.0 / stride;
  bool ok = st[i] == PROJ_OK;
  int col = (int)__dadd_rn(__dmul_rn(u[i], inv_s), 0.5) * stride;
  if (col >= s.W) col = 0;
  int row = (int)__dadd_rn(__dmul_rn((double)v[i], inv_s), 0.5) * stride;
  ok = ok && row >= 0 && row < s.H;
  double q[3] = {0, 0, 0};
  float4 nv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
    const int flat = row * s.W + col;
    nv = surf[flat];
    ok = nv.w > 0.0f;
    const double rq = (double)nv.w;
    double d2 = 0.0;
    for (int c = 0; c < 3; ++c) {
      q[c] = __dadd_rn(__dmul_rn(rq, s.dirs[3 * flat + c]), s.origins[3 * col + c]);
      double dd = __dsub_rn(moved[3 * i + c], q[c]);
      d2 = __dadd_rn(d2, __dmul_rn(dd, dd));
    }
    ok = ok && d2 <= __dmul_rn(max_dist, max_dist);
  }
  keep[i] = ok ? 1 : 0;
  for (int c = 0; c < 3; ++c) target[3 * i + c] = q[c];
  normal[3 * i] = nv.x;
  normal[3 * i + 1] = nv.y;
  normal[3 * i + 2] = nv.z;
}

extern "C" int rk_associate_f64(const rk_sensor* s, const double* moved, const double* u,
                                const int32_t* v, const int8_t* status, int64_t n,
                                const float* dst_surfel, double max_dist, int32_t stride,
                                uint8_t* keep, double* target, double* normal, void* stream) {
  if (n <= 0) return RK_OK;
  k_associate_f64<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(
      s->dev, moved, u, v, status, n, reinterpret_cast<const float4*>(dst_surfel), max_dist, stride,
      keep, target, normal);
  RK_LAUNCHED("k_associate_f64");
  return RK_OK;
}

// float64 robust normal equations of an explicit CorrespondenceSet
// (registration.py:208-234): out[0..20] H upper, [21..26] b, [27] sum(1/w-1),
// [28] sum r^2.  Per-block float64 partials, reduced in fixed order.
constexpr int kNeBlocks = 64;
__global__ void k_normal_eq_f64(const double* __restrict__ pose12, const double* __restrict__ src,
                                const double* __restrict__ tgt, const double* __restrict__ nrm,
                                int64_t n, double kernel, double* partial) {
  double pose[12];
  for (int k = 0; k < 12; ++k) pose[k] = pose12[k];
  double acc[kNumAcc];
  for (int k = 0; k < kNumAcc; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double m[3];
    xform_rows(pose, pose + 9, src[3 * i], src[3 * i + 1], src[3 * i + 2], m, n == 1);
    const double nx = nrm[3 * i], ny = nrm[3 * i + 1], nz = nrm[3 * i + 2];
    const double r = nx * (m[0] - tgt[3 * i]) + ny * (m[1] - tgt[3 * i + 1]) + nz * (m[2] - tgt[3 * i + 2]);
    double J[6] = {m[1] * nz - m[2] * ny, m[2] * nx - m[0] * nz, m[0] * ny - m[1] * nx, nx, ny, nz};
    const double e = r / kernel;
    const double w = 1.0 / sqrt(1.0 + e * e);
    int q = 0;
    for (int a = 0; a < 6; ++a)
      for (int b = a; b < 6; ++b) { acc[q] += J[a] * w * J[b]; ++q; }
    for (int a = 0; a < 6; ++a) acc[21 + a] += -(r * w) * J[a];
    acc[27] += 1.0 / w - 1.0;
    acc[28] += r * r;
  }
  __shared__ double sh[8][kNumAcc];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < kNumAcc; ++k) {
    double v = acc[k];
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) sh[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < kNumAcc) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w][threadIdx.x];
    partial[blockIdx.x * kNumAcc + threadIdx.x] = t;
  }
}

__global__ void k_normal_eq_final(const double* partial, double* out) {
  int k = threadIdx.x;
  if (k >= kNumAcc) return;
  double t = 0.0;
  for (int b = 0; b < kNeBlocks; ++b) t += partial[b * kNumAcc + k];
  out[k] = t;
}

extern "C" int rk_normal_equations_f64(const double* pose12, const double* src, const double* tgt,
                                       const double* nrm, int64_t n, double kernel, double* out29,
                                       double* work, void* stream) {
  cudaStream_t st = S(stream);
  k_normal_eq_f64<<<kNeBlocks, 256, 0, st>>>(pose12, src, tgt, nrm, n, kernel, work);
  k_normal_eq_final<<<1, 32, 0, st>>>(work, out29);
  RK_LAUNCHED("k_normal_eq_f64");
  return RK_OK;
}

// point_to_plane_residuals (registration.py:190-192)
__global__ void k_residuals(const double* __restrict__ pose12, const double* __restrict__ src,
                            const double* __restrict__ tgt, const double* __restrict__ nrm, int64_t n,
                            double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double pose[12];
  for (int k = 0; k < 12; ++k) pose[k] = pose12[k];
  double m[3];
  xform_rows(pose, pose + 9, src[3 * i], src[3 * i + 1], src[3 * i + 2], m, n == 1);
  double acc = __dmul_rn(nrm[3 * i], __dsub_rn(m[0], tgt[3 * i]));
  acc = __dadd_rn(acc, __dmul_rn(nrm[3 * i + 1], __dsub_rn(m[1], tgt[3 * i + 1])));
  acc = __dadd_rn(acc, __dmul_rn(nrm[3 * i + 2], __dsub_rn(m[2], tgt[3 * i + 2])));
  out[i] = acc;
}

extern "C" int rk_point_to_plane_residuals(const double* pose12, const double* src, const double* tgt,
                                           const double* nrm, int64_t n, double* out, void* stream) {
  if (n <= 0) return RK_OK;
  k_residuals<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(pose12, src, tgt, nrm, n, out);
  RK_LAUNCHED("k_residuals");
  return RK_OK;
}

// column means of an (n,3) float64 cloud (initial_translation_by_centroids,
// registration.py:96-102): fixed-order block partials -> deterministic
__global__ void k_colsum(const double* __restrict__ pts, int64_t n, double* partial) {
  double a0 = 0, a1 = 0, a2 = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    a0 += pts[3 * i];
    a1 += pts[3 * i + 1];
    a2 += pts[3 * i + 2];
  }
  __shared__ double sh[8][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off; off >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, off);
    a1 += __shfl_xor_sync(0xffffffffu, a1, off);
    a2 += __shfl_xor_sync(0xffffffffu, a2, off);
  }
  if (lane == 0) { sh[warp][0] = a0; sh[warp][1] = a1; sh[warp][2] = a2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0;
    for (int w = 0; w < 8; ++w) t += sh[w][threadIdx.x];
    partial[blockIdx.x * 3 + threadIdx.x] = t;
  }
}

__global__ void k_centroid_delta(const double* ps, int64_t ns, const double* pd, int64_t nd, double* out) {
  int c = threadIdx.x;
  if (c >= 3) return;
  double a = 0, b = 0;
  for (int k = 0; k < kNeBlocks; ++k) { a += ps[3 * k + c]; b += pd[3 * k + c]; }
  out[c] = b / (double)nd - a / (double)ns;
}

extern "C" int rk_centroid_translation(const double* src, int64_t ns, const double* dst, int64_t nd,
                                       double* out3, double* work, void* stream) {
  if (ns <= 0 || nd <= 0) { rk_set_error("centroid alignment needs non-empty point sets"); return RK_EEMPTY; }
  cudaStream_t st = S(stream);
  k_colsum<<<kNeBlocks, 256, 0, st>>>(src, ns, work);
  k_colsum<<<kNeBlocks, 256, 0, st>>>(dst, nd, work + 3 * kNeBlocks);
  k_centroid_delta<<<1, 32, 0, st>>>(work, ns, work + 3 * kNeBlocks, nd, out3);
  RK_LAUNCHED("rk_centroid_translation");
  return RK_OK;
}
