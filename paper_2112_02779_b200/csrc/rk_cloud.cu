// rk_cloud.cu -- the steps either side of the hot path:
//  * N1 from_point_cloud's z-buffer (range_image.py:170-194): the float64
//    projection comes from rk_project_f64, the nearest range wins each pixel
//    through a 64-bit atomicMin on the (non-negative) double's bit pattern;
//  * N3 windowed-PCA normals (range_image.py:243-283): per pixel, the
//    reference's (2R+1)^2 window sums in its (dv, du) order, the float64
//    covariance, and the smallest-eigenvalue eigenvector by cyclic Jacobi.
#include "rk_common.cuh"

using namespace rk;

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }
static inline unsigned blocks_of(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

namespace {

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;  // +inf

__global__ void k_zb_clear(unsigned long long* zb, int64_t n, long long* stats) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < 4 && stats) stats[i] = 0;
  if (i < n) zb[i] = kInfBits;
}

// np.minimum.at(data, v * W + (floor(u + 0.5) mod W), r) over status == OK
__global__ void k_zb_scatter(SensorDev s, const double* __restrict__ u, const int32_t* __restrict__ v,
                             const double* __restrict__ r, const int8_t* __restrict__ st, int64_t n,
                             unsigned long long* zb, long long* stats) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int ok = 0, oof = 0, deg = 0;
  if (i < n) {
    const int code = st[i];
    ok = code == PROJ_OK;
    oof = code == PROJ_OUT_OF_FOV;
    deg = code == PROJ_DEGENERATE;
    if (ok) {
      long long col = (long long)floor(__dadd_rn(u[i], 0.5)) % s.W;  // round_half_up, np.mod
      if (col < 0) col += s.W;
      const long long flat = (long long)v[i] * s.W + col;
      atomicMin(zb + flat, (unsigned long long)__double_as_longlong(r[i]));
    }
  }
  ok = __reduce_add_sync(0xffffffffu, ok);
  oof = __reduce_add_sync(0xffffffffu, oof);
  deg = __reduce_add_sync(0xffffffffu, deg);
  if ((threadIdx.x & 31) == 0) {
    if (ok) atomicAdd((unsigned long long*)&stats[1], (unsigned long long)ok);    // n_in, -kept later
    if (oof) atomicAdd((unsigned long long*)&stats[2], (unsigned long long)oof);
    if (deg) atomicAdd((unsigned long long*)&stats[3], (unsigned long long)deg);
  }
}

// data[~finite] = 0, float32 image; kept = written pixels; collisions = n_in - kept
__global__ void k_zb_final(const unsigned long long* __restrict__ zb, int64_t n, float* out,
                           long long* stats) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int kept = 0;
  if (i < n) {
    const unsigned long long b = zb[i];
    kept = b != kInfBits;
    out[i] = kept ? (float)__longlong_as_double((long long)b) : 0.0f;
  }
  kept = __reduce_add_sync(0xffffffffu, kept);
  if ((threadIdx.x & 31) == 0 && kept) {
    atomicAdd((unsigned long long*)&stats[0], (unsigned long long)kept);
    atomicAdd((unsigned long long*)&stats[1], (unsigned long long)(-(long long)kept));
  }
}

// ------------------------------------------------------------------ PCA normals
// eigenvector of the smallest eigenvalue of a symmetric 3x3 (cyclic Jacobi)
__device__ void smallest_eigvec3(double a00, double a01, double a02, double a11, double a12,
                                 double a22, double n[3]) {
  double A[3][3] = {{a00, a01, a02}, {a01, a11, a12}, {a02, a12, a22}};
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    const double dg = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
    if (off <= 1e-36 * dg || off == 0.0) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = A[p][q];
      if (apq == 0.0) continue;
      const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
      const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double akp = A[k][p], akq = A[k][q];
        A[k][p] = c * akp - sn * akq;
        A[k][q] = sn * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double apk = A[p][k], aqk = A[q][k];
        A[p][k] = c * apk - sn * aqk;
        A[q][k] = sn * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double vkp = V[k][p], vkq = V[k][q];
        V[k][p] = c * vkp - sn * vkq;
        V[k][q] = sn * vkp + c * vkq;
      }
    }
  }
  int m = 0;
  if (A[1][1] < A[m][m]) m = 1;
  if (A[2][2] < A[m][m]) m = 2;
  const double nn = sqrt(V[0][m] * V[0][m] + V[1][m] * V[1][m] + V[2][m] * V[2][m]);
  n[0] = V[0][m] / nn;
  n[1] = V[1][m] / nn;
  n[2] = V[2][m] / nn;
}

// one thread per pixel; neighbours come through L1 (the window re-reads them)
__global__ void __launch_bounds__(256) k_normals_pca(SensorDev s, const float* __restrict__ range,
                                                     int64_t total, int R, double disc_abs,
                                                     double disc_rel, float* normals, uint8_t* valid,
                                                     float4* surfel) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int W = s.W, H = s.H;
  const int64_t HW = (int64_t)H * W;
  const int64_t img = i / HW;
  const int pix = (int)(i - img * HW);
  const int v = pix / W, u = pix - v * W;
  const float* Rg = range + img * HW;
  const float r32 = Rg[pix];
  const bool ok0 = r32 > 0.0f;
  const double r = (double)r32;
  const double thresh = __dadd_rn(disc_abs, __dmul_rn(disc_rel, r));
  double cnt = 0.0, s1[3] = {0, 0, 0}, s2[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int dv = -R; dv <= R; ++dv) {
    const int vv = v + dv;
    for (int du = -R; du <= R; ++du) {
      int uu = (u + du) % W;  // np.roll along the azimuth
      if (uu < 0) uu += W;
      const bool in = vv >= 0 && vv < H;
      const float q32 = in ? Rg[vv * W + uu] : 0.0f;
      const double qr = (double)q32;
      const bool use = ok0 && in && q32 > 0.0f && fabs(__dsub_rn(qr, r)) <= thresh;
      if (!use) continue;  // the reference adds w = 0 terms: sums unchanged
      double q[3];
      unproject_px(s, vv, uu, q32, q);
      cnt = __dadd_rn(cnt, 1.0);
#pragma unroll
      for (int a = 0; a < 3; ++a) s1[a] = __dadd_rn(s1[a], q[a]);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) s2[3 * a + b] = __dadd_rn(s2[3 * a + b], __dmul_rn(q[a], q[b]));
    }
  }
  const bool ok = ok0 && cnt >= 3.0;
  float n0 = 0.f, n1 = 0.f, n2 = 0.f;
  if (ok) {
    double mean[3], cov[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) mean[a] = __ddiv_rn(s1[a], cnt);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        cov[3 * a + b] = __dsub_rn(__ddiv_rn(s2[3 * a + b], cnt), __dmul_rn(mean[a], mean[b]));
    double n[3];
    smallest_eigvec3(cov[0], cov[1], cov[2], cov[4], cov[5], cov[8], n);
    double p[3];
    unproject_px(s, v, u, r32, p);
    const double facing = __dadd_rn(__dadd_rn(__dmul_rn(n[0], p[0]), __dmul_rn(n[1], p[1])),
                                    __dmul_rn(n[2], p[2]));
    if (facing > 0.0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
    n0 = (float)n[0]; n1 = (float)n[1]; n2 = (float)n[2];
  }
  if (normals) {
    normals[3 * i] = n0;
    normals[3 * i + 1] = n1;
    normals[3 * i + 2] = n2;
  }
  if (valid) valid[i] = ok ? 1 : 0;
  if (surfel) surfel[i] = make_float4(n0, n1, n2, ok ? r32 : 0.f);
}

}  // namespace

extern "C" int rk_zbuffer_image(const rk_sensor* s, const double* u, const int32_t* v, const double* r,
                                const int8_t* status, int64_t n, float* range_out, int64_t* stats4,
                                unsigned long long* zwork, void* stream) {
  cudaStream_t st = S(stream);
  const int64_t px = (int64_t)s->dev.H * s->dev.W;
  long long* stats = reinterpret_cast<long long*>(stats4);
  k_zb_clear<<<blocks_of(px > 4 ? px : 4, 256), 256, 0, st>>>(zwork, px, stats);
  if (n > 0) k_zb_scatter<<<blocks_of(n, 256), 256, 0, st>>>(s->dev, u, v, r, status, n, zwork, stats);
  k_zb_final<<<blocks_of(px, 256), 256, 0, st>>>(zwork, px, range_out, stats);
  RK_LAUNCHED("rk_zbuffer_image");
  return RK_OK;
}

extern "C" int rk_normals_pca(const rk_sensor* s, const float* range, int32_t batch, int32_t radius,
                              double disc_abs, double disc_rel, float* normals, uint8_t* valid,
                              float* surfel, void* stream) {
  const int64_t total = (int64_t)batch * s->dev.H * s->dev.W;
  if (total <= 0) return RK_OK;
  if (radius < 0) {
    rk_set_error("radius must be >= 0");
    return RK_EGENERIC;
  }
  k_normals_pca<<<blocks_of(total, 256), 256, 0, S(stream)>>>(
      s->dev, range, total, radius, disc_abs, disc_rel, normals, valid,
      reinterpret_cast<float4*>(surfel));
  RK_LAUNCHED("k_normals_pca");
  return RK_OK;
}
