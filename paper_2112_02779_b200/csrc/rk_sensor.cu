// rk_sensor.cu -- sensor tables, projection / unprojection, normals, pyramid
// compaction (K1, K2 of DESIGN.md).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "rk_common.cuh"

using namespace rk;

// ------------------------------------------------------------------ errors
static thread_local char g_err[512] = {0};

void rk_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int rk_cuda_status(cudaError_t e, const char* where) {
  rk_set_error("%s: %s", where, cudaGetErrorString(e));
  return RK_ECUDA;
}

extern "C" int rk_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    strncpy(buf, g_err, cap - 1);
    buf[cap - 1] = 0;
  }
  return RK_OK;
}

extern "C" int rk_version(void) { return 1; }
extern "C" int rk_struct_size(int which) {
  return which == 0 ? (int)sizeof(rk_sensor_desc) : which == 1 ? (int)sizeof(rk_icp_config) : -1;
}

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }
static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// ------------------------------------------------------------------ sensor
// VRSQRT14PS table for MATH_NP's arcsin (rk_svml.cuh); generated at build time
// from data/vrsqrt14.u16 (scripts/gen_vrsqrt14.c) by __graft_entry__.build()
static const uint16_t kVrsqrt14[65536] = {
#include "rk_vrsqrt14.inc"
};

extern "C" int rk_sensor_create(const rk_sensor_desc* d, rk_sensor** out) {
  if (!d || !out) { rk_set_error("null argument"); return RK_EGENERIC; }
  const int H = d->height, W = d->width, K = d->inv_size;
  if (H < 2 || W < 2 || K < 2) { rk_set_error("bad sensor dimensions"); return RK_EINTRINSICS; }
  const size_t HW = (size_t)H * W;
  // layout of the single device blob (all offsets 16-byte aligned)
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  size_t o_dirs = take(HW * 3 * sizeof(double));
  size_t o_orig = take((size_t)W * 3 * sizeof(double));
  size_t o_d32 = take(HW * sizeof(float4));
  size_t o_o32 = take((size_t)W * sizeof(float4));
  size_t o_az32 = take(H * sizeof(float));
  size_t o_el32 = take(H * sizeof(float));
  size_t o_az = take(H * sizeof(double));
  size_t o_el = take(H * sizeof(double));
  size_t o_inv = take(K * sizeof(int32_t));
  size_t o_rs14 = take(sizeof(kVrsqrt14));
  std::vector<unsigned char> host(off, 0);
  memcpy(&host[o_dirs], d->dirs_host, HW * 3 * sizeof(double));
  memcpy(&host[o_orig], d->origins_host, (size_t)W * 3 * sizeof(double));
  float4* d32 = reinterpret_cast<float4*>(&host[o_d32]);
  for (size_t i = 0; i < HW; ++i)
    d32[i] = make_float4((float)d->dirs_host[3 * i], (float)d->dirs_host[3 * i + 1],
                         (float)d->dirs_host[3 * i + 2], 0.f);
  float4* o32 = reinterpret_cast<float4*>(&host[o_o32]);
  for (int i = 0; i < W; ++i)
    o32[i] = make_float4((float)d->origins_host[3 * i], (float)d->origins_host[3 * i + 1],
                         (float)d->origins_host[3 * i + 2], 0.f);
  float* az32 = reinterpret_cast<float*>(&host[o_az32]);
  float* el32 = reinterpret_cast<float*>(&host[o_el32]);
  for (int i = 0; i < H; ++i) { az32[i] = (float)d->azimuth_host[i]; el32[i] = (float)d->elevation_host[i]; }
  memcpy(&host[o_az], d->azimuth_host, H * sizeof(double));
  memcpy(&host[o_el], d->elevation_host, H * sizeof(double));
  memcpy(&host[o_inv], d->inv_rows_host, K * sizeof(int32_t));
  memcpy(&host[o_rs14], kVrsqrt14, sizeof(kVrsqrt14));

  rk_sensor* s = new rk_sensor();
  cudaGetDevice(&s->device);
  cudaError_t e = cudaMalloc(&s->blob, off);
  if (e != cudaSuccess) { delete s; return rk_cuda_status(e, "rk_sensor_create cudaMalloc"); }
  e = cudaMemcpy(s->blob, host.data(), off, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(s->blob); delete s; return rk_cuda_status(e, "rk_sensor_create copy"); }
  unsigned char* b = static_cast<unsigned char*>(s->blob);
  SensorDev& v = s->dev;
  v.H = H; v.W = W;
  v.r0 = d->receiver_radius; v.r0f = (float)d->receiver_radius;
  v.dirs = reinterpret_cast<const double*>(b + o_dirs);
  v.origins = reinterpret_cast<const double*>(b + o_orig);
  v.dirs32 = reinterpret_cast<const float4*>(b + o_d32);
  v.origins32 = reinterpret_cast<const float4*>(b + o_o32);
  v.az32 = reinterpret_cast<const float*>(b + o_az32);
  v.el32 = reinterpret_cast<const float*>(b + o_el32);
  v.az = reinterpret_cast<const double*>(b + o_az);
  v.el = reinterpret_cast<const double*>(b + o_el);
  v.inv_rows = reinterpret_cast<const int32_t*>(b + o_inv);
  v.rsqrt14 = reinterpret_cast<const uint16_t*>(b + o_rs14);
  v.K = K;
  v.inv_lo = d->inv_phi_min;
  v.inv_scale = (double)(K - 1) / (d->inv_phi_max - d->inv_phi_min);
  v.inv_lo32 = (float)v.inv_lo;
  v.inv_scale32 = (float)v.inv_scale;
  v.inv_off32 = (float)(0.5 - v.inv_lo * v.inv_scale);
  v.fov_lo = d->fov_lo; v.fov_hi = d->fov_hi;
  v.fov_lo32 = (float)d->fov_lo; v.fov_hi32 = (float)d->fov_hi;
  v.cpr = (double)W / kTwoPi;
  v.cpr32 = (float)v.cpr;
  v.two_pi32 = (float)kTwoPi;
  *out = s;
  return RK_OK;
}

extern "C" int rk_sensor_destroy(rk_sensor* s) {
  if (!s) return RK_OK;
  cudaFree(s->blob);
  delete s;
  return RK_OK;
}

// ------------------------------------------------------------------ projection
template <int MATH, int APPROX = PROJ_EXACT>
__global__ void k_project_f32(SensorDev s, const float* __restrict__ pts, int64_t n, float* u,
                              int32_t* v, float* r, int8_t* st) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Proj32 p = project_f32<MATH, false, APPROX>(s, global_tables(s), pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    if (u) u[i] = p.u;
    if (v) v[i] = p.v;
    if (r) r[i] = p.r;
    if (st) st[i] = (int8_t)p.status;
  }
}

__global__ void k_svml_eval(SensorDev s, int fn, const float* __restrict__ a, const float* __restrict__ b,
                            int64_t n, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fn == 0   ? svml_atan2f(a[i], b[i])
             : fn == 1 ? svml_asinf(a[i], s.rsqrt14)
             : fn == 2 ? div_rn_fast(a[i], b[i])
             : fn == 3 ? __fdiv_rn(a[i], b[i])
             : fn == 4 ? sqrt_rn_normal(a[i])
                       : __fsqrt_rn(a[i]);
}

extern "C" int rk_svml_eval(const rk_sensor* s, int fn, const float* a, const float* b, int64_t n,
                            float* out, void* stream) {
  if (n <= 0) return RK_OK;
  if (fn < 0 || fn > 5) {
    rk_set_error("fn must be 0 (arctan2), 1 (arcsin), 2 / 3 (division), 4 / 5 (square root)");
    return RK_EGENERIC;
  }
  if ((fn == 0 || fn == 2 || fn == 3) && !b) { rk_set_error("arctan2 and division need b"); return RK_EGENERIC; }
  unsigned g = min(blocks_for(n, 256), 148u * 16u);
  k_svml_eval<<<g, 256, 0, S(stream)>>>(s->dev, fn, a, b, n, out);
  RK_LAUNCHED("k_svml_eval");
  return RK_OK;
}

extern "C" int rk_project_f32(const rk_sensor* s, const float* pts, int64_t n, int math,
                              float* u, int32_t* v, float* r, int8_t* status, void* stream) {
  if (n <= 0) return RK_OK;
  unsigned g = min(blocks_for(n, 256), 148u * 16u);
  if (math == MATH_CR)
    k_project_f32<MATH_CR><<<g, 256, 0, S(stream)>>>(s->dev, pts, n, u, v, r, status);
  else if (math == MATH_LIBM)
    k_project_f32<MATH_LIBM><<<g, 256, 0, S(stream)>>>(s->dev, pts, n, u, v, r, status);
  else if (math == MATH_NP)
    k_project_f32<MATH_NP><<<g, 256, 0, S(stream)>>>(s->dev, pts, n, u, v, r, status);
  else if (math == RK_MATH_NP_FINITE)
    k_project_f32<MATH_NP, PROJ_EXACT_FINITE><<<g, 256, 0, S(stream)>>>(s->dev, pts, n, u, v, r, status);
  else
    k_project_f32<MATH_FAST><<<g, 256, 0, S(stream)>>>(s->dev, pts, n, u, v, r, status);
  RK_LAUNCHED("k_project_f32");
  return RK_OK;
}

// float64 fixed-point path (lidar_model.py:287-336).  The reference stops the
// receiver iteration globally once max |du| over non-degenerate points < tol,
// so the loop is split into one launch per iteration with a device flag.
// work layout: [0,n) u_hat, [n,2n) xc, [2n,3n) yc, then 2 x u64 (max du bits, stop)
__device__ __forceinline__ double wrap_cols(double th, double cpr) {
  return __dmul_rn(th < 0.0 ? __dadd_rn(th, kTwoPi) : __dadd_rn(th, 0.0), cpr);
}

__global__ void k_proj64_init(SensorDev s, const double* __restrict__ pts, int64_t n,
                              double* work, unsigned long long* ctl) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i == 0) { ctl[0] = 0ull; ctl[1] = 0ull; }
  if (i >= n) return;
  double x = pts[3 * i], y = pts[3 * i + 1];
  work[i] = wrap_cols(atan2(y, x), s.cpr);
  work[n + i] = x;
  work[2 * n + i] = y;
}

__global__ void k_proj64_iter(SensorDev s, const double* __restrict__ pts, int64_t n,
                              double* work, unsigned long long* ctl, double tol, int last) {
  // ctl[1] != 0: an earlier iteration already met tol -> no-op (reference `break`)
  if (ctl[1]) return;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    double a = __ddiv_rn(work[i], s.cpr);
    double xc = __dsub_rn(x, __dmul_rn(s.r0, cos(a)));
    double yc = __dsub_rn(y, __dmul_rn(s.r0, sin(a)));
    double un = wrap_cols(atan2(yc, xc), s.cpr);
    double du = fabs(__dsub_rn(un, work[i]));
    du = fmin(du, __dsub_rn((double)s.W, du));
    work[i] = un;
    work[n + i] = xc;
    work[2 * n + i] = yc;
    double rho2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    bool deg = __dadd_rn(rho2, __dmul_rn(z, z)) <= __dmul_rn(s.r0, s.r0);
    if (!deg) atomicMax(&ctl[0], (unsigned long long)__double_as_longlong(du));
  }
  (void)last;
}

__global__ void k_proj64_check(unsigned long long* ctl, double tol, int64_t n_live) {
  // decide whether the next iteration runs: max over non-degenerate |du| < tol
  if (ctl[1]) return;
  double m = __longlong_as_double((long long)ctl[0]);
  if (n_live == 0 || m < tol) ctl[1] = 1ull;
  ctl[0] = 0ull;
}

__global__ void k_proj64_final(SensorDev s, const double* __restrict__ pts, int64_t n,
                               const double* work, int refine, double* u_out, int32_t* v_out,
                               double* r_out, int8_t* st_out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
  const double W = (double)s.W;
  double r;
  bool deg;
  if (s.r0 > 0.0) {
    double rho2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    deg = __dadd_rn(rho2, __dmul_rn(z, z)) <= __dmul_rn(s.r0, s.r0);
    double xc = work[n + i], yc = work[2 * n + i];
    r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(xc, xc), __dmul_rn(yc, yc)), __dmul_rn(z, z)));
  } else {
    r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    deg = r <= 0.0;
  }
  double q = fmin(fmax(__ddiv_rn(z, fmax(r, 1e-300)), -1.0), 1.0);
  double phi = asin(q);
  int v = row_from_elevation_f64(s, phi);
  double u = __dsub_rn(work[i], __dmul_rn(s.cpr, s.az[v]));
  if (u < 0.0) u = __dadd_rn(u, W);
  if (u >= W) u = __dsub_rn(u, W);
  if (s.r0 > 0.0 && refine) {
    double a = __ddiv_rn(u, s.cpr);
    double xc = __dsub_rn(x, __dmul_rn(s.r0, cos(a)));
    double yc = __dsub_rn(y, __dmul_rn(s.r0, sin(a)));
    r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(xc, xc), __dmul_rn(yc, yc)), __dmul_rn(z, z)));
    q = fmin(fmax(__ddiv_rn(z, fmax(r, 1e-300)), -1.0), 1.0);
    phi = asin(q);
    v = row_from_elevation_f64(s, phi);
    u = __dsub_rn(wrap_cols(atan2(yc, xc), s.cpr), __dmul_rn(s.cpr, s.az[v]));
    if (u < 0.0) u = __dadd_rn(u, W);
    if (u >= W) u = __dsub_rn(u, W);
  }
  u_out[i] = u;
  v_out[i] = v;
  r_out[i] = r;
  st_out[i] = deg ? PROJ_DEGENERATE : ((phi < s.fov_lo || phi > s.fov_hi) ? PROJ_OUT_OF_FOV : PROJ_OK);
}

__global__ void k_count_live64(SensorDev s, const double* __restrict__ pts, int64_t n,
                               unsigned long long* live) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
  double rho2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
  if (!(__dadd_rn(rho2, __dmul_rn(z, z)) <= __dmul_rn(s.r0, s.r0))) atomicAdd(live, 1ull);
}

extern "C" int rk_project_f64(const rk_sensor* s, const double* pts, int64_t n, int max_iters,
                              double tol, int refine, double* u, int32_t* v, double* r,
                              int8_t* status, double* work, void* stream) {
  if (n <= 0) return RK_OK;
  cudaStream_t st = S(stream);
  unsigned g = blocks_for(n, 256);
  unsigned long long* ctl = reinterpret_cast<unsigned long long*>(work + 3 * n);
  k_proj64_init<<<g, 256, 0, st>>>(s->dev, pts, n, work, ctl);
  if (s->dev.r0 > 0.0 && max_iters > 0) {
    // number of non-degenerate points: the reference breaks immediately when 0
    unsigned long long* live = ctl + 2;
    RK_CUDA(cudaMemsetAsync(live, 0, sizeof(unsigned long long), st));
    k_count_live64<<<g, 256, 0, st>>>(s->dev, pts, n, live);
    unsigned long long h_live = 0;
    RK_CUDA(cudaMemcpyAsync(&h_live, live, sizeof(h_live), cudaMemcpyDeviceToHost, st));
    RK_CUDA(cudaStreamSynchronize(st));
    for (int it = 0; it < max_iters; ++it) {
      k_proj64_iter<<<g, 256, 0, st>>>(s->dev, pts, n, work, ctl, tol, it == max_iters - 1);
      k_proj64_check<<<1, 1, 0, st>>>(ctl, tol, (int64_t)h_live);
    }
  }
  k_proj64_final<<<g, 256, 0, st>>>(s->dev, pts, n, work, refine, u, v, r, status);
  RK_LAUNCHED("rk_project_f64");
  return RK_OK;
}

// ------------------------------------------------------------------ rows
__global__ void k_rows(SensorDev s, const void* phi, int is_f64, int64_t n, int32_t* v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  v[i] = is_f64 ? row_from_elevation_f64(s, static_cast<const double*>(phi)[i])
                : row_from_elevation_f32(s, static_cast<const float*>(phi)[i]);
}

extern "C" int rk_row_from_elevation(const rk_sensor* s, const void* phi, int is_f64, int64_t n,
                                     int32_t* v, void* stream) {
  if (n <= 0) return RK_OK;
  k_rows<<<blocks_for(n, 256), 256, 0, S(stream)>>>(s->dev, phi, is_f64, n, v);
  RK_LAUNCHED("k_rows");
  return RK_OK;
}

__global__ void k_inv_lookup(const int32_t* rows, int k, double lo, double scale, float lo32,
                             float scale32, const void* phi, int is_f64, int64_t n, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int idx;
  if (is_f64) {
    double p = static_cast<const double*>(phi)[i];
    double pos = __dadd_rn(__dmul_rn(__dsub_rn(p, lo), scale), 0.5);
    idx = (int)fmin(fmax(pos, 0.0), (double)(k - 1));
  } else {
    float p = static_cast<const float*>(phi)[i];
    float pos = __fadd_rn(__fmul_rn(__fsub_rn(p, lo32), scale32), 0.5f);
    idx = (int)fminf(fmaxf(pos, 0.f), (float)(k - 1));
  }
  out[i] = rows[idx];
}

extern "C" int rk_inverse_lut_lookup(const int32_t* rows, int32_t k, double phi_min,
                                     double phi_max, const void* phi, int is_f64, int64_t n,
                                     int32_t* out, void* stream) {
  if (n <= 0) return RK_OK;
  double scale = (double)(k - 1) / (phi_max - phi_min);
  k_inv_lookup<<<blocks_for(n, 256), 256, 0, S(stream)>>>(rows, k, phi_min, scale, (float)phi_min,
                                                           (float)scale, phi, is_f64, n, out);
  RK_LAUNCHED("k_inv_lookup");
  return RK_OK;
}

// unproject_many (lidar_model.py:236-250): analytic, float64
__global__ void k_unproject_many(SensorDev s, const double* u, const int64_t* v, const double* r,
                                 int64_t n, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double alpha = __ddiv_rn(__dmul_rn(kTwoPi, u[i]), (double)s.W);
  int64_t row = v[i];
  double theta = __dadd_rn(alpha, s.az[row]);
  double phi = s.el[row];
  double cphi = cos(phi);
  double rr = r[i];
  out[3 * i + 0] = __dadd_rn(__dmul_rn(__dmul_rn(rr, cos(theta)), cphi), __dmul_rn(s.r0, cos(alpha)));
  out[3 * i + 1] = __dadd_rn(__dmul_rn(__dmul_rn(rr, sin(theta)), cphi), __dmul_rn(s.r0, sin(alpha)));
  out[3 * i + 2] = __dadd_rn(__dmul_rn(rr, sin(phi)), 0.0);
}

extern "C" int rk_unproject_many(const rk_sensor* s, const double* u, const int64_t* v,
                                 const double* r, int64_t n, double* out, void* stream) {
  if (n <= 0) return RK_OK;
  k_unproject_many<<<blocks_for(n, 256), 256, 0, S(stream)>>>(s->dev, u, v, r, n, out);
  RK_LAUNCHED("k_unproject_many");
  return RK_OK;
}

// ------------------------------------------------------------------ images
__global__ void k_unproject_image(SensorDev s, const float* __restrict__ range, int64_t total,
                                  double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t HW = (int64_t)s.H * s.W;
  int64_t p = i % HW;
  double q[3];
  unproject_px(s, (int)(p / s.W), (int)(p % s.W), range[i], q);
  out[3 * i] = q[0];
  out[3 * i + 1] = q[1];
  out[3 * i + 2] = q[2];
}

extern "C" int rk_unproject_image(const rk_sensor* s, const float* range, int32_t batch,
                                  double* out, void* stream) {
  int64_t total = (int64_t)batch * s->dev.H * s->dev.W;
  if (total <= 0) return RK_OK;
  k_unproject_image<<<blocks_for(total, 256), 256, 0, S(stream)>>>(s->dev, range, total, out);
  RK_LAUNCHED("k_unproject_image");
  return RK_OK;
}

// K1: cross-product normals (range_image.py:221-240) in the pinned op order
// (SURVEY Appendix A1).  A CTA owns a K1_TH x K1_TW tile of one image and
// unprojects each pixel of the tile plus its right/down halo ONCE into shared
// memory (a per-pixel kernel would unproject every point three times).
constexpr int K1_TW = 128, K1_TH = 8, K1_THREADS = 256;
__global__ void __launch_bounds__(K1_THREADS) k_normals_cross(
    SensorDev s, const float* __restrict__ range, int batch, float* normals, uint8_t* valid,
    float4* surfel, int64_t surfel_pitch, int targets) {
  constexpr int PW = K1_TW + 1, PH = K1_TH + 1;
  __shared__ double sp[3][PH * PW];
  __shared__ float sr[PH * PW];
  const int W = s.W, H = s.H;
  const int tiles_x = (W + K1_TW - 1) / K1_TW, tiles_y = (H + K1_TH - 1) / K1_TH;
  const int64_t HW = (int64_t)H * W;
  const int t = blockIdx.x;
  const int img = t / (tiles_x * tiles_y);
  const int tt = t - img * (tiles_x * tiles_y);
  const int v0 = (tt / tiles_x) * K1_TH, u0 = (tt - (tt / tiles_x) * tiles_x) * K1_TW;
  const float* R = range + img * HW;
  for (int k = threadIdx.x; k < PH * PW; k += K1_THREADS) {
    const int dv = k / PW, du = k - dv * PW;
    const int v = v0 + dv;
    int u = u0 + du;
    if (u >= W) u -= W;  // azimuth wrap (the halo of the last tile is column 0)
    float r = 0.0f;
    double P[3] = {0.0, 0.0, 0.0};
    if (v < H) {
      r = __ldg(R + (int64_t)v * W + u);
      unproject_px(s, v, u, r, P);
    }
    sr[k] = r;
    sp[0][k] = P[0];
    sp[1][k] = P[1];
    sp[2][k] = P[2];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K1_TH * K1_TW; k += K1_THREADS) {
    const int dv = k / K1_TW, du = k - dv * K1_TW;
    const int v = v0 + dv, u = u0 + du;
    if (v >= H || u >= W) continue;
    const int c = dv * PW + du, cr = c + 1, cd = c + PW;
    const float r0 = sr[c];
    const bool has_down = v + 1 < H;
    const bool ok0 = r0 > 0.f && sr[cr] > 0.f && has_down && sr[cd] > 0.f;
    const double P0 = sp[0][c], P1 = sp[1][c], P2 = sp[2][c];
    const double a0 = __dsub_rn(sp[0][cr], P0), a1 = __dsub_rn(sp[1][cr], P1), a2 = __dsub_rn(sp[2][cr], P2);
    // the reference's "down" row below the image is 0.0 (range_image.py:227-228)
    const double d0 = has_down ? sp[0][cd] : 0.0, d1 = has_down ? sp[1][cd] : 0.0,
                 d2 = has_down ? sp[2][cd] : 0.0;
    const double b0 = __dsub_rn(d0, P0), b1 = __dsub_rn(d1, P1), b2 = __dsub_rn(d2, P2);
    const double c0 = __dsub_rn(__dmul_rn(a1, b2), __dmul_rn(a2, b1));
    const double c1 = __dsub_rn(__dmul_rn(a2, b0), __dmul_rn(a0, b2));
    const double c2 = __dsub_rn(__dmul_rn(a0, b1), __dmul_rn(a1, b0));
    const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(c0, c0), __dmul_rn(c1, c1)), __dmul_rn(c2, c2)));
    const bool ok = ok0 && nn > 1e-12;
    float n0 = 0.f, n1 = 0.f, n2 = 0.f;
    if (ok) {
      // c / nn correctly rounded: y = RN(1/nn), q = RN(c*y) plus one residual
      // correction (Markstein; exact for normal operands, |c| <= nn here)
      const double y = __drcp_rn(nn);
      double m0 = __dmul_rn(c0, y), m1 = __dmul_rn(c1, y), m2 = __dmul_rn(c2, y);
      m0 = __fma_rn(__fma_rn(-nn, m0, c0), y, m0);
      m1 = __fma_rn(__fma_rn(-nn, m1, c1), y, m1);
      m2 = __fma_rn(__fma_rn(-nn, m2, c2), y, m2);
      const double facing = __dadd_rn(__dadd_rn(__dmul_rn(m0, P0), __dmul_rn(m1, P1)), __dmul_rn(m2, P2));
      if (facing > 0.0) { m0 = -m0; m1 = -m1; m2 = -m2; }
      n0 = (float)m0; n1 = (float)m1; n2 = (float)m2;
    }
    const int64_t p = (int64_t)v * W + u;
    const int64_t i = img * HW + p;
    if (normals) {
      normals[3 * i] = n0;
      normals[3 * i + 1] = n1;
      normals[3 * i + 2] = n2;
    }
    if (valid) valid[i] = ok ? 1 : 0;
    if (surfel) {
      if (targets && RK_SURFEL_REC == 16) {
        // 16-byte pyramid records {n, range}: the registration forms the
        // target from the (L2-resident, shared) float32 ray tables
        surfel[img * surfel_pitch + p] = make_float4(n0, n1, n2, ok ? r0 : 0.f);
      } else if (targets) {
        // pyramid layout: {n, range} then the association target
        // r * dir32 + origin32 with the reference's separate roundings
        // (registration.py:168-176), so the registration gathers one
        // 32-byte record instead of also reading the ray tables
        const float4 d = __ldg(s.dirs32 + p), o = __ldg(s.origins32 + u);
        float4* rec = surfel + 2 * (img * surfel_pitch + p);
        rec[0] = make_float4(n0, n1, n2, ok ? r0 : 0.f);
        rec[1] = make_float4(__fadd_rn(__fmul_rn(r0, d.x), o.x), __fadd_rn(__fmul_rn(r0, d.y), o.y),
                             __fadd_rn(__fmul_rn(r0, d.z), o.z), 0.f);
      } else {
        surfel[img * surfel_pitch + p] = make_float4(n0, n1, n2, ok ? r0 : 0.f);
      }
    }
  }
}

static void launch_k1(const rk_sensor* s, const float* range, int32_t batch, float* normals,
                      uint8_t* valid, float4* surfel, int64_t pitch, cudaStream_t st, int targets = 0) {
  const int W = s->dev.W, H = s->dev.H;
  const unsigned tiles = (unsigned)(((W + K1_TW - 1) / K1_TW) * ((H + K1_TH - 1) / K1_TH));
  k_normals_cross<<<tiles * (unsigned)batch, K1_THREADS, 0, st>>>(s->dev, range, batch, normals,
                                                                  valid, surfel, pitch, targets);
}

// decimated copies of the full surfel maps (pixel (i, j) of level s = (i*s, j*s))
__global__ void k_surfel_decimate(int H, int W, int batch, float4* pyr, int64_t pitch, int stride,
                                  int64_t off) {
  const int Hs = (H + stride - 1) / stride, Ws = (W + stride - 1) / stride;
  const int64_t per = (int64_t)Hs * Ws, total = per * batch;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t img = k / per;
    const int q = (int)(k - img * per);
    const int i = q / Ws, j = q - i * Ws;
    const int64_t from = (int64_t)i * stride * W + (int64_t)j * stride;
    if (RK_SURFEL_REC == 16) {
      float4* base = pyr + img * pitch;
      base[off + q] = base[from];
    } else {
      float4* base = pyr + 2 * img * pitch;  // 2 float4 records (see k_normals_cross)
      base[2 * (off + q)] = base[2 * from];
      base[2 * (off + q) + 1] = base[2 * from + 1];
    }
  }
}

extern "C" int rk_normals_cross(const rk_sensor* s, const float* range, int32_t batch,
                                float* normals, uint8_t* valid, float* surfel, void* stream) {
  int64_t total = (int64_t)batch * s->dev.H * s->dev.W;
  if (total <= 0) return RK_OK;
  launch_k1(s, range, batch, normals, valid, reinterpret_cast<float4*>(surfel),
            (int64_t)s->dev.H * s->dev.W, S(stream));
  RK_LAUNCHED("k_normals_cross");
  return RK_OK;
}

extern "C" int rk_surfel_record_floats(void) { return RK_SURFEL_REC / 4; }

extern "C" int rk_normals_cross_pyramid(const rk_sensor* s, const float* range, int32_t batch,
                                        const int32_t* strides_host, int32_t n_strides,
                                        float* surfel_pyr, int64_t pitch, void* stream) {
  const int H = s->dev.H, W = s->dev.W;
  const int64_t total = (int64_t)batch * H * W;
  if (total <= 0) return RK_OK;
  int64_t need = (int64_t)H * W;
  for (int k = 0; k < n_strides; ++k) {
    const int st = strides_host[k];
    if (st < 1) { rk_set_error("strides must be >= 1"); return RK_EGENERIC; }
    if (st > 1) need += (int64_t)((H + st - 1) / st) * ((W + st - 1) / st);
  }
  if (pitch < need) { rk_set_error("surfel pyramid pitch %lld < %lld", (long long)pitch, (long long)need); return RK_EGENERIC; }
  float4* pyr = reinterpret_cast<float4*>(surfel_pyr);
  launch_k1(s, range, batch, nullptr, nullptr, pyr, pitch, S(stream), 1);
  int64_t off = (int64_t)H * W;
  for (int k = 0; k < n_strides; ++k) {
    const int st = strides_host[k];
    if (st <= 1) continue;
    const int64_t per = (int64_t)((H + st - 1) / st) * ((W + st - 1) / st);
    k_surfel_decimate<<<blocks_for(per * batch, 256), 256, 0, S(stream)>>>(H, W, batch, pyr, pitch, st, off);
    off += per;
  }
  RK_LAUNCHED("rk_normals_cross_pyramid");
  return RK_OK;
}

// ------------------------------------------------------------------ K2 compaction
// One CTA per image walks the stride-s view in tiles of blockDim pixels;
// warp ballots + a 32-entry scan give each survivor its row-major rank, so
// the output order equals np.nonzero's.
template <int NT>
__global__ void __launch_bounds__(NT) k_stride_compact(SensorDev s, const float* __restrict__ range,
                                                       int stride, float cmin, float cmax,
                                                       int32_t* idx, int32_t* count) {
  const int b = blockIdx.x;
  const int W = s.W, H = s.H;
  const int Hs = (H + stride - 1) / stride, Ws = (W + stride - 1) / stride;
  const int n = Hs * Ws;
  const float* R = range + (int64_t)b * H * W;
  int32_t* out = idx + (int64_t)b * n;
  __shared__ int warp_tot[NT / 32];
  __shared__ int carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < n; base += NT) {
    int k = base + threadIdx.x;
    int flat = 0;
    bool keep = false;
    if (k < n) {
      int vi = k / Ws, ui = k - vi * Ws;
      flat = vi * stride * W + ui * stride;
      keep = range_ok(R[flat], cmin, cmax);
    }
    unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    int carry = carry_s;
    int before = 0;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    if (keep) out[carry + before + __popc(m & ((1u << lane) - 1u))] = flat;
    __syncthreads();
    if (threadIdx.x == NT - 1) {
      int tot = 0;
      for (int w = 0; w < NT / 32; ++w) tot += warp_tot[w];
      carry_s = carry + tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) count[b] = carry_s;
}

extern "C" int rk_stride_compact(const rk_sensor* s, const float* range, int32_t batch,
                                 int32_t stride, float clip_min, float clip_max, int32_t* idx,
                                 int32_t* count, void* stream) {
  if (batch <= 0) return RK_OK;
  if (stride < 1) { rk_set_error("stride must be >= 1"); return RK_EGENERIC; }
  k_stride_compact<512><<<batch, 512, 0, S(stream)>>>(s->dev, range, stride, clip_min, clip_max,
                                                       idx, count);
  RK_LAUNCHED("k_stride_compact");
  return RK_OK;
}

__global__ void k_unproject_pixels(SensorDev s, const float* __restrict__ range,
                                   const int32_t* __restrict__ idx, const int32_t* count,
                                   int64_t cap, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= cap || i >= *count) return;
  int f = idx[i];
  double q[3];
  unproject_px(s, f / s.W, f % s.W, range[f], q);
  out[3 * i] = q[0];
  out[3 * i + 1] = q[1];
  out[3 * i + 2] = q[2];
}

extern "C" int rk_unproject_pixels(const rk_sensor* s, const float* range, const int32_t* idx,
                                   const int32_t* count, int64_t cap, double* out, void* stream) {
  if (cap <= 0) return RK_OK;
  k_unproject_pixels<<<blocks_for(cap, 256), 256, 0, S(stream)>>>(s->dev, range, idx, count, cap, out);
  RK_LAUNCHED("k_unproject_pixels");
  return RK_OK;
}

// generic stable mask compaction: block counts -> single-CTA scan -> scatter
__global__ void k_mask_counts(const uint8_t* __restrict__ mask, int64_t n, int chunk, int32_t* cnt) {
  __shared__ int acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  int c = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) c += mask[i] != 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) atomicAdd(&acc, c);
  __syncthreads();
  if (threadIdx.x == 0) cnt[blockIdx.x] = acc;
}

__global__ void k_scan_counts(int32_t* cnt, int nb, int32_t* total) {
  // tiny: one thread (nb <= a few thousand)
  if (threadIdx.x != 0) return;
  int run = 0;
  for (int i = 0; i < nb; ++i) { int c = cnt[i]; cnt[i] = run; run += c; }
  *total = run;
}

__global__ void k_mask_scatter(const uint8_t* __restrict__ mask, int64_t n, int chunk,
                               const int32_t* offs, int32_t* idx) {
  __shared__ int warp_tot[32];
  __shared__ int carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) carry_s = offs[blockIdx.x];
  __syncthreads();
  int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    bool keep = i < hi && mask[i] != 0;
    unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    int carry = carry_s, before = 0;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    if (keep) idx[carry + before + __popc(m & ((1u << lane) - 1u))] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < nw; ++w) tot += warp_tot[w];
      carry_s = carry + tot;
    }
    __syncthreads();
  }
}

extern "C" int rk_compact_mask(const uint8_t* mask, int64_t n, int32_t* idx, int32_t* count,
                               void* stream) {
  cudaStream_t st = S(stream);
  if (n <= 0) { RK_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), st)); return RK_OK; }
  const int chunk = 8192;
  int nb = (int)((n + chunk - 1) / chunk);
  int32_t* offs = nullptr;
  RK_CUDA(cudaMallocAsync(&offs, sizeof(int32_t) * nb, st));
  k_mask_counts<<<nb, 256, 0, st>>>(mask, n, chunk, offs);
  k_scan_counts<<<1, 32, 0, st>>>(offs, nb, count);
  k_mask_scatter<<<nb, 256, 0, st>>>(mask, n, chunk, offs, idx);
  RK_LAUNCHED("rk_compact_mask");
  RK_CUDA(cudaFreeAsync(offs, st));
  return RK_OK;
}
