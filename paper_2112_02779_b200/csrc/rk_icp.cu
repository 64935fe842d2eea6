// rk_icp.cu -- K3: projective association + point-to-plane normal equations +
// per-pair Gauss-Newton update, the whole multi-scale schedule in one launch.
//
// Layout: one CTA per registration pair (persistent over all levels and
// iterations; the pose lives in shared memory).  Each iteration every thread
// walks a row-major slice of the stride-s source view straight out of the
// zero-copy level-0 image (the "pyramid" is index arithmetic, as in the
// reference's StridedView), accumulates the 21+6 normal-equation terms in
// float32 registers (the reference's sgemm precision), and the CTA reduces
// them in float64 with a fixed shuffle/shared-memory tree -- deterministic,
// no float atomics.  Thread 0 then solves the 6x6 system, applies the twist,
// and decides the level's early exit (registration.py:261-282).
#include "rk_common.cuh"
#include "rk_linalg.cuh"

using namespace rk;

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

namespace {

struct IcpArgs {
  SensorDev s;
  const float* src_range;
  const float* dst_range;
  const float4* dst_surfel;
  const int32_t* pair_src;
  const int32_t* pair_dst;
  const double* init12;
  double* out12;
  int32_t* status;
  int32_t* n_iters;
  double* stats;
  int stats_stride;
  rk_icp_config cfg;
  unsigned long long* pt_iters;
};

constexpr int kNumAcc = 29;  // 21 H (upper) + 6 b + cost + sumsq

// One source pixel's contribution (registration.py:145-187 + 339-354).
// Returns false when the point has no surviving correspondence.
template <int MATH>
__device__ __forceinline__ bool associate(const SensorDev& s, const double* pose, const float4* surf,
                                          int v, int u, float r, int stride, float inv_s,
                                          float gate2, float& mx, float& my, float& mz, float& qx,
                                          float& qy, float& qz, float4& nrm) {
  double p[3], m[3];
  unproject_px(s, v, u, r, p);
  xform_rows(pose, pose + 9, p[0], p[1], p[2], m);
  mx = (float)m[0];
  my = (float)m[1];
  mz = (float)m[2];
  Proj32 pr = project_f32<MATH>(s, mx, my, mz);
  if (pr.status != PROJ_OK) return false;
  int col = (int)__fadd_rn(__fmul_rn(pr.u, inv_s), 0.5f) * stride;
  if (col >= s.W) col = 0;
  int row = (int)__fadd_rn(__fmul_rn((float)pr.v, inv_s), 0.5f) * stride;
  if (row >= s.H) return false;  // dropped, not clamped (registration.py:157-159)
  const int flat = row * s.W + col;
  nrm = __ldg(surf + flat);
  if (!(nrm.w > 0.0f)) return false;  // range > 0 and normal valid
  float4 d = __ldg(s.dirs32 + flat);
  float4 o = __ldg(s.origins32 + col);
  qx = __fadd_rn(__fmul_rn(nrm.w, d.x), o.x);
  qy = __fadd_rn(__fmul_rn(nrm.w, d.y), o.y);
  qz = __fadd_rn(__fmul_rn(nrm.w, d.z), o.z);
  float dx = __fsub_rn(mx, qx), dy = __fsub_rn(my, qy), dz = __fsub_rn(mz, qz);
  float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
  return d2 <= gate2;
}

// Thread 0's per-iteration update (registration.py:266-282): the 6x6 checks,
// the float64 solve, the twist update and the early-exit test.  Kept out of
// line so its scratch arrays do not inflate the kernel's register budget.
// Returns 0 iterate, 1 level done, 2 stop (status set).
__device__ __noinline__ int solve_step(const double* tot, int n_corr, double* sh_pose,
                                       const rk_icp_config* cfg, int* status, double* xi) {
  if (n_corr < cfg->min_corr) {
    *status = RK_ICP_TOO_FEW;
    return 2;
  }
  double Hm[36], L[36], piv[6], b[6];
  int q = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) { Hm[i * 6 + j] = Hm[j * 6 + i] = tot[q]; ++q; }
  for (int i = 0; i < 6; ++i) b[i] = tot[21 + i];
  bool ok = chol6(Hm, L, piv);
  if (cond_exceeds6(Hm, L, ok, piv, 1e12)) {
    *status = RK_ICP_DEGENERATE;
    return 2;
  }
  chol_solve6(L, b, xi);
  double P[12];
  for (int i = 0; i < 12; ++i) P[i] = sh_pose[i];
  se3_left_update(xi, P);
  if (orth_defect(P) > 1e-12) reorthonormalize(P);
  for (int i = 0; i < 12; ++i) sh_pose[i] = P[i];
  const double nr = sqrt(xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
  const double nt = sqrt(xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5]);
  return (nr < cfg->rot_eps && nt < cfg->trans_eps) ? 1 : 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

template <int MATH, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_register(IcpArgs A) {
  constexpr int NW = NT / 32;
  const int pair = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SensorDev& s = A.s;
  const int H = s.H, W = s.W;
  const size_t HW = (size_t)H * W;
  const float* src = A.src_range + (size_t)A.pair_src[pair] * HW;
  const float4* surf = A.dst_surfel + (size_t)A.pair_dst[pair] * HW;

  __shared__ double sh_pose[12];
  __shared__ double sh_red[NW][kNumAcc];
  __shared__ double sh_tot[kNumAcc];
  __shared__ int sh_cnt[NW];
  __shared__ int sh_ctrl;  // 0 iterate, 1 level done, 2 stop everything
  if (tid < 12) sh_pose[tid] = A.init12[pair * 12 + tid];
  int n_done = 0, status = RK_ICP_CONVERGED;
  unsigned work = 0;  // valid source points visited (all iterations)

  for (int lv = 0; lv < A.cfg.n_levels; ++lv) {
    const int stride = A.cfg.strides[lv];
    const double level = A.cfg.scale_with_stride ? (double)stride : 1.0;
    const double gate = A.cfg.max_dist * level;
    const double kern = A.cfg.kernel_scale * level;
    const float gate32 = (float)gate;
    const float gate2 = __fmul_rn(gate32, gate32);
    const float k32 = (float)kern;
    const float inv_s = (float)(1.0 / stride);
    const int Hs = (H + stride - 1) / stride, Ws = (W + stride - 1) / stride;
    const int npix = Hs * Ws;
    for (int it = 0; it < A.cfg.iters[lv]; ++it) {
      __syncthreads();  // pose (and sh_ctrl reuse) ready
      double pose[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) pose[i] = sh_pose[i];
      float acc[27];
#pragma unroll
      for (int i = 0; i < 27; ++i) acc[i] = 0.0f;
      double cost = 0.0;
      float sumsq = 0.0f;
      int cnt = 0;
      // row-major walk of the stride view without a per-point division
      int vi = tid / Ws, ui = tid - (tid / Ws) * Ws;
      const int dv = NT / Ws, du = NT - (NT / Ws) * Ws;
      for (int k = tid; k < npix; k += NT) {
        const int v = vi * stride, u = ui * stride;
        vi += dv;
        ui += du;
        if (ui >= Ws) { ui -= Ws; ++vi; }
        const float r = __ldg(src + v * W + u);
        if (!range_ok(r, A.cfg.clip_min, A.cfg.clip_max)) continue;
        ++work;
        float mx, my, mz, qx, qy, qz;
        float4 n;
        if (!associate<MATH>(s, pose, surf, v, u, r, stride, inv_s, gate2, mx, my, mz, qx, qy, qz, n))
          continue;
        // residual, Jacobian, pseudo-Huber IRLS weight (registration.py:339-352)
        const float dx = __fsub_rn(mx, qx), dy = __fsub_rn(my, qy), dz = __fsub_rn(mz, qz);
        const float res = __fadd_rn(__fadd_rn(__fmul_rn(n.x, dx), __fmul_rn(n.y, dy)), __fmul_rn(n.z, dz));
        float J[6];
        J[0] = __fsub_rn(__fmul_rn(my, n.z), __fmul_rn(mz, n.y));
        J[1] = __fsub_rn(__fmul_rn(mz, n.x), __fmul_rn(mx, n.z));
        J[2] = __fsub_rn(__fmul_rn(mx, n.y), __fmul_rn(my, n.x));
        J[3] = n.x;
        J[4] = n.y;
        J[5] = n.z;
        const float e = __fdiv_rn(res, k32);
        const float w = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(1.0f, __fmul_rn(e, e))));
        const float rw = -__fmul_rn(res, w);
        int q = 0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const float jw = __fmul_rn(J[i], w);
#pragma unroll
          for (int j = i; j < 6; ++j) { acc[q] = __fmaf_rn(jw, J[j], acc[q]); ++q; }
        }
#pragma unroll
        for (int i = 0; i < 6; ++i) acc[21 + i] = __fmaf_rn(rw, J[i], acc[21 + i]);
        cost += (double)__fsub_rn(__fdiv_rn(1.0f, w), 1.0f);
        sumsq = __fmaf_rn(res, res, sumsq);
        ++cnt;
      }
      // ---- deterministic CTA reduction in float64, one quantity at a time
#pragma unroll
      for (int i = 0; i < 27; ++i) {
        const double v = warp_sum((double)acc[i]);
        if (lane == 0) sh_red[warp][i] = v;
      }
      {
        const double c = warp_sum(cost);
        const double q2 = warp_sum((double)sumsq);
        const int n = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) {
          sh_red[warp][27] = c;
          sh_red[warp][28] = q2;
          sh_cnt[warp] = n;
        }
      }
      __syncthreads();
      if (tid < kNumAcc) {
        double t = 0.0;
        for (int w2 = 0; w2 < NW; ++w2) t += sh_red[w2][tid];
        sh_tot[tid] = t;
      }
      __syncthreads();
      if (tid == 0) {
        int n_corr = 0;
        for (int w2 = 0; w2 < NW; ++w2) n_corr += sh_cnt[w2];
        double xi[6];
        const int ctrl = solve_step(sh_tot, n_corr, sh_pose, &A.cfg, &status, xi);
        if (ctrl != 2) {
          if (A.stats && n_done < A.stats_stride) {
            double* row = A.stats + ((size_t)pair * A.stats_stride + n_done) * 5;
            row[0] = stride;
            row[1] = it;
            row[2] = n_corr;
            row[3] = kern * kern * sh_tot[27];
            row[4] = sqrt(sh_tot[28] / n_corr);
          }
          ++n_done;
        }
        sh_ctrl = ctrl;
      }
      __syncthreads();
      const int ctrl = sh_ctrl;
      if (ctrl == 2) goto finish;
      if (ctrl == 1) break;
    }
  }
finish:
  if (A.pt_iters) {
    unsigned w = __reduce_add_sync(0xffffffffu, work);
    if (lane == 0 && w) atomicAdd(A.pt_iters, (unsigned long long)w);
  }
  __syncthreads();
  if (tid < 12) A.out12[pair * 12 + tid] = sh_pose[tid];
  if (tid == 0) {
    A.status[pair] = status;
    A.n_iters[pair] = n_done;
  }
}

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
  else
    k_correspondences<MATH_FAST><<<blocks, 256, 0, S(stream)>>>(s->dev, src_pts, n, surf, pose12, gate2,
                                                                stride, inv_s, keep, target, normal);
  RK_LAUNCHED("k_correspondences");
  return RK_OK;
}

extern "C" int rk_register_batch(const rk_sensor* s, const float* src_range, const float* dst_range,
                                 const float* dst_surfel, const int32_t* pair_src,
                                 const int32_t* pair_dst, int32_t batch, const double* init12,
                                 const rk_icp_config* cfg, double* out12, int32_t* status,
                                 int32_t* n_iters, double* stats, int32_t stats_stride,
                                 unsigned long long* pt_iters, void* stream) {
  (void)dst_range;
  if (batch <= 0) return RK_OK;
  if (!cfg || cfg->n_levels < 1 || cfg->n_levels > 8) {
    rk_set_error("schedule must have 1..8 levels");
    return RK_EGENERIC;
  }
  for (int l = 0; l < cfg->n_levels; ++l)
    if (cfg->strides[l] < 1 || cfg->iters[l] < 1) {
      rk_set_error("strides and iteration counts must be >= 1");
      return RK_EGENERIC;
    }
  IcpArgs a;
  a.s = s->dev;
  a.src_range = src_range;
  a.dst_range = dst_range;
  a.dst_surfel = reinterpret_cast<const float4*>(dst_surfel);
  a.pair_src = pair_src;
  a.pair_dst = pair_dst;
  a.init12 = init12;
  a.out12 = out12;
  a.status = status;
  a.n_iters = n_iters;
  a.stats = stats;
  a.stats_stride = stats ? stats_stride : 0;
  a.cfg = *cfg;
  a.pt_iters = pt_iters;
#ifndef RK_ICP_MINB
#define RK_ICP_MINB 3
#endif
  constexpr int NT = 256, MINB = RK_ICP_MINB;
  if (cfg->math == MATH_CR)
    k_register<MATH_CR, NT, MINB><<<batch, NT, 0, S(stream)>>>(a);
  else
    k_register<MATH_FAST, NT, MINB><<<batch, NT, 0, S(stream)>>>(a);
  RK_LAUNCHED("k_register");
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
