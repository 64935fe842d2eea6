// rk_register.cu -- K3: the whole multi-scale projective point-to-plane ICP
// schedule (registration.py:237-289) for a batch of independent pairs, one
// launch.
//
// A "group" of WPP warps owns one registration pair for its whole schedule;
// the pose lives in shared memory.  Every iteration each lane walks a
// row-major slice of the stride-s source view straight out of the level-0
// image (the reference's zero-copy StridedView, range_image.py:69-116),
// associates it projectively (registration.py:117-187), and accumulates the
// 21 + 6 normal-equation terms in float32 registers (the reference's sgemm
// precision).  The group then reduces them in float64 with a fixed
// shuffle/shared-memory tree -- deterministic, no float atomics -- and one
// lane solves the 6x6 system, applies the twist and decides the early exit
// (registration.py:261-282).
//
// WPP = 8 (one 256-thread CTA per pair, 4 CTAs per SM) is the default: it
// measured fastest at every batch size (fewer distinct pairs per SM keep the
// surfel gathers cache-local).  WPP = 1/2/4 (several pairs per CTA, no
// CTA-wide barrier) remain selectable with RK_ICP_WPP for experiments.
#include "rk_common.cuh"
#include "rk_linalg.cuh"
#include <cooperative_groups.h>
#if RK_ICP_TIME_SOLVE
#include <cstdio>
#endif

using namespace rk;

#ifndef RK_ICP_MINB_NP  // CTAs per SM for the numpy-exact kernel
#define RK_ICP_MINB_NP 3  // 85 registers: the exact float64 walk spills at 64 (A/B: +7%)
#endif
#ifndef RK_ICP_MINB
#define RK_ICP_MINB 4
#endif
#ifndef RK_ICP_F32X
#define RK_ICP_F32X 1
#endif
#ifndef RK_ICP_FUSED
#define RK_ICP_FUSED 1
#endif
// RK_ICP_F64_AHEAD (exact modes' float64 walk): hold the next row's float64
// ray in registers (1) or load the ray and origin at use (0)
#ifndef RK_ICP_F64_AHEAD
#define RK_ICP_F64_AHEAD 1
#endif
#ifndef RK_ICP_TRANSPOSE  // recursive-halving warp reduction of the partials (1) or 29 butterfly sums (0)
#define RK_ICP_TRANSPOSE 1
#endif
#ifndef RK_ICP_ELEV_ONLY
#define RK_ICP_ELEV_ONLY 1
#endif

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

namespace {

constexpr int kNumAcc = 29;  // 21 H (upper) + 6 b + cost + sumsq
// RK_ICP_LVL_SMEM: the per-level constants (gate^2, 1/k, 1/s, stride, surfel
// level offset/width) live in shared memory, so under the 64-register cap the
// compiler re-reads them with one LDS instead of re-deriving them per point
// cluster tiers: all-to-all partials, every CTA solves its own update (one
// cluster barrier per iteration, no pose broadcast): one pair, NP, K3 x8
// 0.416 -> 0.372 ms, x16 0.384 -> 0.301 ms (scripts/latency_probe.py)
#ifndef RK_ICP_CLUSTER_REDUNDANT
#define RK_ICP_CLUSTER_REDUNDANT 1
#endif
#ifndef RK_ICP_CLUSTER16  // the launcher may take 16-CTA clusters (non-portable size)
#define RK_ICP_CLUSTER16 1
#endif
#ifndef RK_ICP_LVL_SMEM
#define RK_ICP_LVL_SMEM 1
#endif
// RK_ICP_PREFETCH: after a point's gather, prefetch the records one view row
// below it (1 = into L1, 2 = into L2): the column walk's next point projects
// close to there, so its dependent gather finds the line on chip
#ifndef RK_ICP_PREFETCH
#define RK_ICP_PREFETCH 1
#endif
#ifndef RK_ICP_PF_ROWS
#define RK_ICP_PF_ROWS 1  // how many view rows ahead (1..3 measured equal)
#endif
#ifndef RK_ICP_THREADS
#define RK_ICP_THREADS 256
#endif
constexpr int kThreads = RK_ICP_THREADS;  // one CTA per pair by default (WPP = kThreads / 32)
constexpr int kWide = 1024;               // latency-mode CTA (small batches)
// the numpy-exact walk needs ~80 registers: at 1024 threads (64 registers)
// it spills ~70 values in the hot loop, so its latency-mode CTAs are 512
// threads (128 registers): one pair, cluster x8: K3 0.594 -> 0.433 ms
// (768: 0.479 ms; scripts/latency_probe.py)
#ifndef RK_ICP_LAT_NT_NP
#define RK_ICP_LAT_NT_NP 512
#endif
template <int MATH>
constexpr int lat_nt() { return MATH == MATH_NP ? RK_ICP_LAT_NT_NP : kWide; }

struct IcpArgs {
  SensorDev s;
  const float* src_range;
  const float4* dst_surfel;
  const int32_t* pair_src;
  const int32_t* pair_dst;
  const double* init12;
  double* out12;
  int32_t* status;
  int32_t* n_iters;
  double* stats;
  int stats_stride;
  int batch;
  rk_icp_config cfg;
  unsigned long long* pt_iters;
};

// Per-iteration update by one lane (registration.py:266-282): the 6x6 checks,
// the float64 solve, the twist update and the early-exit test.  Out of line so
// its scratch arrays do not inflate the hot loop's register budget.
// Returns 0 iterate, 1 level done, 2 stop (status set).
__device__ __noinline__ int solve_step(const double* tot, int n_corr, double* pose, int min_corr,
                                       double rot_eps, double trans_eps, int* status) {
  if (n_corr < min_corr) {
    *status = RK_ICP_TOO_FEW;
    return 2;
  }
  double Hm[36], L[36], piv[6], b[6], xi[6];
  int q = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) { Hm[i * 6 + j] = Hm[j * 6 + i] = tot[q]; ++q; }
  for (int i = 0; i < 6; ++i) b[i] = tot[21 + i];
  double dinv[6];
  bool ok = chol6(Hm, L, piv, dinv);
  if (cond_exceeds6(Hm, L, dinv, ok, piv, 1e12)) {
    *status = RK_ICP_DEGENERATE;
    return 2;
  }
  chol_solve6(L, dinv, b, xi);
  double P[12];
  for (int i = 0; i < 12; ++i) P[i] = pose[i];
  se3_left_update(xi, P);
  if (orth_defect(P) > 1e-12) reorthonormalize(P);
  for (int i = 0; i < 12; ++i) pose[i] = P[i];
  const double nr = sqrt(xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
  const double nt = sqrt(xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5]);
  return (nr < rot_eps && nt < trans_eps) ? 1 : 0;
}

// pose <- exp(xi) pose and the early-exit test, by one lane.  Out of line: its
// own register allocation (inlined under the walk's register cap, the float64
// temporaries live across the division / sqrt / sincos slow-path call sites
// were spilled: ~60 local stores and reloads per update)
__device__ __noinline__ int pose_update(double x0, double x1, double x2, double x3, double x4, double x5,
                                        double* pose, double rot_eps, double trans_eps) {
  const double xi[6] = {x0, x1, x2, x3, x4, x5};
  double P[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) P[i] = pose[i];
  se3_left_update(xi, P);
  if (orth_defect(P) > 1e-12) reorthonormalize(P);
#pragma unroll
  for (int i = 0; i < 12; ++i) pose[i] = P[i];
  const double nr = sqrt(xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
  const double nt = sqrt(xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5]);
  return (nr < rot_eps && nt < trans_eps) ? 1 : 0;
}

// The per-iteration update (registration.py:266-282) by one warp: the common
// case -- an SPD system whose condition number the cheap bounds already
// settle -- runs lane-parallel in registers (right-looking Cholesky with one
// lower-triangle entry per lane, L^-1 by per-lane column substitution for the
// trace(H^-1) bound, x = M^T M b), then lane 0 applies the twist.  Anything
// else (non-positive pivot, a condition number inside the bounds' band) takes
// the exact serial solve_step.  Returns the warp-uniform control word.
__device__ __forceinline__ int warp_solve_step(const double* tot, int n_corr, double* pose,
                                               int min_corr, double rot_eps, double trans_eps,
                                               int* status) {
  const int lane = threadIdx.x & 31;
  if (n_corr < min_corr) {
    if (lane == 0) *status = RK_ICP_TOO_FEW;
    return 2;
  }
  // lane t < 21 owns lower entry (li, lj), t = li (li + 1) / 2 + lj
  int li = 0;
  while ((li + 1) * (li + 2) / 2 <= lane) ++li;
  const int lj = lane - li * (li + 1) / 2;
  const bool own = lane < 21;
  // H[li][lj] = upper entry (lj, li) in tot's row-major upper enumeration
  const double h0 = own ? tot[lj * (11 - lj) / 2 + li] : 0.0;
  double a = h0;
  double pmax = 0.0, pmin = 0.0, dinv[6];
  bool ok = true;
  // no early exit: with a break dinv[] lived in local memory (a store and a
  // reload per pivot); after a non-positive pivot the remaining steps run on
  // a dummy pivot and the serial path below decides
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double d = __shfl_sync(0xffffffffu, a, k * (k + 1) / 2 + k);
    ok = ok && d > 0.0;
    if (!ok) d = 1.0;
    pmax = k ? fmax(pmax, d) : d;
    pmin = k ? fmin(pmin, d) : d;
    const double inv = rsqrt(d);
    dinv[k] = inv;
    if (own && lj == k) a = (li == k) ? d * inv : a * inv;
    const int s1 = own && li > k ? li * (li + 1) / 2 + k : 0;
    const int s2 = own && lj > k ? lj * (lj + 1) / 2 + k : 0;
    const double lik = __shfl_sync(0xffffffffu, a, s1);
    const double ljk = __shfl_sync(0xffffffffu, a, s2);
    if (own && lj > k) a = __fma_rn(-lik, ljk, a);
  }
  if (!ok || pmax > 1e12 * pmin) {
    // degenerate for sure (pivot ratio bounds cond from below) or not SPD:
    // the exact serial path decides
    int ctrl = 0;
    if (lane == 0) ctrl = solve_step(tot, n_corr, pose, min_corr, rot_eps, trans_eps, status);
    return __shfl_sync(0xffffffffu, ctrl, 0);
  }
  // ||H||_F^2 (off-diagonal entries twice)
  double fh = own ? (li == lj ? h0 * h0 : 2.0 * h0 * h0) : 0.0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) fh += __shfl_xor_sync(0xffffffffu, fh, off);
  // column j = lane of M = L^-1: M_jj = dinv_j, M_ij = -dinv_i sum_{k=j}^{i-1} L_ik M_kj
  double m[6];
  const int j = lane < 6 ? lane : 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) m[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double acc = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) {
      const double lik = __shfl_sync(0xffffffffu, a, i * (i + 1) / 2 + k);
      if (k >= j) acc = __fma_rn(-lik, m[k], acc);
    }
    m[i] = i >= j ? acc * dinv[i] : 0.0;
  }
  double tr = 0.0;
  if (lane < 6)
#pragma unroll
    for (int i = 0; i < 6; ++i) tr = __fma_rn(m[i], m[i], tr);
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, off);
  // the xor tree sums lanes 0-7 only: broadcast lane 0's total so the branch
  // below is warp-uniform (lanes >= 8 held 0 and would skip the exact
  // fallback while lanes 0-7 take it -- diverged full-mask shuffles, a hang)
  tr = __shfl_sync(0xffffffffu, tr, 0);
  if (!(sqrt(fh) * tr <= 1e12)) {  // inside the bounds' band: exact eigenvalues decide
    int ctrl = 0;
    if (lane == 0) ctrl = solve_step(tot, n_corr, pose, min_corr, rot_eps, trans_eps, status);
    return __shfl_sync(0xffffffffu, ctrl, 0);
  }
  // x = H^-1 b = M^T (M b): y_i = sum_j M_ij b_j over lanes j < 6
  const double bj = lane < 6 ? tot[21 + lane] : 0.0;
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double v = lane < 6 ? m[i] * bj : 0.0;
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    y[i] = v;
  }
  double xj = 0.0;  // lane j: x_j = sum_i M_ij y_i
#pragma unroll
  for (int i = 0; i < 6; ++i) xj = __fma_rn(m[i], y[i], xj);
  double xi[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) xi[i] = __shfl_sync(0xffffffffu, xj, i);
  int ctrl = 0;
  if (lane == 0) ctrl = pose_update(xi[0], xi[1], xi[2], xi[3], xi[4], xi[5], pose, rot_eps, trans_eps);
  return __shfl_sync(0xffffffffu, ctrl, 0);
}

// The warp's 29 per-lane partials (27 normal-equation terms, cost, sum of
// squares) reduced by recursive halving: at each step a lane keeps one half
// of its values and adds the partner's copy of the same half, so after five
// steps lane L holds the warp total of value L.  46 shuffles instead of the
// 290 of 29 separate butterfly sums (the shuffle pipe moves one warp per
// clock per SM).  The first step adds the float32 partials in float32, the
// rest run in float64; the tree is fixed, so the result is deterministic.
// Returns lane L's total (L < 29; lanes 29-31 hold zero padding).
template <bool STATS>
__device__ __forceinline__ double warp_transpose_sum(const float* acc, float cost, float sumsq) {
  const int lane = threadIdx.x & 31;
  auto val = [&](int i) -> float {
    return i < 27 ? acc[i] : (i == 27 ? (STATS ? cost : 0.0f) : (i == 28 ? (STATS ? sumsq : 0.0f) : 0.0f));
  };
  double v[16];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float lo = val(i), hi = val(i + 16);
      const float r = __shfl_xor_sync(0xffffffffu, up ? lo : hi, 16);
      v[i] = (double)__fadd_rn(up ? hi : lo, r);
    }
  }
#pragma unroll
  for (int k = 8; k >= 1; k >>= 1) {
    const bool up = lane & k;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const double r = __shfl_xor_sync(0xffffffffu, up ? v[i] : v[i + k], k);
      v[i] = (up ? v[i + k] : v[i]) + r;
    }
  }
  return v[0];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// association tail + point-to-plane terms of one correspondence
// (registration.py:168-183, 339-352): gate on the stored target, residual,
// Jacobian, pseudo-Huber IRLS weight, 27 float32 accumulations.
// FUSED (K3 in MATH_FAST): the same expressions as FMA chains (~1 ulp, the
// tolerance class of the float32 move); otherwise the reference's separate
// roundings, so MATH_CR associates exactly like the oracle.
// q: the association target {x, y, z} (registration.py:168-176), from the
// surfel pyramid record or formed from the ray tables by the caller.
// EXACT (the exact modes): the IRLS weight is the reference's own float32
// expression w = 1 / sqrt(1 + (r/k)^2) (robust_weight32, registration.py:
// 357-358; IEEE division and square root), so every per-point term equals
// the reference's and only the summation order differs; the IterationStats
// cost term is its 1/w - 1 (registration.py:352), cancellation included.
template <bool STATS, bool FUSED = false, bool EXACT = false>
__device__ __forceinline__ void accumulate_point(float mx, float my, float mz, const float4& n,
                                                 const float4& q, float gate2, float inv_k, float k32,
                                                 float* acc, float& cost, float& sumsq, int& cnt) {
  if (!(n.w > 0.0f)) return;  // stored range > 0 and normal valid
  float dx, dy, dz, d2, res;
  float J[6];
  if (FUSED) {
    dx = __fsub_rn(mx, q.x);
    dy = __fsub_rn(my, q.y);
    dz = __fsub_rn(mz, q.z);
    d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    if (!(d2 <= gate2)) return;
    res = __fmaf_rn(n.z, dz, __fmaf_rn(n.y, dy, __fmul_rn(n.x, dx)));
    J[0] = __fmaf_rn(my, n.z, -__fmul_rn(mz, n.y));
    J[1] = __fmaf_rn(mz, n.x, -__fmul_rn(mx, n.z));
    J[2] = __fmaf_rn(mx, n.y, -__fmul_rn(my, n.x));
  } else {
    dx = __fsub_rn(mx, q.x);
    dy = __fsub_rn(my, q.y);
    dz = __fsub_rn(mz, q.z);
    d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
    if (!(d2 <= gate2)) return;
    // ---- residual, Jacobian, pseudo-Huber IRLS weight (registration.py:339-352).
    // Only the reduced sums matter here (pose tolerance 1e-5), so the
    // weight uses the fast reciprocal square root.
    res = __fadd_rn(__fadd_rn(__fmul_rn(n.x, dx), __fmul_rn(n.y, dy)), __fmul_rn(n.z, dz));
    J[0] = __fsub_rn(__fmul_rn(my, n.z), __fmul_rn(mz, n.y));
    J[1] = __fsub_rn(__fmul_rn(mz, n.x), __fmul_rn(mx, n.z));
    J[2] = __fsub_rn(__fmul_rn(mx, n.y), __fmul_rn(my, n.x));
  }
  J[3] = n.x;
  J[4] = n.y;
  J[5] = n.z;
  float e, s1, w;
  if (EXACT) {
    e = div_rn_fast(res, k32);
    s1 = __fadd_rn(1.0f, __fmul_rn(e, e));
    w = rcp_rn_fast(RK_SQRT_FAST == 2 ? sqrt_rn_normal(s1)
                          : (RK_SQRT_FAST == 1 && s1 < 3.0e38f) ? sqrt_rn_normal(s1) : __fsqrt_rn(s1));  // s1 >= 1
  } else {
    e = res * inv_k;
    s1 = __fmaf_rn(e, e, 1.0f);
    w = rsqrtf(s1);
  }
  const float rw = -res * w;
  int h = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const float jw = J[i] * w;
#pragma unroll
    for (int j = i; j < 6; ++j) { acc[h] = __fmaf_rn(jw, J[j], acc[h]); ++h; }
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) acc[21 + i] = __fmaf_rn(rw, J[i], acc[21 + i]);
  if (STATS) {
    if (EXACT) {
      cost = __fadd_rn(cost, __fsub_rn(rcp_rn_fast(w), 1.0f));
    } else {
      // rho/k^2 = 1/w - 1 = e^2 / (sqrt(1+e^2) + 1), cancellation-free
      cost += __fdividef(e * e, __fmaf_rn(s1, w, 1.0f));
    }
    sumsq = __fmaf_rn(res, res, sumsq);
  }
  ++cnt;
}

template <int MATH, bool SMEM, bool STATS>
__device__ __forceinline__ void associate_moved(const SensorDev& s, const RowTables& tb, float mx,
                                                float my, float mz, const float4* surf, bool lvl_rec,
                                                int stride, int lvl_off, int lvl_w, float inv_s,
                                                float gate2, float inv_k, float k32, float* acc, float& cost,
                                                float& sumsq, int& cnt);

__device__ __forceinline__ void prefetch_line(const void* p) {
  if (RK_ICP_PREFETCH == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
  if (RK_ICP_PREFETCH == 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// float32 unprojection r * dir + origin and rigid move R p + t (FMA chains),
// P = {R row-major, t} in float32
__device__ __forceinline__ void move_f32(const float* P, float r, const float4& d, const float4& o,
                                         float& mx, float& my, float& mz) {
  const float px = __fmaf_rn(r, d.x, o.x), py = __fmaf_rn(r, d.y, o.y), pz = __fmaf_rn(r, d.z, o.z);
  mx = __fmaf_rn(pz, P[2], __fmaf_rn(py, P[1], __fmaf_rn(px, P[0], P[9])));
  my = __fmaf_rn(pz, P[5], __fmaf_rn(py, P[4], __fmaf_rn(px, P[3], P[10])));
  mz = __fmaf_rn(pz, P[8], __fmaf_rn(py, P[7], __fmaf_rn(px, P[6], P[11])));
}

// one source point against the destination (registration.py:145-183): the
// bit-exact float64 unprojection + FMA-chain transform, float32 projection,
// stride-aligned pixel, then accumulate_point.
template <int MATH, bool SMEM, bool STATS>
__device__ __forceinline__ void associate_point(const SensorDev& s, const RowTables& tb,
                                                const double* pose, float r, const double3& dcur,
                                                const double3& ocur, const float4* surf, bool lvl_rec,
                                                int stride, int lvl_off, int lvl_w, float inv_s,
                                                float gate2, float inv_k, float k32, float* acc, float& cost,
                                                float& sumsq, int& cnt) {
  const double rd = (double)r;
  double m[3];
  xform_rows(pose, pose + 9, __dadd_rn(__dmul_rn(rd, dcur.x), ocur.x),
             __dadd_rn(__dmul_rn(rd, dcur.y), ocur.y), __dadd_rn(__dmul_rn(rd, dcur.z), ocur.z), m);
  associate_moved<MATH, SMEM, STATS>(s, tb, (float)m[0], (float)m[1], (float)m[2], surf, lvl_rec, stride, lvl_off,
                                     lvl_w, inv_s, gate2, inv_k, k32, acc, cost, sumsq, cnt);
}

// the association of an already transformed (float32) source point
template <int MATH, bool SMEM, bool STATS>
__device__ __forceinline__ void associate_moved(const SensorDev& s, const RowTables& tb, float mx,
                                                float my, float mz, const float4* surf, bool lvl_rec,
                                                int stride, int lvl_off, int lvl_w, float inv_s,
                                                float gate2, float inv_k, float k32, float* acc, float& cost,
                                                float& sumsq, int& cnt) {
  constexpr int PROJ = MATH == MATH_FAST ? (RK_ICP_ELEV_ONLY ? PROJ_NO_R : PROJ_EXACT) : PROJ_EXACT_FINITE;
  const Proj32 pr = project_f32<MATH, SMEM, PROJ>(s, tb, mx, my, mz);
  if (pr.status != PROJ_OK) return;
  int ci = (int)__fadd_rn(__fmul_rn(pr.u, inv_s), 0.5f);
  if (ci * stride >= s.W) ci = 0;
  const int ri = (int)__fadd_rn(__fmul_rn((float)pr.v, inv_s), 0.5f);
  const int col = ci * stride, row = ri * stride;
  if (row >= s.H) return;  // dropped, not clamped (registration.py:157-159)
  const int flat = row * s.W + col;
  RK_DCHECK(pr.v >= 0 && pr.v < s.H && ci >= 0 && col < s.W && row >= 0, "K3 pixel", pr.v, col);
  RK_DCHECK(!lvl_w || (ci < lvl_w && lvl_off + ri * lvl_w + ci >= lvl_off), "K3 level index", ci, lvl_w);
  constexpr bool FUSED = RK_ICP_FUSED && MATH == MATH_FAST;
  float4 n, q;
  if (lvl_rec && RK_SURFEL_REC == 16) {
    // 16-byte pyramid records {n, range}; the target from the shared ray tables
    const int idx = lvl_w ? lvl_off + ri * lvl_w + ci : flat;
    n = __ldg(surf + idx);
    const float4 d = __ldg(s.dirs32 + flat);
    const float4 o = __ldg(s.origins32 + col);
    if (RK_ICP_PREFETCH && row + RK_ICP_PF_ROWS * stride < s.H) {
      prefetch_line(surf + (lvl_w ? idx + RK_ICP_PF_ROWS * lvl_w : flat + RK_ICP_PF_ROWS * stride * s.W));
      prefetch_line(s.dirs32 + flat + RK_ICP_PF_ROWS * stride * s.W);
    }
    q = make_float4(__fadd_rn(__fmul_rn(n.w, d.x), o.x), __fadd_rn(__fmul_rn(n.w, d.y), o.y),
                    __fadd_rn(__fmul_rn(n.w, d.z), o.z), 0.f);
  } else if (lvl_rec) {
    // RK_SURFEL_REC=32 pyramid: {n, range} + {target} records; the level's
    // compact decimated map (lvl_w > 0) or the full map (level stride 1)
    const int idx = lvl_w ? lvl_off + ri * lvl_w + ci : flat;
    n = __ldg(surf + 2 * idx);
    q = __ldg(surf + 2 * idx + 1);
  } else {
    n = __ldg(surf + flat);
    const float4 d = __ldg(s.dirs32 + flat);
    const float4 o = __ldg(s.origins32 + col);
    // the reference's target (registration.py:168-176), exactly as the
    // pyramid records hold it, so both layouts associate identically
    q = make_float4(__fadd_rn(__fmul_rn(n.w, d.x), o.x), __fadd_rn(__fmul_rn(n.w, d.y), o.y),
                    __fadd_rn(__fmul_rn(n.w, d.z), o.z), 0.f);
  }
  accumulate_point<STATS, FUSED, MATH != MATH_FAST>(mx, my, mz, n, q, gate2, inv_k, k32, acc, cost,
                                                          sumsq, cnt);
}

template <int WPP, int NT>
__device__ __forceinline__ void group_sync(int g) {
  if (WPP == 1) {
    __syncwarp();
  } else if (WPP * 32 == NT) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(WPP * 32) : "memory");
  }
}

// STATS: accumulate the robust cost and squared residuals (IterationStats
// rows); the pose update needs neither, so batch runs without stats skip them.
//
// CL > 1 (latency mode for a handful of pairs): one pair per thread-block
// cluster of CL CTAs.  The point walk spans the cluster (walk index wtid over
// WGT = CL * GT threads); each CTA reduces its slice as usual, then CTA rank 0
// sums the CL partial systems through distributed shared memory in rank
// order (deterministic), solves, and stores the pose and the control word
// into every CTA's shared memory before the cluster barrier.
template <int MATH, int WPP, int MINB, bool SMEM, bool STATS, int NT = kThreads, int CL = 1>
__global__ void __launch_bounds__(NT, MINB) k_register(IcpArgs A) {
  constexpr int NW = NT / 32, GROUPS = NW / WPP, GT = WPP * 32, WGT = GT * CL;
  static_assert(CL == 1 || GROUPS == 1, "a cluster holds one pair");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp / WPP;
  const int gtid = tid - g * GT;
  const int crank = CL > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const bool lead = crank == 0;  // the cluster CTA that solves and writes the outputs
  const int wtid = crank * GT + gtid;
  const int pair = CL > 1 ? (int)(blockIdx.x / CL) : blockIdx.x * GROUPS + g;
  const SensorDev& s = A.s;
  __shared__ RowTablesSmem sh_tab;
  if (SMEM) {
    stage_tables(s, sh_tab, tid, NT);
    __syncthreads();
  }
  if (pair >= A.batch) return;  // whole groups only (no CTA-wide barrier when GROUPS > 1)
  const RowTables tb = SMEM ? RowTables{sh_tab.el32, sh_tab.az32, sh_tab.inv_rows} : global_tables(s);
  const int H = s.H, W = s.W;
  const size_t HW = (size_t)H * W;
  const int ps = A.pair_src[pair], pd = A.pair_dst[pair];
  if ((A.cfg.n_src_images > 0 && (unsigned)ps >= (unsigned)A.cfg.n_src_images) ||
      (A.cfg.n_dst_images > 0 && (unsigned)pd >= (unsigned)A.cfg.n_dst_images)) {
    // an index outside the pools: no reads, a defined result (group-uniform exit)
    if (lead && gtid < 12) A.out12[pair * 12 + gtid] = A.init12[pair * 12 + gtid];
    if (lead && gtid == 0) {
      A.status[pair] = RK_ICP_BAD_PAIR;
      A.n_iters[pair] = 0;
    }
    return;
  }
  const float* src = A.src_range + (size_t)ps * HW;
  // a surfel pyramid (surfel_pitch != 0) holds RK_SURFEL_REC-byte records {n, range}(, {target});
  // {target}; a plain surfel map 16-byte {n, range}
  const bool rec = A.cfg.surfel_pitch != 0;
  const long long surf_pitch = rec ? (RK_SURFEL_REC / 16) * A.cfg.surfel_pitch : (long long)HW;
  const float4* surf = A.dst_surfel + (size_t)pd * surf_pitch;

  __shared__ double sh_pose[GROUPS][12];
  __shared__ double sh_red[NW][kNumAcc];
  __shared__ double sh_tot[GROUPS][kNumAcc];
  // CL > 1: the cluster's partial systems.  RK_ICP_CLUSTER_REDUNDANT: every
  // CTA receives all CL partials (double-buffered by iteration parity) and
  // solves the update itself; otherwise the lead CTA alone receives them
  constexpr int NPART = RK_ICP_CLUSTER_REDUNDANT ? 2 : 1;
  __shared__ double sh_part[NPART][CL][kNumAcc + 1];
  int parity = 0;
  __shared__ int sh_cnt[NW];
  __shared__ int sh_ctrl[GROUPS];
  __shared__ float sh_pose32[GROUPS][12];
  __shared__ float4 sh_lvl[GROUPS][2];  // RK_ICP_LVL_SMEM: {gate2, 1/k, 1/s, stride}, {level off, level w}
  __shared__ const float4* sh_surf[GROUPS];  // RK_ICP_LVL_SMEM: this pair's surfel base
  if (gtid < 12) sh_pose[g][gtid] = A.init12[pair * 12 + gtid];
  int n_done = 0, status = RK_ICP_CONVERGED;
#if RK_ICP_TIME_SOLVE
  long long t_solve_acc = 0;
  const long long t_kernel0 = clock64();
#endif
  unsigned work = 0;  // valid source points visited (all iterations), per thread
  const float cmin = A.cfg.clip_min, cmax = A.cfg.clip_max;

  for (int lv = 0; lv < A.cfg.n_levels; ++lv) {
    const int stride = A.cfg.strides[lv];
    const double level = A.cfg.scale_with_stride ? (double)stride : 1.0;
    const double kern = A.cfg.kernel_scale * level;
    const float gate32 = (float)(A.cfg.max_dist * level);
    const float gate2 = __fmul_rn(gate32, gate32);
    const float inv_k = (float)(1.0 / kern);
    const float k32 = (float)kern;  // np.float32(kernel_scale) (registration.py:350)
    const float inv_s = (float)(1.0 / stride);
    const int Hs = (H + stride - 1) / stride, Ws = (W + stride - 1) / stride;
    const int npix = Hs * Ws;
    // row-major walk of the stride view (the reference's zero-copy StridedView,
    // range_image.py:69-116) by GT-point steps, as running pixel offsets:
    // one step advances (dv rows, du view columns), wrapping at Ws
    const int dv = WGT / Ws, du = WGT - dv * Ws;
    const int step_off = dv * stride * W + du * stride;
    const int wrap_off = stride * W - Ws * stride;
    const int vi0 = wtid / Ws, ui0 = wtid - vi0 * Ws;
    const int off0 = vi0 * stride * W + ui0 * stride;
    const bool col_mode = Ws % WGT == 0;
    const int lvl_off = A.cfg.surfel_pitch ? A.cfg.surfel_level_off[lv] : 0;
    const int lvl_w = (A.cfg.surfel_pitch && lvl_off > 0) ? Ws : 0;
    const int row_step = stride * W;
    if (RK_ICP_LVL_SMEM && gtid == 0) {
      sh_lvl[g][0] = make_float4(gate2, inv_k, inv_s, __int_as_float(stride));
      sh_lvl[g][1] = make_float4(__int_as_float(lvl_off), __int_as_float(lvl_w), k32, 0.f);
      sh_surf[g] = surf;
    }
    // executed work (the roofline's unit) = valid points of this level x the
    // iterations run; counted once per level, outside the hot loop
    unsigned valid_lv = 0;
    if (A.pt_iters) {
      int off = off0, ui = ui0;
      for (int k = wtid; k < npix; k += WGT) {
        valid_lv += range_ok(__ldg(src + off), cmin, cmax) ? 1u : 0u;
        off += step_off;
        ui += du;
        if (ui >= Ws) { ui -= Ws; off += wrap_off; }
      }
    }
    int executed = 0;
    for (int it = 0; it < A.cfg.iters[lv]; ++it) {
      ++executed;
      group_sync<WPP, NT>(g);  // pose (and sh_ctrl reuse) ready
      // the pose is read from shared memory at every use (broadcast LDS):
      // holding it in registers would cost 24 of the registers the occupancy allows
      const double* pose = sh_pose[g];
      float acc[27];
#pragma unroll
      for (int i = 0; i < 27; ++i) acc[i] = 0.0f;
      float cost = 0.0f, sumsq = 0.0f;
      int cnt = 0;
      // FAST: the source point is unprojected and moved in float32 with FMAs
      // from the float32 ray tables and a float32 copy of the pose (a few ulp
      // from the reference's float64-then-round point; tolerance contract,
      // DESIGN.md §4).  CR keeps the bit-exact float64 restatement.
      constexpr bool F32X = RK_ICP_F32X && MATH == MATH_FAST;
      const float* P = sh_pose32[g];
      if (F32X) {
        if (gtid < 12) sh_pose32[g][gtid] = (float)pose[gtid];
        group_sync<WPP, NT>(g);
      }
      if (F32X && col_mode) {
        for (int cj = wtid; cj < Ws; cj += WGT) {
          const int u = cj * stride;
          const float4 o4 = __ldg(s.origins32 + u);
          const float* sp = src + u;
          const float4* dp = s.dirs32 + u;
          float r_next = __ldg(sp);
          float4 d_next = __ldg(dp);
          for (int vi = 0; vi < Hs; ++vi) {
            const float r = r_next;
            const float4 d4 = d_next;
            sp += row_step;
            dp += row_step;
            if (vi + 1 < Hs) {
              r_next = __ldg(sp);
              d_next = __ldg(dp);
            }
            if (!range_ok(r, cmin, cmax)) continue;
            float mx, my, mz;
            move_f32(P, r, d4, o4, mx, my, mz);
            if (RK_ICP_LVL_SMEM) {
              const float4 L0 = sh_lvl[g][0], L1 = sh_lvl[g][1];
              associate_moved<MATH, SMEM, STATS>(s, tb, mx, my, mz, sh_surf[g], rec, __float_as_int(L0.w),
                                                 __float_as_int(L1.x), __float_as_int(L1.y), L0.z, L0.x,
                                                 L0.y, L1.z, acc, cost, sumsq, cnt);
            } else {
              associate_moved<MATH, SMEM, STATS>(s, tb, mx, my, mz, surf, rec, stride, lvl_off, lvl_w, inv_s,
                                                 gate2, inv_k, k32, acc, cost, sumsq, cnt);
            }
          }
        }
      } else if (F32X) {
        // generic row-major walk, float32 transform
        int off = off0, ui = ui0;
        for (int k = wtid; k < npix; k += WGT) {
          const float r = __ldg(src + off);
          const float4 d4 = __ldg(s.dirs32 + off);
          const int u = ui * stride;
          off += step_off;
          ui += du;
          if (ui >= Ws) { ui -= Ws; off += wrap_off; }
          if (!range_ok(r, cmin, cmax)) continue;
          float mx, my, mz;
          move_f32(P, r, d4, __ldg(s.origins32 + u), mx, my, mz);
          associate_moved<MATH, SMEM, STATS>(s, tb, mx, my, mz, surf, rec, stride, lvl_off, lvl_w, inv_s,
                                             gate2, inv_k, k32, acc, cost, sumsq, cnt);
        }
      } else if (col_mode && RK_ICP_F64_AHEAD) {
        // column-owner walk (Ws % GT == 0): each lane owns view columns
        // gtid, gtid + GT, ... and walks them down the rows with a constant
        // pointer step; the receiver origin depends on the column only
        for (int cj = wtid; cj < Ws; cj += WGT) {
          const int u = cj * stride;
          const double3 ocur = make_double3(__ldg(s.origins + 3 * u), __ldg(s.origins + 3 * u + 1),
                                            __ldg(s.origins + 3 * u + 2));
          const float* sp = src + u;
          const double* dp = s.dirs + 3 * (size_t)u;
          float r_next = __ldg(sp);
          double3 d_next = make_double3(__ldg(dp), __ldg(dp + 1), __ldg(dp + 2));
          for (int vi = 0; vi < Hs; ++vi) {
            const float r = r_next;
            const double3 dcur = d_next;
            RK_DCHECK(sp >= src && sp < src + HW, "K3 source walk", (long long)(sp - src), (long long)HW);
            sp += row_step;
            dp += 3 * (size_t)row_step;
            if (vi + 1 < Hs) {  // next row's range and ray, one point ahead
              r_next = __ldg(sp);
              d_next = make_double3(__ldg(dp), __ldg(dp + 1), __ldg(dp + 2));
            }
            if (!range_ok(r, cmin, cmax)) continue;
            if (RK_ICP_LVL_SMEM) {
              // the level constants from shared memory (under the register
              // cap the compiler would otherwise re-derive them per point)
              const float4 L0 = sh_lvl[g][0], L1 = sh_lvl[g][1];
              associate_point<MATH, SMEM, STATS>(s, tb, pose, r, dcur, ocur, sh_surf[g], rec,
                                                 __float_as_int(L0.w), __float_as_int(L1.x),
                                                 __float_as_int(L1.y), L0.z, L0.x, L0.y, L1.z, acc, cost,
                                                 sumsq, cnt);
            } else {
              associate_point<MATH, SMEM, STATS>(s, tb, pose, r, dcur, ocur, surf, rec, stride, lvl_off,
                                                 lvl_w, inv_s, gate2, inv_k, k32, acc, cost, sumsq, cnt);
            }
          }
        }
      } else if (col_mode) {
        // the same walk with the float64 ray and receiver origin loaded at
        // use (L1 hits) instead of held in registers a row ahead: under the
        // 64-register cap the held float64 values spill
        for (int cj = wtid; cj < Ws; cj += WGT) {
          const int u = cj * stride;
          const float* sp = src + u;
          const double* dp = s.dirs + 3 * (size_t)u;
          float r_next = __ldg(sp);
          for (int vi = 0; vi < Hs; ++vi) {
            const float r = r_next;
            const double* dcp = dp;
            sp += row_step;
            dp += 3 * (size_t)row_step;
            if (vi + 1 < Hs) r_next = __ldg(sp);
            if (!range_ok(r, cmin, cmax)) continue;
            const double3 dcur = make_double3(__ldg(dcp), __ldg(dcp + 1), __ldg(dcp + 2));
            const double3 ocur = make_double3(__ldg(s.origins + 3 * u), __ldg(s.origins + 3 * u + 1),
                                              __ldg(s.origins + 3 * u + 2));
            associate_point<MATH, SMEM, STATS>(s, tb, pose, r, dcur, ocur, surf, rec, stride, lvl_off,
                                               lvl_w, inv_s, gate2, inv_k, k32, acc, cost, sumsq, cnt);
          }
        }
      } else {
        // generic row-major walk of the stride view by GT-point steps
        int off = off0, ui = ui0;
        float r_next = 0.0f;
        double3 d_next = make_double3(0.0, 0.0, 0.0);
        if (wtid < npix) {
          r_next = __ldg(src + off);
          const double* dp = s.dirs + 3 * (size_t)off;
          d_next = make_double3(__ldg(dp), __ldg(dp + 1), __ldg(dp + 2));
        }
        for (int k = wtid; k < npix; k += WGT) {
          const float r = r_next;
          const double3 dcur = d_next;
          const int u = ui * stride;
          off += step_off;
          ui += du;
          if (ui >= Ws) { ui -= Ws; off += wrap_off; }
          if (k + WGT < npix) {
            r_next = __ldg(src + off);
            const double* dp = s.dirs + 3 * (size_t)off;
            d_next = make_double3(__ldg(dp), __ldg(dp + 1), __ldg(dp + 2));
          }
          if (!range_ok(r, cmin, cmax)) continue;
          const double3 ocur = make_double3(__ldg(s.origins + 3 * u), __ldg(s.origins + 3 * u + 1),
                                            __ldg(s.origins + 3 * u + 2));
          associate_point<MATH, SMEM, STATS>(s, tb, pose, r, dcur, ocur, surf, rec, stride, lvl_off,
                                             lvl_w, inv_s, gate2, inv_k, k32, acc, cost, sumsq, cnt);
        }
      }
      // ---- deterministic group reduction in float64
      double* tot = sh_tot[g];
      if (!RK_ICP_TRANSPOSE) {
#pragma unroll
        for (int i = 0; i < 27; ++i) {
          const double v = warp_sum((double)acc[i]);
          if (lane == 0) sh_red[warp][i] = v;
        }
        const double c = warp_sum((double)cost), q2 = warp_sum((double)sumsq);
        const int nc = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) {
          sh_red[warp][27] = c;
          sh_red[warp][28] = q2;
          sh_cnt[warp] = nc;
        }
        if (WPP == 1 && lane < kNumAcc) tot[lane] = sh_red[warp][lane];
        if (WPP > 1) {
          group_sync<WPP, NT>(g);
          if (gtid < kNumAcc) {
            double t = 0.0;
            for (int w2 = 0; w2 < WPP; ++w2) t += sh_red[g * WPP + w2][gtid];
            tot[gtid] = t;
          }
          if (gtid == 0)
            for (int w2 = 1; w2 < WPP; ++w2) sh_cnt[g * WPP] += sh_cnt[g * WPP + w2];
        }
      } else if (WPP == 1) {
        const double v = warp_transpose_sum<STATS>(acc, cost, sumsq);
        const int nc = __reduce_add_sync(0xffffffffu, cnt);
        if (lane < kNumAcc) tot[lane] = v;
        if (lane == 0) sh_cnt[warp] = nc;
      } else {
        const double v = warp_transpose_sum<STATS>(acc, cost, sumsq);
        const int nc = __reduce_add_sync(0xffffffffu, cnt);
        if (lane < kNumAcc) sh_red[warp][lane] = v;
        if (lane == 0) sh_cnt[warp] = nc;
        group_sync<WPP, NT>(g);
        if (gtid < kNumAcc) {
          double t = 0.0;
          for (int w2 = 0; w2 < WPP; ++w2) t += sh_red[g * WPP + w2][gtid];
          tot[gtid] = t;
        }
        if (gtid == 0)
          for (int w2 = 1; w2 < WPP; ++w2) sh_cnt[g * WPP] += sh_cnt[g * WPP + w2];
      }
      group_sync<WPP, NT>(g);
      if (CL > 1 && RK_ICP_CLUSTER_REDUNDANT) {
        // every CTA stores its partial system into slot [crank] of every
        // CTA's buffer for this iteration's parity (posted DSMEM stores), one
        // cluster barrier publishes them, and every CTA sums the CL partials
        // in rank order -- the lead's sum, bit for bit -- and solves the
        // update itself: no pose broadcast, no second barrier.  A buffer is
        // rewritten two iterations later, after the next barrier, which no
        // CTA passes before every CTA has read it.
        cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
        if (gtid <= kNumAcc) {
          const double v = gtid < kNumAcc ? tot[gtid] : (double)sh_cnt[0];
#pragma unroll
          for (int r = 0; r < CL; ++r)
            cl.map_shared_rank(&sh_part[parity][0][0], r)[crank * (kNumAcc + 1) + gtid] = v;
        }
        cl.sync();
        if (gtid < kNumAcc) {
          double t = sh_part[parity][0][gtid];
          for (int r = 1; r < CL; ++r) t += sh_part[parity][r][gtid];
          tot[gtid] = t;
        } else if (gtid == kNumAcc) {
          int c = (int)sh_part[parity][0][kNumAcc];
          for (int r = 1; r < CL; ++r) c += (int)sh_part[parity][r][kNumAcc];
          sh_cnt[0] = c;
        }
        parity ^= 1;
        group_sync<WPP, NT>(g);
      } else if (CL > 1) {
        // the cluster's partial systems -> the lead CTA: every other CTA
        // stores its partial into the lead's shared memory (posted DSMEM
        // stores, no round trips), the cluster barrier publishes them, and
        // the lead sums them in rank order (deterministic)
        cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
        if (!lead && gtid <= kNumAcc) {
          if (gtid < kNumAcc)
            cl.map_shared_rank(&sh_part[0][0][0], 0)[crank * (kNumAcc + 1) + gtid] = tot[gtid];
          else
            cl.map_shared_rank(&sh_part[0][0][0], 0)[crank * (kNumAcc + 1) + kNumAcc] = (double)sh_cnt[0];
        }
        cl.sync();
        if (lead && gtid <= kNumAcc) {
          if (gtid < kNumAcc) {
            double t = tot[gtid];
            for (int r = 1; r < CL; ++r) t += sh_part[0][r][gtid];
            tot[gtid] = t;
          } else {
            int c = sh_cnt[0];
            for (int r = 1; r < CL; ++r) c += (int)sh_part[0][r][kNumAcc];
            sh_cnt[0] = c;
          }
        }
        group_sync<WPP, NT>(g);
      }
#if RK_ICP_TRACE
      if (gtid == 0) printf("pair %d lv %d it %d reduced n %d\n", pair, lv, it, sh_cnt[g * WPP]);
#endif
      // the group's first warp updates the pose (in a cluster: every CTA's
      // first warp with RK_ICP_CLUSTER_REDUNDANT, else the lead's)
      if ((lead || (CL > 1 && RK_ICP_CLUSTER_REDUNDANT)) && gtid < 32) {
        const int n_corr = sh_cnt[g * WPP];
        // (cfg fields by value: taking a kernel parameter's address would
        // spill the whole argument block to local memory)
#if RK_ICP_TIME_SOLVE
        const long long t_solve0 = clock64();
#endif
#if RK_ICP_SERIAL_SOLVE
        int ctrl = 0;
        if (gtid == 0) ctrl = solve_step(tot, n_corr, sh_pose[g], A.cfg.min_corr, A.cfg.rot_eps,
                                         A.cfg.trans_eps, &status);
#else
        const int ctrl = warp_solve_step(tot, n_corr, sh_pose[g], A.cfg.min_corr, A.cfg.rot_eps,
                                         A.cfg.trans_eps, &status);
#endif
#if RK_ICP_TIME_SOLVE
        t_solve_acc += clock64() - t_solve0;
#endif
        if (gtid == 0) {
          if (ctrl != 2) {
            if (lead && A.stats && n_done < A.stats_stride) {
              double* row = A.stats + ((size_t)pair * A.stats_stride + n_done) * 5;
              row[0] = stride;
              row[1] = it;
              row[2] = n_corr;
              row[3] = kern * kern * tot[27];
              row[4] = sqrt(tot[28] / n_corr);
            }
            ++n_done;
          }
          sh_ctrl[g] = ctrl;
        }
        if (CL > 1 && !RK_ICP_CLUSTER_REDUNDANT) {
          // broadcast the pose and the control word to the other CTAs
          __syncwarp();
          cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
          for (int r = 1; r < CL; ++r) {
            if (gtid < 12) cl.map_shared_rank(&sh_pose[0][0], r)[gtid] = sh_pose[0][gtid];
            if (gtid == 12) cl.map_shared_rank(&sh_ctrl[0], r)[0] = sh_ctrl[0];
          }
        }
      }
      if (CL > 1 && !RK_ICP_CLUSTER_REDUNDANT)
        cooperative_groups::this_cluster().sync();
      else
        group_sync<WPP, NT>(g);
      const int ctrl = sh_ctrl[g];
#if RK_ICP_TRACE
      if (gtid == 0) printf("pair %d lv %d it %d n %d ctrl %d t %.6f %.6f %.6f\n", pair, lv, it, sh_cnt[g * WPP], ctrl,
                            sh_pose[g][9], sh_pose[g][10], sh_pose[g][11]);
#endif
      if (ctrl == 2) {
        work += valid_lv * executed;
        goto finish;
      }
      if (ctrl == 1) break;
    }
    work += valid_lv * executed;
  }
finish:
#if RK_ICP_TIME_SOLVE
  if (gtid == 0 && pair < 4)
    printf("pair %d: solve %lld cycles of %lld total, %d iterations\n", pair, t_solve_acc,
           clock64() - t_kernel0, n_done);
#endif
  if (A.pt_iters) {
    const unsigned w = __reduce_add_sync(0xffffffffu, work);
    if (lane == 0 && w) atomicAdd(A.pt_iters, (unsigned long long)w);
  }
  group_sync<WPP, NT>(g);
  if (lead && gtid < 12) A.out12[pair * 12 + gtid] = sh_pose[g][gtid];
  if (lead && gtid == 0) {
    A.status[pair] = status;
    A.n_iters[pair] = n_done;
  }
}

// Shared-memory carveout: the driver's default gave the 256-thread K3 a
// 64 KB shared configuration for its ~28 KB of CTAs (3 x 9.4 KB).  Ask for
// just what MINB resident CTAs need (rounded up by the driver to the next
// supported configuration), so the rest of the SM's 256 KB serves L1 and the
// surfel gathers: NP +1.0 % (A/B x2; a 0 % hint collapses occupancy, -54 %).
#ifndef RK_ICP_CARVEOUT
#define RK_ICP_CARVEOUT 1
#endif
template <typename K>
void set_carveout(K kernel, int ctas_per_sm) {
  if (!RK_ICP_CARVEOUT) return;
  cudaFuncAttributes fa;
  int dev = 0, max_sm = 0;
  if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&max_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess ||
      max_sm <= 0) {
    cudaGetLastError();
    return;
  }
  const long long need = (long long)ctas_per_sm * ((long long)fa.sharedSizeBytes + 1024);  // + reserved per CTA
  const int pct = (int)((need * 100 + max_sm - 1) / max_sm) + 1;
  if (pct < 100) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
}

template <int MATH, int WPP, int MINB, int NT = kThreads>
int launch(const IcpArgs& a, cudaStream_t st) {
  constexpr int GROUPS = NT / 32 / WPP;
  const unsigned grid = (unsigned)((a.batch + GROUPS - 1) / GROUPS);
  const bool smem = a.s.H <= kMaxRowsSmem && a.s.K <= kMaxInvSmem;
  static bool carve = false;  // per instantiation (one device: the hint is per function)
  if (!carve) {
    set_carveout(k_register<MATH, WPP, MINB, true, true, NT>, MINB);
    set_carveout(k_register<MATH, WPP, MINB, false, true, NT>, MINB);
    set_carveout(k_register<MATH, WPP, MINB, true, false, NT>, MINB);
    set_carveout(k_register<MATH, WPP, MINB, false, false, NT>, MINB);
    carve = true;
  }
  if (a.stats) {
    if (smem)
      k_register<MATH, WPP, MINB, true, true, NT><<<grid, NT, 0, st>>>(a);
    else
      k_register<MATH, WPP, MINB, false, true, NT><<<grid, NT, 0, st>>>(a);
  } else {
    if (smem)
      k_register<MATH, WPP, MINB, true, false, NT><<<grid, NT, 0, st>>>(a);
    else
      k_register<MATH, WPP, MINB, false, false, NT><<<grid, NT, 0, st>>>(a);
  }
  RK_LAUNCHED("k_register");
  return RK_OK;
}

// latency mode over clusters: CL CTAs of NT threads per pair
template <int CL, int NT = kWide>
cudaLaunchConfig_t cluster_config(int batch, cudaStream_t st, cudaLaunchAttribute* at) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)batch * CL);
  lc.blockDim = dim3(NT);
  lc.dynamicSmemBytes = 0;
  lc.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return lc;
}

// how many CL-CTA clusters are co-resident on this device (GPC packing:
// 148 SMs do not hold 18 clusters of 8 full-SM CTAs); cached per device
// clusters above the portable size 8 need the per-kernel opt-in
template <int MATH, int CL, int NT = kWide>
void allow_cluster_size() {
  if (CL <= 8) return;
  constexpr int WPP = NT / 32;
  cudaFuncSetAttribute(k_register<MATH, WPP, 1, true, true, NT, CL>,
                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_register<MATH, WPP, 1, false, true, NT, CL>,
                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_register<MATH, WPP, 1, true, false, NT, CL>,
                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_register<MATH, WPP, 1, false, false, NT, CL>,
                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

template <int MATH, int CL>
int max_active_clusters() {
  constexpr int NT = lat_nt<MATH>();
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  if (!cache[dev]) {
    allow_cluster_size<MATH, CL, NT>();
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t lc = cluster_config<CL, NT>(1, nullptr, at);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_register<MATH, NT / 32, 1, true, false, NT, CL>, &lc) !=
            cudaSuccess || n < 1) {
      cudaGetLastError();
      n = -1;  // clusters unavailable: never chosen
    }
    cache[dev] = n;
  }
  return cache[dev];
}

template <int MATH, int CL, int NT = kWide>
int launch_cluster(const IcpArgs& a, cudaStream_t st) {
  constexpr int WPP = NT / 32;
  const bool smem = a.s.H <= kMaxRowsSmem && a.s.K <= kMaxInvSmem;
  if (CL > 8) {
    static bool allowed[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !allowed[dev]) {
      allow_cluster_size<MATH, CL, NT>();
      allowed[dev] = true;
    }
  }
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t lc = cluster_config<CL, NT>(a.batch, st, at);
  cudaError_t e;
  if (a.stats)
    e = smem ? cudaLaunchKernelEx(&lc, k_register<MATH, WPP, 1, true, true, NT, CL>, a)
             : cudaLaunchKernelEx(&lc, k_register<MATH, WPP, 1, false, true, NT, CL>, a);
  else
    e = smem ? cudaLaunchKernelEx(&lc, k_register<MATH, WPP, 1, true, false, NT, CL>, a)
             : cudaLaunchKernelEx(&lc, k_register<MATH, WPP, 1, false, false, NT, CL>, a);
  if (e != cudaSuccess) return rk_cuda_status(e, "k_register (cluster)");
  RK_LAUNCHED("k_register");
  return RK_OK;
}

// SMs of the current device (cached per device)
int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// tier selection by batch size (the latency modes for batches that cannot
// fill the GPU with 256-thread CTAs)
template <int MATH>
int launch_tiers(const IcpArgs& a, cudaStream_t st, const char* force, int wpp) {
  constexpr int MINB = MATH == MATH_FAST ? RK_ICP_MINB : RK_ICP_MINB_NP;
  constexpr int WFULL = kThreads / 32;
  constexpr int LNT = lat_nt<MATH>();
  const int batch = a.batch;
  // latency mode: a batch that cannot fill the GPU with 256-thread CTAs
  // (online odometry, one register() call, a short sequence) runs each pair
  // on a 1024-thread CTA (<= one pair per SM) or a 512-thread CTA (<= two):
  // more warps per pair to hide the gather latency
  const char* wide = getenv("RK_ICP_WIDE");
  const char* fnt = getenv("RK_ICP_NT");  // experiment knob: force the CTA size
  if (!force && fnt) {
    const int nt = atoi(fnt);
    if (nt == 1024) return launch<MATH, kWide / 32, 1, kWide>(a, st);
    if (nt == 512) return launch<MATH, kWide / 64, 2, kWide / 2>(a, st);
  }
  if (!force && (!wide || atoi(wide))) {
    // a few pairs: a cluster of CTAs per pair (RK_ICP_CLUSTER=0 disables,
    // =2|4|8 forces the size)
    const char* fcl = getenv("RK_ICP_CLUSTER");
    const int want = fcl ? atoi(fcl) : -1;
    if (want != 0) {
      // the largest cluster whose batch fits in one wave of co-resident
      // clusters (cudaOccupancyMaxActiveClusters; B200, 512-thread CTAs:
      // 7 x16, 15 x8, 33 x4, 74 x2); x4 up to two such waves (the query is
      // conservative for x4 -- 37 pairs ran in one wave, 0.86 ms against
      // x2's 1.40 -- and even two waves of x4 beat x2), and x2 up to 2.75
      // pairs per SM: its waves still beat one wide CTA per pair or the
      // throughput kernel (99 pairs 1.86 vs 2.46 ms, 149: 2.17 vs 4.00,
      // 296: 3.97 vs 4.52, 400: 4.90 vs 5.12; at 444 the throughput kernel
      // wins, 5.53 vs 5.72; scripts/cluster_latency.py, tier_probe.py)
      const int cl = want > 0 ? want
                              : (RK_ICP_CLUSTER16 && batch <= max_active_clusters<MATH, 16>() ? 16
                                 : batch <= max_active_clusters<MATH, 8>()   ? 8
                                 : batch <= 2 * max_active_clusters<MATH, 4>() ? 4
                                 : (batch <= max_active_clusters<MATH, 2>() ||
                                    (max_active_clusters<MATH, 2>() > 0 && 4 * batch <= 11 * sm_count()))
                                     ? 2
                                     : 1);
      if (cl == 16) return launch_cluster<MATH, 16, LNT>(a, st);
      if (cl == 8) return launch_cluster<MATH, 8, LNT>(a, st);
      if (cl == 4) return launch_cluster<MATH, 4, LNT>(a, st);
      if (cl == 2) return launch_cluster<MATH, 2, LNT>(a, st);
    }
    if (batch <= sm_count()) return launch<MATH, LNT / 32, 1, LNT>(a, st);
    if (batch <= 2 * sm_count()) return launch<MATH, LNT / 64, 2, LNT / 2>(a, st);
  }
  if constexpr (MATH == MATH_FAST) {  // experiment layouts (RK_ICP_WPP), FAST only
    switch (wpp) {
      case 1: return launch<MATH, 1, MINB>(a, st);
      case 2: return launch<MATH, 2, MINB>(a, st);
      case 4: return launch<MATH, 4, MINB>(a, st);
      default: break;
    }
  }
  return launch<MATH, WFULL, MINB>(a, st);
}

}  // namespace


// diagnostic: co-resident clusters of cl CTAs the launcher assumes (the
// occupancy query, cached per device); -1 when clusters are unavailable
extern "C" int rk_icp_cluster_capacity(int math, int cl) {
  if (math == MATH_NP) {
    if (cl == 16) return max_active_clusters<MATH_NP, 16>();
    if (cl == 8) return max_active_clusters<MATH_NP, 8>();
    if (cl == 4) return max_active_clusters<MATH_NP, 4>();
    if (cl == 2) return max_active_clusters<MATH_NP, 2>();
  } else {
    if (cl == 16) return max_active_clusters<MATH_FAST, 16>();
    if (cl == 8) return max_active_clusters<MATH_FAST, 8>();
    if (cl == 4) return max_active_clusters<MATH_FAST, 4>();
    if (cl == 2) return max_active_clusters<MATH_FAST, 2>();
  }
  return -1;
}

extern "C" int rk_register_batch(const rk_sensor* s, const float* src_range, const float* dst_range,
                                 const float* dst_surfel, const int32_t* pair_src,
                                 const int32_t* pair_dst, int32_t batch, const double* init12,
                                 const rk_icp_config* cfg, double* out12, int32_t* status,
                                 int32_t* n_iters, double* stats, int32_t stats_stride,
                                 unsigned long long* pt_iters, void* stream) {
  (void)dst_range;  // the surfel map carries the stored range of every valid pixel
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
  a.dst_surfel = reinterpret_cast<const float4*>(dst_surfel);
  a.pair_src = pair_src;
  a.pair_dst = pair_dst;
  a.init12 = init12;
  a.out12 = out12;
  a.status = status;
  a.n_iters = n_iters;
  a.stats = stats;
  a.stats_stride = stats ? stats_stride : 0;
  a.batch = batch;
  a.cfg = *cfg;
  a.pt_iters = pt_iters;
  // CTA-per-pair (WPP = 8 at 256 threads) measured fastest on B200 (DESIGN.md
  // §3: 4 warps per pair -23%, 2 -25%): fewer distinct pairs per SM keep each
  // pair's surfel gathers L1/L2-local.  RK_ICP_WPP=1|2|4 selects the other
  // layouts for experiments.
  const char* force = getenv("RK_ICP_WPP");
  const int wpp = force ? atoi(force) : kThreads / 32;
  cudaStream_t st = S(stream);
  constexpr int MINB = RK_ICP_MINB;
  constexpr int WFULL = kThreads / 32;
  (void)wpp;
  if (cfg->math == MATH_CR)
    return wpp == 1 ? launch<MATH_CR, 1, MINB>(a, st) : launch<MATH_CR, WFULL, MINB>(a, st);
  if (cfg->math == MATH_NP) return launch_tiers<MATH_NP>(a, st, force, wpp);
  return launch_tiers<MATH_FAST>(a, st, force, wpp);
}
