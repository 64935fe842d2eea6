// rk_linalg.cuh -- tiny float64 linear algebra for the per-pair ICP update
// (registration.py:266-282 and se3.py:22-102), run by one thread per pair.
#pragma once
#include <cuda_runtime.h>

namespace rk {

// Cholesky H = L L^T (6x6, row-major); dinv = 1 / diag(L), piv = diag(L)^2.
// Returns false on a non-positive pivot.  Reciprocal diagonals keep the
// single-lane solve to six float64 divisions.
__device__ inline bool chol6(const double* A, double* L, double* piv, double* dinv) {
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  for (int j = 0; j < 6; ++j) {
    double d = A[j * 6 + j];
    for (int k = 0; k < j; ++k) d -= L[j * 6 + k] * L[j * 6 + k];
    if (!(d > 0.0)) return false;
    piv[j] = d;
    const double ljj = sqrt(d);
    const double inv = 1.0 / ljj;
    L[j * 6 + j] = ljj;
    dinv[j] = inv;
    for (int i = j + 1; i < 6; ++i) {
      double s = A[i * 6 + j];
      for (int k = 0; k < j; ++k) s -= L[i * 6 + k] * L[j * 6 + k];
      L[i * 6 + j] = s * inv;
    }
  }
  return true;
}

__device__ inline void chol_solve6(const double* L, const double* dinv, const double* b, double* x) {
  double y[6];
  for (int i = 0; i < 6; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[i * 6 + k] * y[k];
    y[i] = s * dinv[i];
  }
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 6; ++k) s -= L[k * 6 + i] * x[k];
    x[i] = s * dinv[i];
  }
}

// eigenvalues of a symmetric 6x6 by cyclic Jacobi (the exact fallback for cond)
__device__ inline void jacobi_eig6(const double* A, double* ev) {
  double a[36];
  for (int i = 0; i < 36; ++i) a[i] = A[i];
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < 6; ++p) {
      diag += a[p * 6 + p] * a[p * 6 + p];
      for (int q = p + 1; q < 6; ++q) off += a[p * 6 + q] * a[p * 6 + q];
    }
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int p = 0; p < 5; ++p)
      for (int q = p + 1; q < 6; ++q) {
        double apq = a[p * 6 + q];
        if (apq == 0.0) continue;
        double theta = (a[q * 6 + q] - a[p * 6 + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 6; ++k) {  // columns p, q
          double akp = a[k * 6 + p], akq = a[k * 6 + q];
          a[k * 6 + p] = c * akp - s * akq;
          a[k * 6 + q] = s * akp + c * akq;
        }
        for (int k = 0; k < 6; ++k) {  // rows p, q
          double apk = a[p * 6 + k], aqk = a[q * 6 + k];
          a[p * 6 + k] = c * apk - s * aqk;
          a[q * 6 + k] = s * apk + c * aqk;
        }
      }
  }
  for (int i = 0; i < 6; ++i) ev[i] = a[i * 6 + i];
}

// numpy.linalg.cond(H) > thresh (2-norm, via singular values) for symmetric H.
// Cheap exact screening: Cholesky pivots lie inside [lambda_min, lambda_max],
// so max/min pivot <= cond; and ||H||_F * trace(H^-1) >= lambda_max/lambda_min
// = cond, with trace(H^-1) = ||L^-1||_F^2.  Only the band between the two
// bounds (a factor <= 6*sqrt(6)) pays for the Jacobi eigen solve.
__device__ inline bool cond_exceeds6(const double* H, const double* L, const double* dinv,
                                     bool chol_ok, const double* piv, double thresh) {
  if (chol_ok) {
    double pmax = piv[0], pmin = piv[0];
    for (int i = 1; i < 6; ++i) { pmax = fmax(pmax, piv[i]); pmin = fmin(pmin, piv[i]); }
    if (pmax > thresh * pmin) return true;
    double fh = 0.0;
    for (int i = 0; i < 36; ++i) fh += H[i] * H[i];
    double M[36];  // L^-1, lower triangular
    double tr = 0.0;
    for (int i = 0; i < 6; ++i) {
      M[i * 6 + i] = dinv[i];
      tr += dinv[i] * dinv[i];
      for (int j = 0; j < i; ++j) {
        double s = 0.0;
        for (int k = j; k < i; ++k) s += L[i * 6 + k] * M[k * 6 + j];
        const double mij = -s * dinv[i];
        M[i * 6 + j] = mij;
        tr += mij * mij;
      }
    }
    if (sqrt(fh) * tr <= thresh) return false;
  }
  double ev[6];
  jacobi_eig6(H, ev);
  double smax = 0.0, smin = INFINITY;
  for (int i = 0; i < 6; ++i) { double a = fabs(ev[i]); smax = fmax(smax, a); smin = fmin(smin, a); }
  if (smin == 0.0) return true;
  return smax / smin > thresh;
}

// ---------------------------------------------------------------- SE(3)
__device__ inline void mat3_mul(const double* A, const double* B, double* C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}

__device__ inline void hat3(double x, double y, double z, double* K) {
  K[0] = 0.0; K[1] = -z;  K[2] = y;
  K[3] = z;   K[4] = 0.0; K[5] = -x;
  K[6] = -y;  K[7] = x;   K[8] = 0.0;
}

// pose <- exp(xi) @ pose, pose = [R row-major (9), t (3)]  (se3.py:22-67)
__device__ inline void se3_left_update(const double* xi, double* pose) {
  const double w0 = xi[0], w1 = xi[1], w2 = xi[2];
  const double th = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
  double Re[9], V[9], K[9], K2[9];
  if (th < 1e-12) {
    hat3(w0, w1, w2, K);
    mat3_mul(K, K, K2);
    for (int i = 0; i < 9; ++i) {
      double I = (i % 4 == 0) ? 1.0 : 0.0;
      Re[i] = I + K[i] + 0.5 * K2[i];
      V[i] = I + 0.5 * K[i];
    }
  } else {
    double s, c;
    sincos(th, &s, &c);  // one shared argument reduction (same values as sin / cos)
    hat3(w0 / th, w1 / th, w2 / th, K);
    mat3_mul(K, K, K2);
    double Kw[9], Kw2[9];
    hat3(w0, w1, w2, Kw);
    mat3_mul(Kw, Kw, Kw2);
    const double a = (1.0 - c) / (th * th), bcoef = (th - s) / (th * th * th);
    for (int i = 0; i < 9; ++i) {
      double I = (i % 4 == 0) ? 1.0 : 0.0;
      Re[i] = I + s * K[i] + (1.0 - c) * K2[i];
      V[i] = I + a * Kw[i] + bcoef * Kw2[i];
    }
  }
  double te[3];
  for (int i = 0; i < 3; ++i) te[i] = V[3 * i] * xi[3] + V[3 * i + 1] * xi[4] + V[3 * i + 2] * xi[5];
  double Rn[9];
  mat3_mul(Re, pose, Rn);
  double tn[3];
  for (int i = 0; i < 3; ++i)
    tn[i] = Re[3 * i] * pose[9] + Re[3 * i + 1] * pose[10] + Re[3 * i + 2] * pose[11] + te[i];
  for (int i = 0; i < 9; ++i) pose[i] = Rn[i];
  for (int i = 0; i < 3; ++i) pose[9 + i] = tn[i];
}

// ||R^T R - I||_F  (se3.py:92-93)
__device__ inline double orth_defect(const double* R) {
  double acc = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double d = R[i] * R[j] + R[3 + i] * R[3 + j] + R[6 + i] * R[6 + j] - (i == j ? 1.0 : 0.0);
      acc += d * d;
    }
  return sqrt(acc);
}

// nearest rotation (polar factor == U V^T of the SVD, se3.py:95-102) by the
// Newton iteration Q <- (Q + Q^-T)/2, quadratically convergent from near-SO(3)
__device__ inline void reorthonormalize(double* R) {
  for (int it = 0; it < 8; ++it) {
    double c[9];  // cofactor matrix = det * Q^-T
    c[0] = R[4] * R[8] - R[5] * R[7];
    c[1] = R[5] * R[6] - R[3] * R[8];
    c[2] = R[3] * R[7] - R[4] * R[6];
    c[3] = R[2] * R[7] - R[1] * R[8];
    c[4] = R[0] * R[8] - R[2] * R[6];
    c[5] = R[1] * R[6] - R[0] * R[7];
    c[6] = R[1] * R[5] - R[2] * R[4];
    c[7] = R[2] * R[3] - R[0] * R[5];
    c[8] = R[0] * R[4] - R[1] * R[3];
    double det = R[0] * c[0] + R[1] * c[1] + R[2] * c[2];
    double delta = 0.0;
    for (int i = 0; i < 9; ++i) {
      double q = 0.5 * (R[i] + c[i] / det);
      delta = fmax(delta, fabs(q - R[i]));
      R[i] = q;
    }
    if (delta < 1e-17) break;
  }
}

}  // namespace rk
