/* Host-independent restatement of numpy 2.x's float32 np.arctan2 / np.arcsin
 * on AVX-512 hosts (Intel SVML __svml_atan2f16 / __svml_asinf16 main paths,
 * vendored in numpy; constants = the bit patterns of its
 * __svml_satan2_data_internal / __svml_sasin_data_internal tables).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the oracle's
 * math="svml" mode, so the GPU's RK_MATH_NP results can be checked on a host
 * whose own numpy does not dispatch to SVML.  Same operation sequence as
 * paper_2112_02779_b200/csrc/rk_svml.cuh; every multiply-add is C99 fmaf
 * (correctly rounded on any host), compiled with -ffp-contract=off.
 * tests/test_oracle_golden.py pins it against numpy's outputs (goldens).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static float f_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t u_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

static float atan2_one(float y, float x) {
  const uint32_t ux = u_of(x) & 0x7fffffffu, uy = u_of(y) & 0x7fffffffu;
  const int main_x = (ux - 0x01000000u) < (0x7d000000u - 0x01000000u);
  const int main_y = (uy - 0x01000000u) < (0x7d000000u - 0x01000000u);
  if (!(main_x && main_y)) return (float)atan2((double)y, (double)x);  /* SVML's scalar path */
  const float ax = f_of(ux), ay = f_of(uy);
  const int k1 = ay < ax;
  const float a = k1 ? ay : -ax, b = k1 ? ax : ay;
  float r = 1.0f / b;  /* stands in for VRCP14PS: the Markstein step removes its low bits */
  const float e = fmaf(-b, r, 1.0f);
  r = fmaf(e, r, r);
  const float q = a * r;
  const float e2 = fmaf(-q, b, a);
  const float s = fmaf(e2, r, q);
  const float s2 = s * s, s4 = s2 * s2;
  float P = fmaf(f_of(0x3b322cc0u), s4, f_of(0x3d2bc384u));
  float Q = fmaf(f_of(0xbc7f2631u), s4, f_of(0xbd987629u));
  P = fmaf(s4, P, f_of(0x3dd96474u));
  Q = fmaf(s4, Q, f_of(0xbe1161f8u));
  P = fmaf(s4, P, f_of(0x3e4cb79fu));
  Q = fmaf(s4, Q, f_of(0xbeaaaa49u));
  P = fmaf(s4, P, 1.0f);
  float R = fmaf(s2, Q, P);
  R = fmaf(s, R, k1 ? 0.0f : f_of(0x3fc90fdbu));
  R = f_of(u_of(R) | (u_of(x) & 0x80000000u));
  if (x <= 0.0f) R = R + f_of(0x40490fdbu);
  return f_of(u_of(R) | (u_of(y) & 0x80000000u));
}

static float vrsqrt14(float w, const uint16_t* tab) {
  const uint32_t u = u_of(w);
  const int e = (int)(u >> 23) - 127;
  const int par = e & 1;
  const int k = (e - par) / 2;
  const uint32_t m = u & 0x7fffffu;
  if (m == 0 && par == 0) return f_of((uint32_t)(127 - k) << 23);
  return f_of(((uint32_t)(126 - k) << 23) | ((uint32_t)tab[(par << 15) | (m >> 8)] << 7));
}

static float asin_one(float x, const uint16_t* tab) {
  const float ax = fabsf(x);
  const uint32_t sg = u_of(x) & 0x80000000u;
  if (ax > 1.0f || x != x) return (float)asin((double)x);
  const float x2 = ax * ax;
  float q;
  if (ax < 0.5f) {
    const float z = x2, z2 = z * z;
    float p7 = fmaf(f_of(0x3d2edc07u), z, f_of(0x3cc32a6bu));
    const float p5 = fmaf(f_of(0x3d3a9ab4u), z, f_of(0x3d997c12u));
    p7 = fmaf(z2, p7, p5);
    p7 = fmaf(z, p7, f_of(0x3e2aaaffu));
    q = fmaf(ax, p7 * z, ax);
  } else {
    const float w = fmaf(-0.5f, ax, 0.5f);
    const float r = w < f_of(0x2f800000u) ? 0.0f : vrsqrt14(w, tab);
    const float z = x2 < w ? x2 : w;
    const float w2 = w + w;
    const float s0 = w2 * r;
    const float e = fmaf(r * r, w2, -2.0f);
    const float t = s0 * e;
    float c = fmaf(f_of(0xbdc00004u), e, f_of(0x3e800001u));
    c = fmaf(t, c, -s0);
    const float z2 = z * z;
    float p7 = fmaf(f_of(0x3d2edc07u), z, f_of(0x3cc32a6bu));
    const float p5 = fmaf(f_of(0x3d3a9ab4u), z, f_of(0x3d997c12u));
    p7 = fmaf(z2, p7, p5);
    p7 = fmaf(z, p7, f_of(0x3e2aaaffu));
    q = fmaf(c, p7 * z, c);
    q = q + f_of(0x3fc90fdbu);
  }
  return f_of(u_of(q) ^ sg);
}

void svml_atan2f_n(const float* y, const float* x, float* out, long n) {
  for (long i = 0; i < n; ++i) out[i] = atan2_one(y[i], x[i]);
}

void svml_asinf_n(const float* q, const uint16_t* tab, float* out, long n) {
  for (long i = 0; i < n; ++i) out[i] = asin_one(q[i], tab);
}
