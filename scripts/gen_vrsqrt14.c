// Dump the AVX-512 VRSQRT14PS result table used by numpy's SVML arcsin
// (__svml_asinf16, |x| >= 0.5 branch) for the device emulation (rk_svml.cuh).
//
// VRSQRT14PS(y * 4^k) = VRSQRT14PS(y) * 2^-k for normal inputs, and for
// y in [1, 4) the result depends only on the exponent parity and the top 15
// mantissa bits (verified exhaustively below); every result has >= 7 trailing
// zero mantissa bits.  Table entry i = (parity << 15) | (mantissa >> 8), value
// = the result's mantissa bits [22:7] (uint16); the exponent is 126 except
// for y == 1.0 exactly (result 1.0), which the device code special-cases.
//
//   gcc -O2 -mavx512f -o /tmp/gen_vrsqrt14 scripts/gen_vrsqrt14.c
//   /tmp/gen_vrsqrt14 paper_2112_02779_b200/data/vrsqrt14.u16
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static uint32_t rs14(uint32_t in) {
  __m512 x = _mm512_castsi512_ps(_mm512_set1_epi32((int)in));
  uint32_t o[16];
  _mm512_storeu_si512(o, _mm512_castps_si512(_mm512_rsqrt14_ps(x)));
  return o[0];
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  static uint16_t tab[65536];
  long bad = 0;
  for (uint32_t par = 0; par < 2; ++par)
    for (uint32_t m = 0; m < (1u << 23); ++m) {
      const uint32_t in = ((127u + par) << 23) | m;  // y in [1,2) or [2,4)
      const uint32_t o = rs14(in);
      const uint32_t idx = (par << 15) | (m >> 8);
      const uint32_t hi = (o >> 7) & 0xffffu;
      const uint32_t ex = o >> 23;
      if (in == 0x3f800000u) { if (o != 0x3f800000u) ++bad; continue; }  // 1.0 -> 1.0
      if (ex != 126 || (o & 0x7fu)) ++bad;
      if ((m & 0xffu) == 0 || (par == 0 && m == 1)) tab[idx] = (uint16_t)hi;
      else if (tab[idx] != hi) ++bad;  // not a function of (parity, top 15 bits)
    }
  // power-of-4 scaling over the exponents numpy's arcsin feeds it ((1-|x|)/2 in (2^-32, 0.25])
  for (int e = 127 - 34; e <= 127 + 4; ++e)
    for (uint32_t m = 0; m < (1u << 23); m += 4099) {
      const uint32_t in = ((uint32_t)e << 23) | m;
      const int par = (e - 127) & 1, k = (e - 127 - par) / 2;
      uint32_t want;
      if (m == 0 && par == 0) want = (uint32_t)(127 - k) << 23;
      else want = ((uint32_t)(126 - k) << 23) | ((uint32_t)tab[(par << 15) | (m >> 8)] << 7);
      if (rs14(in) != want) ++bad;
    }
  if (bad) { fprintf(stderr, "table hypothesis violated at %ld inputs\n", bad); return 1; }
  FILE* f = fopen(argv[1], "wb");
  if (!f || fwrite(tab, 2, 65536, f) != 65536) return 1;
  fclose(f);
  printf("wrote %s (65536 entries, hypothesis verified)\n", argv[1]);
  return 0;
}
