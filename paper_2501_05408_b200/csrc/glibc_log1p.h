// log1p, bit-identical to the host libm numpy calls in the ziggurat tail.
//
// numpy's random_standard_normal (numpy/random/src/distributions/
// distributions.c) draws its tail from npy_log1p = the C library's log1p.
// On the x86-64 hosts of this image that is glibc 2.39's FMA variant
// (ifunc-selected __log1p_fma: sysdeps/ieee754/dbl-64/s_log1p.c built with
// -mfma -mavx2, i.e. the fdlibm algorithm with gcc's FMA contractions).
// This is a restatement of that algorithm with each contraction spelled out
// as an explicit fused multiply-add (read off the ifunc target's machine
// code), and every other operation explicitly unfused — so the device result
// equals the host's bit for bit, where CUDA's libdevice log1p differs in the
// last place for about 1% of tail draws.
//
// The same text compiles as C on the host (tests/test_rng_log1p.py runs it
// against glibc on 10^8 arguments; build with -ffp-contract=off).
#pragma once

#ifdef __CUDACC__
#define L1P_DEV __device__ __forceinline__
#define L1P_MUL(a, b) __dmul_rn(a, b)
#define L1P_ADD(a, b) __dadd_rn(a, b)
#define L1P_SUB(a, b) __dsub_rn(a, b)
#define L1P_DIV(a, b) __ddiv_rn(a, b)
#define L1P_FMA(a, b, c) __fma_rn(a, b, c)
#define L1P_HI(x) ((int)__double2hiint(x))
#define L1P_SETHI(x, h) __hiloint2double((h), __double2loint(x))
#define L1P_INF __longlong_as_double(0x7ff0000000000000LL)
#define L1P_NAN __longlong_as_double(0x7ff8000000000000LL)
#else
#include <math.h>
#include <stdint.h>
#include <string.h>
#define L1P_DEV static inline
#define L1P_MUL(a, b) ((a) * (b))
#define L1P_ADD(a, b) ((a) + (b))
#define L1P_SUB(a, b) ((a) - (b))
#define L1P_DIV(a, b) ((a) / (b))
#define L1P_FMA(a, b, c) fma(a, b, c)
static inline int l1p_hi(double x) { uint64_t u; memcpy(&u, &x, 8); return (int)(int32_t)(u >> 32); }
static inline double l1p_sethi(double x, int h) {
  uint64_t u; memcpy(&u, &x, 8);
  u = (u & 0xffffffffull) | ((uint64_t)(uint32_t)h << 32);
  memcpy(&x, &u, 8);
  return x;
}
#define L1P_HI(x) l1p_hi(x)
#define L1P_SETHI(x, h) l1p_sethi(x, h)
#define L1P_INF INFINITY
#define L1P_NAN NAN
#endif

L1P_DEV double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  int hx = L1P_HI(x);
  int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {                          // x < 0.41422
    if (ax >= 0x3ff00000) {                       // x <= -1
      if (x == -1.0) return -L1P_INF;
      return L1P_NAN;
    }
    if (ax < 0x3e200000) {                        // |x| < 2^-29
      if (ax < 0x3c900000) return x;
      return L1P_FMA(-L1P_MUL(x, x), 0.5, x);     // x - x*x*0.5 (fused)
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {        // -0.2929 < x < 0.41422
      k = 0; f = x; hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return L1P_ADD(x, x);
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = L1P_ADD(1.0, x);
      hu = L1P_HI(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? L1P_SUB(1.0, L1P_SUB(u, x)) : L1P_SUB(x, L1P_SUB(u, 1.0));
      c = L1P_DIV(c, u);
    } else {
      u = x;
      hu = L1P_HI(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = L1P_SETHI(u, hu | 0x3ff00000);          // normalize u
    } else {
      k += 1;
      u = L1P_SETHI(u, hu | 0x3fe00000);          // normalize u/2
      hu = (0x00100000 - hu) >> 2;
    }
    f = L1P_SUB(u, 1.0);
  }
  const double hfsq = L1P_MUL(L1P_MUL(0.5, f), f);
  const double dk = (double)k;
  if (hu == 0) {                                  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return L1P_FMA(dk, ln2_hi, L1P_FMA(dk, ln2_lo, c));
    }
    const double R = L1P_MUL(L1P_FMA(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return L1P_SUB(f, R);
    return L1P_FMA(dk, ln2_hi, -L1P_SUB(L1P_SUB(R, L1P_FMA(dk, ln2_lo, c)), f));
  }
  const double s = L1P_DIV(f, L1P_ADD(2.0, f));
  const double z = L1P_MUL(s, s);
  const double R2 = L1P_FMA(z, Lp3, Lp2), R3 = L1P_FMA(z, Lp5, Lp4), R4 = L1P_FMA(z, Lp7, Lp6);
  const double z2 = L1P_MUL(z, z), z4 = L1P_MUL(z2, z2), z6 = L1P_MUL(z2, z4);
  const double R = L1P_FMA(z6, R4, L1P_FMA(z4, R3, L1P_FMA(z, Lp1, L1P_MUL(z2, R2))));
  const double t = L1P_MUL(L1P_ADD(R, hfsq), s);   // s*(hfsq+R)
  if (k == 0) return L1P_SUB(f, L1P_SUB(hfsq, t));
  const double w = L1P_SUB(L1P_SUB(hfsq, L1P_ADD(L1P_FMA(dk, ln2_lo, c), t)), f);
  return L1P_FMA(dk, ln2_hi, -w);
}
