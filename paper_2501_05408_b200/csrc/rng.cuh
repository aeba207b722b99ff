// numpy-exact per-point random streams on device.
//
// The reference draws every rng/udf point from
//   np.random.default_rng((seed, tag, *point))      (runtime.py:50-55, 391-394)
// i.e. SeedSequence(entropy) -> generate_state(4, uint64) -> PCG64 (XSL-RR
// 128/64) -> Generator.standard_normal (256-layer ziggurat) / .uniform.
// This header restates those algorithms (numpy 2.3.5; SeedSequence in
// numpy/random/bit_generator.pyx, PCG64 in numpy/random/src/pcg64/pcg64.h,
// random_standard_normal in numpy/random/src/distributions/distributions.c)
// so every draw is bit-identical to the reference's.  Tables come from the
// numpy binary (tools/gen_ziggurat_tables.py).  Validated against numpy
// itself (every draw of 10 M, including ~2.6 k ziggurat-tail draws) in
// tests/test_gpu_parity.py::test_rng_bit_exact_vs_numpy.
#pragma once
#ifndef __CUDACC_RTC__
#include <stdint.h>
#endif
#include "ziggurat_tables.h"
#include "glibc_log1p.h"

#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

struct rt_pcg64 {
  unsigned __int128 state, inc;
};

__device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= SS_MULT_A;
  v *= hc;
  v ^= v >> 16;
  return v;
}

__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}

// words: the assembled entropy (each python int -> little-endian u32 words;
// 0 -> [0]).  n may exceed the pool size (4).
__device__ __forceinline__ void pcg64_seed(rt_pcg64& g, const uint32_t* words, int n) {
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
#pragma unroll
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? words[i] : 0u, hc);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < n; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], hc));
  // generate_state(4, uint64): 8 u32 words cycling over the pool
  uint32_t st[8];
  uint32_t hb = SS_INIT_B;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  uint64_t v0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  uint64_t v1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  uint64_t v2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
  uint64_t v3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
  unsigned __int128 s = ((unsigned __int128)v0 << 64) | v1;
  unsigned __int128 inc = ((unsigned __int128)v2 << 64) | v3;
  const unsigned __int128 mult =
      ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
  g.inc = (inc << 1) | 1u;
  g.state = 0;
  g.state = g.state * mult + g.inc;
  g.state += s;
  g.state = g.state * mult + g.inc;
}

__device__ __forceinline__ uint64_t pcg64_next(rt_pcg64& g) {
  const unsigned __int128 mult =
      ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
  g.state = g.state * mult + g.inc;
  uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(g.state >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ double pcg64_double(rt_pcg64& g) {
  return (double)(pcg64_next(g) >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double pcg64_normal(rt_pcg64& g) {
  const double zr = 3.6541528853610087963519472518;
  const double zinvr = 0.27366123732975827203338247596;
  for (;;) {
    uint64_t r = pcg64_next(g);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 0x1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * zig_wi[idx];
    if (sign & 0x1) x = -x;
    if (rabs < zig_ki[idx]) return x;
    // numpy distributions.c random_standard_normal, operation for operation;
    // no contraction (numpy's baseline x86-64 build has none): the tail's
    // log1p is glibc's own (glibc_log1p.h); the wedge test's exp can only
    // flip an accept when both sides agree to within an ulp
    if (idx == 0) {
      for (;;) {
        double xx = __dmul_rn(-zinvr, glibc_log1p(-pcg64_double(g)));
        double yy = -glibc_log1p(-pcg64_double(g));
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
          return ((rabs >> 8) & 0x1) ? -__dadd_rn(zr, xx) : __dadd_rn(zr, xx);
      }
    } else {
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(zig_fi[idx - 1], zig_fi[idx]),
                                             pcg64_double(g)), zig_fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x)))
        return x;
    }
  }
}
