// Fused acting step of an MLP policy inside the persistent loop kernel
// (jit_mlp.py generates the kernel around these pieces).
//
// The reference evaluates the acting recurrence point by point
// (runtime.py:344-389): per (b, t) the observation merge, h1 = tanh(o W1 +
// b1), h2 = tanh(h1 W2 + b2), mu = h2 W3 + b3, a = mu + eps and the
// synthetic env step (dsl.py:288-307).  Here one CTA of 256 threads owns
// R <= 8 env rows for the whole horizon and runs a step as
//
//   obs (generic EW)                                              | barrier
//   h1   thread (row half, 2 columns), K = DO from shared memory  | barrier
//   h2   hyb_core (loop_lib.cuh): thread (K half, 2 columns), 64 weight
//        rows per column in registers, 64 in shared memory, all rows; the
//        halves exchange rows through shared memory               | barrier x2
//   tail one warp per row: policy head (warp reduction), action, env
//        (numpy pairwise means in fp64), next observation carried in smem
//                                                                 | barrier
// i.e. five CTA barriers per step (the op-by-op JIT loop: eleven), no global
// round trip between ops, and the narrow head as a warp reduction instead of
// a 32-long dependent FMA chain per thread.
#pragma once
#include "loop_lib.cuh"

#define MLP_THREADS 256

RT_DEV float4 lds4f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// acc[r] += a[r] * w over HR = MRP/2 rows of one column (FFMA2 row pairs).
template <int HR>
RT_DEV void mlp_rows_fma(float (&acc)[HR], const float (&a)[HR], float w) {
#pragma unroll
  for (int r = 0; r + 1 < HR; r += 2) fma2(acc[r], acc[r + 1], a[r], a[r + 1], w);
  if constexpr (HR % 2) acc[HR - 1] = fmaf(a[HR - 1], w, acc[HR - 1]);
}

// h1 pre-activation of rows [rh*MRP/2, +MRP/2), columns c0, c0+1:
// sum_k o[r][k] W1[k][c]  (o k-major in sO: sO[k*MRP + r]; W1 row-major in
// sW1: [DO][NH]); no K split (K = DO is small), so no reduction barrier.
template <int MRP, int DO, int NH>
RT_DEV void mlp_h1(uint32_t sO, uint32_t sW1, int c0, int rh, float (&acc)[2][MRP / 2]) {
  constexpr int HR = MRP / 2, KG = DO % 4 == 0 ? 4 : 1;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int r = 0; r < HR; ++r) acc[j][r] = 0.f;
#pragma unroll
  for (int k0 = 0; k0 < DO; k0 += KG) {
    float a[KG][HR], w[KG][2];
#pragma unroll
    for (int u = 0; u < KG; ++u) {
      lds_rows<HR>(sO + (uint32_t)(((k0 + u) * MRP + rh * HR) * 4), a[u]);
      lds_cols<2>(sW1 + (uint32_t)(((k0 + u) * NH + c0) * 4), w[u]);
    }
#pragma unroll
    for (int u = 0; u < KG; ++u) {
      mlp_rows_fma<HR>(acc[0], a[u], w[u][0]);
      mlp_rows_fma<HR>(acc[1], a[u], w[u][1]);
    }
  }
}

// Policy head of one row, one warp: mu[n] = sum_k h2[k] W3[k][n], n < DA
// (h2 row-major in sH: NH floats; W3 transposed in sW3T: [DA][NH]).  Lane l
// covers k in [4l, 4l+4) and [NH/2 + 4l, ...); every lane ends with all DA sums.
template <int DA, int NH>
RT_DEV void mlp_head(uint32_t sH, uint32_t sW3T, int lane, float (&mu)[DA]) {
  static_assert(NH == 256, "a warp covers 256 inputs as 2 x 32 x float4");
  const float4 h0 = lds4f(sH + (uint32_t)(16 * lane)), h1 = lds4f(sH + (uint32_t)(512 + 16 * lane));
#pragma unroll
  for (int n = 0; n < DA; ++n) {
    const float4 w0 = lds4f(sW3T + (uint32_t)(n * NH * 4 + 16 * lane));
    const float4 w1 = lds4f(sW3T + (uint32_t)(n * NH * 4 + 512 + 16 * lane));
    float s = h0.x * w0.x;
    s = fmaf(h0.y, w0.y, s);
    s = fmaf(h0.z, w0.z, s);
    s = fmaf(h0.w, w0.w, s);
    float s2 = h1.x * w1.x;
    s2 = fmaf(h1.y, w1.y, s2);
    s2 = fmaf(h1.z, w1.z, s2);
    s2 = fmaf(h1.w, w1.w, s2);
    mu[n] = s + s2;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int n = 0; n < DA; ++n) mu[n] += __shfl_xor_sync(0xffffffffu, mu[n], o);
}

// h2 core, four columns per thread (the shared-memory wavefronts of the
// two-column hyb_core bound the step: every thread of a part loads the same
// A rows, so A traffic per FMA halves with twice the columns per thread).
// 256 threads = 4 K parts x 64 threads; thread (part p = tid / 64, columns
// c0 = 4 (tid % 64) .. +4) sums k in [64p, 64p + 64): the first KR rows of
// its columns from registers (w), the other 64 - KR from shared memory
// (sW: [4][64 - KR][NH], row-major).  A (h1) is k-major: sX[k*MRP + r].
// Then every part finalises MRP/4 rows: rows [p*RQ, (p+1)*RQ), RQ = MRP/4,
// summing the four parts' partials in part order through red
// ([4][MRP][NH] floats).  out[j][q] = row p*RQ + q, column c0 + j.
template <int MRP, int NR, int KR, int NH>
RT_DEV void mlp_h2q(const float (&w)[4][KR], uint32_t sW, uint32_t sX, uint32_t red,
                    float (&out)[4][MRP / 4]) {
  constexpr int KP = 64, KS = KP - KR, RQ = MRP / 4;
  const int tid = (int)threadIdx.x, part = tid >> 6, c0 = 4 * (tid & 63);
  float acc[4][MRP];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int r = 0; r < MRP; ++r) acc[j][r] = 0.f;
  const uint32_t a0 = sX + (uint32_t)(part * KP * MRP * 4);
#pragma unroll
  for (int kk = 0; kk < KR; ++kk) {
    float a[MRP];
    lds_rows<MRP>(a0 + (uint32_t)(kk * MRP * 4), a);
#pragma unroll
    for (int j = 0; j < 4; ++j) fma_rows_n<MRP, NR>(acc[j], a, w[j][kk]);
  }
  const uint32_t b0 = sW + (uint32_t)((part * KS * NH + c0) * 4);
#pragma unroll 4
  for (int kk = 0; kk < KS; ++kk) {
    float a[MRP];
    lds_rows<MRP>(a0 + (uint32_t)((KR + kk) * MRP * 4), a);
    const float4 b = lds4f(b0 + (uint32_t)(kk * NH * 4));
    fma_rows_n<MRP, NR>(acc[0], a, b.x);
    fma_rows_n<MRP, NR>(acc[1], a, b.y);
    fma_rows_n<MRP, NR>(acc[2], a, b.z);
    fma_rows_n<MRP, NR>(acc[3], a, b.w);
  }
  // partials of the rows other parts finalise -> red[part][r][c0..c0+4)
#pragma unroll
  for (int r = 0; r < MRP; ++r) {
    if (r / RQ == part) continue;
    sts4(red + (uint32_t)(((part * MRP + r) * NH + c0) * 4),
         make_float4(acc[0][r], acc[1][r], acc[2][r], acc[3][r]));
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int r = part * RQ + q;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) {
      // own partial: row pp*RQ + q is a static register index only for pp == part
      const float4 mine = make_float4(acc[0][pp * RQ + q], acc[1][pp * RQ + q],
                                      acc[2][pp * RQ + q], acc[3][pp * RQ + q]);
      const float4 x = pp == part ? mine : lds4f(red + (uint32_t)(((pp * MRP + r) * NH + c0) * 4));
      s[0] += x.x; s[1] += x.y; s[2] += x.z; s[3] += x.w;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) out[j][q] = s[j];
  }
}
