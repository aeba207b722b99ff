// RT_K_THIN — the HBM-bound GEMMs of the MLP backward over T*E points.
//
// The symbolic backward (reference frontend.py:766-776, 984-989) turns every
// per-point matmul into weight gradients summed over all T*E points.  When one
// side is narrow (the 16-wide observation layer, the 4-wide action head) the
// product is a stream over a [points, wide] activation with a handful of FMAs
// per element: tensor-core tiles would mostly multiply padding, so these run
// as coalesced streams at HBM speed instead.
//
//   variant 1  C[w,r] = sum_k X[k,w] * Y[k,r]   narrow contraction, K split
//              over blockIdx.y; per-split partials -> RT_K_SPLITK
//   variant 2  C[w,r] = epi(sum_k X[w,k] * Y[k,r] + bias[r]) for K <= 32
//              (d(hidden) = d(logits) @ W^T: write-bound)
#include "common.cuh"

namespace {

constexpr int THREADS = 256;
constexpr int KT = 64;

RT_DEV float mul_rn(float a, float b) { return __fmul_rn(a, b); }
RT_DEV double mul_rn(double a, double b) { return __dmul_rn(a, b); }
RT_DEV float sub_rn(float a, float b) { return __fsub_rn(a, b); }
RT_DEV float add_rn(float a, float b) { return __fadd_rn(a, b); }
RT_DEV double add_rn(double a, double b) { return __dadd_rn(a, b); }
RT_DEV double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// offset of flat row index `flat` over box b (nd <= 1: flat * s[0])
RT_DEV int64_t wdec(const rt_gbox& b, int64_t flat, const int64_t* s) {
  if (b.nd <= 1) return flat * s[0];
  int64_t o = 0;
  if (flat < (1ll << 32)) {
    // 32-bit divisions (a 64-bit division is a ~100-instruction call):
    // gathered minibatch rows decompose every row of every tile
    uint32_t f = (uint32_t)flat;
    for (int d = b.nd - 1; d >= 0; --d) {
      const uint32_t e = (uint32_t)b.ext[d];
      const uint32_t q = f / e;
      o += (int64_t)(f - q * e) * s[d];
      f = q;
    }
    return o;
  }
  for (int d = b.nd - 1; d >= 0; --d) {
    const int64_t e = b.ext[d];
    const int64_t q = flat / e;
    o += (flat - q * e) * s[d];
    flat = q;
  }
  return o;
}


template <typename T, int R, bool ONES = false>
__global__ void __launch_bounds__(THREADS) k_thin_contract(const __grid_constant__ rt_thin_params p) {
  // 256-row Y chunks when they fit in 16 KB: 4x fewer barrier + Y-latency
  // exposures per split than 64-row chunks
  constexpr int KT = (R * (int)sizeof(T) <= 64 && R * (int)sizeof(T) >= 32) ? 256 : 64;
  __shared__ __align__(16) T ys[KT][R];
  const int64_t w = (int64_t)blockIdx.x * THREADS + threadIdx.x;
  const bool wok = w < p.w;
  const int s = blockIdx.y;
  const int64_t per = ((p.k + p.splits - 1) / p.splits + KT - 1) / KT * KT;
  const int64_t k0 = (int64_t)s * per;
  const int64_t k1 = k0 + per < p.k ? k0 + per : p.k;
  const T* X = (const T*)p.X.ptr + p.X.off;
  const T* Y = (const T*)p.Y.ptr + p.Y.off;
  const int64_t xk = p.X.s1[0], yk = p.Y.s1[0], yr = p.Y.s2[0];
  const int nr = (int)p.r;
  const T* xp = X + (wok ? w : 0) * p.X.s2[0];
  T acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = (T)0;
  T acc1 = (T)0;   // ONES: the sum of X over k (a column of ones in Y)
  for (int64_t kb = k0; kb < k1; kb += KT) {
    const int nk = (int)(k1 - kb < KT ? k1 - kb : KT);
    __syncthreads();
    for (int i = threadIdx.x; i < KT * R; i += THREADS) {
      const int kk = i / R, r = i - kk * R;
      ys[kk][r] = (kk < nk && r < nr) ? __ldg(Y + (kb + kk) * yk + r * yr) : (T)0;
    }
    __syncthreads();
    if (!wok) continue;
    const T* xb = xp + kb * xk;
    if (nk == KT) {
#pragma unroll 16
      for (int kk = 0; kk < KT; ++kk) {
        const T x = __ldcs(xb + kk * xk);
        fma_bcast<R>(acc, ys[kk], x);
        if constexpr (ONES) acc1 += x;
      }
    } else {
      for (int kk = 0; kk < nk; ++kk) {
        const T x = __ldcs(xb + kk * xk);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma(x, ys[kk][r], acc[r]);
        if constexpr (ONES) acc1 += x;
      }
    }
  }
  if (!wok) return;
  if constexpr (ONES) ((T*)p.part2)[(int64_t)s * p.w + w] = acc1;
  T* part = (T*)p.part + (int64_t)s * p.w * p.r;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r < nr) part[w * p.part_w + r * p.part_r] = acc[r];
}

// variant 1, bulk-streamed (p.vec, fp32): the same per-thread sums as
// k_thin_contract -- thread (blockIdx.x, tid) owns column w of X and sums
// x[k] * y[k, r] over its split's rows in k order -- but the rows arrive by
// cp.async.bulk into a 3-stage shared-memory ring (32 rows of the block's
// 256-column slice of X + the rows' Y per stage, one mbarrier each) instead
// of per-thread 4-byte loads behind a Y-tile barrier: the bulk engine keeps
// ~200 KB per SM in flight (2 CTAs), and the splits are sized to one wave.
// Requires 16-byte aligned rows (X columns contiguous, w % 4 == 0, Y
// columns contiguous, r % 4 == 0); the lowering checks and otherwise keeps
// k_thin_contract.
constexpr int BK_SR = 32, BK_ST = 3;

RT_DEV uint32_t bk_su32(const void* q) { return (uint32_t)__cvta_generic_to_shared(q); }
RT_DEV void bk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
RT_DEV void bk_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  }
}

template <int R, bool ONES>
__global__ void __launch_bounds__(THREADS, 2) k_thin_contract_bulk(const __grid_constant__ rt_thin_params p) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  float* xs = (float*)sm_raw;                          // [ST][SR][256]
  float* ys = xs + BK_ST * BK_SR * THREADS;            // [ST][SR][R]
  uint64_t* bars = (uint64_t*)(ys + BK_ST * BK_SR * R);
  const int tid = (int)threadIdx.x, lane = tid & 31;
  const int64_t w0 = (int64_t)blockIdx.x * THREADS;
  const int W = (int)(p.w - w0 < THREADS ? p.w - w0 : THREADS);
  const int s = blockIdx.y;
  const int64_t per = (p.k + p.splits - 1) / p.splits;
  const int64_t k0 = (int64_t)s * per;
  const int64_t k1 = k0 + per < p.k ? k0 + per : p.k;
  const int nst = k1 > k0 ? (int)((k1 - k0 + BK_SR - 1) / BK_SR) : 0;
  const float* X = (const float*)p.X.ptr + p.X.off + w0;
  const float* Y = (const float*)p.Y.ptr + p.Y.off;
  const int64_t xk = p.X.s1[0], yk = p.Y.s1[0];
  const int nr = (int)p.r;
  const bool xdense = xk == W && W == THREADS, ydense = yk == R && nr == R;
  if (tid == 0) {
    for (int i = 0; i < BK_ST; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bk_su32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // warp 0 fills stage st with rows [kb, kb + n)
  auto issue = [&](int it, int st) {
    const int64_t kb = k0 + (int64_t)it * BK_SR;
    const int n = (int)(k1 - kb < BK_SR ? k1 - kb : BK_SR);
    const uint32_t bar = bk_su32(bars + st);
    float* xd = xs + st * BK_SR * THREADS;
    float* yd = ys + st * BK_SR * R;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   ::"r"(bar), "r"((uint32_t)(n * (W + nr) * 4)) : "memory");
    __syncwarp();
    if (xdense) {
      if (lane == 0) bk_copy(bk_su32(xd), X + kb * xk, (uint32_t)(n * W * 4), bar);
    } else {
      for (int i = lane; i < n; i += 32) bk_copy(bk_su32(xd + i * THREADS), X + (kb + i) * xk, (uint32_t)(W * 4), bar);
    }
    if (ydense) {
      if (lane == 0) bk_copy(bk_su32(yd), Y + kb * yk, (uint32_t)(n * R * 4), bar);
    } else {
      for (int i = lane; i < n; i += 32) bk_copy(bk_su32(yd + i * R), Y + (kb + i) * yk, (uint32_t)(nr * 4), bar);
    }
  };
  if (tid < 32)
    for (int it = 0; it < BK_ST && it < nst; ++it) issue(it, it);
  // thread (g, c4): columns c4 .. c4 + 3 of the slice over the stage rows
  // kk = g, g + 4, ...; the four row groups' sums are added in group order
  // at the end.  (Four columns per thread: the broadcast Y row is read once
  // per 4 columns -- with one column per thread the Y reads were 4/5 of the
  // shared-memory wavefronts and paced the kernel.)
  const int g = tid >> 6, c4 = 4 * (tid & 63);
  const bool cok = c4 < W;                   // W % 4 == 0
  float acc[4][R], acc1[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc1[j] = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) acc[j][r] = 0.f;
  }
  for (int it = 0; it < nst; ++it) {
    const int st = it % BK_ST;
    bk_wait(bk_su32(bars + st), (uint32_t)((it / BK_ST) & 1));
    const int64_t kb = k0 + (int64_t)it * BK_SR;
    const int n = (int)(k1 - kb < BK_SR ? k1 - kb : BK_SR);
    const float* xr = xs + st * BK_SR * THREADS + c4;
    const float4* yr = (const float4*)(ys + st * BK_SR * R);
    if (cok) {
#pragma unroll 2
      for (int kk = g; kk < n; kk += 4) {
        const float4 x = *(const float4*)(xr + kk * THREADS);
        float y[R];
#pragma unroll
        for (int q = 0; q < R / 4; ++q) {
          const float4 v = yr[kk * (R / 4) + q];
          y[4 * q] = v.x; y[4 * q + 1] = v.y; y[4 * q + 2] = v.z; y[4 * q + 3] = v.w;
        }
        fma_bcast<R>(acc[0], y, x.x);
        fma_bcast<R>(acc[1], y, x.y);
        fma_bcast<R>(acc[2], y, x.z);
        fma_bcast<R>(acc[3], y, x.w);
        if constexpr (ONES) { acc1[0] += x.x; acc1[1] += x.y; acc1[2] += x.z; acc1[3] += x.w; }
      }
    }
    __syncthreads();   // every thread is done with stage st
    if (tid < 32 && it + BK_ST < nst) issue(it + BK_ST, st);
  }
  // row groups -> one sum per column, RC outputs at a time through the
  // (now idle) ring: red[g][rc][256]
  constexpr int RC = R < 8 ? R : 8;
  float* red = xs;
  float* part = (float*)p.part + (int64_t)s * p.w * p.r;
  const int64_t w = w0 + tid;
#pragma unroll
  for (int rb = 0; rb < R; rb += RC) {
    if (cok)
#pragma unroll
      for (int r = 0; r < RC; ++r)
        *(float4*)(red + (g * RC + r) * THREADS + c4) =
            make_float4(acc[0][rb + r], acc[1][rb + r], acc[2][rb + r], acc[3][rb + r]);
    if (ONES && rb == 0 && cok)
      *(float4*)(red + 4 * RC * THREADS + g * THREADS + c4) = make_float4(acc1[0], acc1[1], acc1[2], acc1[3]);
    __syncthreads();
    if (tid < W) {
#pragma unroll
      for (int r = 0; r < RC; ++r) {
        if (rb + r >= nr) break;
        float v = red[r * THREADS + tid];
#pragma unroll
        for (int gg = 1; gg < 4; ++gg) v += red[(gg * RC + r) * THREADS + tid];
        part[w * p.part_w + (rb + r) * p.part_r] = v;
      }
      if (ONES && rb == 0) {
        const float* r1 = red + 4 * RC * THREADS;
        ((float*)p.part2)[(int64_t)s * p.w + w] = ((r1[tid] + r1[THREADS + tid]) + r1[2 * THREADS + tid]) + r1[3 * THREADS + tid];
      }
    }
    __syncthreads();
  }
}

// variant 2: rows of X (K <= KP values each, zero-padded to KP) times a
// resident [KP, R] Y; each thread owns output columns, rows stream through
// a shared-memory tile, stores are coalesced along r.
// GATE: the epilogue-2 instantiation (its 16-row h prefetch is kept out of
// the plain kernel's register budget)
// KP2 > 0 (GATE only): a second product X2 Y2 (K2 <= KP2) summed before the
// gate, in the reference's order: a = X Y, b = X2 Y2, then a + b, then the
// gate (the PPO trunk's d(h2) = (dmu W3^T + dV Wv^T) * (1 - h2*h2)).
template <typename T, int KP, bool GATE = false, int KP2 = 0>
__global__ void __launch_bounds__(THREADS) k_thin_smallk(const __grid_constant__ rt_thin_params p) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  constexpr int RT = 64;  // rows per tile
  const int K = (int)p.k, R = (int)p.r;
  T* ys = (T*)sm_raw;             // [KP][R]
  T* xs = ys + KP * R;            // [RT][KP]
  T* bs = xs + RT * KP;           // [R]
  T* ys2 = bs + R;                // KP2: [KP2][R]
  T* xs2 = ys2 + KP2 * R;         // KP2: [RT][KP2]
  __shared__ int64_t coff[RT];    // output row offsets of the tile
  const T* X = (const T*)p.X.ptr + p.X.off;
  const T* Y = (const T*)p.Y.ptr + p.Y.off;
  T* Cp = (T*)p.C.ptr + p.C.off;
  for (int i = threadIdx.x; i < KP * R; i += THREADS) {
    const int k = i / R, r = i - k * R;
    ys[i] = k < K ? Y[k * p.Y.s1[0] + r * p.Y.s2[0]] : (T)0;
  }
  const int K2 = (int)p.k2;
  const T* X2 = KP2 ? (const T*)p.X2.ptr + p.X2.off : nullptr;
  if constexpr (KP2 > 0) {
    const T* Y2 = (const T*)p.Y2.ptr + p.Y2.off;
    for (int i = threadIdx.x; i < KP2 * R; i += THREADS) {
      const int k = i / R, r = i - k * R;
      ys2[i] = k < K2 ? Y2[k * p.Y2.s1[0] + r * p.Y2.s2[0]] : (T)0;
    }
  }
  // epilogue 2 (tanh-VJP gate, executor.find_gate_epilogues): C = acc * (1 - h*h)
  // with h in the bias slot, laid out exactly like C; no bias then
  constexpr bool gate = GATE;
  const T* Hg = gate ? (const T*)p.bias.ptr + p.bias.off : nullptr;
  for (int r = threadIdx.x; r < R; r += THREADS)
    bs[r] = (p.bias.ptr && !gate)
                ? load_as<T>((const void*)p.bias.ptr, p.bias.dtype, p.bias.off + r * p.bias.s2[0])
                : (T)0;
  const int64_t xk = p.X.s1[0], cr = p.C.s2[0];
  const int64_t ntiles = (p.w + RT - 1) / RT;
  const bool acc_in = p.accumulate != 0, tanh_epi = p.epilogue == 1;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t w0 = tile * RT;
    const int nrow = (int)(p.w - w0 < RT ? p.w - w0 : RT);
    __syncthreads();
    if (threadIdx.x < RT) {
      const int rr = threadIdx.x;
      const int64_t w = w0 + (rr < nrow ? rr : 0);
      coff[rr] = wdec(p.W, w, p.C.s1);
      const T* xr = X + wdec(p.W, w, p.X.s2);
#pragma unroll
      for (int k = 0; k < KP; ++k) xs[rr * KP + k] = (rr < nrow && k < K) ? __ldcs(xr + k * xk) : (T)0;
      if constexpr (KP2 > 0) {
        const T* xr2 = X2 + wdec(p.W, w, p.X2.s2);
#pragma unroll
        for (int k = 0; k < KP2; ++k)
          xs2[rr * KP2 + k] = (rr < nrow && k < K2) ? __ldcs(xr2 + k * p.X2.s1[0]) : (T)0;
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < R; r += THREADS) {
      T yreg[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) yreg[k] = ys[k * R + r];
      T yreg2[KP2 > 0 ? KP2 : 1];
#pragma unroll
      for (int k = 0; k < KP2; ++k) yreg2[k] = ys2[k * R + r];
      const T b = bs[r];
      T* cbase = Cp + r * cr;
      if constexpr (GATE) {
        // 16 rows per chunk: their h loads are issued together (a load per
        // output row one at a time left the kernel latency-bound)
        for (int rr0 = 0; rr0 < nrow; rr0 += 16) {
          T hv[16];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            hv[u] = rr0 + u < nrow ? __ldcs(Hg + coff[rr0 + u] + r * cr) : (T)0;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            if (rr0 + u >= nrow) break;
            const int rr = rr0 + u;
            T a = (T)0;
#pragma unroll
            for (int k = 0; k < KP; ++k) a = fma(xs[rr * KP + k], yreg[k], a);
            if constexpr (KP2 > 0) {
              T b = (T)0;
#pragma unroll
              for (int k = 0; k < KP2; ++k) b = fma(xs2[rr * KP2 + k], yreg2[k], b);
              a = add_rn(a, b);
            }
            // numpy order, no contraction: gy * (1 - h*h)
            __stcs(cbase + coff[rr], mul_rn(a, sub_rn((T)1, mul_rn(hv[u], hv[u]))));
          }
        }
        continue;
      }
#pragma unroll 4
      for (int rr = 0; rr < nrow; ++rr) {
        T a = (T)0;
#pragma unroll
        for (int k = 0; k < KP; ++k) a = fma(xs[rr * KP + k], yreg[k], a);
        T* cptr = cbase + coff[rr];
        if (acc_in) a += *cptr;
        a += b;
        if (tanh_epi) a = epi_tanh<T>(a);
        __stcs(cptr, a);
      }
    }
  }
}

// variant 2, vectorised (p.vec != 0): a thread owns VW adjacent output
// columns (one 16-byte store per row) and walks every RL-th row of the tile
// (RL = 256 / (R / VW) row lanes), with its Y columns in registers; the
// K-chain per output is the scalar kernel's (fma from 0 in k order, FFMA2 on
// column pairs: bit-identical), so only the instruction count changes (the
// scalar form issued ~45 instructions per output of the tanh layer over
// gathered minibatch rows, 1.9 TB/s; here the x loads and the address math
// are shared by VW outputs).  Needs R % VW == 0, 256 % (R / VW) == 0, C (and
// the gate operand) 16-byte aligned rows; lower.py _gemm_smallk checks.
template <typename T> struct svec2;
template <> struct svec2<float> { using V = float4; static constexpr int W = 4; };
template <> struct svec2<double> { using V = double2; static constexpr int W = 2; };
RT_DEV void v_unpack(const float4& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
RT_DEV void v_unpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
RT_DEV float4 v_pack(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
RT_DEV double2 v_pack(const double* o) { return make_double2(o[0], o[1]); }

template <int VW>
RT_DEV void vfma(float (&acc)[VW], const float (&y)[VW], float x) {
#pragma unroll
  for (int j = 0; j + 1 < VW; j += 2) fma2(acc[j], acc[j + 1], y[j], y[j + 1], x);
}
template <int VW>
RT_DEV void vfma(double (&acc)[VW], const double (&y)[VW], double x) {
#pragma unroll
  for (int j = 0; j < VW; ++j) acc[j] = fma(x, y[j], acc[j]);
}

template <typename T, int KP, bool GATE = false, int KP2 = 0>
__global__ void __launch_bounds__(THREADS, KP2 > 0 ? 2 : 1) k_thin_smallv(const __grid_constant__ rt_thin_params p) {
  using V = typename svec2<T>::V;
  constexpr int VW = svec2<T>::W;
  constexpr int RT = 64;  // rows per tile
  __shared__ __align__(16) T xs[RT * KP];
  __shared__ __align__(16) T xs2[RT * (KP2 > 0 ? KP2 : 1)];
  __shared__ int64_t coff[RT];
  __shared__ double csum[THREADS * VW];   // colsum: per-lane column partials
  const int K = (int)p.k, R = (int)p.r, K2 = (int)p.k2;
  const int G = R / VW, RL = THREADS / G;
  double cs[VW];
#pragma unroll
  for (int j = 0; j < VW; ++j) cs[j] = 0.0;
  const bool colsum = p.colsum != 0;
  // dw (GATE): sum_rows h[c] * x[k] -- the first operand's weight gradient
  constexpr int DK = GATE ? KP : 1, DK2 = GATE ? (KP2 > 0 ? KP2 : 1) : 1;
  T dwa[VW][DK], dwb[VW][DK2];
#pragma unroll
  for (int j = 0; j < VW; ++j) {
#pragma unroll
    for (int k = 0; k < DK; ++k) dwa[j][k] = (T)0;
#pragma unroll
    for (int k = 0; k < DK2; ++k) dwb[j][k] = (T)0;
  }
  const bool dw = GATE && p.dw != 0, dw2 = GATE && KP2 > 0 && p.dw2 != 0;
  const int cg = (int)threadIdx.x % G, rl = (int)threadIdx.x / G;
  const T* X = (const T*)p.X.ptr + p.X.off;
  const T* Y = (const T*)p.Y.ptr + p.Y.off;
  T* Cp = (T*)p.C.ptr + p.C.off;
  const T* Hg = GATE ? (const T*)p.bias.ptr + p.bias.off : nullptr;
  const int c0 = cg * VW;
  T yreg[KP][VW], breg[VW];
#pragma unroll
  for (int k = 0; k < KP; ++k)
#pragma unroll
    for (int j = 0; j < VW; ++j)
      yreg[k][j] = k < K ? Y[k * p.Y.s1[0] + (c0 + j) * p.Y.s2[0]] : (T)0;
  T yreg2[KP2 > 0 ? KP2 : 1][VW];
  if constexpr (KP2 > 0) {
    const T* Y2 = (const T*)p.Y2.ptr + p.Y2.off;
#pragma unroll
    for (int k = 0; k < KP2; ++k)
#pragma unroll
      for (int j = 0; j < VW; ++j)
        yreg2[k][j] = k < K2 ? Y2[k * p.Y2.s1[0] + (c0 + j) * p.Y2.s2[0]] : (T)0;
  }
#pragma unroll
  for (int j = 0; j < VW; ++j)
    breg[j] = (p.bias.ptr && !GATE)
                  ? load_as<T>((const void*)p.bias.ptr, p.bias.dtype, p.bias.off + (c0 + j) * p.bias.s2[0])
                  : (T)0;
  const T* X2 = KP2 ? (const T*)p.X2.ptr + p.X2.off : nullptr;
  const int64_t xk = p.X.s1[0];
  const int64_t ntiles = (p.w + RT - 1) / RT;
  const bool acc_in = p.accumulate != 0, tanh_epi = p.epilogue == 1;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t w0 = tile * RT;
    const int nrow = (int)(p.w - w0 < RT ? p.w - w0 : RT);
    __syncthreads();
    if (threadIdx.x < RT) {
      const int rr = threadIdx.x;
      const int64_t w = w0 + (rr < nrow ? rr : 0);
      coff[rr] = wdec(p.W, w, p.C.s1);
      const T* xr = X + wdec(p.W, w, p.X.s2);
#pragma unroll
      for (int k = 0; k < KP; ++k) xs[rr * KP + k] = (rr < nrow && k < K) ? __ldcs(xr + k * xk) : (T)0;
      if constexpr (KP2 > 0) {
        const T* xr2 = X2 + wdec(p.W, w, p.X2.s2);
#pragma unroll
        for (int k = 0; k < KP2; ++k)
          xs2[rr * KP2 + k] = (rr < nrow && k < K2) ? __ldcs(xr2 + k * p.X2.s1[0]) : (T)0;
      }
    }
    __syncthreads();
    // GATE: the h rows of HB row steps are loaded together (one 16-byte load
    // per row in flight per thread left the kernel latency-bound, ~3 TB/s)
    constexpr int HB = GATE ? (KP2 > 0 ? 4 : 8) : 1;   // KP2: 2 CTAs per SM in 128 registers
    for (int rb = rl; rb < nrow; rb += HB * RL) {
    V hvb[HB];
    if constexpr (GATE) {
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        const int rr = rb + u * RL;
        if (rr < nrow) hvb[u] = __ldcs(reinterpret_cast<const V*>(Hg + coff[rr] + c0));
      }
    }
#pragma unroll
    for (int u = 0; u < HB; ++u) {
      const int rr = rb + u * RL;
      if (rr >= nrow) break;
      const int64_t co = coff[rr] + c0;
      V hv = hvb[u];
      T a[VW];
#pragma unroll
      for (int j = 0; j < VW; ++j) a[j] = (T)0;
#pragma unroll
      for (int k = 0; k < KP; ++k) vfma<VW>(a, yreg[k], xs[rr * KP + k]);
      if constexpr (KP2 > 0) {
        T b[VW];
#pragma unroll
        for (int j = 0; j < VW; ++j) b[j] = (T)0;
#pragma unroll
        for (int k = 0; k < KP2; ++k) vfma<VW>(b, yreg2[k], xs2[rr * KP2 + k]);
#pragma unroll
        for (int j = 0; j < VW; ++j) a[j] = add_rn(a[j], b[j]);
      }
      if constexpr (GATE) {
        T h[VW];
        v_unpack(hv, h);
        if (dw) {
#pragma unroll
          for (int k = 0; k < DK; ++k) {
            const T xk_ = xs[rr * KP + k];
#pragma unroll
            for (int j = 0; j < VW; ++j) dwa[j][k] = fma(h[j], xk_, dwa[j][k]);
          }
        }
        if constexpr (KP2 > 0) {
          if (dw2) {
#pragma unroll
            for (int k = 0; k < DK2; ++k) {
              const T xk_ = xs2[rr * KP2 + k];
#pragma unroll
              for (int j = 0; j < VW; ++j) dwb[j][k] = fma(h[j], xk_, dwb[j][k]);
            }
          }
        }
        // numpy order, no contraction: gy * (1 - h*h)
#pragma unroll
        for (int j = 0; j < VW; ++j) a[j] = mul_rn(a[j], sub_rn((T)1, mul_rn(h[j], h[j])));
      } else {
        if (acc_in) {
          T o[VW];
          v_unpack(*reinterpret_cast<const V*>(Cp + co), o);
#pragma unroll
          for (int j = 0; j < VW; ++j) a[j] += o[j];
        }
#pragma unroll
        for (int j = 0; j < VW; ++j) a[j] += breg[j];
        if (tanh_epi) {
#pragma unroll
          for (int j = 0; j < VW; ++j) a[j] = epi_tanh<T>(a[j]);
        }
      }
      __stcs(reinterpret_cast<V*>(Cp + co), v_pack(a));
      if (colsum) {     // fp64 per row: the sum keeps the reference's accuracy
#pragma unroll
        for (int j = 0; j < VW; ++j) cs[j] += (double)a[j];
      }
    }
    }
  }
  if (dw || dw2) {
    // this CTA's weight-gradient partials: row lanes in order, fp64
    for (int which = 0; which < 2; ++which) {
      const int KK = which ? K2 : K;
      if (which ? !dw2 : !dw) continue;
      for (int k = 0; k < KK; ++k) {
        __syncthreads();
#pragma unroll
        for (int j = 0; j < VW; ++j) {
          T v = (T)0;
#pragma unroll
          for (int kk = 0; kk < (DK > DK2 ? DK : DK2); ++kk)
            if (kk == k) v = which ? (kk < DK2 ? dwb[j][kk < DK2 ? kk : 0] : (T)0)
                                   : (kk < DK ? dwa[j][kk < DK ? kk : 0] : (T)0);
          csum[rl * R + c0 + j] = (double)v;
        }
        __syncthreads();
        for (int c = (int)threadIdx.x; c < R; c += THREADS) {
          double t = 0.0;
          for (int l = 0; l < RL; ++l) t += csum[l * R + c];
          ((double*)(which ? p.part4 : p.part3))[((int64_t)blockIdx.x * R + c) * KK + k] = t;
        }
      }
    }
  }
  if (colsum) {
    // this CTA's column sums: lanes rl = 0.. RL-1 in order (deterministic)
    __syncthreads();
#pragma unroll
    for (int j = 0; j < VW; ++j) csum[rl * R + c0 + j] = cs[j];
    __syncthreads();
    for (int c = (int)threadIdx.x; c < R; c += THREADS) {
      double t = 0.0;
      for (int l = 0; l < RL; ++l) t += csum[l * R + c];
      ((double*)p.part2)[(int64_t)blockIdx.x * R + c] = t;
    }
  }
}

// variant 3: narrow-N row products C[w, 0:R] = X[w, 0:K] @ Y[0:K, 0:R].
// One warp per RW (4 or 8) rows per iteration; lane l owns k in {l*VW + 32*VW*i}
// for i < KI, with the matching Y rows held in registers for the whole
// kernel.  Rows stream through 16-byte loads (RW rows x KI vectors in
// flight per lane), partial dots reduce with xor shuffles, and lane
// rr*R + r stores element (rr, r).
template <typename T> struct vec16;
template <> struct vec16<float> { using V = float4; static constexpr int W = 4; };
template <> struct vec16<double> { using V = double2; static constexpr int W = 2; };

template <typename T>
RT_DEV void unpack(const typename vec16<T>::V& v, T* out);
template <> RT_DEV void unpack<float>(const float4& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
template <> RT_DEV void unpack<double>(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
RT_DEV void unpack_zero(float4& v) { v = make_float4(0.f, 0.f, 0.f, 0.f); }
RT_DEV void unpack_zero(double2& v) { v = make_double2(0.0, 0.0); }

// the RW x R dot products of a warp (lane partials in acc) reduced and
// stored with the bias / accumulate / tanh epilogue (k_thin_rows)
template <typename T, int R, int RW>
RT_DEV void rows_reduce_store(const rt_thin_params& p, int64_t w0, T (&acc)[RW][R], const T (&bias)[R],
                              int lane, int r1, T* Cp, int64_t wlim) {
    // the RW x R dot products across the warp by recursive halving: at each
    // level a lane keeps half of its values and receives the partner's copy
    // of that half (NV - 1 + 5 - log2 NV shuffles instead of 5 NV)
    constexpr int NV = RW * R;
    constexpr int LG = NV >= 32 ? 5 : NV >= 16 ? 4 : NV >= 8 ? 3 : NV >= 4 ? 2 : NV >= 2 ? 1 : 0;
    static_assert((1 << LG) == NV, "power-of-two row x output count");
    T v[NV];
#pragma unroll
    for (int rr = 0; rr < RW; ++rr)
#pragma unroll
      for (int r = 0; r < R; ++r) v[rr * R + r] = acc[rr][r];
#pragma unroll
    for (int sl = 0; sl < LG; ++sl) {
      const int n = NV >> sl, o = 16 >> sl;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < n / 2; ++i) {
        const T send = up ? v[i] : v[i + n / 2];
        const T keep = up ? v[i + n / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
#pragma unroll
    for (int o = 16 >> LG; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    const T mine = v[0];
    int idx = 0;
#pragma unroll
    for (int sl = 0; sl < LG; ++sl) idx |= ((lane >> (4 - sl)) & 1) << (LG - 1 - sl);
    if ((lane & ((1 << (5 - LG)) - 1)) == 0) {
      const int rr = idx / R, r = idx - rr * R;
      const int64_t w = w0 + rr;
      if (w < wlim && r < p.r) {
        T* cptr = r < r1 ? Cp + wdec(p.W, w, p.C.s1) + r * p.C.s2[0]
                         : (T*)p.C2.ptr + p.C2.off + wdec(p.W, w, p.C2.s1) + (r - r1) * p.C2.s2[0];
        T a = mine;
        if (p.accumulate) a += *cptr;
        a += bias[r];
        if (p.epilogue == 1) a = epi_tanh<T>(a);
        *cptr = a;
      }
    }
}

template <typename T, int R, int KI>
__global__ void __launch_bounds__(THREADS) k_thin_rows(const __grid_constant__ rt_thin_params p) {
  using V = typename vec16<T>::V;
  constexpr int VW = vec16<T>::W;
  constexpr int RW = (R * KI * VW >= 16) ? 4 : 8;   // rows per warp iteration
  const int lane = threadIdx.x & 31;
  const int K = (int)p.k;
  const T* X = (const T*)p.X.ptr + p.X.off;
  const T* Y = (const T*)p.Y.ptr + p.Y.off;
  T* Cp = (T*)p.C.ptr + p.C.off;
  const int64_t xk = p.X.s1[0];
  // outputs r < r1 from (Y, bias, C); r1 <= r < r from the sibling (Y2, bias2, C2)
  const int r1 = (int)(p.r - p.r2);
  const T* Y2 = (const T*)p.Y2.ptr + p.Y2.off;
  T y[KI][VW][R];
#pragma unroll
  for (int i = 0; i < KI; ++i)
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      const int k = (i * 32 + lane) * VW + j;
#pragma unroll
      for (int r = 0; r < R; ++r)
        y[i][j][r] = !(k < K && r < p.r) ? (T)0
                     : r < r1 ? Y[k * p.Y.s1[0] + r * p.Y.s2[0]]
                              : Y2[k * p.Y2.s1[0] + (r - r1) * p.Y2.s2[0]];
    }
  T bias[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    bias[r] = r < r1 ? (p.bias.ptr ? load_as<T>((const void*)p.bias.ptr, p.bias.dtype,
                                                 p.bias.off + r * p.bias.s2[0]) : (T)0)
            : r < p.r ? (p.bias2.ptr ? load_as<T>((const void*)p.bias2.ptr, p.bias2.dtype,
                                                   p.bias2.off + (r - r1) * p.bias2.s2[0]) : (T)0)
                      : (T)0;
  const int64_t gw = (int64_t)blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (THREADS / 32);
  for (int64_t w0 = gw * RW; w0 < p.w; w0 += nw * RW) {
    T acc[RW][R];
#pragma unroll
    for (int rr = 0; rr < RW; ++rr)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[rr][r] = (T)0;
    int64_t xo[RW];
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      const int64_t w = w0 + rr < p.w ? w0 + rr : p.w - 1;
      xo[rr] = wdec(p.W, w, p.X.s2);
    }
    if (p.vec) {
      V xv[RW][KI];
#pragma unroll
      for (int rr = 0; rr < RW; ++rr)
#pragma unroll
        for (int i = 0; i < KI; ++i) {
          const int k = (i * 32 + lane) * VW;
          if (k < K) xv[rr][i] = __ldcs(reinterpret_cast<const V*>(X + xo[rr] + k));
          else unpack_zero(xv[rr][i]);
        }
#pragma unroll
      for (int rr = 0; rr < RW; ++rr)
#pragma unroll
        for (int i = 0; i < KI; ++i) {
          T xs[VW];
          unpack<T>(xv[rr][i], xs);
          // acc[rr][r] = fma(x, y[r], acc[rr][r]) per r (FFMA2 on r pairs)
#pragma unroll
          for (int j = 0; j < VW; ++j) fma_bcast<R>(acc[rr], y[i][j], xs[j]);
        }
    } else {
#pragma unroll
      for (int rr = 0; rr < RW; ++rr)
#pragma unroll
        for (int i = 0; i < KI; ++i)
#pragma unroll
          for (int j = 0; j < VW; ++j) {
            const int k = (i * 32 + lane) * VW + j;
            const T x = k < K ? __ldcs(X + xo[rr] + k * xk) : (T)0;
            fma_bcast<R>(acc[rr], y[i][j], x);
          }
    }
    rows_reduce_store<T, R, RW>(p, w0, acc, bias, lane, r1, Cp, p.w);
  }
}

}  // namespace

// variant 3 with its rows streamed by cp.async.bulk (p.vec == 2, fp32,
// K <= 256 contiguous 16-byte-aligned floats per row): the per-warp
// 16-byte row loads of k_thin_rows left the kernel memory-latency bound
// (ncu: 41% of DRAM peak, 128 registers for the loads in flight).  CTA s
// takes a contiguous range of rows; a stage is 8 warps x RW rows, copied
// one row per lane of warp 0 into a 3-stage mbarrier ring; every warp then
// runs k_thin_rows' arithmetic on its RW rows from shared memory (same
// fma order, same reduction: bit-identical outputs).
template <int R, int KI>
__global__ void __launch_bounds__(THREADS, 2) k_thin_rows_bulk(const __grid_constant__ rt_thin_params p) {
  using T = float;
  using V = float4;
  constexpr int VW = 4, KP = KI * 32 * VW;
  constexpr int RW = (R * KI * VW >= 16) ? 4 : 8;
  constexpr int SR = (THREADS / 32) * RW;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  float* xs = (float*)sm_raw;                          // [ST][SR][KP]
  uint64_t* bars = (uint64_t*)(xs + BK_ST * SR * KP);
  const int tid = (int)threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int K = (int)p.k;
  const T* X = (const T*)p.X.ptr + p.X.off;
  const T* Y = (const T*)p.Y.ptr + p.Y.off;
  T* Cp = (T*)p.C.ptr + p.C.off;
  const int r1 = (int)(p.r - p.r2);
  const T* Y2 = (const T*)p.Y2.ptr + p.Y2.off;
  T y[KI][VW][R];
#pragma unroll
  for (int i = 0; i < KI; ++i)
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      const int k = (i * 32 + lane) * VW + j;
#pragma unroll
      for (int r = 0; r < R; ++r)
        y[i][j][r] = !(k < K && r < p.r) ? (T)0
                     : r < r1 ? Y[k * p.Y.s1[0] + r * p.Y.s2[0]]
                              : Y2[k * p.Y2.s1[0] + (r - r1) * p.Y2.s2[0]];
    }
  T bias[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    bias[r] = r < r1 ? (p.bias.ptr ? load_as<T>((const void*)p.bias.ptr, p.bias.dtype,
                                                 p.bias.off + r * p.bias.s2[0]) : (T)0)
            : r < p.r ? (p.bias2.ptr ? load_as<T>((const void*)p.bias2.ptr, p.bias2.dtype,
                                                   p.bias2.off + (r - r1) * p.bias2.s2[0]) : (T)0)
                      : (T)0;
  const int64_t per = (p.w + gridDim.x - 1) / gridDim.x;
  const int64_t q0 = (int64_t)blockIdx.x * per;
  const int64_t q1 = q0 + per < p.w ? q0 + per : p.w;
  const int nst = q1 > q0 ? (int)((q1 - q0 + SR - 1) / SR) : 0;
  if (tid == 0) {
    for (int i = 0; i < BK_ST; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bk_su32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int it, int st) {       // warp 0: one row per lane
    const int64_t wb = q0 + (int64_t)it * SR;
    const int n = (int)(q1 - wb < SR ? q1 - wb : SR);
    const uint32_t bar = bk_su32(bars + st);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   ::"r"(bar), "r"((uint32_t)(n * K * 4)) : "memory");
    __syncwarp();
    for (int i = lane; i < n; i += 32)
      bk_copy(bk_su32(xs + (st * SR + i) * KP), X + wdec(p.W, wb + i, p.X.s2), (uint32_t)(K * 4), bar);
  };
  if (tid < 32)
    for (int it = 0; it < BK_ST && it < nst; ++it) issue(it, it);
  for (int it = 0; it < nst; ++it) {
    const int st = it % BK_ST;
    bk_wait(bk_su32(bars + st), (uint32_t)((it / BK_ST) & 1));
    const int64_t w0 = q0 + (int64_t)it * SR + wp * RW;
    if (w0 < q1) {
      T acc[RW][R];
#pragma unroll
      for (int rr = 0; rr < RW; ++rr)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[rr][r] = (T)0;
#pragma unroll
      for (int rr = 0; rr < RW; ++rr) {
        const float* xr = xs + (st * SR + wp * RW + rr) * KP;
#pragma unroll
        for (int i = 0; i < KI; ++i) {
          const int k = (i * 32 + lane) * VW;
          // rows past q1 hold stale data: their outputs are not stored
          V xv;
          if (k < K) xv = *reinterpret_cast<const V*>(xr + k);
          else unpack_zero(xv);
          T xv_[VW];
          unpack<T>(xv, xv_);
#pragma unroll
          for (int j = 0; j < VW; ++j) fma_bcast<R>(acc[rr], y[i][j], xv_[j]);
        }
      }
      // rows in [q1, p.w) belong to the next CTA: stored only below q1
      rows_reduce_store<T, R, RW>(p, w0, acc, bias, lane, r1, Cp, q1);
    }
    __syncthreads();
    if (tid < 32 && it + BK_ST < nst) issue(it + BK_ST, st);
  }
}

extern "C" void* rt_kernel_thin_rows_bulk(int r, int k) {
  if (k > 256) return nullptr;
#define RB(R) if (r <= R) return k <= 128 ? (void*)k_thin_rows_bulk<R, 1> : (void*)k_thin_rows_bulk<R, 2>;
  RB(1) RB(2) RB(4) RB(8)
#undef RB
  return nullptr;
}

extern "C" void* rt_kernel_thin_rows(int f64, int r, int k) {
#define RT_ROWS(T, R)                                            \
  if (r <= R) {                                                  \
    constexpr int C = 32 * vec16<T>::W;                          \
    if (k <= C) return (void*)k_thin_rows<T, R, 1>;              \
    if (k <= 2 * C) return (void*)k_thin_rows<T, R, 2>;          \
    if (k <= 4 * C) return (void*)k_thin_rows<T, R, 4>;          \
    return (void*)k_thin_rows<T, R, 8>;                          \
  }
  if (f64) {
    RT_ROWS(double, 1) RT_ROWS(double, 2) RT_ROWS(double, 4) RT_ROWS(double, 8)
  } else {
    RT_ROWS(float, 1) RT_ROWS(float, 2) RT_ROWS(float, 4) RT_ROWS(float, 8)
  }
#undef RT_ROWS
  return nullptr;
}

// vectorised variant 2 (p.vec): mode 0 plain/tanh/accumulate, 1 gate, 2
// gate + a second product (K2 <= 4); k = K (KP <= 16 fp32, <= 8 fp64)
extern "C" void* rt_kernel_thin_vec(int mode, int f64, int k) {
#define SV(T, KP)                                                              \
  (mode == 0 ? (void*)k_thin_smallv<T, KP> : mode == 1 ? (void*)k_thin_smallv<T, KP, true> \
                                                         : (void*)k_thin_smallv<T, KP, true, 4>)
  if (f64) {
    if (k <= 4) return SV(double, 4);
    if (k <= 8) return SV(double, 8);
    return nullptr;
  }
  if (k <= 4) return SV(float, 4);
  if (k <= 8) return SV(float, 8);
  if (k <= 16) return SV(float, 16);
  return nullptr;
#undef SV
}

extern "C" void* rt_kernel_thin_bulk(int r, int ones) {
#define BK(R) (ones ? (void*)k_thin_contract_bulk<R, true> : (void*)k_thin_contract_bulk<R, false>)
  if (r <= 4) return BK(4);
  if (r <= 8) return BK(8);
  if (r <= 16) return BK(16);
  return nullptr;   // r > 16: k_thin_contract (4 x 32 accumulators would spill)
#undef BK
}

extern "C" void* rt_kernel_thin(int variant, int f64, int r) {
  if (variant == 6) {
    // variant 1 with the ones column (bias gradient of the same contraction)
    if (f64) {
      if (r <= 4) return (void*)k_thin_contract<double, 4, true>;
      if (r <= 8) return (void*)k_thin_contract<double, 8, true>;
      if (r <= 16) return (void*)k_thin_contract<double, 16, true>;
      return (void*)k_thin_contract<double, 32, true>;
    }
    if (r <= 4) return (void*)k_thin_contract<float, 4, true>;
    if (r <= 8) return (void*)k_thin_contract<float, 8, true>;
    if (r <= 16) return (void*)k_thin_contract<float, 16, true>;
    return (void*)k_thin_contract<float, 32, true>;
  }
  if (variant == 5) {
    // variant 2 + gate + a second product with K2 <= 4 (runtime.cu passes 5)
    if (f64) {
      if (r <= 4) return (void*)k_thin_smallk<double, 4, true, 4>;
      if (r <= 8) return (void*)k_thin_smallk<double, 8, true, 4>;
      return nullptr;
    }
    if (r <= 4) return (void*)k_thin_smallk<float, 4, true, 4>;
    if (r <= 8) return (void*)k_thin_smallk<float, 8, true, 4>;
    if (r <= 16) return (void*)k_thin_smallk<float, 16, true, 4>;
    return nullptr;
  }
  if (variant == 4) {
    // variant 2 with the tanh-VJP gate epilogue (runtime.cu passes 4)
    if (f64) {
      if (r <= 4) return (void*)k_thin_smallk<double, 4, true>;
      if (r <= 8) return (void*)k_thin_smallk<double, 8, true>;
      if (r <= 16) return (void*)k_thin_smallk<double, 16, true>;
      return (void*)k_thin_smallk<double, 32, true>;
    }
    if (r <= 4) return (void*)k_thin_smallk<float, 4, true>;
    if (r <= 8) return (void*)k_thin_smallk<float, 8, true>;
    if (r <= 16) return (void*)k_thin_smallk<float, 16, true>;
    return (void*)k_thin_smallk<float, 32, true>;
  }
  if (variant == 2) {
    // r carries K for this variant (see lower.py _gemm_thin)
    if (f64) {
      if (r <= 4) return (void*)k_thin_smallk<double, 4>;
      if (r <= 8) return (void*)k_thin_smallk<double, 8>;
      if (r <= 16) return (void*)k_thin_smallk<double, 16>;
      return (void*)k_thin_smallk<double, 32>;
    }
    if (r <= 4) return (void*)k_thin_smallk<float, 4>;
    if (r <= 8) return (void*)k_thin_smallk<float, 8>;
    if (r <= 16) return (void*)k_thin_smallk<float, 16>;
    return (void*)k_thin_smallk<float, 32>;
  }
  if (f64) {
    if (r <= 4) return (void*)k_thin_contract<double, 4>;
    if (r <= 8) return (void*)k_thin_contract<double, 8>;
    if (r <= 16) return (void*)k_thin_contract<double, 16>;
    return (void*)k_thin_contract<double, 32>;
  }
  if (r <= 4) return (void*)k_thin_contract<float, 4>;
  if (r <= 8) return (void*)k_thin_contract<float, 8>;
  if (r <= 16) return (void*)k_thin_contract<float, 16>;
  return (void*)k_thin_contract<float, 32>;
}
