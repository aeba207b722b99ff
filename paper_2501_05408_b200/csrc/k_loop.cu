// RT_K_LOOP — a whole row-local loop in one persistent launch.
//
// The reference runs a recurrence such as the acting loop
//     o[b,t] -> policy MLP -> a[b,t] -> env -> o[b,t+1]
// one (node, point) at a time (runtime.py:344-389).  The planner turns it
// into a loop over t whose body evaluates every node for all envs b; here
// that whole loop is ONE kernel: each CTA owns a block of rows (envs) and
// steps through t itself, running every body op on its rows with a
// __syncthreads between ops.  Rows never read other rows (checked by the
// planner), so no grid-wide synchronisation is needed and the per-step cost
// is the ops' latency, not ~6 kernel launches.
//
// Ops: the EW program VM, a row-block GEMM (+bias, tanh) streaming the
// weights from L2, the synthetic env (with its normals pre-drawn by an RNG
// launch hoisted out of the loop), and per-row RNG draws.
#include "common.cuh"
#include "rng.cuh"

#define LOOP_THREADS 256
#define LOOP_MAXR 16   // max GEMM rows held per thread (rows_per_cta * m)

RT_DEV int64_t fold_gop_off(const rt_gop& g, const int64_t* env) {
  int64_t o = g.off;
  for (int e = 0; e < RT_MAXENV; ++e) o += env[e] * g.off_env[e];
  return o;
}

RT_DEV int64_t gdec32(const rt_gbox& b, int64_t flat, const int64_t* s) {
  uint32_t f = (uint32_t)flat;
  int64_t o = 0;
  for (int d = b.nd - 1; d >= 0; --d) {
    uint32_t e = (uint32_t)b.ext[d];
    uint32_t q = f / e;
    o += (int64_t)(f - q * e) * s[d];
    f = q;
  }
  return o;
}

// ---------------------------------------------------------------- EW rows

template <typename T>
RT_DEV void ew_rows(const rt_ew_params& p, const int64_t* env, int64_t f0, int64_t f1,
                    rt_fold* sfold) {
  // fold every view once per step (thread i -> view i; slot 0 = output)
  const int nv = p.nin + 1;
  if (threadIdx.x < nv) sfold[threadIdx.x] = fold_of(threadIdx.x == 0 ? p.out : p.in[threadIdx.x - 1], env);
  __syncthreads();
  int64_t idx[RT_MAXD];
  const int nd = p.box.nd;
  for (int64_t f = f0 + threadIdx.x; f < f1; f += blockDim.x) {
    decompose(p.box, f, idx);
    T v = (T)0;
    int64_t dummy;
    vm_run_env<T>(p.code, 0, p.konst, p.h, env, idx, nd, p.in, sfold + 1, &v, &dummy);
    store_as<T>((void*)p.out.ptr, p.out.dtype, fview_off(p.out, sfold, nd, idx), v);
  }
}

// ---------------------------------------------------------------- GEMM rows
// C[r, n] = sum_k A[r, k] B[k, n] for the CTA's rows r in [m0, m1) of M
// (M = slab rows x m), all n.  A rows are staged in shared memory; B is
// streamed from L2 with each thread owning columns and all rows (B reuse).

template <typename T>
RT_DEV void gemm_rows(const rt_gemm_params& p, const int64_t* env, int64_t m0, int64_t m1,
                      unsigned char* smem) {
  const int64_t K = p.k, Nn = p.n;
  const int mr = (int)(m1 - m0);
  T* As = (T*)smem;                                        // [mr][K]
  int64_t* kB = (int64_t*)(smem + ((mr * K * sizeof(T) + 15) / 16) * 16);   // [K]
  const int64_t aoff = fold_gop_off(p.A, env);
  const int64_t boff = fold_gop_off(p.B, env);
  const int64_t coff = fold_gop_off(p.C, env);
  const int64_t biasoff = p.bias.ptr ? fold_gop_off(p.bias, env) : 0;
  // stage A rows
  for (int64_t i = threadIdx.x; i < (int64_t)mr * K; i += blockDim.x) {
    int r = (int)(i / K);
    int64_t k = i - (int64_t)r * K;
    int64_t o = aoff + gdec32(p.M, m0 + r, p.A.s1) + gdec32(p.K, k, p.A.s2);
    As[i] = load_as<T>((const void*)p.A.ptr, p.A.dtype, o);
  }
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) kB[k] = gdec32(p.K, k, p.B.s1);
  __syncthreads();
  const void* Bp = (const void*)p.B.ptr;
  if (Nn >= 64 || mr * Nn >= (int64_t)blockDim.x) {
    // thread owns column n, all rows
    for (int64_t n = threadIdx.x; n < Nn; n += blockDim.x) {
      T acc[LOOP_MAXR];
#pragma unroll
      for (int r = 0; r < LOOP_MAXR; ++r) acc[r] = (T)0;
      const int64_t cb = boff + gdec32(p.N, n, p.B.s2);
      for (int64_t k = 0; k < K; ++k) {
        T b = load_as<T>(Bp, p.B.dtype, cb + kB[k]);
#pragma unroll
        for (int r = 0; r < LOOP_MAXR; ++r)
          if (r < mr) acc[r] = fma(As[r * K + k], b, acc[r]);
      }
      T bias = p.bias.ptr ? load_as<T>((const void*)p.bias.ptr, p.bias.dtype,
                                       biasoff + gdec32(p.N, n, p.bias.s2)) : (T)0;
      const int64_t cn = gdec32(p.N, n, p.C.s2);
#pragma unroll
      for (int r = 0; r < LOOP_MAXR; ++r) {
        if (r >= mr) break;
        T v = acc[r] + bias;
        if (p.epilogue == 1) v = vm_tanh<T>(v);
        store_as<T>((void*)p.C.ptr, p.C.dtype, coff + gdec32(p.M, m0 + r, p.C.s1) + cn, v);
      }
    }
  } else {
    // few outputs: a group of lanes splits K for each output, shuffle-reduce
    const int outs = (int)(mr * Nn);
    int g = 1;
    while (g * 2 * outs <= (int)blockDim.x && g < 32) g *= 2;
    const int lane_in = threadIdx.x % g;
    const int per = (int)blockDim.x / g;
    for (int base = 0; base < outs; base += per) {
      const int o = base + (int)threadIdx.x / g;
      const bool act = o < outs;
      const int r = act ? o / (int)Nn : 0;
      const int64_t n = act ? o - (int64_t)r * Nn : 0;
      const int64_t cb = boff + gdec32(p.N, n, p.B.s2);
      T acc = (T)0;
      if (act)
        for (int64_t k = lane_in; k < K; k += g)
          acc = fma(As[r * K + k], load_as<T>(Bp, p.B.dtype, cb + kB[k]), acc);
      for (int sft = g / 2; sft > 0; sft >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, sft, g);
      if (act && lane_in == 0) {
        T v = acc;
        if (p.bias.ptr)
          v += load_as<T>((const void*)p.bias.ptr, p.bias.dtype, biasoff + gdec32(p.N, n, p.bias.s2));
        if (p.epilogue == 1) v = vm_tanh<T>(v);
        store_as<T>((void*)p.C.ptr, p.C.dtype, coff + gdec32(p.M, m0 + r, p.C.s1) + gdec32(p.N, n, p.C.s2), v);
      }
    }
  }
}

// ---------------------------------------------------------------- UDF rows

RT_DEV double pairwise_sum_l(const void* base, int dtype, int64_t off, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += load_as<double>(base, dtype, off + i);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = load_as<double>(base, dtype, off + j);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += load_as<double>(base, dtype, off + i + j);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += load_as<double>(base, dtype, off + i);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum_l(base, dtype, off, n2) + pairwise_sum_l(base, dtype, off + n2, n - n2);
}

RT_DEV int push_words_l(uint32_t* w, int n, int64_t v) {
  uint64_t u = (uint64_t)v;
  if (u == 0) { w[n++] = 0; return n; }
  while (u) { w[n++] = (uint32_t)(u & 0xffffffffu); u >>= 32; }
  return n;
}

RT_DEV void udf_rows(const rt_udf_params& p, const rt_loop_op& op, const int64_t* env,
                     int64_t r0, int64_t r1, int64_t tix) {
  int64_t idx[RT_MAXD];
  for (int64_t row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
    decompose(p.box, row, idx);
    double base = p.salt;
    for (int k = 0; k < p.nin; ++k) {
      int64_t c = p.in_count[k];
      if (c == 0) continue;
      rt_fold f = fold_of(p.in[k], env);
      int64_t o = fview_off(p.in[k], &f, p.box.nd, idx);
      base = base + pairwise_sum_l((const void*)p.in[k].ptr, p.in[k].dtype, o, c) / (double)c;
    }
    const double* noise = (const double*)op.noise;
    int64_t nz = op.noise_off + row * op.noise_row + tix * op.noise_step;
    rt_pcg64 g;
    if (!noise) {
      uint32_t words[8 + 2 * RT_MAXD];
      int n = 0;
      for (int i = 0; i < p.nprefix; ++i) words[n++] = p.prefix[i];
      for (int j = 0; j < p.ncoord; ++j) {
        int s = p.coord_src[j];
        n = push_words_l(words, n, s >= 0 ? idx[s] : env[-1 - s]);
      }
      pcg64_seed(g, words, n);
    }
    for (int j = 0; j < p.nout; ++j) {
      rt_fold f = fold_of(p.out[j], env);
      int64_t o = fview_off(p.out[j], &f, p.box.nd, idx);
      int kind = p.out_kind[j];
      double tb = kind == RT_BOOL ? tanh(base) : 0.0;
      for (int e = 0; e < p.out_count[j]; ++e) {
        double z = noise ? noise[nz++] : pcg64_normal(g);
        double v;
        if (kind == RT_BOOL) v = (tb + z > 0.8) ? 1.0 : 0.0;
        else if (kind == RT_I64) v = floor(3.0 * tanh(base + z));
        else v = tanh(base + 0.3 * z);
        store_as<double>((void*)p.out[j].ptr, p.out[j].dtype, o + e, v);
      }
    }
  }
}

RT_DEV void rng_rows(const rt_rng_params& p, const int64_t* env, int64_t r0, int64_t r1) {
  int64_t idx[RT_MAXD];
  uint32_t words[8 + 2 * RT_MAXD];
  for (int64_t row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
    decompose(p.box, row, idx);
    int n = 0;
    for (int i = 0; i < p.nprefix; ++i) words[n++] = p.prefix[i];
    for (int j = 0; j < p.ncoord; ++j) {
      int s = p.coord_src[j];
      n = push_words_l(words, n, s >= 0 ? idx[s] : env[-1 - s]);
    }
    rt_pcg64 g;
    pcg64_seed(g, words, n);
    rt_fold f = fold_of(p.out, env);
    int64_t o = fview_off(p.out, &f, p.box.nd, idx);
    for (int j = 0; j < p.count; ++j) {
      double v = p.dist == 0 ? pcg64_normal(g) : pcg64_double(g);
      store_as<double>((void*)p.out.ptr, p.out.dtype, o + j, v);
    }
  }
}

// ---------------------------------------------------------------- the loop

__global__ void __launch_bounds__(LOOP_THREADS) k_loop(const __grid_constant__ rt_loop_params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ rt_fold sfold[RT_MAXIN + 1];
  int64_t env[RT_MAXENV];
  for (int e = 0; e < RT_MAXENV; ++e) env[e] = p.h.env[e];
  const int64_t r0 = (int64_t)blockIdx.x * p.rows_per_cta;
  const int64_t r1 = min(p.rows, r0 + p.rows_per_cta);
  if (r0 >= r1) return;
  const rt_loop_op* ops = (const rt_loop_op*)p.ops;
  int64_t tix = 0;
  for (int64_t t = p.start; p.step > 0 ? t < p.stop : t > p.stop; t += p.step, ++tix) {
    env[p.slot] = t;
    for (int i = 0; i < p.nops; ++i) {
      const rt_loop_op& op = ops[i];
      switch (op.kernel) {
        case RT_K_EW: {
          const rt_ew_params& q = *(const rt_ew_params*)op.params;
          if (op.f64) ew_rows<double>(q, env, r0 * op.row_elems, r1 * op.row_elems, sfold);
          else ew_rows<float>(q, env, r0 * op.row_elems, r1 * op.row_elems, sfold);
          break;
        }
        case RT_K_GEMM: {
          const rt_gemm_params& q = *(const rt_gemm_params*)op.params;
          if (op.f64) gemm_rows<double>(q, env, r0 * op.row_elems, r1 * op.row_elems, smem);
          else gemm_rows<float>(q, env, r0 * op.row_elems, r1 * op.row_elems, smem);
          break;
        }
        case RT_K_UDF:
          udf_rows(*(const rt_udf_params*)op.params, op, env, r0, r1, t);
          break;
        case RT_K_RNG:
          rng_rows(*(const rt_rng_params*)op.params, env, r0, r1);
          break;
        default:
          break;
      }
      __syncthreads();
    }
  }
}

extern "C" void* rt_kernel_loop() { return (void*)k_loop; }
