// RT_K_RNG and RT_K_UDF — per-point seeded draws and the synthetic
// environment body, batched over whole slabs.
//   rng nodes: runtime.py:50-55 (`default_rng((seed, tag, *point))` then
//              standard_normal(shape) / uniform(0, 1, shape));
//   udf nodes: runtime.py:153-158 with the body of dsl.make_udf_fn
//              (dsl.py:288-307): base = salt + sum_k mean(float64(x_k));
//              per output: noise = standard_normal(shape) from the same
//              stream; f -> tanh(base + 0.3 noise), bool -> tanh(base) +
//              noise > 0.8, i64 -> floor(3 tanh(base + noise)).
#include "common.cuh"
#include "rng.cuh"

// Python int -> little-endian u32 words (0 -> [0]); bit_generator.pyx
// _int_to_uint32_array.
RT_DEV int push_words(uint32_t* w, int n, int64_t v) {
  uint64_t u = (uint64_t)v;
  if (u == 0) { w[n++] = 0; return n; }
  while (u) { w[n++] = (uint32_t)(u & 0xffffffffu); u >>= 32; }
  return n;
}

RT_DEV int assemble_words(uint32_t* w, const uint32_t* prefix, int nprefix, const int32_t* src,
                          int ncoord, const int64_t* idx, const int64_t* env, const int64_t* add) {
  int n = 0;
  for (int i = 0; i < nprefix; ++i) w[n++] = prefix[i];
  for (int j = 0; j < ncoord; ++j) {
    int s = src[j];
    int64_t c = s >= 0 ? idx[s] : env[-1 - s];
    n = push_words(w, n, c + add[j]);
  }
  return n;
}

__global__ void __launch_bounds__(128) k_rng(const __grid_constant__ rt_rng_params p) {
  int64_t idx[RT_MAXD];
  uint32_t words[8 + 2 * RT_MAXD];
  for (int64_t flat = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; flat < p.total;
       flat += (int64_t)gridDim.x * blockDim.x) {
    decompose(p.box, flat, idx);
    int n = assemble_words(words, p.prefix, p.nprefix, p.coord_src, p.ncoord, idx, p.h.env,
                           p.coord_add);
    rt_pcg64 g;
    pcg64_seed(g, words, n);
    int64_t o = view_off(p.out, p.box.nd, idx);
    for (int j = 0; j < p.count; ++j) {
      double v = p.dist == 0 ? pcg64_normal(g) : pcg64_double(g);
      store_as<double>((void*)p.out.ptr, p.out.dtype, o + j, v);
    }
  }
}

// numpy pairwise summation (umath loops_utils pairwise_sum), fp64
RT_DEV double pairwise_sum(const void* base, int dtype, int64_t off, int64_t n) {
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
  return pairwise_sum(base, dtype, off, n2) + pairwise_sum(base, dtype, off + n2, n - n2);
}

__global__ void __launch_bounds__(128) k_udf(const __grid_constant__ rt_udf_params p) {
  int64_t idx[RT_MAXD];
  uint32_t words[8 + 2 * RT_MAXD];
  for (int64_t flat = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; flat < p.total;
       flat += (int64_t)gridDim.x * blockDim.x) {
    decompose(p.box, flat, idx);
    double base = p.salt;
    for (int k = 0; k < p.nin; ++k) {
      int64_t c = p.in_count[k];
      if (c == 0) continue;
      int64_t o = view_off(p.in[k], p.box.nd, idx);
      base = base + pairwise_sum((const void*)p.in[k].ptr, p.in[k].dtype, o, c) / (double)c;
    }
    int n = assemble_words(words, p.prefix, p.nprefix, p.coord_src, p.ncoord, idx, p.h.env,
                           p.coord_add);
    rt_pcg64 g;
    pcg64_seed(g, words, n);
    for (int j = 0; j < p.nout; ++j) {
      int64_t o = view_off(p.out[j], p.box.nd, idx);
      int kind = p.out_kind[j];
      double tb = kind == RT_BOOL ? tanh(base) : 0.0;
      for (int e = 0; e < p.out_count[j]; ++e) {
        double noise = pcg64_normal(g);
        double v;
        if (kind == RT_BOOL) v = (tb + noise > 0.8) ? 1.0 : 0.0;
        else if (kind == RT_I64) v = floor(3.0 * tanh(base + noise));
        else v = tanh(base + 0.3 * noise);
        store_as<double>((void*)p.out[j].ptr, p.out[j].dtype, o + e, v);
      }
    }
  }
}

// standalone fill for tests: rows x count draws, entropy = prefix + coords[row]
__global__ void k_rng_fill(double* out, const uint32_t* prefix, int nprefix, const int64_t* coords,
                           int ncoord, int64_t rows, int count, int dist) {
  uint32_t words[8 + 2 * RT_MAXD];
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int n = 0;
    for (int i = 0; i < nprefix; ++i) words[n++] = prefix[i];
    for (int j = 0; j < ncoord; ++j) n = push_words(words, n, coords[r * ncoord + j]);
    rt_pcg64 g;
    pcg64_seed(g, words, n);
    for (int j = 0; j < count; ++j) out[r * count + j] = dist == 0 ? pcg64_normal(g) : pcg64_double(g);
  }
}

extern "C" void* rt_kernel_rng() { return (void*)k_rng; }
extern "C" void* rt_kernel_udf() { return (void*)k_udf; }
extern "C" void* rt_kernel_rng_fill() { return (void*)k_rng_fill; }
