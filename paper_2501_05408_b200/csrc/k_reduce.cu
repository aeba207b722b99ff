// RT_K_REDUCE — sums and discounted sums over payload axes and over gathered
// (possibly ragged) index ranges.  Replaces the reference's per-point
// `_k_sum` (runtime.py:95-96), `_k_discounted_sum` (runtime.py:108-122),
// `_k_window_reduce` (runtime.py:192-211, direct form for short windows) and
// the slice gather of `_Oracle.read` (runtime.py:414-425) feeding them: the
// gathered range is never materialised, the reduction walks it in place.
// Accumulation is in fp64 for every input type.
#include "common.cuh"

template <typename T>
RT_DEV double red_weight(const rt_reduce_params& p, int64_t k, int64_t n) {
  if (p.op == 0) return 1.0;
  int64_t e = p.reverse ? (n - 1 - k) : k;
  // runtime.py:108-112: f64 gamma**arange, cast to the input dtype
  return (double)(T)pow(p.gamma, (double)e);
}

template <typename T>
RT_DEV void red_setup(const rt_reduce_params& p, const int64_t* idx, int64_t* len,
                      int64_t* base, int64_t* total) {
  const int nd = p.box.nd;
  int64_t off = view_off(p.in, nd, idx);
  int64_t tot = 1;
  for (int j = 0; j < p.nred; ++j) {
    int64_t L;
    if (p.len_prog[j] < 0) {
      L = p.len0[j];
      for (int d = 0; d < nd; ++d) L += p.len_a[j][d] * idx[d];
    } else {
      T dv;
      vm_run<T>(p.code, p.len_prog[j], p.konst, p.h, idx, nd, &p.in, &dv, &L);
    }
    if (L < 0) L = 0;
    len[j] = L;
    tot *= L;
    if (p.lo_prog[j] >= 0) {
      int64_t lo = 0;
      T dv;
      vm_run<T>(p.code, p.lo_prog[j], p.konst, p.h, idx, nd, &p.in, &dv, &lo);
      off += lo * p.red_stride[j];
    }
  }
  *base = off;
  *total = tot;
}

template <typename T>
RT_DEV double red_term(const rt_reduce_params& p, int64_t base, const int64_t* len, int64_t k) {
  if (p.nred == 1 && p.op == 0)
    return (double)load_as<T>((const void*)p.in.ptr, p.in.dtype, base + k * p.red_stride[0]);
  int64_t off = base;
  int64_t r = k, k0 = 0;
  for (int j = p.nred - 1; j >= 0; --j) {
    int64_t q = r / len[j];
    int64_t kj = r - q * len[j];
    r = q;
    off += kj * p.red_stride[j];
    if (j == 0) k0 = kj;
  }
  T x = load_as<T>((const void*)p.in.ptr, p.in.dtype, off);
  if (p.op == 0) return (double)x;
  T w = (T)red_weight<T>(p, k0, len[0]);
  return (double)(T)(x * w);
}

template <typename T>
__global__ void __launch_bounds__(256) k_reduce_thread(const __grid_constant__ rt_reduce_params p) {
  int64_t idx[RT_MAXD];
  int64_t len[4];
  const int nd = p.box.nd;
  // plain sum over one contiguous fp32 dim of constant length 4n (e.g. the
  // per-point mean of a 16-wide observation): vector loads
  bool vec4 = p.nred == 1 && p.op == 0 && p.len_prog[0] < 0 && p.lo_prog[0] < 0 &&
              p.red_stride[0] == 1 && p.in.dtype == RT_F32 && (p.len0[0] & 3) == 0 &&
              (p.in.ptr & 15) == 0;
  for (int d = 0; d < nd; ++d) vec4 = vec4 && p.len_a[0][d] == 0;
  for (int64_t flat = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; flat < p.total;
       flat += (int64_t)gridDim.x * blockDim.x) {
    decompose(p.box, flat, idx);
    int64_t base, tot;
    red_setup<T>(p, idx, len, &base, &tot);
    double acc = 0.0;
    if (vec4 && (base & 3) == 0) {
      // contiguous fp32 run of constant length: 16-byte loads, same order
      const float4* q = reinterpret_cast<const float4*>((const float*)p.in.ptr + base);
      for (int64_t k4 = 0; k4 < tot / 4; ++k4) {
        const float4 v = __ldg(q + k4);
        acc += (double)v.x; acc += (double)v.y; acc += (double)v.z; acc += (double)v.w;
      }
    } else {
      for (int64_t k = 0; k < tot; ++k) acc += red_term<T>(p, base, len, k);
    }
    store_as<double>((void*)p.out.ptr, p.out.dtype, view_off(p.out, nd, idx), acc);
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) k_reduce_block(const __grid_constant__ rt_reduce_params p) {
  __shared__ double sh[32];
  int64_t idx[RT_MAXD];
  int64_t len[4];
  const int nd = p.box.nd;
  for (int64_t flat = blockIdx.x; flat < p.total; flat += gridDim.x) {
    decompose(p.box, flat, idx);
    int64_t base, tot;
    red_setup<T>(p, idx, len, &base, &tot);
    double acc = 0.0;
    for (int64_t k = threadIdx.x; k < tot; k += blockDim.x) acc += red_term<T>(p, base, len, k);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = acc;
    __syncthreads();
    if (w == 0) {
      int nw = blockDim.x >> 5;
      double v = l < nw ? sh[l] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (l == 0) store_as<double>((void*)p.out.ptr, p.out.dtype, view_off(p.out, nd, idx), v);
    }
    __syncthreads();
  }
}

// Warp mode: one warp per output for medium contiguous ranges (e.g. the
// per-point sum over a 256-wide payload axis): lanes read consecutive
// elements, fixed shuffle tree (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) k_reduce_warp(const __grid_constant__ rt_reduce_params p) {
  int64_t idx[RT_MAXD];
  int64_t len[4];
  const int nd = p.box.nd;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool fast = p.nred == 1 && p.op == 0 && p.in.dtype == (sizeof(T) == 8 ? RT_F64 : RT_F32);
  for (int64_t flat = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); flat < p.total;
       flat += nw) {
    decompose(p.box, flat, idx);
    int64_t base, tot;
    red_setup<T>(p, idx, len, &base, &tot);
    double acc = 0.0;
    if (fast) {
      const T* src = (const T*)p.in.ptr + base;
      const int64_t st = p.red_stride[0];
      int64_t k = lane;
      for (; k + 96 < tot; k += 128) {
        T x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = src[(k + 32 * u) * st];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += (double)x[u];
      }
      for (; k < tot; k += 32) acc += (double)src[k * st];
    } else {
      for (int64_t k = lane; k < tot; k += 32) acc += red_term<T>(p, base, len, k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) store_as<double>((void*)p.out.ptr, p.out.dtype, view_off(p.out, nd, idx), acc);
  }
}

// Column mode: outputs contiguous in the input (e.g. a bias gradient summed
// over all T*E points of a [points, 256] tensor).  Pass 1: a block covers up
// to 256 outputs; with fewer outputs, 256/total lanes per output walk the
// rows interleaved and are combined in a fixed order in shared memory.  Each
// blockIdx.y takes one slice of the reduced range.  Pass 2 sums the fp64
// partials in a fixed order (deterministic).
#ifndef RT_REDUCE_RU
#define RT_REDUCE_RU 32
#endif
constexpr int RU = RT_REDUCE_RU;
template <typename T>
__global__ void __launch_bounds__(256) k_reduce_cols(const __grid_constant__ rt_reduce_params p) {
  __shared__ double red[256];
  int64_t idx[RT_MAXD];
  int64_t len[4];
  const int per_blk = p.total < 256 ? (int)p.total : 256;
  const int lanes = 256 / per_blk;
  const int oi = threadIdx.x % per_blk, lane = threadIdx.x / per_blk;
  const int64_t o = (int64_t)blockIdx.x * per_blk + oi;
  const int s = blockIdx.y;
  double acc = 0.0;
  if (lane < lanes && o < p.total) {
    decompose(p.box, o, idx);
    int64_t base, tot;
    red_setup<T>(p, idx, len, &base, &tot);
    const int64_t per = (tot + p.splits - 1) / p.splits;
    const int64_t k0 = s * per, k1 = min(tot, k0 + per);
    const bool fast = p.nred == 1 && p.op == 0 &&
                      p.in.dtype == (sizeof(T) == 8 ? RT_F64 : RT_F32);
    if (fast) {
      const T* src = (const T*)p.in.ptr + base;
      const int64_t st = p.red_stride[0];
      int64_t k = k0 + lane;
      // RU rows in flight per thread (8 left HBM short of bytes in flight:
      // 3.4 TB/s on the 1 GB bias-gradient sums; 16: 4.6 TB/s)
      for (; k + (RU - 1) * lanes < k1; k += RU * lanes) {
        T x[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) x[u] = __ldcs(src + (k + u * lanes) * st);
#pragma unroll
        for (int u = 0; u < RU; ++u) acc += (double)x[u];
      }
      for (; k < k1; k += lanes) acc += (double)src[k * st];
    } else {
      for (int64_t k = k0 + lane; k < k1; k += lanes) acc += red_term<T>(p, base, len, k);
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (lane == 0 && o < p.total) {
    double v = 0.0;
    for (int l = 0; l < lanes; ++l) v += red[l * per_blk + oi];
    ((double*)p.part)[(int64_t)s * p.total + o] = v;
  }
}

// Pass 2: one warp per output; lane l sums splits l, l+32, ... in order,
// then a fixed xor tree (deterministic; a thread per output walking up to
// 1024 partials serially took ~90 us per launch)
__global__ void __launch_bounds__(256) k_reduce_cols_fin(const __grid_constant__ rt_reduce_params p) {
  int64_t idx[RT_MAXD];
  const double* part = (const double*)p.part;
  const int lane = threadIdx.x & 31;
  for (int64_t o = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < p.total;
       o += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double acc = 0.0;
    for (int s = lane; s < p.splits; s += 32) acc += part[(int64_t)s * p.total + o];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (lane == 0) {
      decompose(p.box, o, idx);
      store_as<double>((void*)p.out.ptr, p.out.dtype, view_off(p.out, p.box.nd, idx), acc);
    }
  }
}

extern "C" void* rt_kernel_reduce_cols(int f64, int fin) {
  if (fin) return (void*)k_reduce_cols_fin;
  return f64 ? (void*)k_reduce_cols<double> : (void*)k_reduce_cols<float>;
}

extern "C" void* rt_kernel_reduce(int f64, int tpo) {
  if (tpo == 32) return f64 ? (void*)k_reduce_warp<double> : (void*)k_reduce_warp<float>;
  if (tpo > 1) return f64 ? (void*)k_reduce_block<double> : (void*)k_reduce_block<float>;
  return f64 ? (void*)k_reduce_thread<double> : (void*)k_reduce_thread<float>;
}
