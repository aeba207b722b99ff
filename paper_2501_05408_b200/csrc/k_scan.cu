// RT_K_SCAN — linear recurrence y[j] = x[j] + gamma * y[j -/+ 1] along one
// dim of a box.  One kernel serves the lifted scans and their vectorised
// forms (`_k_scan`/`_k_cumsum`/`_k_discounted_cumsum`, reference
// runtime.py:99-105, 125-146) and the suffix discounted return
// G[t] = dsum(r[t:T]) (runtime.py:115-122 gathered by runtime.py:414-425,
// O(T^2) in the reference), which is the reverse scan with the same gamma.
//
// Contiguous lines: one warp per line, 8 chunks of 32 elements in flight
// per batch, warp-shuffle scan of (A, B) affine pairs, carry across chunks.
// Strided lines: one thread per line (coalesced across lines), 8-deep
// prefetch.  Accumulation in fp64.
#include "common.cuh"

#define SCAN_UNROLL 8

RT_DEV void line_base(const rt_scan_params& p, int64_t line, int64_t* in0, int64_t* out0,
                      int64_t* sin, int64_t* sout, int64_t* L) {
  // decompose `line` over all dims except sdim
  int64_t r = line;
  int64_t oi = p.in.off, oo = p.out.off;
  for (int d = p.box.nd - 1; d >= 0; --d) {
    if (d == p.sdim) continue;
    int64_t e = p.box.ext[d];
    int64_t q = r / e;
    int64_t c = r - q * e;
    r = q;
    oi += c * p.in.stride[d];
    oo += c * p.out.stride[d];
  }
  *in0 = oi;
  *out0 = oo;
  *sin = p.in.stride[p.sdim];
  *sout = p.out.stride[p.sdim];
  *L = p.box.ext[p.sdim];
}

template <typename T>
__global__ void __launch_bounds__(256) k_scan_warp(const __grid_constant__ rt_scan_params p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double g = p.gamma;
  for (int64_t line = warp; line < p.total_lines; line += nwarps) {
    int64_t i0, o0, si, so, L;
    line_base(p, line, &i0, &o0, &si, &so, &L);
    double carry = 0.0;
    bool have = false;
    const int64_t nchunks = (L + 31) / 32;
    for (int64_t cb = 0; cb < nchunks; cb += SCAN_UNROLL) {
      double x[SCAN_UNROLL];
#pragma unroll
      for (int u = 0; u < SCAN_UNROLL; ++u) {
        int64_t c = cb + u;
        // element position along the line in processing order
        int64_t pos = c * 32 + lane;
        int64_t j = p.reverse ? (L - 1 - pos) : pos;
        x[u] = (c < nchunks && pos < L) ? (double)load_as<T>((const void*)p.in.ptr, p.in.dtype, i0 + j * si)
                                         : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SCAN_UNROLL; ++u) {
        int64_t c = cb + u;
        if (c >= nchunks) break;
        int64_t pos = c * 32 + lane;
        // inclusive scan of (A, B): y = A*y_in + B, element: (g, x)
        double A = g, B = x[u];
        if (pos >= L) { A = 1.0; B = 0.0; }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          double Ap = __shfl_up_sync(0xffffffffu, A, o);
          double Bp = __shfl_up_sync(0xffffffffu, B, o);
          if (lane >= o) { B = A * Bp + B; A = A * Ap; }
        }
        // the chain head takes x as is (runtime.py:141: acc = x[j].copy())
        double y = have ? (A * carry + B) : B;
        if (pos < L) {
          int64_t j = p.reverse ? (L - 1 - pos) : pos;
          store_as<double>((void*)p.out.ptr, p.out.dtype, o0 + j * so, y);
        }
        int last = (int)((L - c * 32) < 32 ? (L - c * 32 - 1) : 31);
        carry = __shfl_sync(0xffffffffu, y, last);
        have = true;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_scan_thread(const __grid_constant__ rt_scan_params p) {
  const double g = p.gamma;
  for (int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; line < p.total_lines;
       line += (int64_t)gridDim.x * blockDim.x) {
    int64_t i0, o0, si, so, L;
    line_base(p, line, &i0, &o0, &si, &so, &L);
    double acc = 0.0;
    for (int64_t jb = 0; jb < L; jb += SCAN_UNROLL) {
      double x[SCAN_UNROLL];
#pragma unroll
      for (int u = 0; u < SCAN_UNROLL; ++u) {
        int64_t pos = jb + u;
        int64_t j = p.reverse ? (L - 1 - pos) : pos;
        x[u] = pos < L ? (double)load_as<T>((const void*)p.in.ptr, p.in.dtype, i0 + j * si) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SCAN_UNROLL; ++u) {
        int64_t pos = jb + u;
        if (pos >= L) break;
        int64_t j = p.reverse ? (L - 1 - pos) : pos;
        acc = pos == 0 ? x[u] : x[u] + g * acc;
        store_as<double>((void*)p.out.ptr, p.out.dtype, o0 + j * so, acc);
      }
    }
  }
}

extern "C" void* rt_kernel_scan(int f64, int warp) {
  if (warp) return f64 ? (void*)k_scan_warp<double> : (void*)k_scan_warp<float>;
  return f64 ? (void*)k_scan_thread<double> : (void*)k_scan_thread<float>;
}
