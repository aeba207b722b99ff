// RT_K_GEMM — the reference's `matmul` kernel (np.matmul, runtime.py:249)
// evaluated over whole slabs of points at once, fp32 (FFMA) or fp64 (DFMA).
//
// Every operand index is a flat index decomposed over a small box with its
// own strides, which covers the three shapes the PDG produces:
//   * per-point matmuls sharing one weight:  M = points x m        (acting,
//     dX of the backward: frontend.py:972-989)
//   * per-point matmuls summed over points:   K = points x r        (dW: the
//     `sum(matmul(permute(x), g)[i,0:B,0:T])` contraction the symbolic
//     backward emits, frontend.py:766-776 + 984-989) — never materialising
//     the per-point outer products
//   * batched matmuls (numpy broadcasting over leading payload axes): Z.
// 64x64x16 tiles, 256 threads, 4x4 register blocking, optional split-K with
// a deterministic second pass, fused bias + tanh epilogue.
#include "common.cuh"

#define BM 64
#define BN 64
#define BK 16

RT_DEV int64_t gdecomp(const rt_gbox& b, int64_t flat, const int64_t* s) {
  // all extents and flat indices are < 2^31 (checked by the planner)
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

template <typename T>
RT_DEV T gload(const rt_gop& o, int64_t off) {
  return load_as<T>((const void*)o.ptr, o.dtype, off);
}

template <typename T>
RT_DEV T gload_f(const void* base, int dtype, int64_t off) {
  if (dtype == RT_F32) return (T)((const float*)base)[off];
  if (dtype == RT_F64) return (T)((const double*)base)[off];
  return load_as<T>(base, dtype, off);
}

template <typename T>
__global__ void __launch_bounds__(256) k_gemm(const __grid_constant__ rt_gemm_params p) {
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  __shared__ int64_t rowA[BM], rowC[BM], colB[BN], colC[BN], colBias[BN], kA[BK], kB[BK];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * BN;
  const int64_t zs = blockIdx.z;
  const int64_t zi = zs / p.splits;
  const int split = (int)(zs - zi * p.splits);
  const void* Ap = (const void*)p.A.ptr;
  const void* Bp = (const void*)p.B.ptr;
  const int adt = p.A.dtype, bdt = p.B.dtype;

  if (tid < BM) {
    int64_t m = m0 + tid;
    bool ok = m < p.m;
    rowA[tid] = ok ? p.A.off + gdecomp(p.Z, zi, p.A.sz) + gdecomp(p.M, m, p.A.s1) : 0;
    rowC[tid] = ok ? p.C.off + gdecomp(p.Z, zi, p.C.sz) + gdecomp(p.M, m, p.C.s1) : -1;
  } else if (tid < BM + BN) {
    int c = tid - BM;
    int64_t n = n0 + c;
    bool ok = n < p.n;
    colB[c] = ok ? p.B.off + gdecomp(p.Z, zi, p.B.sz) + gdecomp(p.N, n, p.B.s2) : 0;
    colC[c] = ok ? gdecomp(p.N, n, p.C.s2) : -1;
    colBias[c] = (ok && p.bias.ptr) ? p.bias.off + gdecomp(p.Z, zi, p.bias.sz) +
                                          gdecomp(p.N, n, p.bias.s2) : 0;
  }
  // K range of this split
  const int64_t kper = ((p.k + p.splits - 1) / p.splits + BK - 1) / BK * BK;
  const int64_t kbeg = split * kper;
  const int64_t kend = min(p.k, kbeg + kper);

  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = (T)0;

  const bool a_kfast = (p.K.nd > 0 && p.A.s2[p.K.nd - 1] == 1);
  const bool b_nfast = (p.N.nd > 0 && p.B.s2[p.N.nd - 1] == 1);
  const bool m_in = m0 + BM <= p.m, n_in = n0 + BN <= p.n;

  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    __syncthreads();
    if (tid < BK) {
      int64_t k = k0 + tid;
      kA[tid] = k < kend ? gdecomp(p.K, k, p.A.s2) : 0;
    } else if (tid >= 32 && tid < 32 + BK) {
      int64_t k = k0 + tid - 32;
      kB[tid - 32] = k < kend ? gdecomp(p.K, k, p.B.s1) : 0;
    }
    __syncthreads();
    const bool k_in = k0 + BK <= kend;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + 256 * i;
      int r, kk;
      if (a_kfast) { r = e >> 4; kk = e & 15; } else { kk = e >> 6; r = e & 63; }
      bool ok = (m_in || m0 + r < p.m) && (k_in || k0 + kk < kend);
      As[kk][r] = ok ? gload_f<T>(Ap, adt, rowA[r] + kA[kk]) : (T)0;
      int c, kb;
      if (b_nfast) { kb = e >> 6; c = e & 63; } else { c = e >> 4; kb = e & 15; }
      bool okb = (n_in || n0 + c < p.n) && (k_in || k0 + kb < kend);
      Bs[kb][c] = okb ? gload_f<T>(Bp, bdt, colB[c] + kB[kb]) : (T)0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = ty * 4 + i;
    int64_t m = m0 + r;
    if (m >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = tx * 4 + j;
      int64_t n = n0 + c;
      if (n >= p.n) continue;
      T v = acc[i][j];
      if (p.splits > 1) {
        T* part = (T*)p.part;
        part[((split * p.z + zi) * p.m + m) * p.n + n] = v;
        continue;
      }
      int64_t oc = rowC[r] + colC[c];
      if (p.accumulate) v += gload<T>(p.C, oc);
      if (p.bias.ptr) v += gload<T>(p.bias, colBias[c]);
      if (p.epilogue == 1) v = vm_tanh<T>(v);
      store_as<T>((void*)p.C.ptr, p.C.dtype, oc, v);
    }
  }
}

// Split-K reduction.  One warp per output (grid-stride over outputs by
// warp): lane l sums splits l, l+32, ... in order, then a fixed xor tree —
// deterministic; a thread walking ~1000 partials serially per output was
// latency-bound (~90 GB/s on the narrow dW contractions).
template <typename T>
__global__ void __launch_bounds__(256) k_splitk(const __grid_constant__ rt_splitk_params p) {
  const int64_t total = p.z * p.m * p.n;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t f = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; f < total; f += nw) {
    const T* part = (const T*)p.part;
    T v = (T)0;
    for (int s = lane; s < p.splits; s += 32) v += part[s * total + f];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane != 0) continue;
    int64_t n = f % p.n, r = f / p.n;
    int64_t m = r % p.m, zi = r / p.m;
    int64_t oc = p.C.off + gdecomp(p.Z, zi, p.C.sz) + gdecomp(p.M, m, p.C.s1) +
                 gdecomp(p.N, n, p.C.s2);
    if (p.accumulate) v += load_as<T>((const void*)p.C.ptr, p.C.dtype, oc);
    if (p.bias.ptr) {
      int64_t ob = p.bias.off + gdecomp(p.Z, zi, p.bias.sz) + gdecomp(p.M, m, p.bias.s1) +
                   gdecomp(p.N, n, p.bias.s2);
      v += load_as<T>((const void*)p.bias.ptr, p.bias.dtype, ob);
    }
    if (p.epilogue == 1) v = vm_tanh<T>(v);
    store_as<T>((void*)p.C.ptr, p.C.dtype, oc, v);
  }
}

extern "C" void* rt_kernel_gemm(int f64) {
  return f64 ? (void*)k_gemm<double> : (void*)k_gemm<float>;
}
extern "C" void* rt_kernel_splitk(int f64) {
  return f64 ? (void*)k_splitk<double> : (void*)k_splitk<float>;
}
