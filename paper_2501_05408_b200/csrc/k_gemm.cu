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
  int64_t o = 0;
  for (int d = b.nd - 1; d >= 0; --d) {
    int64_t e = b.ext[d];
    int64_t q = flat / e;
    o += (flat - q * e) * s[d];
    flat = q;
  }
  return o;
}

template <typename T>
RT_DEV T gload(const rt_gop& o, int64_t off) {
  return load_as<T>((const void*)o.ptr, o.dtype, off);
}

template <typename T>
RT_DEV T epi(const rt_gemm_params& p, T v) {
  if (p.epilogue == 1) return vm_tanh<T>(v);
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) k_gemm(const __grid_constant__ rt_gemm_params p) {
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  __shared__ int64_t offA_row[BM], offB_col[BN], offA_k[BK], offB_k[BK];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t zs = blockIdx.z;
  const int64_t zi = zs / p.splits;
  const int split = (int)(zs - zi * p.splits);

  const int64_t zA = p.A.off + gdecomp(p.Z, zi, p.A.sz);
  const int64_t zB = p.B.off + gdecomp(p.Z, zi, p.B.sz);
  if (tid < BM) {
    int64_t m = m0 + tid;
    offA_row[tid] = m < p.m ? zA + gdecomp(p.M, m, p.A.s1) : 0;
  } else if (tid < BM + BN) {
    int64_t n = n0 + (tid - BM);
    offB_col[tid - BM] = n < p.n ? zB + gdecomp(p.N, n, p.B.s2) : 0;
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

  // A tile mapping: k-fast when the A operand is contiguous along K
  const bool a_kfast = (p.K.nd > 0 && p.A.s2[p.K.nd - 1] == 1);
  const bool b_nfast = (p.N.nd > 0 && p.B.s2[p.N.nd - 1] == 1);

  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    __syncthreads();
    if (tid < BK) {
      int64_t k = k0 + tid;
      offA_k[tid] = k < kend ? gdecomp(p.K, k, p.A.s2) : 0;
    } else if (tid < 2 * BK) {
      int64_t k = k0 + tid - BK;
      offB_k[tid - BK] = k < kend ? gdecomp(p.K, k, p.B.s1) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + 256 * i;
      int r, kk;
      if (a_kfast) { r = e / BK; kk = e % BK; } else { kk = e / BM; r = e % BM; }
      int64_t m = m0 + r, k = k0 + kk;
      As[kk][r] = (m < p.m && k < kend) ? gload<T>(p.A, offA_row[r] + offA_k[kk]) : (T)0;
      int c, kb;
      if (b_nfast) { kb = e / BN; c = e % BN; } else { c = e / BK; kb = e % BK; }
      int64_t n = n0 + c, k2 = k0 + kb;
      Bs[kb][c] = (n < p.n && k2 < kend) ? gload<T>(p.B, offB_col[c] + offB_k[kb]) : (T)0;
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
  const int64_t zC = p.C.off + gdecomp(p.Z, zi, p.C.sz);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= p.m) continue;
    int64_t rowC = zC + gdecomp(p.M, m, p.C.s1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n >= p.n) continue;
      T v = acc[i][j];
      if (p.splits > 1) {
        T* part = (T*)p.part;
        part[((split * p.z + zi) * p.m + m) * p.n + n] = v;
        continue;
      }
      int64_t oc = rowC + gdecomp(p.N, n, p.C.s2);
      if (p.accumulate) v += gload<T>(p.C, oc);
      if (p.bias.ptr) {
        int64_t ob = p.bias.off + gdecomp(p.Z, zi, p.bias.sz) + gdecomp(p.M, m, p.bias.s1) +
                     gdecomp(p.N, n, p.bias.s2);
        v += gload<T>(p.bias, ob);
      }
      store_as<T>((void*)p.C.ptr, p.C.dtype, oc, epi<T>(p, v));
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_splitk(const __grid_constant__ rt_splitk_params p) {
  const int64_t total = p.z * p.m * p.n;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const T* part = (const T*)p.part;
    T v = (T)0;
    for (int s = 0; s < p.splits; ++s) v += part[s * total + f];
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
