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

#define SCAN_DEPTH 16   // loads in flight per thread on strided lines

template <typename T>
__global__ void __launch_bounds__(256) k_scan_thread(const __grid_constant__ rt_scan_params p) {
  const double g = p.gamma;
  for (int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; line < p.total_lines;
       line += (int64_t)gridDim.x * blockDim.x) {
    int64_t i0, o0, si, so, L;
    line_base(p, line, &i0, &o0, &si, &so, &L);
    double acc = 0.0;
    for (int64_t jb = 0; jb < L; jb += SCAN_DEPTH) {
      double x[SCAN_DEPTH];
#pragma unroll
      for (int u = 0; u < SCAN_DEPTH; ++u) {
        int64_t pos = jb + u;
        int64_t j = p.reverse ? (L - 1 - pos) : pos;
        x[u] = pos < L ? (double)load_as<T>((const void*)p.in.ptr, p.in.dtype, i0 + j * si) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SCAN_DEPTH; ++u) {
        int64_t pos = jb + u;
        if (pos >= L) break;
        int64_t j = p.reverse ? (L - 1 - pos) : pos;
        acc = pos == 0 ? x[u] : x[u] + g * acc;
        store_as<double>((void*)p.out.ptr, p.out.dtype, o0 + j * so, acc);
      }
    }
  }
}

template <typename T> struct svec;
template <> struct svec<float> { using V = float4; static constexpr int W = 4; };
template <> struct svec<double> { using V = double2; static constexpr int W = 2; };

RT_DEV void sunpack(const float4& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
RT_DEV void sunpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
RT_DEV float4 spack(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
RT_DEV double2 spack(const double* o) { return make_double2(o[0], o[1]); }

#define SCAN_LB 64

// Pipelined tiled scan: the same 64-line CTA tiles, but chunks land in a
// 3-stage shared-memory ring through cp.async 16-byte copies (two chunks in
// flight while the third is scanned), so HBM sees a steady stream instead
// of one register-prefetched chunk per CTA.
//   STEP_MAJOR = false: lines contiguous (x[b, t], scan along t); a tile
//     row is one line's chunk, vector slots XOR-swizzled by (line & 7) so the
//     scan phase's 16-byte reads are bank-conflict free.
//   STEP_MAJOR = true: the 64 lines of a CTA are adjacent in memory (x[t, b],
//     scan along t with stride S); a tile row is one step of 64 lines.
RT_DEV void cp16(void* smem, const void* gmem, bool valid) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;   // src-size 0: zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
RT_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RT_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

#define SCAN_NS 3

template <typename T, bool STEP_MAJOR>
__global__ void __launch_bounds__(SCAN_LB) k_scan_pipe(const __grid_constant__ rt_scan_params p) {
  using V = typename svec<T>::V;
  constexpr int VW = svec<T>::W;
  constexpr int VPL = 16;                      // vectors per line per chunk
  constexpr int TC = VPL * VW;                 // steps per chunk
  constexpr int NVEC = SCAN_LB * TC / VW;      // vectors per stage (1024)
  constexpr int NV = NVEC / SCAN_LB;           // per thread (16)
  constexpr int VPR = SCAN_LB / VW;            // step-major: vectors per row of 64 lines
  extern __shared__ __align__(16) unsigned char sraw[];
  V* ring = reinterpret_cast<V*>(sraw);        // [NS][NVEC], then the line bases
  int64_t* ib = reinterpret_cast<int64_t*>(ring + SCAN_NS * NVEC);
  int64_t* ob = ib + SCAN_LB;
  const int tid = threadIdx.x;
  const double g = p.gamma;
  const T* X = (const T*)p.in.ptr;
  T* Y = (T*)p.out.ptr;
  const int64_t L = p.box.ext[p.sdim];
  const int64_t si = p.in.stride[p.sdim], so = p.out.stride[p.sdim];
  const int64_t nch = (L + TC - 1) / TC;
  const int64_t l0 = (int64_t)blockIdx.x * SCAN_LB;
  const int nl = (int)(p.total_lines - l0 < SCAN_LB ? p.total_lines - l0 : SCAN_LB);
  {
    int64_t i0, o0, a, b, LL;
    line_base(p, l0 + (tid < nl ? tid : 0), &i0, &o0, &a, &b, &LL);
    ib[tid] = i0;
    ob[tid] = o0;
  }
  __syncthreads();
  auto chunk = [&](int64_t c, int64_t& j0, int& cnt) {
    const int64_t a = c * TC, b = (c + 1) * TC < L ? (c + 1) * TC : L;
    cnt = (int)(b - a);
    j0 = p.reverse ? L - b : a;
  };
  // tile vector v of a stage -> (row, vector-in-row) and its smem slot
  auto issue = [&](int64_t c) {
    int64_t j0;
    int cnt;
    chunk(c, j0, cnt);
    V* st = ring + (c % SCAN_NS) * NVEC;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int v = tid + SCAN_LB * q;
      if (!STEP_MAJOR) {
        const int ln = v / VPL, pc = v % VPL;
        const bool ok = ln < nl && pc * VW < cnt;
        cp16(st + ln * VPL + (pc ^ (ln & 7)), X + ib[ok ? ln : 0] + (ok ? j0 + pc * VW : 0), ok);
      } else {
        const int k = v / VPR, pc = v % VPR;
        const bool ok = k < cnt;
        cp16(st + v, X + ib[0] + pc * VW + (ok ? (j0 + k) * si : 0), ok);
      }
    }
  };
  issue(0);
  cp_commit();
  if (nch > 1) issue(1);
  cp_commit();
  double acc = 0.0;
  for (int64_t c = 0; c < nch; ++c) {
    int64_t j0;
    int cnt;
    chunk(c, j0, cnt);
    cp_wait<1>();
    __syncthreads();
    V* st = ring + (c % SCAN_NS) * NVEC;
    if (!STEP_MAJOR) {
      V* row = st + tid * VPL;
      const int nv = cnt / VW;
      if (p.reverse) {
        for (int pc = nv - 1; pc >= 0; --pc) {
          V* slot = row + (pc ^ (tid & 7));
          T e[VW];
          sunpack(*slot, e);
#pragma unroll
          for (int q = VW - 1; q >= 0; --q) {
            const double x = (double)e[q];
            acc = (c == 0 && pc == nv - 1 && q == VW - 1) ? x : x + g * acc;
            e[q] = (T)acc;
          }
          *slot = spack(e);
        }
      } else {
        for (int pc = 0; pc < nv; ++pc) {
          V* slot = row + (pc ^ (tid & 7));
          T e[VW];
          sunpack(*slot, e);
#pragma unroll
          for (int q = 0; q < VW; ++q) {
            const double x = (double)e[q];
            acc = (c == 0 && pc == 0 && q == 0) ? x : x + g * acc;
            e[q] = (T)acc;
          }
          *slot = spack(e);
        }
      }
    } else {
      T* t = reinterpret_cast<T*>(st);
      if (p.reverse) {
        for (int k = cnt - 1; k >= 0; --k) {
          const double x = (double)t[k * SCAN_LB + tid];
          acc = (c == 0 && k == cnt - 1) ? x : x + g * acc;
          t[k * SCAN_LB + tid] = (T)acc;
        }
      } else {
        for (int k = 0; k < cnt; ++k) {
          const double x = (double)t[k * SCAN_LB + tid];
          acc = (c == 0 && k == 0) ? x : x + g * acc;
          t[k * SCAN_LB + tid] = (T)acc;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int v = tid + SCAN_LB * q;
      if (!STEP_MAJOR) {
        const int ln = v / VPL, pc = v % VPL;
        if (ln < nl && pc * VW < cnt)
          __stcs(reinterpret_cast<V*>(Y + ob[ln] + j0 + pc * VW), st[ln * VPL + (pc ^ (ln & 7))]);
      } else {
        const int k = v / VPR, pc = v % VPR;
        if (k < cnt) __stcs(reinterpret_cast<V*>(Y + ob[0] + pc * VW + (j0 + k) * so), st[v]);
      }
    }
    if (c + 2 < nch) issue(c + 2);
    cp_commit();
  }
}

RT_DEV float rn_add(float a, float b) { return __fadd_rn(a, b); }
RT_DEV double rn_add(double a, double b) { return __dadd_rn(a, b); }
RT_DEV float rn_sub(float a, float b) { return __fsub_rn(a, b); }
RT_DEV double rn_sub(double a, double b) { return __dsub_rn(a, b); }
RT_DEV float rn_mul(float a, float b) { return __fmul_rn(a, b); }
RT_DEV double rn_mul(double a, double b) { return __dmul_rn(a, b); }

// GAE-fused pipelined scan (line-major, reverse): two input rings (r and V),
// the TD residual delta = (r + c * V[t+1]) - V is formed in the scan phase in
// the program's precision with the reference's operation order (no FMA
// contraction: numpy evaluates add(r, mul(Vn, c)) then sub(.., V)), V[t+1]
// across a chunk boundary comes from the previously processed chunk (carried
// per line), and the bootstrap value vb stands in for V[T].
template <typename T>
__global__ void __launch_bounds__(SCAN_LB) k_scan_gae(const __grid_constant__ rt_scan_params p) {
  using V = typename svec<T>::V;
  constexpr int VW = svec<T>::W;
  constexpr int VPL = 8;                       // vectors per line per chunk
  constexpr int TC = VPL * VW;
  constexpr int NVEC = SCAN_LB * TC / VW;
  constexpr int NV = NVEC / SCAN_LB;
  extern __shared__ __align__(16) unsigned char sraw[];
  V* ring = reinterpret_cast<V*>(sraw);                 // r: [NS][NVEC]
  V* ring2 = ring + SCAN_NS * NVEC;                     // V: [NS][NVEC]
  int64_t* ib = reinterpret_cast<int64_t*>(ring2 + SCAN_NS * NVEC);
  int64_t* ib2 = ib + SCAN_LB;
  int64_t* ob = ib2 + SCAN_LB;
  const int tid = threadIdx.x;
  const double g = p.gamma;
  const T c = (T)p.gae_c;
  const T* X = (const T*)p.in.ptr;
  const T* X2 = (const T*)p.in2.ptr;
  T* Y = (T*)p.out.ptr;
  const int64_t L = p.box.ext[p.sdim];
  const int64_t nch = (L + TC - 1) / TC;
  const int64_t l0 = (int64_t)blockIdx.x * SCAN_LB;
  const int nl = (int)(p.total_lines - l0 < SCAN_LB ? p.total_lines - l0 : SCAN_LB);
  {
    int64_t i0, o0, a, b, LL;
    line_base(p, l0 + (tid < nl ? tid : 0), &i0, &o0, &a, &b, &LL);
    ib[tid] = i0;
    ob[tid] = o0;
    // second input: same decomposition over its own strides
    int64_t r = l0 + (tid < nl ? tid : 0), o2 = p.in2.off;
    for (int d = p.box.nd - 1; d >= 0; --d) {
      if (d == p.sdim) continue;
      const int64_t e = p.box.ext[d], q = r / e;
      o2 += (r - q * e) * p.in2.stride[d];
      r = q;
    }
    ib2[tid] = o2;
  }
  __syncthreads();
  auto chunk = [&](int64_t cc, int64_t& j0, int& cnt) {   // reverse order
    const int64_t a = cc * TC, b = (cc + 1) * TC < L ? (cc + 1) * TC : L;
    cnt = (int)(b - a);
    j0 = L - b;
  };
  auto issue = [&](int64_t cc) {
    int64_t j0;
    int cnt;
    chunk(cc, j0, cnt);
    V* st = ring + (cc % SCAN_NS) * NVEC;
    V* st2 = ring2 + (cc % SCAN_NS) * NVEC;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int v = tid + SCAN_LB * q;
      const int ln = v / VPL, pc = v % VPL;
      const bool ok = ln < nl && pc * VW < cnt;
      const int slot = ln * VPL + (pc ^ (ln & 7));
      cp16(st + slot, X + ib[ok ? ln : 0] + (ok ? j0 + pc * VW : 0), ok);
      cp16(st2 + slot, X2 + ib2[ok ? ln : 0] + (ok ? j0 + pc * VW : 0), ok);
    }
  };
  issue(0);
  cp_commit();
  if (nch > 1) issue(1);
  cp_commit();
  double acc = 0.0;
  T vnext = (T)p.gae_vb;
  for (int64_t cc = 0; cc < nch; ++cc) {
    int64_t j0;
    int cnt;
    chunk(cc, j0, cnt);
    cp_wait<1>();
    __syncthreads();
    V* st = ring + (cc % SCAN_NS) * NVEC;
    V* st2 = ring2 + (cc % SCAN_NS) * NVEC;
    V* row = st + tid * VPL;
    V* row2 = st2 + tid * VPL;
    const int nv = cnt / VW;
    for (int pc = nv - 1; pc >= 0; --pc) {
      V* slot = row + (pc ^ (tid & 7));
      T e[VW], w[VW];
      sunpack(*slot, e);
      sunpack(row2[pc ^ (tid & 7)], w);
#pragma unroll
      for (int q = VW - 1; q >= 0; --q) {
        T d = rn_add(e[q], rn_mul(vnext, c));   // add(r, mul(Vn, c)), no contraction
        d = rn_sub(d, w[q]);                    // sub(.., V)
        vnext = w[q];
        const double x = (double)d;
        acc = (cc == 0 && pc == nv - 1 && q == VW - 1) ? x : x + g * acc;
        e[q] = (T)acc;
      }
      *slot = spack(e);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int v = tid + SCAN_LB * q;
      const int ln = v / VPL, pc = v % VPL;
      if (ln < nl && pc * VW < cnt)
        __stcs(reinterpret_cast<V*>(Y + ob[ln] + j0 + pc * VW), st[ln * VPL + (pc ^ (ln & 7))]);
    }
    if (cc + 2 < nch) issue(cc + 2);
    cp_commit();
  }
}

extern "C" void* rt_kernel_scan_gae(int f64) {
  return f64 ? (void*)k_scan_gae<double> : (void*)k_scan_gae<float>;
}

// tile == 2: pipelined line-major, tile == 3: pipelined step-major
extern "C" void* rt_kernel_scan_pipe(int f64, int step_major) {
  if (step_major) return f64 ? (void*)k_scan_pipe<double, true> : (void*)k_scan_pipe<float, true>;
  return f64 ? (void*)k_scan_pipe<double, false> : (void*)k_scan_pipe<float, false>;
}

extern "C" void* rt_kernel_scan(int f64, int warp) {
  if (warp) return f64 ? (void*)k_scan_warp<double> : (void*)k_scan_warp<float>;
  return f64 ? (void*)k_scan_thread<double> : (void*)k_scan_thread<float>;
}

