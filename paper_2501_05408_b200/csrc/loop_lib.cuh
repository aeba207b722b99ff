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
#pragma once
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


// ---------------------------------------------------------------- TMA bulk
// 1-D bulk async copies global -> shared with mbarrier completion (sm_90+;
// UBLKCP in SASS), used to stream dense weight panels through a smem ring.

RT_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

RT_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

RT_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}

RT_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

RT_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  }
}

#define RING 4

// ---------------------------------------------------------------- cp.async
// 8-byte global -> shared async copies (LDGSTS): completion is tracked per
// thread by commit groups, not by register scoreboards.
RT_DEV void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
RT_DEV void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
RT_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
RT_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------- clusters
// A CTA pair of the persistent acting loop keeps one K-half of a large
// weight matrix resident in each SM's shared memory and exchanges operand
// rows / partial sums through distributed shared memory (DSMEM).
RT_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
RT_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
RT_DEV uint32_t dsmem_map(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
RT_DEV float dsmem_ld(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
RT_DEV float4 dsmem_ld4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}
RT_DEV void sts4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

template <int MRP>
RT_DEV void fma_rows(float (&acc)[MRP], const float (&a)[MRP], float b) {
  static_assert(MRP % 2 == 0, "row blocks are padded to even counts");
#pragma unroll
  for (int r = 0; r < MRP; r += 2) fma2(acc[r], acc[r + 1], a[r], a[r + 1], b);
}
template <int MRP>
RT_DEV void fma_rows(double (&acc)[MRP], const double (&a)[MRP], double b) {
#pragma unroll
  for (int r = 0; r < MRP; ++r) acc[r] = fma(a[r], b, acc[r]);
}


struct loop_ring {
  uint64_t* bar;       // [RING] mbarriers
  unsigned char* buf;  // [RING][stage_bytes]
  uint32_t stage_bytes;
  uint32_t seq;        // chunks consumed so far (uniform across the CTA)
};

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


// A loads for MRP rows at one k: float4 / double2 vector broadcasts from smem
template <typename T, int MRP>
RT_DEV void load_a(const T* ak, T (&a)[MRP]) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int q = 0; q < MRP / 4; ++q) {
      float4 v = reinterpret_cast<const float4*>(ak)[q];
      a[4 * q] = v.x; a[4 * q + 1] = v.y; a[4 * q + 2] = v.z; a[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < MRP / 2; ++q) {
      double2 v = reinterpret_cast<const double2*>(ak)[q];
      a[2 * q] = v.x; a[2 * q + 1] = v.y;
    }
  }
}

// chunk loop + epilogue with the padded row count MRP and the columns per
// thread NC known at compile time; k unrolled by 4 with loads batched ahead
// of the FMAs (the loop is issue/latency bound, not bandwidth bound).
template <typename T, int MRP, int NC>
RT_DEV void tma_body(const rt_gemm_params& p, const T* As, const T* Bg, int64_t K, int64_t Nn,
                     int64_t kc, int64_t nch, int mr, int64_t m0, int64_t coff, int64_t biasoff,
                     loop_ring& ring) {
  const int nn = (int)Nn;
  T acc[NC][MRP];
#pragma unroll
  for (int j = 0; j < NC; ++j)
#pragma unroll
    for (int r = 0; r < MRP; ++r) acc[j][r] = (T)0;
  int col[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    col[j] = (int)threadIdx.x + j * (int)blockDim.x;
    if (col[j] >= nn) col[j] = nn - 1;   // duplicate work, never stored
  }
  auto issue = [&](int c) {
    uint32_t st = (ring.seq + (uint32_t)c) % RING;
    int64_t k0 = (int64_t)c * kc;
    int64_t rows = min(kc, K - k0);
    uint32_t bytes = (uint32_t)(rows * Nn * sizeof(T));
    mbar_expect_tx(&ring.bar[st], bytes);
    bulk_g2s(ring.buf + (size_t)st * ring.stage_bytes, Bg + k0 * Nn, bytes, &ring.bar[st]);
  };
  for (int c = 0; c < (int)nch; ++c) {
    uint32_t g = ring.seq + (uint32_t)c;
    uint32_t st = g % RING;
    mbar_wait(&ring.bar[st], (g / RING) & 1);
    const T* Bs = (const T*)(ring.buf + (size_t)st * ring.stage_bytes);
    const int k0 = c * (int)kc;
    const int rows = (int)min(kc, K - (int64_t)k0);
    const T* ak = As + (size_t)k0 * MRP;
    int kk = 0;
    for (; kk + 4 <= rows; kk += 4, ak += 4 * MRP) {
      T b[4][NC];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < NC; ++j) b[u][j] = Bs[(kk + u) * nn + col[j]];
      T a[4][MRP];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_a<T, MRP>(ak + u * MRP, a[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < NC; ++j) fma_rows<MRP>(acc[j], a[u], b[u][j]);
    }
    for (; kk < rows; ++kk, ak += MRP) {
      T a[MRP];
      load_a<T, MRP>(ak, a);
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const T bb = Bs[kk * nn + col[j]];
#pragma unroll
        for (int r = 0; r < MRP; ++r) acc[j][r] = fma(a[r], bb, acc[j][r]);
      }
    }
    __syncthreads();   // everyone is done with stage st
    if (threadIdx.x == 0 && c + RING < (int)nch) issue(c + RING);
  }
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int64_t n = threadIdx.x + j * (int64_t)blockDim.x;
    if (n >= Nn) break;
    T bias = p.bias.ptr ? load_as<T>((const void*)p.bias.ptr, p.bias.dtype,
                                     biasoff + gdec32(p.N, n, p.bias.s2)) : (T)0;
    const int64_t cn = gdec32(p.N, n, p.C.s2);
#pragma unroll
    for (int r = 0; r < MRP; ++r) {
      if (r >= mr) break;
      T v = acc[j][r] + bias;
      if (p.epilogue == 1) v = vm_tanh<T>(v);
      store_as<T>((void*)p.C.ptr, p.C.dtype, coff + gdec32(p.M, m0 + r, p.C.s1) + cn, v);
    }
  }
}

template <typename T, int MRP>
RT_DEV void tma_body_nc(const rt_gemm_params& p, const T* As, const T* Bg, int64_t K, int64_t Nn,
                        int64_t kc, int64_t nch, int mr, int64_t m0, int64_t coff,
                        int64_t biasoff, loop_ring& ring) {
  const int nc = (int)((Nn + blockDim.x - 1) / blockDim.x);
  if (nc <= 1 || sizeof(T) == 8) tma_body<T, MRP, 1>(p, As, Bg, K, Nn, kc, nch, mr, m0, coff, biasoff, ring);
  else tma_body<T, MRP, 2>(p, As, Bg, K, Nn, kc, nch, mr, m0, coff, biasoff, ring);
}

template <typename T>
RT_DEV bool gemm_rows_tma(const rt_gemm_params& p, const int64_t* env, int64_t m0, int64_t m1,
                          unsigned char* smem, loop_ring& ring) {
  // dense row-major weights B[K][N] of type T: stream K-panels with TMA bulk copies
  const int64_t K = p.k, Nn = p.n;
  if (p.B.dtype != (sizeof(T) == 8 ? RT_F64 : RT_F32) || p.N.nd != 1 || p.K.nd != 1 ||
      p.B.s2[0] != 1 || p.B.s1[0] != Nn || p.Z.nd > 1)
    return false;
  const int64_t kc = ring.stage_bytes / (Nn * (int64_t)sizeof(T));
  const int mr = (int)(m1 - m0);
  if (kc < 1 || Nn < 64 || mr > 8 || Nn > (sizeof(T) == 8 ? 1 : 2) * (int64_t)blockDim.x)
    return false;
  const int mrp = (mr + 3) & ~3;                           // rows padded to a multiple of 4
  T* As = (T*)smem;                                        // k-major: As[k * mrp + r]
  const int64_t aoff = fold_gop_off(p.A, env);
  const int64_t boff = fold_gop_off(p.B, env);
  const int64_t coff = fold_gop_off(p.C, env);
  const int64_t biasoff = p.bias.ptr ? fold_gop_off(p.bias, env) : 0;
  const T* Bg = (const T*)p.B.ptr + boff;
  if ((((uintptr_t)Bg) & 15) != 0 || ((Nn * (int64_t)sizeof(T)) & 15) != 0) return false;
  const int64_t nch = (K + kc - 1) / kc;
  auto issue = [&](int64_t c) {
    uint32_t st = (ring.seq + (uint32_t)c) % RING;
    int64_t k0 = c * kc;
    int64_t rows = min(kc, K - k0);
    uint32_t bytes = (uint32_t)(rows * Nn * sizeof(T));
    mbar_expect_tx(&ring.bar[st], bytes);
    bulk_g2s(ring.buf + (size_t)st * ring.stage_bytes, Bg + k0 * Nn, bytes, &ring.bar[st]);
  };
  if (threadIdx.x == 0)
    for (int64_t c = 0; c < (nch < RING ? nch : (int64_t)RING); ++c) issue(c);
  // stage A rows meanwhile (k-major, zero-padded rows)
  {
    const int64_t sk = p.A.s2[0];
    for (int64_t i = threadIdx.x; i < (int64_t)mrp * K; i += blockDim.x) {
      int r = (int)(i / K);
      int64_t k = i - (int64_t)r * K;
      As[k * mrp + r] = r < mr ? load_as<T>((const void*)p.A.ptr, p.A.dtype,
                                            aoff + gdec32(p.M, m0 + r, p.A.s1) + k * sk) : (T)0;
    }
  }
  __syncthreads();
  if (mrp <= 4) tma_body_nc<T, 4>(p, As, Bg, K, Nn, kc, nch, mr, m0, coff, biasoff, ring);
  else tma_body_nc<T, 8>(p, As, Bg, K, Nn, kc, nch, mr, m0, coff, biasoff, ring);
  ring.seq += (uint32_t)nch;
  return true;
}

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

// mean of n values in numpy's pairwise order (umath pairwise_sum, n <= 128:
// 8 strided accumulators, tree-combined, remainder added in order); lane j of
// the warp owns accumulator j, so the result is bit-identical to numpy's.
RT_DEV double warp_pairwise_sum(const void* base, int dtype, int64_t off, int64_t n, int lane) {
  if (n > 128) {
    double v = lane == 0 ? pairwise_sum_l(base, dtype, off, n) : 0.0;
    return __shfl_sync(0xffffffffu, v, 0);
  }
  if (n < 8) {
    double v = 0.0;
    if (lane == 0)
      for (int64_t i = 0; i < n; ++i) v += load_as<double>(base, dtype, off + i);
    return __shfl_sync(0xffffffffu, v, 0);
  }
  const int64_t body = n - (n % 8);
  double r = 0.0;
  if (lane < 8) {
    r = load_as<double>(base, dtype, off + lane);
    for (int64_t i = 8 + lane; i < body; i += 8) r += load_as<double>(base, dtype, off + i);
  }
  double r1 = __shfl_down_sync(0xffffffffu, r, 1);   // pairs (0,1) (2,3) (4,5) (6,7)
  double p01 = r + r1;
  double p23 = __shfl_down_sync(0xffffffffu, p01, 2);
  double q = p01 + p23;                               // lane 0: (r0+r1)+(r2+r3); lane 4: (r4+r5)+(r6+r7)
  double q4 = __shfl_down_sync(0xffffffffu, q, 4);
  double res = q + q4;
  if (lane == 0)
    for (int64_t i = body; i < n; ++i) res += load_as<double>(base, dtype, off + i);
  return __shfl_sync(0xffffffffu, res, 0);
}

RT_DEV void udf_rows(const rt_udf_params& p, const rt_loop_op& op, const int64_t* env,
                     int64_t r0, int64_t r1, int64_t tix) {
  int64_t idx[RT_MAXD];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int64_t row = r0 + warp; row < r1; row += nwarps) {
    decompose(p.box, row, idx);
    double base = p.salt;
    for (int k = 0; k < p.nin; ++k) {
      int64_t c = p.in_count[k];
      if (c == 0) continue;
      rt_fold f = fold_of(p.in[k], env);
      int64_t o = fview_off(p.in[k], &f, p.box.nd, idx);
      base = base + warp_pairwise_sum((const void*)p.in[k].ptr, p.in[k].dtype, o, c, lane) / (double)c;
    }
    const double* noise = (const double*)op.noise;
    if (noise) {
      int64_t nz = op.noise_off + row * op.noise_row + tix * op.noise_step;
      for (int j = 0; j < p.nout; ++j) {
        rt_fold f = fold_of(p.out[j], env);
        int64_t o = fview_off(p.out[j], &f, p.box.nd, idx);
        int kind = p.out_kind[j];
        double tb = kind == RT_BOOL ? tanh(base) : 0.0;
        for (int e = lane; e < p.out_count[j]; e += 32) {
          double z = noise[nz + e];
          double v;
          if (kind == RT_BOOL) v = (tb + z > 0.8) ? 1.0 : 0.0;
          else if (kind == RT_I64) v = floor(3.0 * tanh(base + z));
          else v = tanh(base + 0.3 * z);
          store_as<double>((void*)p.out[j].ptr, p.out[j].dtype, o + e, v);
        }
        nz += p.out_count[j];
      }
      continue;
    }
    if (lane != 0) continue;
    uint32_t words[8 + 2 * RT_MAXD];
    int n = 0;
    for (int i = 0; i < p.nprefix; ++i) words[n++] = p.prefix[i];
    for (int j = 0; j < p.ncoord; ++j) {
      int s = p.coord_src[j];
      n = push_words_l(words, n, (s >= 0 ? idx[s] : env[-1 - s]) + p.coord_add[j]);
    }
    rt_pcg64 g;
    pcg64_seed(g, words, n);
    for (int j = 0; j < p.nout; ++j) {
      rt_fold f = fold_of(p.out[j], env);
      int64_t o = fview_off(p.out[j], &f, p.box.nd, idx);
      int kind = p.out_kind[j];
      double tb = kind == RT_BOOL ? tanh(base) : 0.0;
      for (int e = 0; e < p.out_count[j]; ++e) {
        double z = pcg64_normal(g);
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
      n = push_words_l(words, n, (s >= 0 ? idx[s] : env[-1 - s]) + p.coord_add[j]);
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


// ---------------------------------------------------------------- prologue
// Copy every op descriptor into shared memory and set up the TMA ring.

RT_DEV void loop_prologue(const rt_loop_params& p, unsigned char* smem, uint64_t* bars,
                          loop_ring& ring) {
  const rt_loop_op* ops = (const rt_loop_op*)p.ops;
  for (int i = 0; i < p.nops; ++i) {
    const int4* src = (const int4*)ops[i].params;
    int4* dst = (int4*)(smem + ops[i].smem_off);
    for (int w = threadIdx.x; w < (ops[i].param_bytes + 15) / 16; w += blockDim.x) dst[w] = src[w];
  }
  const uint32_t ring_off = (uint32_t)p.ring_off;
  ring.bar = bars;
  ring.buf = smem + ring_off;
  ring.stage_bytes = p.smem_bytes > (int)ring_off
                         ? (uint32_t)((p.smem_bytes - (int)ring_off) / RING) & ~127u : 0u;
  ring.seq = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RING; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
}

// out-of-line op entry points: compiled once per kernel however many ops call
// them (keeps the JIT-specialised loop kernels small and quick to build)
template <typename T>
__device__ __noinline__ void gemm_op(const rt_gemm_params& q, const int64_t* env, int64_t m0,
                                     int64_t m1, unsigned char* sA, loop_ring& ring) {
  if (ring.stage_bytes == 0 || !gemm_rows_tma<T>(q, env, m0, m1, sA, ring))
    gemm_rows<T>(q, env, m0, m1, sA);
}

__device__ __noinline__ void udf_op(const rt_udf_params& p, const rt_loop_op& op, const int64_t* env,
                                    int64_t r0, int64_t r1, int64_t tix) {
  udf_rows(p, op, env, r0, r1, tix);
}

__device__ __noinline__ void rng_op(const rt_rng_params& p, const int64_t* env, int64_t r0,
                                    int64_t r1) {
  rng_rows(p, env, r0, r1);
}

// ================================================================ JIT ops
// Shape-specialised op bodies for JIT-compiled loop kernels: K, N, rows and
// panel sizes are template constants, shared memory is addressed with
// explicit ld.shared (the generic-pointer path costs an LD.E + 64-bit address
// math per operand), and every op is a single inlined instantiation.

RT_DEV float lds1(uint32_t a, float) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v; }
RT_DEV double lds1(uint32_t a, double) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a)); return v; }

// warp_pairwise_sum over n <= 128 fp32 values staged in shared memory at
// byte address a (same summation order: numpy's pairwise sum)
RT_DEV double warp_pairwise_sum_s(uint32_t a, int n, int lane) {
  auto ld = [&](int i) { return (double)lds1(a + 4u * (uint32_t)i, 0.f); };
  if (n < 8) {
    double v = 0.0;
    if (lane == 0)
      for (int i = 0; i < n; ++i) v += ld(i);
    return __shfl_sync(0xffffffffu, v, 0);
  }
  const int body = n - (n % 8);
  double r = 0.0;
  if (lane < 8) {
    r = ld(lane);
    for (int i = 8 + lane; i < body; i += 8) r += ld(i);
  }
  double r1 = __shfl_down_sync(0xffffffffu, r, 1);
  double p01 = r + r1;
  double p23 = __shfl_down_sync(0xffffffffu, p01, 2);
  double q = p01 + p23;
  double q4 = __shfl_down_sync(0xffffffffu, q, 4);
  double res = q + q4;
  if (lane == 0)
    for (int i = body; i < n; ++i) res += ld(i);
  return __shfl_sync(0xffffffffu, res, 0);
}

RT_DEV void sts1(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }
RT_DEV void sts1(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }

template <int MRP>
RT_DEV void lds_rows(uint32_t a, float (&x)[MRP]) {
#pragma unroll
  for (int q = 0; q < MRP / 4; ++q)
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(x[4 * q]), "=f"(x[4 * q + 1]), "=f"(x[4 * q + 2]), "=f"(x[4 * q + 3])
                 : "r"(a + 16 * q));
}
template <int MRP>
RT_DEV void lds_rows(uint32_t a, double (&x)[MRP]) {
#pragma unroll
  for (int q = 0; q < MRP / 2; ++q)
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(x[2 * q]), "=d"(x[2 * q + 1]) : "r"(a + 16 * q));
}

// stage A rows [m0, m0+mr) x K into shared memory k-major (As[k*MRP + r]),
// zero-padded to MRP rows; the K stride of A is the compile-time KS.
template <typename T, int MRP, int K>
RT_DEV void stage_a(const rt_gemm_params& p, const int64_t* env, int64_t m0, int mr, uint32_t sA) {
  const int64_t aoff = fold_gop_off(p.A, env);
  const int64_t ks = p.A.s2[0];
  for (int i = threadIdx.x; i < MRP * K; i += blockDim.x) {
    const int r = i / K, k = i - r * K;
    T v = (T)0;
    if (r < mr) v = load_as<T>((const void*)p.A.ptr, p.A.dtype, aoff + gdec32(p.M, m0 + r, p.A.s1) + k * ks);
    sts1(sA + (uint32_t)((k * MRP + r) * sizeof(T)), v);
  }
}

// C[r, n] = act(sum_k A[r,k] B[k,n] + bias[n]) with dense row-major B[K][N]
// streamed by TMA bulk copies in KC-row panels through the ring.
template <typename T, int MRP, int NC, int K, int N, int KC>
RT_DEV void gemm_tma_fixed(const rt_gemm_params& p, const int64_t* env, int64_t m0, int64_t m1,
                           uint32_t sA, loop_ring& ring) {
  constexpr int NCH = (K + KC - 1) / KC;
  const int mr = (int)(m1 - m0);
  const T* Bg = (const T*)p.B.ptr + fold_gop_off(p.B, env);
  auto issue = [&](int c) {
    const uint32_t st = (ring.seq + (uint32_t)c) % RING;
    const int rows = (c + 1) * KC <= K ? KC : K - c * KC;
    const uint32_t bytes = (uint32_t)(rows * N * sizeof(T));
    mbar_expect_tx(&ring.bar[st], bytes);
    bulk_g2s(ring.buf + (size_t)st * ring.stage_bytes, Bg + (size_t)c * KC * N, bytes, &ring.bar[st]);
  };
  if (threadIdx.x == 0)
#pragma unroll
    for (int c = 0; c < (NCH < RING ? NCH : RING); ++c) issue(c);
  stage_a<T, MRP, K>(p, env, m0, mr, sA);
  __syncthreads();
  T acc[NC][MRP];
#pragma unroll
  for (int j = 0; j < NC; ++j)
#pragma unroll
    for (int r = 0; r < MRP; ++r) acc[j][r] = (T)0;
  int col[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    col[j] = (int)threadIdx.x + j * (int)blockDim.x;
    if (col[j] >= N) col[j] = N - 1;
  }
  const uint32_t ring_base = smem_u32(ring.buf);
  for (int c = 0; c < NCH; ++c) {
    const uint32_t g = ring.seq + (uint32_t)c;
    const uint32_t st = g % RING;
    mbar_wait(&ring.bar[st], (g / RING) & 1);
    const uint32_t bs = ring_base + st * ring.stage_bytes;
    const int rows = (c + 1) * KC <= K ? KC : K - c * KC;
    uint32_t ak = sA + (uint32_t)(c * KC * MRP * sizeof(T));
#pragma unroll 2
    for (int kk = 0; kk < rows; kk += 4) {
      T b[4][NC];
      T a[4][MRP];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int j = 0; j < NC; ++j)
          b[u][j] = kk + u < rows ? lds1(bs + (uint32_t)(((kk + u) * N + col[j]) * sizeof(T)), (T)0) : (T)0;
        lds_rows<MRP>(ak + (uint32_t)((kk + u) * MRP * sizeof(T)), a[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < NC; ++j) fma_rows<MRP>(acc[j], a[u], b[u][j]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + RING < NCH) issue(c + RING);
  }
  ring.seq += NCH;
  const int64_t coff = fold_gop_off(p.C, env);
  const int64_t boff = p.bias.ptr ? fold_gop_off(p.bias, env) : 0;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int n = (int)threadIdx.x + j * (int)blockDim.x;
    if (n >= N) break;
    const T bias = p.bias.ptr ? load_as<T>((const void*)p.bias.ptr, p.bias.dtype,
                                           boff + (int64_t)n * p.bias.s2[0]) : (T)0;
    const int64_t cn = (int64_t)n * p.C.s2[0];
#pragma unroll
    for (int r = 0; r < MRP; ++r) {
      if (r >= mr) break;
      T v = acc[j][r] + bias;
      if (p.epilogue == 1) v = vm_tanh<T>(v);
      store_as<T>((void*)p.C.ptr, p.C.dtype, coff + gdec32(p.M, m0 + r, p.C.s1) + cn, v);
    }
  }
}

// small N (< 64): B[K][N] staged whole in shared memory, each output's K
// range split over G lanes and shuffle-reduced.
template <typename T, int MRP, int K, int N>
RT_DEV void gemm_small_fixed(const rt_gemm_params& p, const int64_t* env, int64_t m0, int64_t m1,
                             uint32_t sA, uint32_t sB) {
  const int mr = (int)(m1 - m0);
  const int64_t boff = fold_gop_off(p.B, env);
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i - k * N;
    sts1(sB + (uint32_t)(i * sizeof(T)),
         load_as<T>((const void*)p.B.ptr, p.B.dtype, boff + gdec32(p.K, k, p.B.s1) + gdec32(p.N, n, p.B.s2)));
  }
  stage_a<T, MRP, K>(p, env, m0, mr, sA);
  __syncthreads();
  constexpr int OUTS = MRP * N;
  constexpr int G0 = 256 / OUTS;
  constexpr int G = G0 >= 32 ? 32 : G0 >= 16 ? 16 : G0 >= 8 ? 8 : G0 >= 4 ? 4 : G0 >= 2 ? 2 : 1;
  const int lane_in = threadIdx.x % G;
  const int64_t coff = fold_gop_off(p.C, env);
  const int64_t bo = p.bias.ptr ? fold_gop_off(p.bias, env) : 0;
  for (int base = 0; base < OUTS; base += 256 / G) {
    const int o = base + (int)threadIdx.x / G;
    const bool act = o < OUTS && (o / N) < mr;
    const int r = act ? o / N : 0, n = act ? o % N : 0;
    T acc = (T)0;
    if (act)
#pragma unroll 4
      for (int k = lane_in; k < K; k += G)
        acc = fma(lds1(sA + (uint32_t)((k * MRP + r) * sizeof(T)), (T)0),
                  lds1(sB + (uint32_t)((k * N + n) * sizeof(T)), (T)0), acc);
#pragma unroll
    for (int s = G / 2; s > 0; s >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, s, G);
    if (act && lane_in == 0) {
      T v = acc;
      if (p.bias.ptr) v += load_as<T>((const void*)p.bias.ptr, p.bias.dtype, bo + (int64_t)n * p.bias.s2[0]);
      if (p.epilogue == 1) v = vm_tanh<T>(v);
      store_as<T>((void*)p.C.ptr, p.C.dtype, coff + gdec32(p.M, m0 + r, p.C.s1) + (int64_t)n * p.C.s2[0], v);
    }
  }
}

// synthetic env with hoisted normals: one warp per row, numpy pairwise means
// of the inputs, one lane per output element.
template <int NIN, int NOUT>
RT_DEV void udf_fixed(const rt_udf_params& p, const rt_loop_op& op, const int64_t* env,
                      int64_t r0, int64_t r1, int64_t t) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int64_t idx[RT_MAXD];
  for (int64_t row = r0 + warp; row < r1; row += nwarps) {
    decompose(p.box, row, idx);
    double base = p.salt;
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      const int64_t c = p.in_count[k];
      rt_fold f = fold_of(p.in[k], env);
      const int64_t o = fview_off(p.in[k], &f, p.box.nd, idx);
      base = base + warp_pairwise_sum((const void*)p.in[k].ptr, p.in[k].dtype, o, c, lane) / (double)c;
    }
    const double* noise = (const double*)op.noise;
    int64_t nz = op.noise_off + row * op.noise_row + t * op.noise_step;
#pragma unroll
    for (int j = 0; j < NOUT; ++j) {
      rt_fold f = fold_of(p.out[j], env);
      const int64_t o = fview_off(p.out[j], &f, p.box.nd, idx);
      const int kind = p.out_kind[j];
      const double tb = kind == RT_BOOL ? tanh(base) : 0.0;
      for (int e = lane; e < p.out_count[j]; e += 32) {
        const double z = noise[nz + e];
        double v;
        if (kind == RT_BOOL) v = (tb + z > 0.8) ? 1.0 : 0.0;
        else if (kind == RT_I64) v = floor(3.0 * tanh(base + z));
        else v = tanh(base + 0.3 * z);
        store_as<double>((void*)p.out[j].ptr, p.out[j].dtype, o + e, v);
      }
      nz += p.out_count[j];
    }
  }
}

// pair GEMM core: acc_own[r] += sum_{k in my half} A_own[k][r] B[k][col],
// acc_par[r] likewise for the partner's rows (A_par = its k-half, copied).
template <int MRP, int KH, int N>
RT_DEV void pair_core(uint32_t sA_own, uint32_t sA_par, uint32_t sB, int col, float (&ao)[MRP],
                      float (&ap)[MRP]) {
#pragma unroll 4
  for (int kk = 0; kk < KH; ++kk) {
    const float b = lds1(sB + (uint32_t)((kk * N + col) * 4), 0.f);
    float a1[MRP], a2[MRP];
    lds_rows<MRP>(sA_own + (uint32_t)(kk * MRP * 4), a1);
    lds_rows<MRP>(sA_par + (uint32_t)(kk * MRP * 4), a2);
#pragma unroll
    for (int r = 0; r < MRP; ++r) {
      ao[r] = fma(a1[r], b, ao[r]);
      ap[r] = fma(a2[r], b, ap[r]);
    }
  }
}

// ---------------------------------------------------------------- warp MMA
// 3xTF32 warp-level tensor-core core for the in-loop GEMM: few rows (<= 8,
// padded to the m16 tile), wide N.  C = A_hi B_hi + A_hi B_lo + A_lo B_hi
// with mma.sync.m16n8k8 tf32 (fp32 accumulate): the dropped A_lo B_lo term
// is ~2^-22 relative, i.e. fp32-grade products for the 1e-5 parity bar.
// Warp w owns columns [w*N/8, (w+1)*N/8) as N/64 n8 tiles; rows 8..15 of
// the A tile are zero (R <= 8), so only c0/c1 (row g = lane/4) are kept.
RT_DEV uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
RT_DEV void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - __uint_as_float(hi));
}
RT_DEV void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  // A rows 8..15 (a1, a3) are the zero padding of an 8-row block
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// acc[j][0..1] = C[row g][n0_j + 2t + {0,1}] for the warp's NT = N/64 tiles
template <int MRP, int K, int N, int KC>
RT_DEV void mma_core(const float* Bg, uint32_t sA, loop_ring& ring, float (&acc)[N / 64][4]) {
  static_assert(MRP == 8 && N % 64 == 0 && K % 8 == 0 && KC % 8 == 0, "mma core shape");
  constexpr int NCH = (K + KC - 1) / KC;
  constexpr int NT = N / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nw0 = warp * (N / 8);
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q] = 0.f;
  const uint32_t ring_base = smem_u32(ring.buf);
  for (int c = 0; c < NCH; ++c) {
    const uint32_t gq = ring.seq + (uint32_t)c;
    const uint32_t st = gq % RING;
    mbar_wait(&ring.bar[st], (gq / RING) & 1);
    const uint32_t bs = ring_base + st * ring.stage_bytes;
    const int rows = (c + 1) * KC <= K ? KC : K - c * KC;
    const uint32_t ak = sA + (uint32_t)(c * KC * MRP * 4);
#pragma unroll 2
    for (int k8 = 0; k8 < rows; k8 += 8) {
      // A[row g][k8 + t], A[row g][k8 + t + 4]   (sA is k-major [k][MRP])
      uint32_t ah0, al0, ah2, al2;
      split_tf32(lds1(ak + (uint32_t)(((k8 + t) * MRP + g) * 4), 0.f), ah0, al0);
      split_tf32(lds1(ak + (uint32_t)(((k8 + t + 4) * MRP + g) * 4), 0.f), ah2, al2);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int n = nw0 + j * 8 + g;
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(lds1(bs + (uint32_t)(((k8 + t) * N + n) * 4), 0.f), bh0, bl0);
        split_tf32(lds1(bs + (uint32_t)(((k8 + t + 4) * N + n) * 4), 0.f), bh1, bl1);
        mma_tf32(acc[j], ah0, ah2, bl0, bl1);
        mma_tf32(acc[j], al0, al2, bh0, bh1);
        mma_tf32(acc[j], ah0, ah2, bh0, bh1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + RING < NCH) {
      const int cc = c + RING;
      const uint32_t st2 = (ring.seq + (uint32_t)cc) % RING;
      const int rows2 = (cc + 1) * KC <= K ? KC : K - cc * KC;
      const uint32_t bytes = (uint32_t)(rows2 * N * 4);
      mbar_expect_tx(&ring.bar[st2], bytes);
      bulk_g2s(ring.buf + (size_t)st2 * ring.stage_bytes, Bg + (size_t)cc * KC * N, bytes, &ring.bar[st2]);
    }
  }
  ring.seq += NCH;
}

// ---------------------------------------------------------------- JIT cores
// Raw-pointer cores: all descriptor values are supplied by the generated code
// as literals or registers, so nothing is re-read from shared memory after a
// global store.

// acc[j][r] += sum_k A_s[k][r] * B[k][col_j]; A staged k-major in smem at sA,
// B[K][N] dense in global memory at Bg, streamed by TMA in KC-row panels.
template <typename T, int MRP, int NC, int K, int N, int KC>
RT_DEV void tma_core(const T* Bg, uint32_t sA, loop_ring& ring, T (&acc)[NC][MRP]) {
  constexpr int NCH = (K + KC - 1) / KC;
  int col[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    col[j] = (int)threadIdx.x + j * (int)blockDim.x;
    if (col[j] >= N) col[j] = N - 1;
  }
  const uint32_t ring_base = smem_u32(ring.buf);
  for (int c = 0; c < NCH; ++c) {
    const uint32_t g = ring.seq + (uint32_t)c;
    const uint32_t st = g % RING;
    mbar_wait(&ring.bar[st], (g / RING) & 1);
    const uint32_t bs = ring_base + st * ring.stage_bytes;
    const int rows = (c + 1) * KC <= K ? KC : K - c * KC;
    const uint32_t ak = sA + (uint32_t)(c * KC * MRP * sizeof(T));
#pragma unroll 2
    for (int kk = 0; kk < rows; kk += 4) {
      T b[4][NC];
      T a[4][MRP];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int j = 0; j < NC; ++j)
          b[u][j] = kk + u < rows ? lds1(bs + (uint32_t)(((kk + u) * N + col[j]) * sizeof(T)), (T)0) : (T)0;
        lds_rows<MRP>(ak + (uint32_t)((kk + u) * MRP * sizeof(T)), a[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < NC; ++j) fma_rows<MRP>(acc[j], a[u], b[u][j]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + RING < NCH) {
      const int cc = c + RING;
      const uint32_t st2 = (ring.seq + (uint32_t)cc) % RING;
      const int rows2 = (cc + 1) * KC <= K ? KC : K - cc * KC;
      const uint32_t bytes = (uint32_t)(rows2 * N * sizeof(T));
      mbar_expect_tx(&ring.bar[st2], bytes);
      bulk_g2s(ring.buf + (size_t)st2 * ring.stage_bytes, Bg + (size_t)cc * KC * N, bytes, &ring.bar[st2]);
    }
  }
  ring.seq += NCH;
}

// K-split variant for wide N (N = 32*CPL, CPL <= 8) and few rows: warp w
// takes rows w, w+W, ... of every streamed panel for ALL N columns (lane l
// owns columns [l*CPL, (l+1)*CPL)), so each k costs CPL/4 + MRP/4 16-byte
// shared loads for CPL*MRP FMAs (the column-per-thread core spends 3 loads
// per MRP*... FMAs and is LSU-bound).  The W per-warp partial tiles are
// summed through `red` ([W][MRP][N] in shared memory) once per step; on
// return acc[q] holds output (row, col) = (o / N, o % N) for
// o = tid * OPT + q, OPT = MRP * N / blockDim.
template <typename T, int MRP, int K, int N, int KC>
RT_DEV void tma_core_ks(const T* Bg, uint32_t sA, loop_ring& ring, uint32_t red,
                        T (&out)[MRP * N / 256]) {
  constexpr int NCH = (K + KC - 1) / KC;
  constexpr int CPL = N / 32;
  constexpr int W = 8;                       // warps (blockDim 256)
  constexpr int OPT = MRP * N / 256;
  static_assert(N % 32 == 0 && CPL <= 8 && CPL % 4 == 0, "K-split core: N = 32*{4,8}");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T acc[MRP][CPL];
#pragma unroll
  for (int r = 0; r < MRP; ++r)
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[r][c] = (T)0;
  const uint32_t ring_base = smem_u32(ring.buf);
  for (int ch = 0; ch < NCH; ++ch) {
    const uint32_t g = ring.seq + (uint32_t)ch;
    const uint32_t st = g % RING;
    mbar_wait(&ring.bar[st], (g / RING) & 1);
    const uint32_t bs = ring_base + st * ring.stage_bytes;
    const int rows = (ch + 1) * KC <= K ? KC : K - ch * KC;
    const uint32_t ak = sA + (uint32_t)(ch * KC * MRP * sizeof(T));
#pragma unroll 2
    for (int kk = warp; kk < rows; kk += W) {
      T a[MRP], b[CPL];
      lds_rows<MRP>(ak + (uint32_t)(kk * MRP * sizeof(T)), a);
      lds_rows<CPL>(bs + (uint32_t)((kk * N + lane * CPL) * sizeof(T)), b);
#pragma unroll
      for (int r = 0; r < MRP; ++r)
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && ch + RING < NCH) {
      const int cc = ch + RING;
      const uint32_t st2 = (ring.seq + (uint32_t)cc) % RING;
      const int rows2 = (cc + 1) * KC <= K ? KC : K - cc * KC;
      const uint32_t bytes = (uint32_t)(rows2 * N * sizeof(T));
      mbar_expect_tx(&ring.bar[st2], bytes);
      bulk_g2s(ring.buf + (size_t)st2 * ring.stage_bytes, Bg + (size_t)cc * KC * N, bytes, &ring.bar[st2]);
    }
  }
  ring.seq += NCH;
  // cross-warp sum: red[w][r][n]
#pragma unroll
  for (int r = 0; r < MRP; ++r)
#pragma unroll
    for (int c = 0; c < CPL; c += 4) {
      const uint32_t a = red + (uint32_t)(((warp * MRP + r) * N + lane * CPL + c) * sizeof(T));
      if constexpr (sizeof(T) == 4)
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(acc[r][c]), "f"(acc[r][c + 1]),
                     "f"(acc[r][c + 2]), "f"(acc[r][c + 3]));
      else {
        sts1(a, acc[r][c]); sts1(a + 8, acc[r][c + 1]); sts1(a + 16, acc[r][c + 2]); sts1(a + 24, acc[r][c + 3]);
      }
    }
  __syncthreads();
  const int o0 = threadIdx.x * OPT;
#pragma unroll
  for (int q = 0; q < OPT; ++q) out[q] = (T)0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    T v[OPT];
    lds_rows<OPT>(red + (uint32_t)((w * MRP * N + o0) * sizeof(T)), v);
#pragma unroll
    for (int q = 0; q < OPT; ++q) out[q] += v[q];
  }
}

// NCOL adjacent columns per thread (threads < N/NCOL compute, the rest
// only join the barriers): per k one NCOL*4-byte B load and MRP/4 16-byte A
// loads feed NCOL*MRP FMAs (the column-per-thread core is shared-memory-issue
// bound at 1 B + MRP/4 A loads per MRP FMAs).
template <int MRP, int K, int N, int KC, int NCOL>
RT_DEV void tma_core2(const float* Bg, uint32_t sA, loop_ring& ring, float (&acc)[NCOL][MRP]) {
  constexpr int NCH = (K + KC - 1) / KC;
  const bool act = (int)threadIdx.x < N / NCOL;
  const int c0 = act ? NCOL * (int)threadIdx.x : 0;
  const uint32_t ring_base = smem_u32(ring.buf);
  for (int c = 0; c < NCH; ++c) {
    const uint32_t g = ring.seq + (uint32_t)c;
    const uint32_t st = g % RING;
    mbar_wait(&ring.bar[st], (g / RING) & 1);
    const uint32_t bs = ring_base + st * ring.stage_bytes;
    const int rows = (c + 1) * KC <= K ? KC : K - c * KC;
    const uint32_t ak = sA + (uint32_t)(c * KC * MRP * 4);
    if (act) {
#pragma unroll 2
      for (int kk = 0; kk < rows; kk += 4) {
        float b[4][NCOL];
        float a[4][MRP];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t ba = bs + (uint32_t)(((kk + u) * N + c0) * 4);
          if (kk + u < rows) {
            if constexpr (NCOL == 4)
              asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                           : "=f"(b[u][0]), "=f"(b[u][1]), "=f"(b[u][2]), "=f"(b[u][3]) : "r"(ba));
            else
              asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(b[u][0]), "=f"(b[u][1]) : "r"(ba));
          } else {
#pragma unroll
            for (int j = 0; j < NCOL; ++j) b[u][j] = 0.f;
          }
          lds_rows<MRP>(ak + (uint32_t)((kk + u) * MRP * 4), a[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < NCOL; ++j) fma_rows<MRP>(acc[j], a[u], b[u][j]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + RING < NCH) {
      const int cc = c + RING;
      const uint32_t st2 = (ring.seq + (uint32_t)cc) % RING;
      const int rows2 = (cc + 1) * KC <= K ? KC : K - cc * KC;
      const uint32_t bytes = (uint32_t)(rows2 * N * 4);
      mbar_expect_tx(&ring.bar[st2], bytes);
      bulk_g2s(ring.buf + (size_t)st2 * ring.stage_bytes, Bg + (size_t)cc * KC * N, bytes, &ring.bar[st2]);
    }
  }
  ring.seq += NCH;
}

// tma_core2 over both thread halves: threads [0, HT) and [HT, 2 HT) (HT =
// N / NCOL) take the lower and upper half of every ring chunk's k rows, so
// all eight warps issue FMAs (with one computing warp per scheduler the
// LDS -> FFMA2 latencies stayed exposed: ncu, profiles/README.md), then the
// upper half's partial sums join the lower half's through shared memory
// (red: MRP x N floats).  The final sums are in threads < HT, as tma_core2's.
template <int MRP, int K, int N, int KC, int NCOL>
RT_DEV void tma_core2k(const float* Bg, uint32_t sA, loop_ring& ring, uint32_t red,
                       float (&acc)[NCOL][MRP]) {
  static_assert(NCOL == 2, "partial sums are exchanged as float2");
  constexpr int NCH = (K + KC - 1) / KC;
  constexpr int HT = N / NCOL;
  const int tid = (int)threadIdx.x;
  const int h = tid >= HT ? 1 : 0;
  const bool act = tid < 2 * HT;
  const int c0 = act ? NCOL * (tid - h * HT) : 0;
  const uint32_t ring_base = smem_u32(ring.buf);
  for (int c = 0; c < NCH; ++c) {
    const uint32_t g = ring.seq + (uint32_t)c;
    const uint32_t st = g % RING;
    mbar_wait(&ring.bar[st], (g / RING) & 1);
    const uint32_t bs = ring_base + st * ring.stage_bytes;
    const int rows = (c + 1) * KC <= K ? KC : K - c * KC;
    const int hr = ((rows + 1) / 2 + 3) / 4 * 4;
    const int lo = h * hr, hi = (h + 1) * hr < rows ? (h + 1) * hr : rows;
    const uint32_t ak = sA + (uint32_t)(c * KC * MRP * 4);
    if (act) {
#pragma unroll 2
      for (int kk = lo; kk < hi; kk += 4) {
        float b[4][NCOL];
        float a[4][MRP];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t ba = bs + (uint32_t)(((kk + u) * N + c0) * 4);
          if (kk + u < hi)
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(b[u][0]), "=f"(b[u][1]) : "r"(ba));
          else
            b[u][0] = b[u][1] = 0.f;
          lds_rows<MRP>(ak + (uint32_t)((kk + u) * MRP * 4), a[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < NCOL; ++j) fma_rows<MRP>(acc[j], a[u], b[u][j]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + RING < NCH) {
      const int cc = c + RING;
      const uint32_t st2 = (ring.seq + (uint32_t)cc) % RING;
      const int rows2 = (cc + 1) * KC <= K ? KC : K - cc * KC;
      const uint32_t bytes = (uint32_t)(rows2 * N * 4);
      mbar_expect_tx(&ring.bar[st2], bytes);
      bulk_g2s(ring.buf + (size_t)st2 * ring.stage_bytes, Bg + (size_t)cc * KC * N, bytes, &ring.bar[st2]);
    }
  }
  ring.seq += NCH;
  if (act && h == 1) {
#pragma unroll
    for (int r = 0; r < MRP; ++r)
      asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(red + (uint32_t)((r * N + c0) * 4)),
                   "f"(acc[0][r]), "f"(acc[1][r]));
  }
  __syncthreads();
  if (act && h == 0) {
#pragma unroll
    for (int r = 0; r < MRP; ++r) {
      float x0, x1;
      asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x0), "=f"(x1) : "r"(red + (uint32_t)((r * N + c0) * 4)));
      acc[0][r] += x0;
      acc[1][r] += x1;
    }
  }
}

// NC adjacent floats from / to shared memory in one access (NC = 1, 2, 4)
template <int NC>
RT_DEV void lds_cols(uint32_t a, float (&x)[NC]) {
  if constexpr (NC == 1) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[0]) : "r"(a));
  else if constexpr (NC == 2) asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x[0]), "=f"(x[1]) : "r"(a));
  else asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]) : "r"(a));
}
template <int NC>
RT_DEV void sts_cols(uint32_t a, const float (&x)[NC]) {
  if constexpr (NC == 1) asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x[0]));
  else if constexpr (NC == 2) asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(a), "f"(x[0]), "f"(x[1]));
  else asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]));
}

// On-chip weights for the widest in-loop layer (N = 256 = blockDim): the
// CTA's threads form P = NCOL parts of N / NCOL threads; part p owns k rows
// [p K/P, (p+1) K/P) and each thread NCOL adjacent columns.  The first KRP
// of a part's rows live in registers (w[j][kk]) for the whole loop, the
// rest in shared memory (sB: part-major, row-major within a part), so a
// step streams nothing from L2 and waits on no ring.  More columns per
// thread divide the A broadcast loads (the same MRP values for every
// thread of a part) by NCOL.  Parts p > 0 hand their partial sums to part
// 0 through red ([P-1][MRP][N] floats); the final sums are in threads
// < N / NCOL.  A is k-major in sA (MRP rows per k).
//
// SPLIT (P = 2, MRP = 8): the two parts instead finalise half of the rows
// each (part p keeps rows [4p, 4p+4) in acc[j][0..3]) so the epilogue
// (bias, tanh, stores) runs on all eight warps.  KRP = 0: no register rows
// (a shared-memory resident layer such as W1 through the same core).
// NR < MRP: only rows [0, NR) are computed (the CTA's real rows; the FMA
// pipe time of a step scales with NR, the padding to MRP only feeds the
// 16-byte row loads).
template <int MRP, int NR>
RT_DEV void fma_rows_n(float (&acc)[MRP], const float (&a)[MRP], float b) {
#pragma unroll
  for (int r = 0; r < NR; r += 2) {
    if (r + 1 < NR) fma2(acc[r], acc[r + 1], a[r], a[r + 1], b);
    else acc[r] = fmaf(a[r], b, acc[r]);
  }
}

template <int MRP, int K, int N, int NCOL, int KRP, bool SPLIT = false, int NR = MRP>
RT_DEV void hyb_core(const float (&w)[NCOL][KRP > 0 ? KRP : 1], uint32_t sB, uint32_t sA, uint32_t red,
                     float (&acc)[NCOL][MRP]) {
  constexpr int P = NCOL, HT = N / NCOL, KP = K / P, KS = KP - KRP;
  static_assert(K % P == 0 && KS >= 0, "K splits evenly over the parts");
  const int tid = (int)threadIdx.x;
  const int part = tid / HT, c0 = NCOL * (tid - part * HT);
  const uint32_t a0 = sA + (uint32_t)(part * KP * MRP * 4);
#pragma unroll
  for (int kk = 0; kk < KRP; ++kk) {
    float a[MRP];
    lds_rows<MRP>(a0 + (uint32_t)(kk * MRP * 4), a);
#pragma unroll
    for (int j = 0; j < NCOL; ++j) fma_rows_n<MRP, NR>(acc[j], a, w[j][kk]);
  }
  const uint32_t bn = sB + (uint32_t)((part * KS * N + c0) * 4);
#pragma unroll 4
  for (int kk = 0; kk < KS; ++kk) {
    float a[MRP], b[NCOL];
    lds_rows<MRP>(a0 + (uint32_t)((KRP + kk) * MRP * 4), a);
    lds_cols<NCOL>(bn + (uint32_t)(kk * N * 4), b);
#pragma unroll
    for (int j = 0; j < NCOL; ++j) fma_rows_n<MRP, NR>(acc[j], a, b[j]);
  }
  if constexpr (SPLIT) {
    static_assert(P == 2 && MRP == 8, "row-split finalisation: two parts, 8 rows");
    constexpr int H = MRP / 2;
    // part p hands the other part's rows to red[p][rr][n], keeps its own
#pragma unroll
    for (int rr = 0; rr < H; ++rr) {
      float x[NCOL];
#pragma unroll
      for (int j = 0; j < NCOL; ++j) x[j] = part == 0 ? acc[j][H + rr] : acc[j][rr];
      sts_cols<NCOL>(red + (uint32_t)(((part * H + rr) * N + c0) * 4), x);
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < H; ++rr) {
      float x[NCOL];
      lds_cols<NCOL>(red + (uint32_t)((((1 - part) * H + rr) * N + c0) * 4), x);
#pragma unroll
      for (int j = 0; j < NCOL; ++j) acc[j][rr] = (part == 0 ? acc[j][rr] : acc[j][H + rr]) + x[j];
    }
  } else if constexpr (P > 1) {
    if (part > 0) {
#pragma unroll
      for (int r = 0; r < MRP; ++r) {
        float x[NCOL];
#pragma unroll
        for (int j = 0; j < NCOL; ++j) x[j] = acc[j][r];
        sts_cols<NCOL>(red + (uint32_t)((((part - 1) * MRP + r) * N + c0) * 4), x);
      }
    }
    __syncthreads();
    if (part == 0) {
#pragma unroll
      for (int q = 1; q < P; ++q)
#pragma unroll
        for (int r = 0; r < MRP; ++r) {
          float x[NCOL];
          lds_cols<NCOL>(red + (uint32_t)((((q - 1) * MRP + r) * N + c0) * 4), x);
#pragma unroll
          for (int j = 0; j < NCOL; ++j) acc[j][r] += x[j];
        }
    }
  }
}

// Same core over a weight matrix that stays resident in shared memory for
// the whole loop (small, loop-invariant B: the observation layer W1, the
// policy head W3): no per-step stream, no ring waits.  Ends with a CTA
// barrier (callers may overwrite the A staging area afterwards).
template <int MRP, int K, int N, int NCOL>
RT_DEV void res_core(uint32_t sB, uint32_t sA, float (&acc)[NCOL][MRP]) {
  const bool act = (int)threadIdx.x < N / NCOL;
  const int c0 = act ? NCOL * (int)threadIdx.x : 0;
  if (act) {
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
      float b[NCOL], a[MRP];
      const uint32_t ba = sB + (uint32_t)((k * N + c0) * 4);
      if constexpr (NCOL == 2)
        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(b[0]), "=f"(b[1]) : "r"(ba));
      else
        b[0] = lds1(ba, 0.f);
      lds_rows<MRP>(sA + (uint32_t)(k * MRP * 4), a);
#pragma unroll
      for (int j = 0; j < NCOL; ++j) fma_rows<MRP>(acc[j], a, b[j]);
    }
  }
  __syncthreads();
}

template <typename T, int K, int N, int KC>
RT_DEV void tma_prefetch(const T* Bg, loop_ring& ring) {
  constexpr int NCH = (K + KC - 1) / KC;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < (NCH < RING ? NCH : RING); ++c) {
      const uint32_t st = (ring.seq + (uint32_t)c) % RING;
      const int rows = (c + 1) * KC <= K ? KC : K - c * KC;
      const uint32_t bytes = (uint32_t)(rows * N * sizeof(T));
      mbar_expect_tx(&ring.bar[st], bytes);
      bulk_g2s(ring.buf + (size_t)st * ring.stage_bytes, Bg + (size_t)c * KC * N, bytes, &ring.bar[st]);
    }
  }
}
