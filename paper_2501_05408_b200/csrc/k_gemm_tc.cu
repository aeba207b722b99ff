// RT_K_GEMM on the 5th-generation tensor cores: tcgen05.mma kind::tf32 with
// a 3xTF32 split (a_hi*b_hi + a_hi*b_lo + a_lo*b_hi) so fp32 programs keep
// fp32-level accuracy (the reference computes these products in fp32 with
// np.matmul, runtime.py:249; north_star tolerance 1e-5 rel).
//
// Used for the learner-side GEMMs of the PDG backward (frontend.py:972-989):
// dX = G @ W^T over all T*E points (M = 1M rows) and the dW contraction
// sum_points x^T g (K = 1M, split-K).  Operands keep the executor's general
// decomposed-stride addressing (rt_gemm_params); CTA threads stage tiles
// into the canonical no-swizzle K-major UMMA layout (8x16B core matrices),
// transposing MN-major sources on the way, and one elected thread issues the
// MMAs; accumulators live in TMEM and are drained with tcgen05.ld.
//
// CTA tile 128 x BN (BN <= 256), BK = 16 (two MMA K-steps of 8), 2-stage
// smem ring with tcgen05.commit -> mbarrier release, 128 threads (4 warps:
// warp w owns TMEM lanes 32w..32w+31 in the epilogue).
#include "common.cuh"

#define TC_BM 128
#define TC_BK 32
#define TC_THREADS 256
#define TC_STAGES 2

RT_DEV uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

RT_DEV uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version 1 (sm_100); SWIZZLE_NONE, base offset 0
  return d;
}

RT_DEV void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

RT_DEV void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(tc_smem(bar)) : "memory");
}

RT_DEV void tc_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(tc_smem(bar)), "r"(phase) : "memory");
  }
}

RT_DEV float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

RT_DEV int64_t tc_decomp(const rt_gbox& b, int64_t flat, const int64_t* s) {
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

// 3xTF32 split of x into (hi, lo) stored at the same offset of the hi and lo
// tiles (lo tile `lo_off` bytes after the hi tile).
RT_DEV void split_store1(unsigned char* base, uint32_t lo_off, uint32_t o, float x) {
  float h = tf32_hi(x);
  *(float*)(base + o) = h;
  *(float*)(base + lo_off + o) = tf32_hi(x - h);
}

RT_DEV void split_store4(unsigned char* base, uint32_t lo_off, uint32_t o, float4 x) {
  float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
  float4 l = make_float4(tf32_hi(x.x - h.x), tf32_hi(x.y - h.y), tf32_hi(x.z - h.z),
                         tf32_hi(x.w - h.w));
  *(float4*)(base + o) = h;
  *(float4*)(base + lo_off + o) = l;
}

// byte offset of element (row r, k) in a K-major no-swizzle tile with BK
// columns: core matrix (r/8, k/4) of 8 rows x 16 bytes.
RT_DEV uint32_t tc_off(int r, int k) {
  return (uint32_t)((r >> 3) * (TC_BK * 32) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__global__ void __launch_bounds__(TC_THREADS, 1) k_gemm_tc(const __grid_constant__ rt_gemm_params p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[TC_STAGES];
  __shared__ uint32_t tmem_base_s;
  __shared__ int64_t rowA[TC_BM], rowC[TC_BM];
  __shared__ int64_t colB[256], colC[256], colBias[256];
  __shared__ int64_t kA[TC_BK], kB[TC_BK];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * TC_BM;
  const int64_t n0 = (int64_t)blockIdx.y * 256;
  const int64_t nrem = p.n - n0;
  const int BN = nrem >= 256 ? 256 : (int)((nrem + 15) / 16 * 16);   // MMA N: multiple of 16
  const int64_t zs = blockIdx.z;
  const int64_t zi = zs / p.splits;
  const int split = (int)(zs - zi * p.splits);
  // stage layout: A_hi, A_lo [128 x BK], B_hi, B_lo [256 x BK]
  const uint32_t a_bytes = TC_BM * TC_BK * 4, b_bytes = 256 * TC_BK * 4;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;

  if (tid == 0) {
    for (int i = 0; i < TC_STAGES; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    // 256 fp32 accumulator columns (power of two >= 32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;"
                 ::"r"(tc_smem(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // row / column offsets
  for (int r = tid; r < TC_BM; r += TC_THREADS) {
    int64_t m = m0 + r;
    bool ok = m < p.m;
    rowA[r] = ok ? p.A.off + tc_decomp(p.Z, zi, p.A.sz) + tc_decomp(p.M, m, p.A.s1) : 0;
    rowC[r] = ok ? p.C.off + tc_decomp(p.Z, zi, p.C.sz) + tc_decomp(p.M, m, p.C.s1) : -1;
  }
  for (int c = tid; c < 256; c += TC_THREADS) {
    int64_t n = n0 + c;
    bool ok = n < p.n;
    colB[c] = ok ? p.B.off + tc_decomp(p.Z, zi, p.B.sz) + tc_decomp(p.N, n, p.B.s2) : 0;
    colC[c] = ok ? tc_decomp(p.N, n, p.C.s2) : -1;
    colBias[c] = (ok && p.bias.ptr) ? p.bias.off + tc_decomp(p.Z, zi, p.bias.sz) +
                                          tc_decomp(p.N, n, p.bias.s2) : 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  const int64_t kper = ((p.k + p.splits - 1) / p.splits + TC_BK - 1) / TC_BK * TC_BK;
  const int64_t kbeg = split * kper;
  const int64_t kend = min(p.k, kbeg + kper);
  const int64_t ntiles = kend > kbeg ? (kend - kbeg + TC_BK - 1) / TC_BK : 0;
  const bool a_kfast = (p.K.nd > 0 && p.A.s2[p.K.nd - 1] == 1);
  const bool b_kfast = (p.K.nd > 0 && p.B.s1[p.K.nd - 1] == 1);
  // 128-bit loads: 4 consecutive elements along the contiguous dim, all groups
  // 16-byte aligned (every offset a multiple of 4 elements)
  const bool a_mfast = (p.M.nd > 0 && p.A.s1[p.M.nd - 1] == 1);
  const bool b_nfast = (p.N.nd > 0 && p.B.s2[p.N.nd - 1] == 1);
  bool a_vec = false, b_vec = false;
  {
    bool a_al = ((p.A.ptr + 4 * (uint64_t)p.A.off) & 15) == 0;
    bool b_al = ((p.B.ptr + 4 * (uint64_t)p.B.off) & 15) == 0;
    bool ka = a_kfast && (p.K.ext[p.K.nd - 1] % 4 == 0);
    for (int d = 0; d < p.K.nd - 1 && ka; ++d) ka = (p.A.s2[d] % 4 == 0);
    for (int d = 0; d < p.M.nd && ka; ++d) ka = (p.A.s1[d] % 4 == 0);
    bool ma = !a_kfast && a_mfast && (p.M.ext[p.M.nd - 1] % 4 == 0);
    for (int d = 0; d < p.M.nd - 1 && ma; ++d) ma = (p.A.s1[d] % 4 == 0);
    for (int d = 0; d < p.K.nd && ma; ++d) ma = (p.A.s2[d] % 4 == 0);
    for (int d = 0; d < p.Z.nd; ++d) a_al = a_al && (p.A.sz[d] % 4 == 0);
    a_vec = a_al && (ka || ma) && p.A.dtype == RT_F32;
    bool kb = b_kfast && (p.K.ext[p.K.nd - 1] % 4 == 0);
    for (int d = 0; d < p.K.nd - 1 && kb; ++d) kb = (p.B.s1[d] % 4 == 0);
    for (int d = 0; d < p.N.nd && kb; ++d) kb = (p.B.s2[d] % 4 == 0);
    bool nb = !b_kfast && b_nfast && (p.N.ext[p.N.nd - 1] % 4 == 0);
    for (int d = 0; d < p.N.nd - 1 && nb; ++d) nb = (p.B.s2[d] % 4 == 0);
    for (int d = 0; d < p.K.nd && nb; ++d) nb = (p.B.s1[d] % 4 == 0);
    for (int d = 0; d < p.Z.nd; ++d) b_al = b_al && (p.B.sz[d] % 4 == 0);
    b_vec = b_al && (kb || nb) && p.B.dtype == RT_F32;
    if (a_vec && !a_kfast) { /* M-contiguous */ }
  }
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(TC_BM >> 4) << 24);
  const float* Ap = (const float*)p.A.ptr;
  const float* Bp = (const float*)p.B.ptr;

  for (int64_t kt = 0; kt < ntiles; ++kt) {
    const int st = (int)(kt % TC_STAGES);
    unsigned char* sb = smem + st * stage_bytes;
    if (kt >= TC_STAGES) tc_wait(&bars[st], (uint32_t)(((kt / TC_STAGES) - 1) & 1));
    const int64_t k0 = kbeg + kt * TC_BK;
    if (tid < TC_BK) {
      int64_t k = k0 + tid;
      kA[tid] = k < kend ? tc_decomp(p.K, k, p.A.s2) : 0;
    } else if (tid >= 64 && tid < 64 + TC_BK) {
      int64_t k = k0 + tid - 64;
      kB[tid - 64] = k < kend ? tc_decomp(p.K, k, p.B.s1) : 0;
    }
    __syncthreads();
    // A tile: 128 x BK, 128-bit loads along the operand's contiguous dim
    if (a_vec) {
      if (a_kfast) {
#pragma unroll
        for (int i = 0; i < (TC_BM * TC_BK / 4) / TC_THREADS; ++i) {
          int e = tid + TC_THREADS * i;
          int r = e / (TC_BK / 4), k4 = (e % (TC_BK / 4)) * 4;
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (m0 + r < p.m && k0 + k4 + 3 < kend)
            x = *(const float4*)(Ap + rowA[r] + kA[k4]);
          else if (m0 + r < p.m)
            for (int j = 0; j < 4; ++j)
              if (k0 + k4 + j < kend) (&x.x)[j] = Ap[rowA[r] + kA[k4 + j]];
          split_store4(sb, a_bytes, tc_off(r, k4), x);
        }
      } else {
#pragma unroll
        for (int i = 0; i < (TC_BM * TC_BK / 4) / TC_THREADS; ++i) {
          int e = tid + TC_THREADS * i;
          int k = e / (TC_BM / 4), r4 = (e % (TC_BM / 4)) * 4;
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (k0 + k < kend) {
            if (m0 + r4 + 3 < p.m) x = *(const float4*)(Ap + rowA[r4] + kA[k]);
            else
              for (int j = 0; j < 4; ++j)
                if (m0 + r4 + j < p.m) (&x.x)[j] = Ap[rowA[r4 + j] + kA[k]];
          }
          for (int j = 0; j < 4; ++j) split_store1(sb, a_bytes, tc_off(r4 + j, k), (&x.x)[j]);
        }
      }
    } else {
      for (int i = 0; i < (TC_BM * TC_BK) / TC_THREADS; ++i) {
        int e = tid + TC_THREADS * i;
        int r, k;
        if (a_kfast) { r = e / TC_BK; k = e % TC_BK; } else { k = e / TC_BM; r = e % TC_BM; }
        bool ok = (m0 + r < p.m) && (k0 + k < kend);
        split_store1(sb, a_bytes, tc_off(r, k), ok ? Ap[rowA[r] + kA[k]] : 0.f);
      }
    }
    // B tile: BN x BK (rows = n)
    unsigned char* sbB = sb + 2 * a_bytes;
    if (b_vec) {
      if (b_kfast) {
        for (int i = 0; i < (256 * TC_BK / 4) / TC_THREADS; ++i) {
          int e = tid + TC_THREADS * i;
          int c = e / (TC_BK / 4), k4 = (e % (TC_BK / 4)) * 4;
          if (c >= BN) continue;
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (n0 + c < p.n && k0 + k4 + 3 < kend)
            x = *(const float4*)(Bp + colB[c] + kB[k4]);
          else if (n0 + c < p.n)
            for (int j = 0; j < 4; ++j)
              if (k0 + k4 + j < kend) (&x.x)[j] = Bp[colB[c] + kB[k4 + j]];
          split_store4(sbB, b_bytes, tc_off(c, k4), x);
        }
      } else {
        for (int i = 0; i < (256 * TC_BK / 4) / TC_THREADS; ++i) {
          int e = tid + TC_THREADS * i;
          int k = e / 64, c4 = (e % 64) * 4;
          if (c4 >= BN) continue;
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (k0 + k < kend) {
            if (n0 + c4 + 3 < p.n) x = *(const float4*)(Bp + colB[c4] + kB[k]);
            else
              for (int j = 0; j < 4; ++j)
                if (n0 + c4 + j < p.n) (&x.x)[j] = Bp[colB[c4 + j] + kB[k]];
          }
          for (int j = 0; j < 4; ++j) split_store1(sbB, b_bytes, tc_off(c4 + j, k), (&x.x)[j]);
        }
      }
    } else {
      for (int i = 0; i < (256 * TC_BK) / TC_THREADS; ++i) {
        int e = tid + TC_THREADS * i;
        int c, k;
        if (b_kfast) { c = e / TC_BK; k = e % TC_BK; } else { k = e / 256; c = e % 256; }
        if (c >= BN) continue;
        bool ok = (n0 + c < p.n) && (k0 + k < kend);
        split_store1(sbB, b_bytes, tc_off(c, k), ok ? Bp[colB[c] + kB[k]] : 0.f);
      }
    }
    // make the generic-proxy smem writes visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = tc_smem(sb);
      const uint32_t sbo = TC_BK * 32;   // 8-row group stride (BK/4 core matrices of 128 B)
#pragma unroll
      for (int s = 0; s < TC_BK / 8; ++s) {
        const uint32_t ko = s * 256;      // two 16B core matrices along K per MMA
        uint64_t ahi = tc_desc(base + ko, 128, sbo);
        uint64_t alo = tc_desc(base + a_bytes + ko, 128, sbo);
        uint64_t bhi = tc_desc(base + 2 * a_bytes + ko, 128, sbo);
        uint64_t blo = tc_desc(base + 2 * a_bytes + b_bytes + ko, 128, sbo);
        uint32_t acc = (kt > 0 || s > 0) ? 1u : 0u;
        tc_mma(tmem, ahi, bhi, idesc, acc);
        tc_mma(tmem, ahi, blo, idesc, 1u);
        tc_mma(tmem, alo, bhi, idesc, 1u);
      }
      tc_commit(&bars[st]);
    }
  }
  // drain: wait for the last commit of every stage in flight
  if (ntiles > 0) {
    int64_t last = ntiles - 1;
    tc_wait(&bars[last % TC_STAGES], (uint32_t)((last / TC_STAGES) & 1));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");

  // epilogue: warp w reads TMEM lanes [32(w%4), +32) = tile rows, column half w/4
  const int wq = warp & 3, wh = warp >> 2;
  const int r = wq * 32 + lane;
  const int64_t m = m0 + r;
  const int half = ((BN / 2) + 15) / 16 * 16;
  const int cbeg = wh * half, cend = wh ? BN : (half < BN ? half : BN);
  for (int c0 = cbeg; c0 < cend; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (ntiles == 0)
      for (int j = 0; j < 16; ++j) v[j] = 0u;
    if (m >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = c0 + j;
      const int64_t n = n0 + c;
      if (n >= p.n) break;
      float x = __uint_as_float(v[j]);
      if (p.splits > 1) {
        float* part = (float*)p.part;
        part[((split * p.z + zi) * p.m + m) * p.n + n] = x;
        continue;
      }
      int64_t oc = rowC[r] + colC[c];
      if (p.accumulate) x += ((const float*)p.C.ptr)[oc];
      if (p.bias.ptr) x += load_as<float>((const void*)p.bias.ptr, p.bias.dtype, colBias[c]);
      if (p.epilogue == 1) x = tanh_fast(x);
      ((float*)p.C.ptr)[oc] = x;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

extern "C" void* rt_kernel_gemm_tc() { return (void*)k_gemm_tc; }
extern "C" int rt_gemm_tc_smem() { return TC_STAGES * (2 * TC_BM * TC_BK * 4 + 2 * 256 * TC_BK * 4); }
