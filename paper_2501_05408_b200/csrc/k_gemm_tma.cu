// RT_K_GEMM_TMA — the learner GEMMs of the PDG backward on tcgen05 with a
// TMA-fed, warp-specialised pipeline (3xTF32 for fp32 accuracy; reference
// products are fp32 np.matmul, runtime.py:249; north_star tolerance 1e-5).
//
//   dX = G @ W^T over all T*E points   (M = 1M rows, K-major operands)
//   dW = sum_points x^T g              (K = 1M points, MN-major operands, split-K)
//
// Roles (320 threads):
//   warp 8 lane 0  TMA producer: raw fp32 tiles -> smem ring (SWIZZLE_64B
//                  K-major or SWIZZLE_128B_BASE32B MN-major UMMA layouts)
//   warps 0-7      converters: in place hi = tf32(x), lo = tf32(x - hi) into a
//                  twin buffer (elementwise, so layout-agnostic and
//                  conflict-free), then the epilogue (TMEM -> global)
//   warp 9 lane 0  MMA issuer: hi*hi + hi*lo + lo*hi per K=8 step, commit
//                  releases the stage back to the producer
// Stage = A(128 x 16) + B(256 x 16) fp32, hi and lo: 48 KB.
// Operands must be plain 2-D (collapsed boxes), one unit-stride dim, 16-byte
// aligned — lower.py checks that, else RT_K_GEMM_TC (generic staging) runs.
//
// Accumulation bias.  The tensor core's fp32 accumulation truncates (rounds
// toward zero) once per MMA, so a long K chain shrinks |C| systematically by
// about 3e-8 per MMA into the same accumulator (measured, tools/tc_bias.py:
// -2.1e-5 relative at 2 k MMAs per accumulator, -7.9e-5 at 2.6 k — the C2
// dW2 contraction — while fp32 SIMT stays unbiased).  Launches whose K per
// CTA exceeds TM_DRAIN_K therefore run the DRAIN variant: one CTA per SM, two
// TMEM accumulators; every TM_DRAIN_K of K the MMA issuer switches
// accumulator and the converter warps drain the finished one into fp32
// registers (round-to-nearest adds), so no accumulator sees more than
// 3 * TM_DRAIN_K / 8 = 96 MMAs (bias ~2.4e-6, as the K = 256 row GEMMs).
#include <cuda.h>
#include "common.cuh"

#define TM_BM 128
#define TM_BN 256
#define TM_BK 16
#define TM_ST 2   // 2 stages: two CTAs per SM, one's epilogue overlaps the other's mainloop
#define TM_ST_DRAIN 4   // drain variant: one CTA per SM, deeper ring
#define TM_DRAIN_K 256  // K elements per TMEM accumulation chunk (drain variant)
#define TM_CONV 256
#define TM_THREADS (TM_CONV + 64)
#define TM_A_BYTES (TM_BM * TM_BK * 4)
#define TM_B_BYTES (TM_BN * TM_BK * 4)
#define TM_STAGE (2 * TM_A_BYTES + 2 * TM_B_BYTES)
#define TM_SMEM (TM_ST * TM_STAGE + 1024)
#define TM_SMEM_DRAIN (TM_ST_DRAIN * TM_STAGE + 1024)

struct tm_args {
  CUtensorMap ta;
  CUtensorMap tb;
  rt_gemm_params p;
  int32_t a_mn, b_mn;      // operand is MN-major (unit stride along M / N)
  int64_t c_m, c_n;        // collapsed C strides
  int64_t bias_n;          // collapsed bias stride along N
  int64_t g_m, g_n;        // epilogue 2: the gate operand's strides (in p.bias)
  CUtensorMap tbh, tbl;    // PRESPLIT: B's tf32 hi / lo parts (same geometry as tb)
  uint64_t b_base, b_span; // PRESPLIT: B element base address and span (elements)
  int32_t presplit, _pad2; // 1: B split in place; 2: split AND transposed to K-major
  int64_t b_ld, b_kk, b_nn; // presplit 2: the MN-major source's row stride, K, N
  CUtensorMap tc;           // persistent epilogue: C as 16-col x 32-row boxes (SWIZZLE_64B)
  int32_t c_tma, _pad3;     // 1: the epilogue stores C through shared memory + TMA
  int32_t a3d, b3d;         // MN-major operand as ONE 3-D box (32-wide groups on dim 2)
};

namespace {

RT_DEV uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

RT_DEV void mb_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
RT_DEV void mb_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  }
}
RT_DEV void mb_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
RT_DEV void mb_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// L2 prefetch of a TMA box (no shared memory, no barrier): the A operand
// tile a few stages ahead, so the stage's TMA load is an L2 hit
RT_DEV void tma2d_prefetch(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];"
               ::"l"((uint64_t)map), "r"(c0), "r"(c1) : "memory");
}
RT_DEV void tma2d_store(const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"((uint64_t)map), "r"(c0), "r"(c1), "r"(src) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
RT_DEV void tma3d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                  uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
RT_DEV void tma2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
// smem matrix descriptor (sm_100 version 1), layout: 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
RT_DEV uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
RT_DEV void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
RT_DEV void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(bar) : "memory");
}
RT_DEV uint32_t rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// descriptor of operand tile at `base` for MMA K-step ks (8 fp32 of K)
RT_DEV uint64_t op_desc(uint32_t base, int ks, int mn) {
  // MN-major 32-bit operands need SWIZZLE_128B_BASE32B (layout 1; plain
  // SWIZZLE_128B reads as zeros for tf32 — measured, tools/probe/tc_probe2.cu):
  // 128 B MN rows, 4-k atoms 512 B apart (SBO), 32-wide MN groups 2 KB apart
  // (LBO); one K=8 MMA step spans two atoms.
  if (mn)
    return sdesc(base + ks * 1024, 2048, 512, 1);
  // K-major SW64: 64 B rows, 8-row groups 512 B apart; K-step = +32 B
  return sdesc(base + ks * 32, 16, 512, 4);
}

}  // namespace

template <int ST, bool DRAIN>
__device__ __forceinline__ void gemm_tma_body(const tm_args& a) {
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[ST], conv[ST], empty[ST], done, accfull[2], accfree[2];
  __shared__ uint32_t tmem_s;
  const rt_gemm_params& p = a.p;
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = su32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * TM_BM;
  const int64_t n0 = (int64_t)blockIdx.y * TM_BN;
  const int64_t nrem = p.n - n0;
  const int split = blockIdx.z;
  // MMA N: multiple of 16 (K-major B) / of 32 (MN-major B, whole 32-wide atoms)
  const int BN = nrem >= TM_BN ? TM_BN
               : a.b_mn ? (int)((nrem + 31) / 32 * 32) : (int)((nrem + 15) / 16 * 16);
  const int nbB = a.b_mn ? BN / 32 : 1;
  const uint32_t bytesB = a.b_mn && !a.b3d ? nbB * 32 * TM_BK * 4 : TM_B_BYTES;

  constexpr uint32_t TCOLS = DRAIN ? 512 : 256;
  constexpr int KD = TM_DRAIN_K / TM_BK;     // k-tiles per accumulation chunk (DRAIN)
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mb_init(su32(&full[i]), 1);
      mb_init(su32(&conv[i]), TM_CONV);
      mb_init(su32(&empty[i]), 1);
    }
    mb_init(su32(&done), 1);
    for (int i = 0; i < 2; ++i) {
      mb_init(su32(&accfull[i]), 1);
      mb_init(su32(&accfree[i]), TM_CONV);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(su32(&tmem_s)), "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_s;

  const int64_t kper = ((p.k + p.splits - 1) / p.splits + TM_BK - 1) / TM_BK * TM_BK;
  const int64_t kbeg = split * kper;
  const int64_t kend = p.k < kbeg + kper ? p.k : kbeg + kper;
  const int ntiles = kend > kbeg ? (int)((kend - kbeg + TM_BK - 1) / TM_BK) : 0;

  if (warp == 8) {
    if (lane == 0) {
      for (int kt = 0; kt < ntiles; ++kt) {
        const int s = kt % ST;
        if (kt >= ST) mb_wait(su32(&empty[s]), (uint32_t)(((kt / ST) - 1) & 1));
        const uint32_t st = sbase + s * TM_STAGE;
        const uint32_t fb = su32(&full[s]);
        mb_expect(fb, TM_A_BYTES + bytesB);
        const int32_t k0 = (int32_t)(kbeg + (int64_t)kt * TM_BK);
        if (a.a_mn && a.a3d)
          tma3d(st, &a.ta, 0, k0, (int32_t)(m0 / 32), fb);
        else if (a.a_mn)
          for (int j = 0; j < TM_BM / 32; ++j)
            tma2d(st + j * 2048, &a.ta, (int32_t)(m0 + 32 * j), k0, fb);
        else
          tma2d(st, &a.ta, k0, (int32_t)m0, fb);
        const uint32_t sb = st + 2 * TM_A_BYTES;
        if (a.b_mn && a.b3d)
          tma3d(sb, &a.tb, 0, k0, (int32_t)(n0 / 32), fb);
        else if (a.b_mn)
          for (int j = 0; j < nbB; ++j) tma2d(sb + j * 2048, &a.tb, (int32_t)(n0 + 32 * j), k0, fb);
        else
          tma2d(sb, &a.tb, k0, (int32_t)n0, fb);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a.a_mn << 15) |
                             ((uint32_t)a.b_mn << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(TM_BM >> 4) << 24);
      for (int kt = 0; kt < ntiles; ++kt) {
        const int s = kt % ST;
        const int c = DRAIN ? kt / KD : 0, kc = DRAIN ? kt - c * KD : kt;
        const uint32_t acc = tmem + (uint32_t)(256 * (c & 1));
        if (DRAIN && kc == 0 && c >= 2)   // the converters drained this accumulator
          mb_wait(su32(&accfree[c & 1]), (uint32_t)(((c >> 1) - 1) & 1));
        mb_wait(su32(&conv[s]), (uint32_t)((kt / ST) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t st = sbase + s * TM_STAGE;
        const uint32_t ahi = st, alo = st + TM_A_BYTES;
        const uint32_t bhi = st + 2 * TM_A_BYTES, blo = bhi + TM_B_BYTES;
#pragma unroll
        for (int ks = 0; ks < TM_BK / 8; ++ks) {
          const uint64_t dah = op_desc(ahi, ks, a.a_mn), dal = op_desc(alo, ks, a.a_mn);
          const uint64_t dbh = op_desc(bhi, ks, a.b_mn), dbl = op_desc(blo, ks, a.b_mn);
          mma_tf32(acc, dah, dbh, idesc, (kc > 0 || ks > 0) ? 1u : 0u);
          mma_tf32(acc, dah, dbl, idesc, 1u);
          mma_tf32(acc, dal, dbh, idesc, 1u);
        }
        mma_commit(su32(&empty[s]));
        if (DRAIN && (kc == KD - 1 || kt == ntiles - 1)) mma_commit(su32(&accfull[c & 1]));
      }
      mma_commit(su32(&done));
    }
  } else {
    // converters: hi in place, lo into the twin buffer
    const int wq = warp & 3, wh = warp >> 2;
    float racc[DRAIN ? 128 : 1];     // DRAIN: this thread's row, column half wh
#pragma unroll
    for (int j = 0; j < (DRAIN ? 128 : 1); ++j) racc[j] = 0.f;
#define TM_DRAIN(c_)                                                                          \
  do {                                                                                        \
    const int cc_ = (c_);                                                                     \
    mb_wait(su32(&accfull[cc_ & 1]), (uint32_t)((cc_ >> 1) & 1));                             \
    asm volatile("tcgen05.fence::after_thread_sync;");                                        \
    const uint32_t base_ = tmem + (uint32_t)(256 * (cc_ & 1)) + ((uint32_t)(wq * 32) << 16) + \
                           (uint32_t)(128 * wh);                                              \
    _Pragma("unroll") for (int q = 0; q < (DRAIN ? 8 : 0); ++q) {                             \
      uint32_t v[16];                                                                         \
      asm volatile(                                                                           \
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), \
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),       \
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15])                                             \
          : "r"(base_ + 16u * q));                                                            \
      asm volatile("tcgen05.wait::ld.sync.aligned;");                                         \
      _Pragma("unroll") for (int j = 0; j < 16; ++j)                                          \
        racc[(16 * q + j) & (DRAIN ? 127 : 0)] += __uint_as_float(v[j]);                      \
    }                                                                                         \
    asm volatile("tcgen05.fence::before_thread_sync;");                                       \
    mb_arrive(su32(&accfree[cc_ & 1]));                                                       \
  } while (0)
    for (int kt = 0; kt < ntiles; ++kt) {
      const int s = kt % ST;
      mb_wait(su32(&full[s]), (uint32_t)((kt / ST) & 1));
      const uint32_t st = sbase + s * TM_STAGE;
      constexpr int NA = TM_A_BYTES / 16, NB = TM_B_BYTES / 16;
      constexpr int NI = (NA + NB) / TM_CONV;
      static_assert((NA + NB) % TM_CONV == 0 && NA % TM_CONV == 0, "whole conversion rounds");
      // explicit shared-space accesses (generic LD/ST.E here were tracked on
      // the long scoreboard), all of a thread's loads issued before its stores
      // (DRAIN: two half batches — the 128 drain accumulators leave 168 - 128
      // registers, the per-SMSP limit for 10 warps)
      constexpr int NB_ = DRAIN ? NI / 2 : NI;
#pragma unroll
      for (int j0 = 0; j0 < NI; j0 += NB_) {
        float4 xs[NB_];
#pragma unroll
        for (int jj = 0; jj < NB_; ++jj) {
          const int i = tid + (j0 + jj) * TM_CONV;
          const uint32_t off = i < NA ? i * 16 : 2 * TM_A_BYTES + (i - NA) * 16;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(xs[jj].x), "=f"(xs[jj].y), "=f"(xs[jj].z), "=f"(xs[jj].w) : "r"(st + off));
        }
#pragma unroll
        for (int jj = 0; jj < NB_; ++jj) {
          const int i = tid + (j0 + jj) * TM_CONV;
          const uint32_t off = i < NA ? i * 16 : 2 * TM_A_BYTES + (i - NA) * 16;
          const uint32_t lo_off = i < NA ? TM_A_BYTES : TM_B_BYTES;
          const float4 x = xs[jj];
          uint4 h, l;
          h.x = rna(x.x); h.y = rna(x.y); h.z = rna(x.z); h.w = rna(x.w);
          l.x = rna(x.x - __uint_as_float(h.x)); l.y = rna(x.y - __uint_as_float(h.y));
          l.z = rna(x.z - __uint_as_float(h.z)); l.w = rna(x.w - __uint_as_float(h.w));
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(st + off), "r"(h.x), "r"(h.y), "r"(h.z), "r"(h.w));
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(st + off + lo_off), "r"(l.x), "r"(l.y), "r"(l.z), "r"(l.w));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mb_arrive(su32(&conv[s]));
      // DRAIN: the previous chunk, once the first tile of this one is converted
      if (DRAIN && kt % KD == 0 && kt > 0) TM_DRAIN(kt / KD - 1);
    }
    if (DRAIN && ntiles > 0) TM_DRAIN((ntiles - 1) / KD);
    // epilogue: warp w reads TMEM lanes 32(w%4).. (= tile rows), column half w/4
    if (ntiles > 0) mb_wait(su32(&done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int r = wq * 32 + lane;
    const int64_t m = m0 + r;
    const int half = DRAIN ? 128 : ((BN / 2) + 15) / 16 * 16;
    const int cbeg = wh * half;
    const int cend = DRAIN ? (cbeg + 128 < BN ? cbeg + 128 : BN) : (wh ? BN : (half < BN ? half : BN));
    float* Cp = (float*)p.C.ptr;
    const bool vec = p.splits == 1 && a.c_n == 1 && ((p.C.ptr + 4 * (p.C.off + m * a.c_m)) & 15) == 0;
    // (DRAIN: the columns come from racc, so the chunk loop is unrolled
    // with static indices; the 128-column halves start at 128 * wh)
#pragma unroll
    for (int qq = 0; qq < (DRAIN ? 8 : 1); ++qq)
    for (int c0 = DRAIN ? 128 * wh + 16 * qq : cbeg; c0 < (DRAIN ? (128 * wh + 16 * qq + 16 < cend ? 128 * wh + 16 * qq + 16 : cend) : cend); c0 += 16) {
      float x[16];
      // epilogue 2: this row's 16 gate values, issued before the TMEM read
      // (four 16-byte loads when contiguous and aligned)
      float gv[16];
      if (!DRAIN && p.epilogue == 2 && m < p.m) {   // (the gate runs only with K <= 256)
        const float* gp = (const float*)p.bias.ptr + p.bias.off + m * a.g_m + (n0 + c0) * a.g_n;
        if (a.g_n == 1 && n0 + c0 + 16 <= p.n && (reinterpret_cast<uintptr_t>(gp) & 15) == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 g4 = __ldcs(reinterpret_cast<const float4*>(gp) + q);
            gv[4 * q] = g4.x; gv[4 * q + 1] = g4.y; gv[4 * q + 2] = g4.z; gv[4 * q + 3] = g4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) gv[j] = n0 + c0 + j < p.n ? gp[j * a.g_n] : 0.f;
        }
      }
      if constexpr (DRAIN) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = racc[(16 * qq + j) & 127];
      } else {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = ntiles == 0 ? 0.f : __uint_as_float(v[j]);
      }
      if (m >= p.m) continue;
      if (p.splits > 1) {
        float* part = (float*)p.part + ((int64_t)split * p.m + m) * p.n + n0;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (n0 + c0 + j < p.n) part[c0 + j] = x[j];
        continue;
      }
      const int64_t rowoff = p.C.off + m * a.c_m;
      // the 16 bias values of this chunk (the same for every row/thread):
      // four 16-byte loads when contiguous fp32, not a dtype-dispatched load
      // per element (the bias+tanh forward GEMM ran ~30% slower than dX)
      float bv[16];
      if (!DRAIN && p.epilogue == 2) {
        // tanh-VJP gate (frontend.py:961-963): x * (1 - h*h), h laid out like
        // C; each op rounded like numpy's (no contraction into an FMA)
#pragma unroll
        for (int j = 0; j < 16; ++j) bv[j] = __fsub_rn(1.f, __fmul_rn(gv[j], gv[j]));
      } else if (p.bias.ptr) {
        const int64_t b0 = p.bias.off + (n0 + c0) * a.bias_n;
        const float* bp = (const float*)p.bias.ptr + b0;
        if (a.bias_n == 1 && p.bias.dtype == RT_F32 && n0 + c0 + 16 <= p.n &&
            (reinterpret_cast<uintptr_t>(bp) & 15) == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(bp) + q);
            bv[4 * q] = b4.x; bv[4 * q + 1] = b4.y; bv[4 * q + 2] = b4.z; bv[4 * q + 3] = b4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            bv[j] = n0 + c0 + j < p.n
                        ? load_as<float>((const void*)p.bias.ptr, p.bias.dtype, b0 + j * a.bias_n) : 0.f;
        }
      }
      // every column unconditionally (the stores below are guarded): the 16
      // independent epilogue chains unroll and interleave
      if (p.accumulate) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t n = n0 + c0 + j;
          if (n < p.n) x[j] += Cp[rowoff + n * a.c_n];
        }
      }
      if (!DRAIN && p.epilogue == 2) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = __fmul_rn(x[j], bv[j]);
      } else {
        if (p.bias.ptr) {
#pragma unroll
          for (int j = 0; j < 16; ++j) x[j] += bv[j];
        }
        if (p.epilogue == 1) {
#pragma unroll
          for (int j = 0; j < 16; ++j) x[j] = tanh_fast(x[j]);
        }
      }
      if (vec && n0 + c0 + 16 <= p.n) {
        float4* dst = (float4*)(Cp + rowoff + n0 + c0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          __stcs(dst + j, make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]));
      } else {
        for (int j = 0; j < 16; ++j) {
          const int64_t n = n0 + c0 + j;
          if (n >= p.n) break;
          Cp[rowoff + n * a.c_n] = x[j];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
}

__global__ void __launch_bounds__(TM_THREADS, 2) k_gemm_tma(const __grid_constant__ tm_args a) {
  gemm_tma_body<TM_ST, false>(a);
}
// 10 warps, 3 on some SM sub-partition: 16 K registers / 96 threads -> 168
__global__ void __launch_bounds__(TM_THREADS, 1) k_gemm_tma_drain(const __grid_constant__ tm_args a) {
  gemm_tma_body<TM_ST_DRAIN, true>(a);
}


// ---------------------------------------------------------------- persistent
// Warp-specialised persistent variant for launches with one K chunk (K <=
// TM_DRAIN_K, no split): one CTA per SM loops over the output tiles; TMEM
// holds two 256-column accumulators so four epilogue warps drain tile i
// (TMEM -> gate/bias/tanh -> HBM) while the MMA issuer fills tile i+1; the
// operand ring has 4 stages.  PRESPLIT: B (a weight matrix every M tile
// reads) was split into tf32 hi / lo arrays once by k_tf32_split for the
// launch; TMA loads them straight into the stage's hi / lo slots and the
// converters only split A (the converters' shared-memory traffic bounded
// the per-tile variant: ncu tensor pipe 29%, smem 31%, long-scoreboard
// stalls on per-tile prologues).
#define TP_ST 4
#ifndef TM_3D
#define TM_3D 1   // MN-major operands as one 3-D TMA box per stage
#endif
#ifndef TP_TMA_STORE
#define TP_TMA_STORE 1   // persistent epilogue: C through shared memory + TMA store
#endif
#ifndef TM_TRACE
#define TM_TRACE 0
#endif
#if TM_TRACE
// per-role timestamps of CTA 0 (globaltimer ns): [role][event]
__device__ long long g_tm_trace[10][512];
#define TM_TS(role, idx) do { if (blockIdx.x == 0 && (idx) < 512) { long long t_; \
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_tm_trace[role][idx] = t_; } } while (0)
#else
#define TM_TS(role, idx) do {} while (0)
#endif
#ifndef TM_NO_B
#define TM_NO_B 0
#endif
#ifndef TM_PASSES
#define TM_PASSES 3  // 3xTF32 (hi*hi + hi*lo + lo*hi); fewer only for bound experiments (wrong results)
#endif
#ifndef TP_PF
#define TP_PF 0      // A-tile L2 prefetch distance (stages; 8 measured slower: h2_n 0.56 -> 0.74 ms)
#endif
#define TP_CONV 128  // converter threads (warps 0-3; PRESPLIT leaves them only A)
#define TP_EPI 8     // epilogue warps 6-13: two per TMEM lane quarter (column halves)
#define TP_THREADS (TP_CONV + 64 + 32 * TP_EPI)
#define TP_STAGE_EPI (2 * 32 * 16 * 4)   // per epilogue warp: two C chunks of 32 rows x 16 cols
#define TP_SMEM (TP_ST * TM_STAGE + 1024 + TP_EPI * TP_STAGE_EPI)

template <bool PRESPLIT>
__device__ __forceinline__ void gemm_tmap_body(const tm_args& a) {
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[TP_ST], conv[TP_ST], empty[TP_ST], accfull[2], accfree[2];
  __shared__ uint32_t tmem_s;
  const rt_gemm_params& p = a.p;
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = su32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t mt = (p.m + TM_BM - 1) / TM_BM, nt = (p.n + TM_BN - 1) / TM_BN;
  const int64_t ntile = mt * nt;
  const int ktiles = (int)((p.k + TM_BK - 1) / TM_BK);
  if (tid == 0) {
    for (int i = 0; i < TP_ST; ++i) {
      mb_init(su32(&full[i]), 1);
      mb_init(su32(&conv[i]), TP_CONV);
      mb_init(su32(&empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mb_init(su32(&accfull[i]), 1);
      mb_init(su32(&accfree[i]), 32 * TP_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"(su32(&tmem_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_s;
  auto tile_bn = [&](int64_t ni) {
    const int64_t nrem = p.n - ni * TM_BN;
    return nrem >= TM_BN ? TM_BN
           : a.b_mn ? (int)((nrem + 31) / 32 * 32) : (int)((nrem + 15) / 16 * 16);
  };

  if (warp == TP_CONV / 32) {                    // TMA producer
    if (lane == 0) {
      // A tiles TP_PF stages ahead are prefetched into L2 (the ring holds
      // only TP_ST - 1 stages of HBM latency; B is L2-resident anyway)
      auto prefetch_a = [&](int64_t gg) {
        const int64_t lt = gg / ktiles, tile2 = blockIdx.x + lt * gridDim.x;
        if (tile2 >= ntile) return;
        const int64_t m2 = (tile2 % mt) * TM_BM;
        const int32_t k2 = (int32_t)((gg % ktiles) * TM_BK);
        if (a.a_mn)
          for (int j = 0; j < TM_BM / 32; ++j) tma2d_prefetch(&a.ta, (int32_t)(m2 + 32 * j), k2);
        else
          tma2d_prefetch(&a.ta, k2, (int32_t)m2);
      };
      for (int64_t q = 0; q < TP_PF; ++q) prefetch_a(q);
      int64_t g = 0;
      for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int64_t mi = tile % mt, ni = tile / mt;
        const int64_t m0 = mi * TM_BM, n0 = ni * TM_BN;
        const int BN = tile_bn(ni);
        const int nbB = a.b_mn ? BN / 32 : 1;
        const uint32_t bytesB = a.b_mn && !a.b3d ? nbB * 32 * TM_BK * 4 : TM_B_BYTES;
        for (int kt = 0; kt < ktiles; ++kt, ++g) {
          if (TP_PF > 0) prefetch_a(g + TP_PF);
          const int s = (int)(g % TP_ST);
          if (g >= TP_ST) mb_wait(su32(&empty[s]), (uint32_t)(((g / TP_ST) - 1) & 1));
          const uint32_t st = sbase + s * TM_STAGE;
          const uint32_t fb = su32(&full[s]);
#if TM_NO_B   // bound experiment only: B never reloaded (wrong results)
          mb_expect(fb, TM_A_BYTES + ((g < TP_ST) ? (PRESPLIT ? 2 : 1) * bytesB : 0));
#else
          mb_expect(fb, TM_A_BYTES + (PRESPLIT ? 2 : 1) * bytesB);
#endif
          const int32_t k0 = kt * TM_BK;
          if (a.a_mn && a.a3d)
            tma3d(st, &a.ta, 0, k0, (int32_t)(m0 / 32), fb);
          else if (a.a_mn)
            for (int j = 0; j < TM_BM / 32; ++j) tma2d(st + j * 2048, &a.ta, (int32_t)(m0 + 32 * j), k0, fb);
          else
            tma2d(st, &a.ta, k0, (int32_t)m0, fb);
            TM_TS(0, g);
          const uint32_t sb = st + 2 * TM_A_BYTES;
#if TM_NO_B
          if (g >= TP_ST) continue;
#endif
#pragma unroll
          for (int part = 0; part < (PRESPLIT ? 2 : 1); ++part) {
            const CUtensorMap* mb = PRESPLIT ? (part ? &a.tbl : &a.tbh) : &a.tb;
            const uint32_t dst = sb + part * TM_B_BYTES;
            if (a.b_mn && a.b3d && !PRESPLIT)
              tma3d(dst, mb, 0, k0, (int32_t)(n0 / 32), fb);
            else if (a.b_mn)
              for (int j = 0; j < nbB; ++j) tma2d(dst + j * 2048, mb, (int32_t)(n0 + 32 * j), k0, fb);
            else
              tma2d(dst, mb, k0, (int32_t)n0, fb);
          }
        }
      }
    }
  } else if (warp == TP_CONV / 32 + 1) {         // MMA issuer
    if (lane == 0) {
      int64_t g = 0;
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++it) {
        const int BN = tile_bn(tile / mt);
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a.a_mn << 15) |
                               ((uint32_t)a.b_mn << 16) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(TM_BM >> 4) << 24);
        const int b = it & 1;
        const uint32_t acc = tmem + (uint32_t)(256 * b);
        if (it >= 2) mb_wait(su32(&accfree[b]), (uint32_t)(((it >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kt = 0; kt < ktiles; ++kt, ++g) {
          const int s = (int)(g % TP_ST);
          mb_wait(su32(&conv[s]), (uint32_t)((g / TP_ST) & 1));
          TM_TS(2, g);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = sbase + s * TM_STAGE;
          const uint32_t ahi = st, alo = st + TM_A_BYTES;
          const uint32_t bhi = st + 2 * TM_A_BYTES, blo = bhi + TM_B_BYTES;
#pragma unroll
          for (int ks = 0; ks < TM_BK / 8; ++ks) {
            const uint64_t dah = op_desc(ahi, ks, a.a_mn), dal = op_desc(alo, ks, a.a_mn);
            const uint64_t dbh = op_desc(bhi, ks, a.b_mn), dbl = op_desc(blo, ks, a.b_mn);
            mma_tf32(acc, dah, dbh, idesc, (kt > 0 || ks > 0) ? 1u : 0u);
#if TM_PASSES >= 2
            mma_tf32(acc, dah, dbl, idesc, 1u);
#endif
#if TM_PASSES >= 3
            mma_tf32(acc, dal, dbh, idesc, 1u);
#endif
          }
          mma_commit(su32(&empty[s]));
          TM_TS(3, g);
        }
        mma_commit(su32(&accfull[b]));
      }
    }
  } else if (warp < TP_CONV / 32) {              // converters: hi in place, lo into the twin
    int64_t g = 0;
    constexpr int NA = TM_A_BYTES / 16, NB = PRESPLIT ? 0 : TM_B_BYTES / 16;
    constexpr int NI = (NA + NB) / TP_CONV;
    static_assert((NA + NB) % TP_CONV == 0, "whole conversion rounds");
    for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
      for (int kt = 0; kt < ktiles; ++kt, ++g) {
        const int s = (int)(g % TP_ST);
        mb_wait(su32(&full[s]), (uint32_t)((g / TP_ST) & 1));
        if (tid == 0) TM_TS(1, g);
        const uint32_t st = sbase + s * TM_STAGE;
        float4 xs[NI];
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int i = tid + j * TP_CONV;
          const uint32_t off = i < NA ? i * 16 : 2 * TM_A_BYTES + (i - NA) * 16;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(xs[j].x), "=f"(xs[j].y), "=f"(xs[j].z), "=f"(xs[j].w) : "r"(st + off));
        }
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int i = tid + j * TP_CONV;
          const uint32_t off = i < NA ? i * 16 : 2 * TM_A_BYTES + (i - NA) * 16;
          const uint32_t lo_off = i < NA ? TM_A_BYTES : TM_B_BYTES;
          const float4 x = xs[j];
          uint4 h, l;
          h.x = rna(x.x); h.y = rna(x.y); h.z = rna(x.z); h.w = rna(x.w);
          l.x = rna(x.x - __uint_as_float(h.x)); l.y = rna(x.y - __uint_as_float(h.y));
          l.z = rna(x.z - __uint_as_float(h.z)); l.w = rna(x.w - __uint_as_float(h.w));
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(st + off), "r"(h.x), "r"(h.y), "r"(h.z), "r"(h.w));
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(st + off + lo_off), "r"(l.x), "r"(l.y), "r"(l.z), "r"(l.w));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mb_arrive(su32(&conv[s]));
        if (tid == 0) TM_TS(4, g);
      }
    }
  } else {                                       // epilogue warps
    const int wq = warp & 3;                     // TMEM lane quarter of this warp
    const int half = (warp - TP_CONV / 32 - 2) >> 2;   // column half of the tile
    const uint32_t estage = sbase + TP_ST * TM_STAGE;  // the epilogue warps' C chunks
    const int r = wq * 32 + lane;
    float* Cp = (float*)p.C.ptr;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++it) {
      const int64_t mi = tile % mt, ni = tile / mt;
      const int64_t m0 = mi * TM_BM, n0 = ni * TM_BN;
      const int BN = tile_bn(ni);
      const int hw = ((BN / 2) + 15) / 16 * 16;  // columns of half 0
      const int cbeg = half * hw, cend = half ? BN : (hw < BN ? hw : BN);
      const int b = it & 1;
      const int64_t m = m0 + r;
      const bool live = m < p.m;
      const bool gate = p.epilogue == 2 && live;
      const float* gbase = (const float*)p.bias.ptr + p.bias.off + m * a.g_m + n0 * a.g_n;
      const bool gvec = a.g_n == 1 && ((reinterpret_cast<uintptr_t>(gbase) & 15) == 0);
      // this row's gate values one chunk ahead (the HBM latency of chunk c+1
      // overlaps chunk c; before the first, it overlaps the accumulator wait)
      float gn[16];
      auto load_gate = [&](int c0, float (&gv)[16]) {
        if (c0 >= cend) return;
        if (p.epilogue != 2) {
          // no gate: prefetch this chunk's bias instead (row-independent; a
          // load after the accumulator read exposed ~1 us per chunk)
          if (!p.bias.ptr) return;
          const int64_t b0 = p.bias.off + (n0 + c0) * a.bias_n;
          const float* bp = (const float*)p.bias.ptr + b0;
          if (a.bias_n == 1 && p.bias.dtype == RT_F32 && n0 + c0 + 16 <= p.n &&
              (reinterpret_cast<uintptr_t>(bp) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bp) + q);
              gv[4 * q] = b4.x; gv[4 * q + 1] = b4.y; gv[4 * q + 2] = b4.z; gv[4 * q + 3] = b4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              gv[j] = n0 + c0 + j < p.n
                          ? load_as<float>((const void*)p.bias.ptr, p.bias.dtype, b0 + j * a.bias_n) : 0.f;
          }
          return;
        }
        if (!gate) return;
        const float* gp = gbase + c0 * a.g_n;
        if (gvec && n0 + c0 + 16 <= p.n) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 g4 = __ldcs(reinterpret_cast<const float4*>(gp) + q);
            gv[4 * q] = g4.x; gv[4 * q + 1] = g4.y; gv[4 * q + 2] = g4.z; gv[4 * q + 3] = g4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) gv[j] = n0 + c0 + j < p.n ? gp[j * a.g_n] : 0.f;
        }
      };
      // two chunks ahead: 2 x 64 B of HBM reads in flight per thread
      float gn2[16];
      load_gate(cbeg, gn);
      load_gate(cbeg + 16, gn2);
      mb_wait(su32(&accfull[b]), (uint32_t)((it >> 1) & 1));
      if (warp == TP_CONV / 32 + 2 && lane == 0) TM_TS(5, it);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const bool vec = a.c_n == 1 && ((p.C.ptr + 4 * (p.C.off + m * a.c_m)) & 15) == 0;
      const int64_t rowoff = p.C.off + m * a.c_m;
      for (int c0 = cbeg; c0 < cend; c0 += 16) {
        float gv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) { gv[j] = gn[j]; gn[j] = gn2[j]; }
        load_gate(c0 + 32, gn2);
        uint32_t v[16];
        const uint32_t taddr = tmem + (uint32_t)(256 * b) + ((uint32_t)(wq * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (warp == TP_CONV / 32 + 2 && lane == 0) TM_TS(6, it * 16 + ((c0 - cbeg) >> 4));
        if (c0 + 16 >= cend) {     // this warp's reads of the accumulator are done
          asm volatile("tcgen05.fence::before_thread_sync;");
          mb_arrive(su32(&accfree[b]));
        }
        if (!live && !a.c_tma) continue;   // (TMA stores clip the rows past M)
        float x[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = ktiles == 0 ? 0.f : __uint_as_float(v[j]);
        if (p.epilogue == 2) {
#pragma unroll
          for (int j = 0; j < 16; ++j) x[j] = __fmul_rn(x[j], __fsub_rn(1.f, __fmul_rn(gv[j], gv[j])));
        } else {
          const float* bv = gv;      // the prefetched bias chunk (load_gate)
          // all 16 columns unconditionally (past N: clipped by the store), so
          // the 16 independent bias + tanh chains unroll and interleave (a
          // per-column `break` kept them one at a time: ~1.7 us per chunk)
          if (p.accumulate) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int64_t n = n0 + c0 + j;
              if (n < p.n) x[j] += Cp[rowoff + n * a.c_n];
            }
          }
          if (p.bias.ptr) {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] += bv[j];
          }
          if (p.epilogue == 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = tanh_fast(x[j]);
          }
        }
        if (a.c_tma) {
          // the warp's 32 rows x 16 columns through shared memory, one TMA
          // store per chunk (row-per-lane 16-byte stores hit 32 rows per
          // instruction); SWIZZLE_64B: 16-byte chunk q of row l sits at
          // q ^ ((l >> 1) & 3), so the lanes' writes are conflict-free
          const int ew = warp - TP_CONV / 32 - 2;
          const uint32_t buf = estage + (uint32_t)ew * TP_STAGE_EPI +
                               (uint32_t)((((c0 - cbeg) >> 4) & 1) * 2048);
          if (warp == TP_CONV / 32 + 2 && lane == 0) TM_TS(8, it * 16 + ((c0 - cbeg) >> 4));
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          if (warp == TP_CONV / 32 + 2 && lane == 0) TM_TS(9, it * 16 + ((c0 - cbeg) >> 4));
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t sa = buf + (uint32_t)(lane * 64 + ((q ^ ((lane >> 1) & 3)) * 16));
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(sa), "f"(x[4 * q]),
                         "f"(x[4 * q + 1]), "f"(x[4 * q + 2]), "f"(x[4 * q + 3]) : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) tma2d_store(&a.tc, (int32_t)(n0 + c0), (int32_t)(m0 + wq * 32), buf);
          if (warp == TP_CONV / 32 + 2 && lane == 0) TM_TS(7, it * 16 + ((c0 - cbeg) >> 4));
        } else if (vec && n0 + c0 + 16 <= p.n) {
          float4* dst = (float4*)(Cp + rowoff + n0 + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcs(dst + j, make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]));
        } else {
          for (int j = 0; j < 16; ++j) {
            const int64_t n = n0 + c0 + j;
            if (n >= p.n) break;
            Cp[rowoff + n * a.c_n] = x[j];
          }
        }
      }
      if (cbeg >= cend) {          // (a half with no columns still frees its share)
        asm volatile("tcgen05.fence::before_thread_sync;");
        mb_arrive(su32(&accfree[b]));
      }
    }
    if (a.c_tma && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__global__ void __launch_bounds__(TP_THREADS, 1) k_gemm_tmap(const __grid_constant__ tm_args a) {
  gemm_tmap_body<false>(a);
}
__global__ void __launch_bounds__(TP_THREADS, 1) k_gemm_tmap_split(const __grid_constant__ tm_args a) {
  gemm_tmap_body<true>(a);
}

// B -> tf32 hi / lo arrays over its whole element span (same offsets)
__global__ void k_tf32_split(const float* __restrict__ x, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const uint32_t h = rna(v);
    hi[i] = __uint_as_float(h);
    lo[i] = __uint_as_float(rna(v - __uint_as_float(h)));
  }
}

// split + transpose an MN-major [K][N] (row stride ld) fp32 operand into
// K-major [N][K] tf32 hi / lo arrays (32 x 32 tiles through shared memory)
__global__ void k_tf32_split_t(const float* __restrict__ x, int64_t ld, int64_t K, int64_t N,
                               float* __restrict__ hi, float* __restrict__ lo) {
  __shared__ float t[32][33];
  const int64_t n0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t k = k0 + r, n = n0 + threadIdx.x;
    t[r][threadIdx.x] = (k < K && n < N) ? x[k * ld + n] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t n = n0 + r, k = k0 + threadIdx.x;
    if (n < N && k < K) {
      const float v = t[threadIdx.x][r];
      const uint32_t h = rna(v);
      hi[n * K + k] = __uint_as_float(h);
      lo[n * K + k] = __uint_as_float(rna(v - __uint_as_float(h)));
    }
  }
}

typedef CUresult (*encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);

// 2-D fp32 map over (inner, outer) with unit inner stride.
// an MN-major operand [K][MN] (row stride ld) as dims {32, K, MN/32}: one
// box of {32, TM_BK, groups} fills `groups` 2 KB group slots of a stage in a
// single TMA instruction (the 2-D map needed one per 32-wide group: 12 per
// stage of the contraction GEMMs)
static int tm_encode3_mn(encode_fn_t enc, CUtensorMap* map, uint64_t addr, uint64_t mn, uint64_t k,
                         uint64_t ld, uint32_t groups) {
  cuuint64_t dims[3] = {32, k, mn / 32};
  cuuint64_t strides[2] = {ld * 4, 128};
  cuuint32_t box[3] = {32, TM_BK, groups};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)addr, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

static int tm_encode(encode_fn_t enc, CUtensorMap* map, uint64_t addr, uint64_t inner, uint64_t outer,
                     uint64_t outer_stride_elems, uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {outer_stride_elems * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  if (outer == 1) strides[0] = ((inner * 4 + 15) / 16) * 16;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)addr, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

// Pack a folded rt_gemm_params (1-D M/N/K boxes) into the kernel's argument
// block (tensor maps first, 64-byte aligned) in place.  Returns the kernel.
extern "C" void* rt_gemm_tma_pack(void* blk, void* encode) {
  rt_gemm_params p;
  memcpy(&p, blk, sizeof p);
  tm_args a;
  memset(&a, 0, sizeof a);
  a.p = p;
  encode_fn_t enc = (encode_fn_t)encode;
  const int64_t a_m = p.A.s1[0], a_k = p.A.s2[0], b_k = p.B.s1[0], b_n = p.B.s2[0];
  a.c_m = p.C.s1[0];
  a.c_n = p.C.s2[0];
  a.bias_n = p.bias.s2[0];
  a.g_m = p.bias.s1[0];
  a.g_n = p.bias.s2[0];
  const uint64_t abase = p.A.ptr + 4 * (uint64_t)p.A.off, bbase = p.B.ptr + 4 * (uint64_t)p.B.off;
  int rc;
  if (a_k == 1 || p.k == 1) {
    a.a_mn = 0;
    rc = tm_encode(enc, &a.ta, abase, p.k, p.m, a_m, TM_BK, TM_BM, CU_TENSOR_MAP_SWIZZLE_64B);
  } else {
    a.a_mn = 1;
    a.a3d = TM_3D && p.m % 32 == 0 && (abase & 127) == 0 &&
            tm_encode3_mn(enc, &a.ta, abase, p.m, p.k, a_k, TM_BM / 32) == 0;
    rc = a.a3d ? 0 : tm_encode(enc, &a.ta, abase, p.m, p.k, a_k, 32, TM_BK,
                               CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  if (rc) return nullptr;
  if (b_k == 1 || p.k == 1) {
    a.b_mn = 0;
    rc = tm_encode(enc, &a.tb, bbase, p.k, p.n, b_n, TM_BK, TM_BN, CU_TENSOR_MAP_SWIZZLE_64B);
  } else {
    a.b_mn = 1;
    a.b3d = TM_3D && p.n % 32 == 0 && (bbase & 127) == 0 &&
            tm_encode3_mn(enc, &a.tb, bbase, p.n, p.k, b_k, TM_BN / 32) == 0;
    rc = a.b3d ? 0 : tm_encode(enc, &a.tb, bbase, p.n, p.k, b_k, 32, TM_BK,
                               CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  if (rc) return nullptr;
  memcpy(blk, &a, sizeof a);
  // K per CTA past one accumulation chunk: the draining variant (lower.py
  // sizes its shared memory with the same rule, TMA_SMEM_DRAIN)
  const int64_t kper = ((p.k + p.splits - 1) / p.splits + TM_BK - 1) / TM_BK * TM_BK;
  if (kper > TM_DRAIN_K && p.epilogue == 2) return nullptr;   // no gate in the drain variant
  if (kper > TM_DRAIN_K) return (void*)k_gemm_tma_drain;
  if (p.splits != 1 || !p.part) return (void*)k_gemm_tma;      // per-tile variant
  // persistent (lower.py launches TP_THREADS x min(tiles, SMs) when it set
  // `part`: the hi/lo scratch of B, 2 x span floats, or ~0 for no presplit)
  {
    // the epilogue stores C with TMA when C is a plain row-major 2-D tile
    const uint64_t cbase = p.C.ptr + 4 * (uint64_t)p.C.off;
    a.c_tma = 0;
    if (TP_TMA_STORE && !p.accumulate && a.c_n == 1 && (cbase & 15) == 0 &&
        ((a.c_m * 4) & 15) == 0 && a.c_m >= p.n && p.C.dtype == RT_F32)
      a.c_tma = tm_encode(enc, &a.tc, cbase, p.n, p.m, a.c_m, 16, 32,
                          CU_TENSOR_MAP_SWIZZLE_64B) == 0;
  }
  if (p.part != ~0ull) {
    const uint64_t span = a.b_mn ? (uint64_t)(p.k - 1) * (uint64_t)b_k + (uint64_t)p.n
                                 : (uint64_t)(p.n - 1) * (uint64_t)b_n + (uint64_t)p.k;
    const uint64_t hbase = p.part, lbase = p.part + 4 * span;
    a.b_base = bbase;
    a.b_span = span;
    a.presplit = 1;
    if (a.b_mn) {
      // MN-major weights: the split pass also transposes them to K-major, so
      // a stage of B is ONE 64-byte-row box per part instead of eight 32-wide
      // MN groups (per-stage TMA issue bounded the kernel: ~1 us per stage,
      // tools/gemm_trace.py)
      a.presplit = 2;
      a.b_ld = b_k;
      a.b_kk = p.k;
      a.b_nn = p.n;
      a.b_mn = 0;
      rc = tm_encode(enc, &a.tbh, hbase, p.k, p.n, p.k, TM_BK, TM_BN, CU_TENSOR_MAP_SWIZZLE_64B);
      rc |= tm_encode(enc, &a.tbl, lbase, p.k, p.n, p.k, TM_BK, TM_BN, CU_TENSOR_MAP_SWIZZLE_64B);
    } else {
      rc = tm_encode(enc, &a.tbh, hbase, p.k, p.n, b_n, TM_BK, TM_BN, CU_TENSOR_MAP_SWIZZLE_64B);
      rc |= tm_encode(enc, &a.tbl, lbase, p.k, p.n, b_n, TM_BK, TM_BN, CU_TENSOR_MAP_SWIZZLE_64B);
    }
    if (rc) return nullptr;
    memcpy(blk, &a, sizeof a);
    return (void*)k_gemm_tmap_split;
  }
  memcpy(blk, &a, sizeof a);
  return (void*)k_gemm_tmap;
}

// launched before a PRESPLIT GEMM on the same stream (runtime.cu launch_one)
extern "C" int rt_gemm_tma_prepass(const void* blk, void* stream) {
  const tm_args* a = (const tm_args*)blk;
  if (!a->presplit) return 0;
  float* hi = (float*)a->p.part;
  float* lo = hi + a->b_span;
  if (a->presplit == 2) {
    dim3 grid((unsigned)((a->b_nn + 31) / 32), (unsigned)((a->b_kk + 31) / 32));
    k_tf32_split_t<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>((const float*)a->b_base, a->b_ld,
                                                                   a->b_kk, a->b_nn, hi, lo);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  const int64_t n = (int64_t)a->b_span;
  const int grid = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  k_tf32_split<<<grid > 0 ? grid : 1, 256, 0, (cudaStream_t)stream>>>((const float*)a->b_base, hi, lo, n);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int rt_gemm_tma_smem() { return TM_SMEM; }
extern "C" int rt_gemm_tma_smem_persist() { return TP_SMEM; }
extern "C" int rt_gemm_tma_smem_drain() { return TM_SMEM_DRAIN; }
extern "C" int rt_gemm_tma_args_bytes() { return (int)sizeof(tm_args); }

extern "C" int rt_gemm_tma_trace(long long* out, int n) {
#if TM_TRACE
  return cudaMemcpyFromSymbol(out, g_tm_trace, sizeof(long long) * (n < 10 * 512 ? n : 10 * 512)) == cudaSuccess ? 0 : -1;
#else
  (void)out; (void)n;
  return -1;
#endif
}
