// RT_K_SCAN, tile 4 — the reverse discounted return / discounted cumsum
// (reference runtime.py:99-105, 115-146; the suffix window r[t:T] of
// runtime.py:414-425) and the GAE scan with the TD residual formed on the
// fly (as k_scan_gae), fed and drained by 2-D TMA.
//
// Layout: the lines (every dim but the scan dim) collapse to one stride, so
// each operand is a 2-D tensor [lines][L] with unit stride along L; lower.py
// checks that before it picks this kernel.  A CTA is one warp owning 32
// lines.  A stage is one TMA box of 32 lines x TC elements (TC x sizeof(T) =
// 128 bytes, SWIZZLE_128B) per operand, landing on the stage's mbarrier;
// NS stages form a ring (NS - 1 boxes in flight while one is scanned).
// Lane i scans line i of the box sequentially in fp64 — its 16-byte vectors
// sit at (k ^ (i & 7)) under the 128-byte swizzle, so the warp's reads are
// bank-conflict free — writes the results in place, and lane 0 sends the box
// back with one TMA store.  A stage is refilled once the store that read it
// has drained (bulk_group .read).  Chunks are TC-aligned from t = 0; the
// ragged last chunk and the lines past the end are zero-filled on load and
// clipped on store by the TMA unit.  Two TMA operations per 4 KB box instead
// of 256 16-byte cp.async per CTA and chunk (k_scan_pipe).
#include <cuda.h>
#include "common.cuh"

typedef CUresult (*scan_encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct scan_tma_args {
  CUtensorMap tin, tin2, tout;
  rt_scan_params p;
};

namespace {

RT_DEV uint32_t su32s(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
RT_DEV void sm_init(uint32_t bar) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar)); }
RT_DEV void sm_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
RT_DEV void sm_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  }
}
RT_DEV void tma_load2(uint32_t dst, const CUtensorMap* map, int32_t x, int32_t y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"((uint64_t)map), "r"(x), "r"(y), "r"(bar) : "memory");
}
RT_DEV void tma_store2(const CUtensorMap* map, int32_t x, int32_t y, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"((uint64_t)map), "r"(x), "r"(y), "r"(src) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <typename T> struct tvec;
template <> struct tvec<float> { using V = float4; static constexpr int W = 4; };
template <> struct tvec<double> { using V = double2; static constexpr int W = 2; };
RT_DEV void tunpack(const float4& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
RT_DEV void tunpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
RT_DEV float4 tpack(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
RT_DEV double2 tpack(const double* o) { return make_double2(o[0], o[1]); }
RT_DEV float rn_add_(float a, float b) { return __fadd_rn(a, b); }
RT_DEV double rn_add_(double a, double b) { return __dadd_rn(a, b); }
RT_DEV float rn_sub_(float a, float b) { return __fsub_rn(a, b); }
RT_DEV double rn_sub_(double a, double b) { return __dsub_rn(a, b); }
RT_DEV float rn_mul_(float a, float b) { return __fmul_rn(a, b); }
RT_DEV double rn_mul_(double a, double b) { return __dmul_rn(a, b); }

#define ST_LINES 32
#define ST_BOX 4096   // bytes per operand box: 32 lines x 128 bytes

template <typename T, bool GAE>
__global__ void __launch_bounds__(32) k_scan_tma(const __grid_constant__ scan_tma_args a) {
  using V = typename tvec<T>::V;
  constexpr int VW = tvec<T>::W;
  constexpr int TC = 128 / (int)sizeof(T);    // elements per line per box
  constexpr int NV = TC / VW;                 // 16-byte vectors per line per box (8)
  constexpr int NIN = GAE ? 2 : 1;
  const rt_scan_params& p = a.p;
  const int NS = p.stages;
  const int lane = (int)threadIdx.x;
  extern __shared__ __align__(1024) unsigned char sraw[];
  // [NS][NIN][box] (1024-aligned boxes for the 128-byte swizzle), then NS mbarriers
  unsigned char* base = (unsigned char*)(((uintptr_t)sraw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)NS * NIN * ST_BOX);
  auto box = [&](int s, int in) { return base + (size_t)(s * NIN + in) * ST_BOX; };
  const int64_t L = p.box.ext[p.sdim];
  const int64_t nch = (L + TC - 1) / TC;
  const int32_t y0 = (int32_t)((int64_t)blockIdx.x * ST_LINES);
  const bool rev = GAE || p.reverse;
  const bool line_ok = (int64_t)y0 + lane < p.total_lines;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) sm_init(su32s(bars + s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // processing order: chunk q = c (forward) or nch - 1 - c (reverse)
  auto issue = [&](int64_t c) {
    const int64_t q = rev ? nch - 1 - c : c;
    const int s = (int)(c % NS);
    const uint32_t bar = su32s(bars + s);
    sm_expect(bar, NIN * ST_BOX);
    tma_load2(su32s(box(s, 0)), &a.tin, (int32_t)(q * TC), y0, bar);
    if (GAE) tma_load2(su32s(box(s, 1)), &a.tin2, (int32_t)(q * TC), y0, bar);
  };
  if (lane == 0)
    for (int64_t c = 0; c < NS - 1 && c < nch; ++c) issue(c);
  const double g = p.gamma;
  double acc = 0.0;
  bool head = true;
  T vnext = (T)p.gae_vb;
  const T gc = (T)p.gae_c;
  const int sw = lane & 7;
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t q = rev ? nch - 1 - c : c;
    const int s = (int)(c % NS);
    sm_wait(su32s(bars + s), (uint32_t)((c / NS) & 1));
    const int cnt = (int)((q + 1) * TC < L ? TC : L - q * TC);   // valid elements (multiple of VW)
    const int nv = cnt / VW;
    V* row = reinterpret_cast<V*>(box(s, 0) + lane * 128);
    if (line_ok) {
      if (GAE) {
        const V* row2 = reinterpret_cast<const V*>(box(s, 1) + lane * 128);
        for (int k = nv - 1; k >= 0; --k) {
          T e[VW], w[VW];
          tunpack(row[k ^ sw], e);
          tunpack(row2[k ^ sw], w);
#pragma unroll
          for (int u = VW - 1; u >= 0; --u) {
            T d = rn_add_(e[u], rn_mul_(vnext, gc));   // add(r, mul(Vn, c)), no contraction
            d = rn_sub_(d, w[u]);                      // sub(.., V)
            vnext = w[u];
            const double x = (double)d;
            acc = head ? x : x + g * acc;
            head = false;
            e[u] = (T)acc;
          }
          row[k ^ sw] = tpack(e);
        }
      } else if (rev) {
        for (int k = nv - 1; k >= 0; --k) {
          T e[VW];
          tunpack(row[k ^ sw], e);
#pragma unroll
          for (int u = VW - 1; u >= 0; --u) {
            const double x = (double)e[u];
            acc = head ? x : x + g * acc;   // the chain head takes x as is (runtime.py:141)
            head = false;
            e[u] = (T)acc;
          }
          row[k ^ sw] = tpack(e);
        }
      } else {
#pragma unroll 2
        for (int k = 0; k < nv; ++k) {
          T e[VW];
          tunpack(row[k ^ sw], e);
#pragma unroll
          for (int u = 0; u < VW; ++u) {
            const double x = (double)e[u];
            acc = head ? x : x + g * acc;
            head = false;
            e[u] = (T)acc;
          }
          row[k ^ sw] = tpack(e);
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> TMA store
    __syncwarp();
    if (lane == 0) {
      tma_store2(&a.tout, (int32_t)(q * TC), y0, su32s(box(s, 0)));
      if (c + NS - 1 < nch) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");   // store of c-1 left its stage
        issue(c + NS - 1);
      }
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 2-D map [outer lines][inner L] of element type T, 128-byte swizzled boxes
static int st_encode(scan_encode_fn_t enc, CUtensorMap* map, bool f64, uint64_t addr, uint64_t L,
                     uint64_t lines, uint64_t line_stride_elems) {
  const uint64_t es = f64 ? 8 : 4;
  cuuint64_t dims[2] = {L, lines};
  cuuint64_t strides[1] = {line_stride_elems * es};
  if (lines == 1) strides[0] = ((L * es + 15) / 16) * 16;
  cuuint32_t boxd[2] = {(cuuint32_t)(128 / es), ST_LINES};
  cuuint32_t el[2] = {1, 1};
  CUresult r = enc(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   (void*)addr, dims, strides, boxd, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

// stride of line index l in view v when the non-scan dims collapse, else -1
static int64_t line_stride(const rt_scan_params& p, const rt_view& v) {
  int64_t st = -1, span = 1;
  for (int d = p.box.nd - 1; d >= 0; --d) {
    if (d == p.sdim || p.box.ext[d] <= 1) continue;
    if (st < 0) {
      st = v.stride[d];
    } else if (v.stride[d] != st * span) {
      return -1;
    }
    span *= p.box.ext[d];
  }
  return st < 0 ? 1 : st;
}

}  // namespace

// Pack a folded rt_scan_params (tile 4) into scan_tma_args in place.
extern "C" void* rt_scan_tma_pack(void* blk, void* encode) {
  scan_tma_args a;
  memset(&a, 0, sizeof a);
  memcpy(&a.p, blk, sizeof a.p);
  const rt_scan_params& p = a.p;
  scan_encode_fn_t enc = (scan_encode_fn_t)encode;
  const bool f64 = p.f64 != 0;
  const uint64_t es = f64 ? 8 : 4, L = (uint64_t)p.box.ext[p.sdim];
  const uint64_t lines = (uint64_t)p.total_lines;
  const rt_view* vs[3] = {&p.in, p.gae ? &p.in2 : &p.in, &p.out};
  CUtensorMap* maps[3] = {&a.tin, &a.tin2, &a.tout};
  for (int i = 0; i < 3; ++i) {
    const int64_t ls = line_stride(p, *vs[i]);
    if (ls < 0 || vs[i]->stride[p.sdim] != 1) return nullptr;
    if (st_encode(enc, maps[i], f64, vs[i]->ptr + es * (uint64_t)vs[i]->off, L, lines, (uint64_t)ls))
      return nullptr;
  }
  memcpy(blk, &a, sizeof a);
  if (p.gae) return f64 ? (void*)k_scan_tma<double, true> : (void*)k_scan_tma<float, true>;
  return f64 ? (void*)k_scan_tma<double, false> : (void*)k_scan_tma<float, false>;
}

extern "C" int rt_scan_tma_args_bytes() { return (int)sizeof(scan_tma_args); }
