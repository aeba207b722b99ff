// RT_K_LOOP — a whole row-local loop in one persistent launch (interpreting
// form: the op list is dispatched at run time; `jit.loop_source` emits the
// same kernel with the body specialised).  See loop_lib.cuh for the ops.
#include "loop_lib.cuh"

// ---------------------------------------------------------------- the loop

__global__ void __launch_bounds__(LOOP_THREADS) k_loop(const __grid_constant__ rt_loop_params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ rt_fold sfold[RT_MAXIN + 1];
  __shared__ __align__(8) uint64_t bars[RING];
  int64_t env[RT_MAXENV];
  for (int e = 0; e < RT_MAXENV; ++e) env[e] = p.h.env[e];
  const int64_t r0 = (int64_t)blockIdx.x * p.rows_per_cta;
  const int64_t r1 = min(p.rows, r0 + p.rows_per_cta);
  if (r0 >= r1) return;
  const rt_loop_op* ops = (const rt_loop_op*)p.ops;
  // smem: [op descriptors | A rows | TMA ring]
  unsigned char* sA = smem + p.a_off;
  loop_ring ring;
  loop_prologue(p, smem, bars, ring);
  for (int64_t t = p.start; p.step > 0 ? t < p.stop : t > p.stop; t += p.step) {
    env[p.slot] = t;
    for (int i = 0; i < p.nops; ++i) {
      const rt_loop_op& op = ops[i];
      long long c0 = (p.prof && blockIdx.x == 0) ? clock64() : 0;
      switch (op.kernel) {
        case RT_K_EW: {
          const rt_ew_params& q = *(const rt_ew_params*)(smem + op.smem_off);
          if (op.f64) ew_rows<double>(q, env, r0 * op.row_elems, r1 * op.row_elems, sfold);
          else ew_rows<float>(q, env, r0 * op.row_elems, r1 * op.row_elems, sfold);
          break;
        }
        case RT_K_GEMM: {
          const rt_gemm_params& q = *(const rt_gemm_params*)(smem + op.smem_off);
          const int64_t m0 = r0 * op.row_elems, m1 = r1 * op.row_elems;
          if (op.f64) gemm_op<double>(q, env, m0, m1, sA, ring);
          else gemm_op<float>(q, env, m0, m1, sA, ring);
          break;
        }
        case RT_K_UDF:
          udf_rows(*(const rt_udf_params*)(smem + op.smem_off), op, env, r0, r1, t);
          break;
        case RT_K_RNG:
          rng_rows(*(const rt_rng_params*)(smem + op.smem_off), env, r0, r1);
          break;
        default:
          break;
      }
      __syncthreads();
      if (p.prof && blockIdx.x == 0 && threadIdx.x == 0)
        ((long long*)p.prof)[i] += clock64() - c0;
    }
  }
}

extern "C" void* rt_kernel_loop() { return (void*)k_loop; }
