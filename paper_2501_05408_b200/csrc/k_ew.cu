// RT_K_EW — one launch evaluates a node (or a fused chain of nodes) over a
// box = slab of its domain x its payload.  Replaces the per-point dispatch
// of the elementwise/layout/merge/gather kernels of the reference
// (runtime.py:58-93, 161-189, 214-223, 239-259, 362-371): every output
// element runs the node's program, whose LOADs gather operands through
// affine views (index expressions folded into strides, domain checks kept
// as range checks) or through int programs for non-affine indexes.
#include "common.cuh"

template <typename T>
__global__ void __launch_bounds__(256) k_ew(const __grid_constant__ rt_ew_params p) {
  int64_t idx[RT_MAXD];
  const int nd = p.box.nd;
  for (int64_t flat = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; flat < p.total;
       flat += (int64_t)gridDim.x * blockDim.x) {
    decompose(p.box, flat, idx);
    T v = (T)0;
    int64_t dummy;
    vm_run<T>(p.code, 0, p.konst, p.h, idx, nd, p.in, &v, &dummy);
    store_as<T>((void*)p.out.ptr, p.out.dtype, view_off(p.out, nd, idx), v);
  }
}

extern "C" void* rt_kernel_ew(int f64) {
  return f64 ? (void*)k_ew<double> : (void*)k_ew<float>;
}
