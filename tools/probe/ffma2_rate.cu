// FP32 FMA issue-rate probe: scalar FFMA vs packed FFMA2 (fma.rn.f32x2) on
// independent chains, to pin the FP32 SIMT ceiling the acting loop is held to.
#include <cstdio>
#include <cuda_runtime.h>
template <bool PACKED>
__global__ void k(float* out, int iters, float w) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (PACKED) {
        asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %2}; fma.rn.f32x2 z, x, y, x; mov.b64 {%0, %1}, z;}"
                     : "+f"(a[i]), "+f"(a[i + 1]) : "f"(w));
      } else {
        asm volatile("fma.rn.f32 %0, %0, %2, %0; fma.rn.f32 %1, %1, %2, %1;" : "+f"(a[i]), "+f"(a[i + 1]) : "f"(w));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int packed = 0; packed < 2; ++packed)
    for (int tpb : {256, 512, 1024}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (packed) k<true><<<148 * 2, tpb>>>(o, iters, 0.999f); else k<false><<<148 * 2, tpb>>>(o, iters, 0.999f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = 148.0 * 2 * tpb * iters * 16;
        if (rep) printf("packed=%d tpb=%d: %.3f ms, %.1f TFLOP/s fp32\n", packed, tpb, ms, 2 * fmas / ms / 1e9);
      }
    }
  return 0;
}
