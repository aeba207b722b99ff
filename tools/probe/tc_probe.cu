// Minimal tcgen05 kind::tf32 probe: which issue configurations produce D = A*B.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(ph) : "memory");
}

// A: 128 x 8 tf32, B: 16(N) x 8, both K-major no swizzle (core matrices 8 rows x 16B)
__global__ void probe(float* out, int issuer_warp, int use_dyn, int dyn_off) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  __shared__ __align__(1024) unsigned char stat[(128 + 16) * 8 * 4];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  unsigned char* buf = use_dyn ? dyn + dyn_off : stat;
  const int tid = threadIdx.x, warp = tid >> 5;
  // element (r, k): core matrix (r/8, k/4) at (r/8)*256 + (k/4)*128 + (r%8)*16 + (k%4)*4
  for (int i = tid; i < (128 + 16) * 8; i += blockDim.x) {
    int r = i / 8, k = i % 8;
    int rr = r < 128 ? r : r - 128;
    unsigned char* base = buf + (r < 128 ? 0 : 128 * 32);
    *(float*)(base + (rr / 8) * 256 + (k / 4) * 128 + (rr % 8) * 16 + (k % 4) * 4) = 1.0f + (r < 128 ? 0.f : (float)(rr));
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tm;
  if (warp == issuer_warp && (tid & 31) == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t da = desc(su32(buf), 128, 256), db = desc(su32(buf + 128 * 32), 128, 256);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  wait(su32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t v[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 4; ++j) out[(warp * 32 + (tid & 31)) * 4 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 4 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 197632);
  int cfg[][4] = {{128, 0, 0, 0}, {320, 9, 1, 0}, {320, 9, 1, 16384}, {320, 9, 1, 65536}, {320, 9, 1, 131072}, {320, 9, 1, 180224}};
  for (auto& c : cfg) {
    cudaMemset(d, 0, 128 * 16);
    probe<<<1, c[0], c[2] ? 197632 : 0>>>(d, c[1], c[2], c[3]);
    cudaError_t e = cudaDeviceSynchronize();
    float h[8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("off %d threads %d issuer warp %d dyn %d err %s -> D[0][0..3] %g %g %g %g (want 8 16 24 32)\n", c[3], c[0], c[1], c[2],
           cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
  }
  return 0;
}
