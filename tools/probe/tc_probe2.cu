// tcgen05 kind::tf32 layout probe: A 128 x 16 (K), B N x 16, one CTA, two
// K=8 MMAs.  Layouts: 0 = K-major no swizzle, 1 = K-major SW64, 2 = K-major
// SW128 (BK=32 row pitch), 3 = MN-major SW128 (32-wide atoms), 4 = MN-major
// SW128_BASE32B.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)lay << 61);
}
// byte offset of element (row r = m or n, k) for layout L with R rows, BK = 16
__host__ __device__ uint32_t off(int L, int r, int k, int R) {
  switch (L) {
    case 0: return (r / 8) * 512 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4;   // LBO 128, SBO 512
    case 1: { uint32_t a = r * 64 + k * 4; return a ^ (((a >> 7) & 3) << 4); }   // SW64 K-major
    case 2: { uint32_t a = r * 128 + k * 4; return a ^ (((a >> 7) & 7) << 4); }  // SW128 K-major (row 128B, k<16 uses half)
    case 3: { // MN-major SW128: atom = 8 k-rows x 32 mn (128 B); mn groups of 32 at LBO = 16*128
      uint32_t a = (r / 32) * 2048 + k * 128 + (r % 32) * 4; return a ^ (((a >> 7) & 7) << 4); }
    default: { // MN-major SW128_BASE32B: Swizzle<2,5,2>: bits [5,7) ^= bits [7,9)
      uint32_t a = (r / 32) * 2048 + k * 128 + (r % 32) * 4; return a ^ (((a >> 7) & 3) << 5); }
  }
}
__device__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(ph) : "memory");
}

__global__ void probe(const float* A, const float* B, float* out, int N, int LA, int LB) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  unsigned char* sa = sm;
  unsigned char* sb = sm + 65536;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 16; i += blockDim.x) *(float*)(sa + off(LA, i / 16, i % 16, 128)) = A[i];
  for (int i = tid; i < N * 16; i += blockDim.x) *(float*)(sb + off(LB, i / 16, i % 16, N)) = B[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tm;
  if (tid == 0) {
    const int amn = LA >= 3, bmn = LB >= 3;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amn << 15) | (bmn << 16) |
                     ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    for (int ks = 0; ks < 2; ++ks) {
      uint64_t da, db;
      auto mk = [&](int L, uint32_t base) -> uint64_t {
        switch (L) {
          case 0: return desc(base + ks * 256, 128, 512, 0);
          case 1: return desc(base + ks * 32, 16, 512, 4);
          case 2: return desc(base + ks * 32, 16, 1024, 2);
          case 3: return desc(base + ks * 1024, 2048, 1024, 2);
          default: return desc(base + ks * 1024, 2048, 512, 1);
        }
      };
      da = mk(LA, su32(sa));
      db = mk(LB, su32(sb));
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  wait(su32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    for (int c = 0; c < N; c += 4) {
      uint32_t v[4];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 4; ++j) out[(warp * 32 + (tid & 31)) * N + c + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  const int N = 64;
  float hA[128 * 16], hB[N * 16], ref[128 * N], got[128 * N];
  srand(1);
  for (auto& x : hA) x = (float)(rand() % 7 - 3);
  for (auto& x : hB) x = (float)(rand() % 7 - 3);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < 16; ++k) s += hA[m * 16 + k] * hB[n * 16 + k];
      ref[m * N + n] = s;
    }
  float *dA, *dB, *dO;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dO, sizeof got);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  int combos[][2] = {{0, 0}, {1, 1}, {2, 2}, {1, 3}, {3, 3}, {1, 4}, {4, 4}, {3, 1}};
  for (auto& c : combos) {
    cudaMemset(dO, 0, sizeof got);
    probe<<<1, 128, 131072>>>(dA, dB, dO, N, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(got, dO, sizeof got, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * N; ++i) bad += got[i] != ref[i];
    printf("LA %d LB %d err %s bad %d / %d  got[0..3] %g %g %g %g ref %g %g %g %g\n", c[0], c[1],
           cudaGetErrorString(e), bad, 128 * N, got[0], got[1], got[2], got[3], ref[0], ref[1], ref[2], ref[3]);
  }
  return 0;
}
