// The SPEC's runtime Backend and MemorySim at the C ABI (reference SPEC.md
// :541-561, `Backend: allocate, deallocate, move-between-tiers,
// execute-kernel(kind, inputs, params), dynamic-update, stack` and
// `MemorySim: device tier {capacity, live, peak}; host tier {live, peak};
// transfer counters {fetches, offloads, bytes moved}; device overflow is a
// hard error`).  The reference package implements none of it;
// polysched.py:767-1137 only plans the memory ops.
//
//   allocate / deallocate   rt_pool_alloc / rt_pool_free: stream-ordered
//                           (cudaMallocFromPoolAsync / cudaFreeAsync on a
//                           per-device cudaMemPool), live/peak accounting,
//                           capacity overflow -> RT_ERR_OVERFLOW
//   move-between-tiers      rt_offload / rt_fetch: pinned 2-D copies on a
//                           copy stream ordered after an event, recording a
//                           caller-owned completion event
//   execute-kernel          rt_launch (runtime.cu)
//   dynamic-update          rt_block_update: one point's value into slot
//                           `slot` of a pre-allocated block (SPEC BlockStore)
//   stack                   rt_stack: n point values concatenated into one
//                           contiguous tensor (a slice read materialised)
#include <cuda_runtime.h>
#include <mutex>
#include <stdio.h>
#include <string.h>
#include <unordered_map>
#include "../../include/rtb200.h"

extern "C" int rt_set_error(int code, const char* msg);

namespace {

struct Pool {
  cudaMemPool_t pool = nullptr;
  int device = 0;
  uint64_t capacity = 0, live = 0, peak = 0;
  uint64_t host_live = 0, host_peak = 0;
  uint64_t offloads = 0, fetches = 0, bytes_moved = 0;
  std::unordered_map<uint64_t, uint64_t> sizes;
  std::mutex mu;
};

int cuda_rc(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RT_OK;
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return rt_set_error(RT_ERR_CUDA, buf);
}

// element copies of the stack / block-update kernels: 16-byte vectors when
// every pointer and the element size allow it
struct StackArgs {
  uint64_t dst;
  uint64_t elem_bytes;
  int32_t n;
  int32_t vec;
  uint64_t src[240];
};

__global__ void k_stack(const __grid_constant__ StackArgs a) {
  const int i = blockIdx.y;
  if (i >= a.n) return;
  if (a.vec) {
    const int4* s = (const int4*)a.src[i];
    int4* d = (int4*)(a.dst + (uint64_t)i * a.elem_bytes);
    for (uint64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.elem_bytes / 16;
         j += (uint64_t)gridDim.x * blockDim.x)
      d[j] = s[j];
  } else {
    const unsigned char* s = (const unsigned char*)a.src[i];
    unsigned char* d = (unsigned char*)(a.dst + (uint64_t)i * a.elem_bytes);
    for (uint64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.elem_bytes;
         j += (uint64_t)gridDim.x * blockDim.x)
      d[j] = s[j];
  }
}

int launch_stack(uint64_t dst, const uint64_t* srcs, int32_t n, uint64_t elem_bytes,
                 cudaStream_t s) {
  for (int32_t b = 0; b < n; b += 240) {
    StackArgs a;
    memset(&a, 0, sizeof a);
    a.dst = dst + (uint64_t)b * elem_bytes;
    a.elem_bytes = elem_bytes;
    a.n = n - b < 240 ? n - b : 240;
    a.vec = elem_bytes % 16 == 0 && a.dst % 16 == 0;
    for (int i = 0; i < a.n; ++i) {
      a.src[i] = srcs[b + i];
      if (a.src[i] % 16) a.vec = 0;
    }
    const uint64_t units = a.vec ? elem_bytes / 16 : elem_bytes;
    const unsigned gx = (unsigned)((units + 255) / 256 < 64 ? (units + 255) / 256 : 64);
    k_stack<<<dim3(gx > 0 ? gx : 1, (unsigned)a.n), 256, 0, s>>>(a);
    int rc = cuda_rc(cudaGetLastError(), "stack");
    if (rc) return rc;
  }
  return RT_OK;
}

int tier_move(Pool* p, void* dst, uint64_t dpitch, const void* src, uint64_t spitch,
              uint64_t width, uint64_t height, cudaMemcpyKind kind, uint64_t stream,
              uint64_t after_event, uint64_t done_event) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if (after_event && (rc = cuda_rc(cudaStreamWaitEvent(s, (cudaEvent_t)after_event, 0), "wait")))
    return rc;
  if (height == 1)
    rc = cuda_rc(cudaMemcpyAsync(dst, src, width, kind, s), "tier move");
  else
    rc = cuda_rc(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, s), "tier move");
  if (rc) return rc;
  if (done_event && (rc = cuda_rc(cudaEventRecord((cudaEvent_t)done_event, s), "record")))
    return rc;
  if (p) {
    std::lock_guard<std::mutex> g(p->mu);
    (kind == cudaMemcpyDeviceToHost ? p->offloads : p->fetches) += 1;
    p->bytes_moved += width * height;
  }
  return RT_OK;
}

}  // namespace

extern "C" int rt_pool_create(int32_t device, uint64_t capacity, uint64_t* pool_out) {
  Pool* p = new Pool;
  p->device = device;
  p->capacity = capacity;
  cudaMemPoolProps props;
  memset(&props, 0, sizeof props);
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  int rc = cuda_rc(cudaMemPoolCreate(&p->pool, &props), "pool create");
  if (rc) {
    delete p;
    return rc;
  }
  uint64_t keep = UINT64_MAX;   // freed blocks stay reserved for reuse (no OS round trip)
  cudaMemPoolSetAttribute(p->pool, cudaMemPoolAttrReleaseThreshold, &keep);
  *pool_out = (uint64_t)p;
  return RT_OK;
}

extern "C" int rt_pool_destroy(uint64_t pool) {
  Pool* p = (Pool*)pool;
  if (!p) return rt_set_error(RT_ERR_BAD_ARG, "null pool");
  int rc = cuda_rc(cudaMemPoolDestroy(p->pool), "pool destroy");
  delete p;
  return rc;
}

extern "C" int rt_pool_alloc(uint64_t pool, uint64_t bytes, uint64_t stream, uint64_t* dev_out) {
  Pool* p = (Pool*)pool;
  if (!p) return rt_set_error(RT_ERR_BAD_ARG, "null pool");
  {
    std::lock_guard<std::mutex> g(p->mu);
    if (p->capacity && p->live + bytes > p->capacity)
      return rt_set_error(RT_ERR_OVERFLOW, "device tier overflow (MemorySim capacity)");
  }
  void* d = nullptr;
  int rc = cuda_rc(cudaMallocFromPoolAsync(&d, bytes ? bytes : 1, p->pool, (cudaStream_t)stream),
                   "pool alloc");
  if (rc) return rc;
  std::lock_guard<std::mutex> g(p->mu);
  p->sizes[(uint64_t)d] = bytes;
  p->live += bytes;
  if (p->live > p->peak) p->peak = p->live;
  *dev_out = (uint64_t)d;
  return RT_OK;
}

extern "C" int rt_pool_free(uint64_t pool, uint64_t dev, uint64_t stream) {
  Pool* p = (Pool*)pool;
  if (!p) return rt_set_error(RT_ERR_BAD_ARG, "null pool");
  uint64_t bytes;
  {
    std::lock_guard<std::mutex> g(p->mu);
    auto it = p->sizes.find(dev);
    if (it == p->sizes.end()) return rt_set_error(RT_ERR_BAD_ARG, "free of a pointer the pool does not own");
    bytes = it->second;
    p->sizes.erase(it);
    p->live -= bytes;
  }
  return cuda_rc(cudaFreeAsync((void*)dev, (cudaStream_t)stream), "pool free");
}

extern "C" int rt_pool_host(uint64_t pool, int64_t delta_bytes) {
  Pool* p = (Pool*)pool;
  if (!p) return rt_set_error(RT_ERR_BAD_ARG, "null pool");
  std::lock_guard<std::mutex> g(p->mu);
  if (delta_bytes < 0 && (uint64_t)(-delta_bytes) > p->host_live)
    return rt_set_error(RT_ERR_BAD_ARG, "host tier below zero");
  p->host_live += delta_bytes;
  if (p->host_live > p->host_peak) p->host_peak = p->host_live;
  return RT_OK;
}

extern "C" int rt_pool_stats(uint64_t pool, uint64_t* stats8) {
  Pool* p = (Pool*)pool;
  if (!p) return rt_set_error(RT_ERR_BAD_ARG, "null pool");
  std::lock_guard<std::mutex> g(p->mu);
  const uint64_t v[8] = {p->capacity, p->live,     p->peak,     p->host_live,
                         p->host_peak, p->offloads, p->fetches, p->bytes_moved};
  memcpy(stats8, v, sizeof v);
  return RT_OK;
}

extern "C" int rt_offload(uint64_t pool, void* host_pinned, uint64_t hpitch, uint64_t dev,
                          uint64_t dpitch, uint64_t width, uint64_t height, uint64_t stream,
                          uint64_t after_event, uint64_t done_event) {
  return tier_move((Pool*)pool, host_pinned, hpitch, (const void*)dev, dpitch, width, height,
                   cudaMemcpyDeviceToHost, stream, after_event, done_event);
}

extern "C" int rt_fetch(uint64_t pool, uint64_t dev, uint64_t dpitch, const void* host_pinned,
                        uint64_t hpitch, uint64_t width, uint64_t height, uint64_t stream,
                        uint64_t after_event, uint64_t done_event) {
  return tier_move((Pool*)pool, (void*)dev, dpitch, host_pinned, hpitch, width, height,
                   cudaMemcpyHostToDevice, stream, after_event, done_event);
}

extern "C" int rt_block_update(uint64_t block, int64_t slot, uint64_t src, uint64_t elem_bytes,
                               uint64_t stream) {
  if (slot < 0) return rt_set_error(RT_ERR_BAD_ARG, "negative block slot");
  return cuda_rc(cudaMemcpyAsync((void*)(block + (uint64_t)slot * elem_bytes), (const void*)src,
                                 elem_bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
                 "block update");
}

extern "C" int rt_stack(uint64_t dst, const uint64_t* srcs, int32_t n, uint64_t elem_bytes,
                        uint64_t stream) {
  if (n < 0) return rt_set_error(RT_ERR_BAD_ARG, "negative stack count");
  if (n == 0 || elem_bytes == 0) return RT_OK;
  return launch_stack(dst, srcs, n, elem_bytes, (cudaStream_t)stream);
}
