// In-program collectives: the gradient all-reduce of an env-sharded run
// (one sum all-reduce over the flattened gradients per
// optimizer step) issued by the program interpreter itself, on the program's
// stream, through an NCCL communicator owned by this library.  Because the
// interpreter issues it (RT_OP_COLL), a sharded program is captured into ONE
// CUDA graph per step with its collectives inside (NCCL supports stream
// capture) instead of returning to Python at every all-reduce hook.
//
// NCCL is resolved with dlopen at first use (the library that PyTorch already
// loaded when present), so librtb200.so still loads on machines without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>
#include <vector>
#include "../../include/rtb200.h"

extern "C" int rt_set_error(int code, const char* what);

namespace {

typedef struct { char internal[128]; } nccl_id_t;
typedef void* nccl_comm_t;
typedef int nccl_result_t;

struct NcclApi {
  nccl_result_t (*getUniqueId)(nccl_id_t*) = nullptr;
  nccl_result_t (*commInitRank)(nccl_comm_t*, int, nccl_id_t, int) = nullptr;
  nccl_result_t (*allReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_result_t (*groupStart)() = nullptr;
  nccl_result_t (*groupEnd)() = nullptr;
  nccl_result_t (*commDestroy)(nccl_comm_t) = nullptr;
  const char* (*getErrorString)(nccl_result_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // PyTorch's, if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
  a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
  a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
  a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
  a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
  a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
  a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
  a.getErrorString = (decltype(a.getErrorString))dlsym(h, "ncclGetErrorString");
  a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.groupStart && a.groupEnd &&
         a.commDestroy && a.getErrorString;
  return a;
}

int nccl_rc(nccl_result_t r, const char* what) {
  if (r == 0) return RT_OK;
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, nccl().getErrorString ? nccl().getErrorString(r) : "?");
  return rt_set_error(RT_ERR_CUDA, buf);
}

int nccl_type(int dtype) {
  switch (dtype) {
    case RT_F64: return 8;    // ncclFloat64
    case RT_F32: return 7;    // ncclFloat32
    case RT_I64: return 4;    // ncclInt64
    default: return -1;
  }
}

int item(int dtype) { return dtype == RT_F32 ? 4 : dtype == RT_BOOL ? 1 : 8; }

// the collectives of the program about to run (rt_set_collectives), per thread
thread_local nccl_comm_t g_comm = nullptr;
thread_local std::vector<rt_coll> g_colls;
thread_local std::vector<rt_coll> g_pending;   // bucket: reduced at the next flushing op
thread_local std::vector<int64_t> g_pending_off;

}  // namespace

extern "C" int rt_nccl_unique_id(unsigned char* out128) {
  NcclApi& a = nccl();
  if (!a.ok) return rt_set_error(RT_ERR_CUDA, "NCCL not available (libnccl.so.2)");
  nccl_id_t id;
  int rc = nccl_rc(a.getUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(out128, id.internal, 128);
  return RT_OK;
}

extern "C" int rt_nccl_comm_init(int32_t nranks, int32_t rank, const unsigned char* id128,
                                 uint64_t* comm_out) {
  NcclApi& a = nccl();
  if (!a.ok) return rt_set_error(RT_ERR_CUDA, "NCCL not available (libnccl.so.2)");
  nccl_id_t id;
  memcpy(id.internal, id128, 128);
  nccl_comm_t c = nullptr;
  int rc = nccl_rc(a.commInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  if (rc) return rc;
  *comm_out = (uint64_t)c;
  return RT_OK;
}

extern "C" int rt_nccl_comm_destroy(uint64_t comm) {
  NcclApi& a = nccl();
  if (!a.ok || !comm) return RT_OK;
  return nccl_rc(a.commDestroy((nccl_comm_t)comm), "ncclCommDestroy");
}

extern "C" int rt_nccl_allreduce(uint64_t comm, uint64_t ptr, uint64_t count, int32_t dtype,
                                 uint64_t stream) {
  NcclApi& a = nccl();
  if (!a.ok) return rt_set_error(RT_ERR_CUDA, "NCCL not available (libnccl.so.2)");
  const int t = nccl_type(dtype);
  if (t < 0) return rt_set_error(RT_ERR_BAD_ARG, "all-reduce dtype");
  return nccl_rc(a.allReduce((const void*)ptr, (void*)ptr, count, t, 0, (nccl_comm_t)comm,
                             (cudaStream_t)stream), "ncclAllReduce");
}

extern "C" int rt_set_collectives(uint64_t comm, const rt_coll* colls, int32_t ncoll) {
  g_comm = (nccl_comm_t)comm;
  g_colls.assign(colls, colls + (ncoll > 0 ? ncoll : 0));
  g_pending.clear();
  g_pending_off.clear();
  return RT_OK;
}

// RT_OP_COLL: add collective `idx` (its slab at the current env) to the
// bucket; a flushing one reduces the whole bucket as one NCCL group (one
// launch) on the program's stream.
extern "C" int rt_coll_exec(int32_t idx, const int64_t* env, int32_t nenv, uint64_t stream) {
  if (idx < 0 || idx >= (int)g_colls.size() || !g_comm)
    return rt_set_error(RT_ERR_BAD_ARG, "collective out of range (rt_set_collectives)");
  const rt_coll& c = g_colls[idx];
  int64_t off = c.off0;
  for (int e = 0; e < RT_MAXENV && e < nenv; ++e) off += env[e] * c.off_env[e];
  g_pending.push_back(c);
  g_pending_off.push_back(off);
  if (!c.flush) return RT_OK;
  NcclApi& a = nccl();
  if (!a.ok) return rt_set_error(RT_ERR_CUDA, "NCCL not available (libnccl.so.2)");
  int rc = nccl_rc(a.groupStart(), "ncclGroupStart");
  for (size_t i = 0; i < g_pending.size() && !rc; ++i) {
    const rt_coll& p = g_pending[i];
    const int t = nccl_type(p.dtype);
    if (t < 0) {
      rc = rt_set_error(RT_ERR_BAD_ARG, "all-reduce dtype");
      break;
    }
    void* ptr = (void*)(p.ptr + (uint64_t)(g_pending_off[i] * item(p.dtype)));
    rc = nccl_rc(a.allReduce(ptr, ptr, (size_t)p.count, t, 0, g_comm, (cudaStream_t)stream),
                 "ncclAllReduce");
  }
  int rc2 = nccl_rc(a.groupEnd(), "ncclGroupEnd");
  g_pending.clear();
  g_pending_off.clear();
  return rc ? rc : rc2;
}
