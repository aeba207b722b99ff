// C-ABI runtime: kernel table, launch with env patching, the loop-nest
// program interpreter (the executor loop that replaces the reference's
// demand-driven recursion, runtime.py:285-475), status word, tier moves.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <stdio.h>
#include <string.h>
#include <string>
#include <vector>
#include "../../include/rtb200.h"

extern "C" void* rt_kernel_ew(int f64);
extern "C" void* rt_kernel_reduce(int f64, int tpo);
extern "C" void* rt_kernel_reduce_cols(int f64, int fin);
extern "C" void* rt_kernel_scan(int f64, int warp);
extern "C" void* rt_kernel_gemm(int f64);
extern "C" void* rt_kernel_splitk(int f64);
extern "C" void* rt_kernel_rng();
extern "C" void* rt_kernel_udf();
extern "C" void* rt_kernel_rng_fill();
extern "C" void* rt_kernel_loop();
extern "C" void* rt_kernel_gemm_tc();
extern "C" void* rt_kernel_thin(int variant, int f64, int r);
extern "C" void* rt_kernel_thin_bulk(int r, int ones);
extern "C" void* rt_kernel_thin_rows_bulk(int r, int k);
extern "C" void* rt_kernel_thin_vec(int mode, int f64, int k);
extern "C" void* rt_kernel_thin_rows(int f64, int r, int k);
extern "C" void* rt_scan_tma_pack(void* blk, void* encode);
extern "C" void* rt_kernel_scan_pipe(int f64, int step_major);
extern "C" void* rt_kernel_scan_gae(int f64);
extern "C" void* rt_gemm_tma_pack(void* blk, void* encode);
extern "C" int rt_gemm_tma_prepass(const void* blk, void* stream);
extern "C" int rt_coll_exec(int32_t idx, const int64_t* env, int32_t nenv, uint64_t stream);

static thread_local std::string g_err;

// Driver API entry points resolved through the runtime, so the library loads
// (and its CPU-side tests run) on machines without libcuda.so.
struct DriverApi {
  decltype(&cuModuleLoadData) moduleLoadData = nullptr;
  decltype(&cuModuleGetFunction) moduleGetFunction = nullptr;
  decltype(&cuLaunchKernel) launchKernel = nullptr;
  decltype(&cuLaunchKernelEx) launchKernelEx = nullptr;
  decltype(&cuFuncSetAttribute) funcSetAttribute = nullptr;
  decltype(&cuGetErrorString) getErrorString = nullptr;
  void* tensorMapEncodeTiled = nullptr;
  bool ok = false;
};

static DriverApi& drv() {
  static DriverApi d;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    bool all = true;
#define RT_GET(field, name)                                                              \
    if (cudaGetDriverEntryPoint(name, (void**)&d.field, cudaEnableDefault, &q) != cudaSuccess || \
        q != cudaDriverEntryPointSuccess)                                                  \
      all = false;
    RT_GET(moduleLoadData, "cuModuleLoadData")
    RT_GET(moduleGetFunction, "cuModuleGetFunction")
    RT_GET(launchKernel, "cuLaunchKernel")
    RT_GET(launchKernelEx, "cuLaunchKernelEx")
    RT_GET(funcSetAttribute, "cuFuncSetAttribute")
    RT_GET(getErrorString, "cuGetErrorString")
    RT_GET(tensorMapEncodeTiled, "cuTensorMapEncodeTiled")
#undef RT_GET
    d.ok = all;
  }
  return d;
}

static int fail(int code, const char* what) {
  g_err = what;
  return code;
}

// for the other translation units of the library (backend.cu)
extern "C" int rt_set_error(int code, const char* what) { return fail(code, what); }

static int cuda_check(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return RT_OK;
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
  g_err = buf;
  return RT_ERR_CUDA;
}

extern "C" const char* rt_last_error(void) { return g_err.c_str(); }
extern "C" int rt_version(void) { return 1; }

// ------------------------------------------------------------ env folding

static void fold_view(rt_view& v, const int64_t* env, int nenv) {
  for (int e = 0; e < nenv && e < RT_MAXENV; ++e) {
    int64_t x = env[e];
    if (!x) continue;
    v.off += x * v.off_env[e];
    for (int c = 0; c < v.nchk; ++c) v.chk_c0[c] += x * (int64_t)v.chk_env[c][e];
  }
}

static void fold_gop(rt_gop& g, const int64_t* env, int nenv) {
  for (int e = 0; e < nenv && e < RT_MAXENV; ++e) g.off += env[e] * g.off_env[e];
}

static void patch_env(rt_hdr* h, const int64_t* env, int nenv) {
  for (int e = 0; e < RT_MAXENV; ++e) h->env[e] = e < nenv ? env[e] : 0;
}

static char rt_memcpy_marker;

// Fold the launch's env into a private copy of the parameter block and pick
// the kernel variant.  Returns the kernel function or null.
static void* prepare(int kernel, void* blk, const int64_t* env, int nenv) {
  patch_env((rt_hdr*)blk, env, nenv);
  switch (kernel) {
    case RT_K_EW: {
      rt_ew_params* p = (rt_ew_params*)blk;
      fold_view(p->out, env, nenv);
      for (int i = 0; i < p->nin; ++i) fold_view(p->in[i], env, nenv);
      return rt_kernel_ew(p->f64);
    }
    case RT_K_REDUCE: {
      rt_reduce_params* p = (rt_reduce_params*)blk;
      fold_view(p->in, env, nenv);
      fold_view(p->out, env, nenv);
      for (int j = 0; j < p->nred; ++j)
        for (int e = 0; e < nenv && e < RT_MAXENV; ++e) p->len0[j] += env[e] * p->len_env[j][e];
      if (p->part) return rt_kernel_reduce_cols(p->f64, p->threads_per_out == -1);
      return rt_kernel_reduce(p->f64, p->threads_per_out);
    }
    case RT_K_SCAN: {
      rt_scan_params* p = (rt_scan_params*)blk;
      fold_view(p->in, env, nenv);
      fold_view(p->out, env, nenv);
      if (p->gae) fold_view(p->in2, env, nenv);
      if (p->tile == 4) {
        DriverApi& D = drv();
        if (!D.ok) return nullptr;
        return rt_scan_tma_pack(blk, D.tensorMapEncodeTiled);
      }
      if (p->gae) return rt_kernel_scan_gae(p->f64);
      if (p->tile >= 2) return rt_kernel_scan_pipe(p->f64, p->tile == 3);
      int warp = p->in.stride[p->sdim] == 1 && p->out.stride[p->sdim] == 1;
      return rt_kernel_scan(p->f64, warp);
    }
    case RT_K_GEMM: {
      rt_gemm_params* p = (rt_gemm_params*)blk;
      fold_gop(p->A, env, nenv);
      fold_gop(p->B, env, nenv);
      fold_gop(p->C, env, nenv);
      if (p->bias.ptr) fold_gop(p->bias, env, nenv);
      return rt_kernel_gemm(p->f64);
    }
    case RT_K_GEMM_TC: {
      rt_gemm_params* p = (rt_gemm_params*)blk;
      fold_gop(p->A, env, nenv);
      fold_gop(p->B, env, nenv);
      fold_gop(p->C, env, nenv);
      if (p->bias.ptr) fold_gop(p->bias, env, nenv);
      return rt_kernel_gemm_tc();
    }
    case RT_K_GEMM_TMA: {
      rt_gemm_params* p = (rt_gemm_params*)blk;
      fold_gop(p->A, env, nenv);
      fold_gop(p->B, env, nenv);
      fold_gop(p->C, env, nenv);
      if (p->bias.ptr) fold_gop(p->bias, env, nenv);
      DriverApi& D = drv();
      if (!D.ok) return nullptr;
      return rt_gemm_tma_pack(blk, D.tensorMapEncodeTiled);
    }
    case RT_K_THIN: {
      rt_thin_params* p = (rt_thin_params*)blk;
      fold_gop(p->X, env, nenv);
      fold_gop(p->Y, env, nenv);
      fold_gop(p->C, env, nenv);
      if (p->bias.ptr) fold_gop(p->bias, env, nenv);
      if (p->variant == 3) {
        if (p->r2 > 0) {
          fold_gop(p->Y2, env, nenv);
          fold_gop(p->C2, env, nenv);
          if (p->bias2.ptr) fold_gop(p->bias2, env, nenv);
        }
        if (p->vec == 2) return p->f64 ? nullptr : rt_kernel_thin_rows_bulk((int)p->r, (int)p->k);
        return rt_kernel_thin_rows(p->f64, (int)p->r, (int)p->k);
      }
      // variant 2 with epilogue 2 (gate) is a separate instantiation ("4"),
      // with a second summed product ("5")
      if (p->variant == 2 && p->k2 > 0) {
        fold_gop(p->X2, env, nenv);
        fold_gop(p->Y2, env, nenv);
        if (p->epilogue != 2 || p->k2 > 4) return nullptr;
        return p->vec ? rt_kernel_thin_vec(2, p->f64, (int)p->k) : rt_kernel_thin(5, p->f64, (int)p->k);
      }
      if (p->variant == 1 && p->vec) return p->f64 ? nullptr : rt_kernel_thin_bulk((int)p->r, p->ones);
      if (p->variant == 1 && p->ones) return rt_kernel_thin(6, p->f64, (int)p->r);
      if (p->variant == 2 && p->vec)
        return rt_kernel_thin_vec(p->epilogue == 2 ? 1 : 0, p->f64, (int)p->k);
      return rt_kernel_thin(p->variant == 2 && p->epilogue == 2 ? 4 : p->variant, p->f64,
                            (int)(p->variant == 2 ? p->k : p->r));
    }
    case RT_K_SPLITK: {
      rt_splitk_params* p = (rt_splitk_params*)blk;
      fold_gop(p->C, env, nenv);
      if (p->bias.ptr) fold_gop(p->bias, env, nenv);
      return rt_kernel_splitk(p->f64);
    }
    case RT_K_RNG: {
      rt_rng_params* p = (rt_rng_params*)blk;
      fold_view(p->out, env, nenv);
      return rt_kernel_rng();
    }
    case RT_K_UDF: {
      rt_udf_params* p = (rt_udf_params*)blk;
      for (int i = 0; i < p->nin; ++i) fold_view(p->in[i], env, nenv);
      for (int i = 0; i < p->nout; ++i) fold_view(p->out[i], env, nenv);
      return rt_kernel_udf();
    }
    case RT_K_MEMCPY:
      return (void*)&rt_memcpy_marker;   // not a kernel: launch_one copies
    case RT_K_LOOP: {
      rt_loop_params* p = (rt_loop_params*)blk;
      if (p->blk_len > 0) {
        if (p->blk_slot < 0 || p->blk_slot >= nenv) return nullptr;
        p->start = env[p->blk_slot] * p->blk_len;
        p->stop = p->start + p->blk_len;
      }
      return rt_kernel_loop();
    }
    default:
      return nullptr;
  }
}

static int launch_one(const rt_launch_rec* rec, const int64_t* env, int nenv, cudaStream_t s) {
  alignas(128) static thread_local unsigned char blk[32768];
  if (rec->kernel == RT_K_MEMCPY) {
    rt_memcpy_params m;
    if (rec->param_bytes != (int)sizeof m) return fail(RT_ERR_BAD_ARG, "memcpy record size");
    memcpy(&m, (const void*)rec->params, sizeof m);
    if (m.bytes <= 0) return RT_OK;
    return cuda_check(cudaMemcpyAsync((void*)m.dst, (const void*)m.src, (size_t)m.bytes,
                                      cudaMemcpyDefault, s),
                      m.dir ? "swap fetch (cudaMemcpyAsync)" : "swap offload (cudaMemcpyAsync)");
  }
  if (rec->param_bytes <= 0 || rec->param_bytes > (int)sizeof blk)
    return fail(RT_ERR_BAD_ARG, "parameter block size out of range");
  memcpy(blk, (const void*)rec->params, rec->param_bytes);
  void* fn = prepare(rec->kernel, blk, env, nenv);
  if (!fn) return fail(RT_ERR_UNKNOWN_KERNEL, "unknown kernel family");
  if (rec->grid[0] <= 0) return RT_OK;  // empty box
  // a persistent TMA GEMM whose weight operand is split into tf32 hi/lo once
  // per launch: the split pass first, on the same stream
  if (rec->kernel == RT_K_GEMM_TMA && rt_gemm_tma_prepass(blk, (void*)s) != 0)
    return fail(RT_ERR_CUDA, "tf32 split pass");
  void* args[1] = {blk};
  dim3 g(rec->grid[0], rec->grid[1] > 0 ? rec->grid[1] : 1, rec->grid[2] > 0 ? rec->grid[2] : 1);
  dim3 b(rec->block[0], rec->block[1] > 0 ? rec->block[1] : 1, rec->block[2] > 0 ? rec->block[2] : 1);
  if (rec->jit_fn) {
    DriverApi& D = drv();
    if (!D.ok) return fail(RT_ERR_CUDA, "driver API unavailable");
    CUfunction f = (CUfunction)rec->jit_fn;
    if (rec->smem > 48 * 1024)
      D.funcSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, rec->smem);
    CUresult r;
    if (rec->cluster > 1) {
      // thread-block clusters (e.g. a CTA pair splitting a resident weight
      // matrix of the persistent acting loop across its two SMs)
      CUlaunchConfig cfg = {};
      CUlaunchAttribute attr[1];
      attr[0].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
      attr[0].value.clusterDim.x = (unsigned)rec->cluster;
      attr[0].value.clusterDim.y = 1;
      attr[0].value.clusterDim.z = 1;
      cfg.gridDimX = g.x; cfg.gridDimY = g.y; cfg.gridDimZ = g.z;
      cfg.blockDimX = b.x; cfg.blockDimY = b.y; cfg.blockDimZ = b.z;
      cfg.sharedMemBytes = rec->smem;
      cfg.hStream = (CUstream)s;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      r = D.launchKernelEx(&cfg, f, args, nullptr);
    } else {
      r = D.launchKernel(f, g.x, g.y, g.z, b.x, b.y, b.z, rec->smem, (CUstream)s, args, nullptr);
    }
    if (r != CUDA_SUCCESS) {
      const char* m = nullptr;
      D.getErrorString(r, &m);
      return fail(RT_ERR_CUDA, m ? m : "cuLaunchKernel failed");
    }
    return RT_OK;
  }
  if (rec->smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, rec->smem);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute");
  }
  return cuda_check(cudaLaunchKernel(fn, g, b, args, rec->smem, s), "cudaLaunchKernel");
}

extern "C" int rt_launch(const rt_launch_rec* rec, const int64_t* env, int32_t nenv, uint64_t stream) {
  return launch_one(rec, env, nenv, (cudaStream_t)stream);
}

// ------------------------------------------------------------ programs

extern "C" int rt_run(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs, int32_t nrec,
                      int64_t* env, int32_t nenv, uint64_t stream, const uint64_t* events,
                      int32_t nevents) {
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int64_t> ends(nprog, 0);
  int pc = 0;
  while (pc < nprog) {
    const rt_instr& in = prog[pc];
    switch (in.op) {
      case RT_OP_LAUNCH: {
        if (in.a < 0 || in.a >= nrec) return fail(RT_ERR_BAD_ARG, "launch record out of range");
        int rc = launch_one(&recs[in.a], env, nenv, s);
        if (rc) return rc;
        ++pc;
        break;
      }
      case RT_OP_FOR: {
        // b = first value, c = bound (exclusive in the direction of d), d = step
        if (in.a < 0 || in.a >= nenv) return fail(RT_ERR_BAD_ARG, "loop slot out of range");
        bool empty = in.d > 0 ? (in.b >= in.c) : (in.b <= in.c);
        if (empty) {
          pc = in.e;
        } else {
          env[in.a] = in.b;
          ++pc;
        }
        break;
      }
      case RT_OP_END: {
        const rt_instr& f = prog[in.a];
        int64_t v = env[f.a] + f.d;
        bool more = f.d > 0 ? (v < f.c) : (v > f.c);
        if (more) {
          env[f.a] = v;
          pc = in.a + 1;
        } else {
          ++pc;
        }
        break;
      }
      case RT_OP_EVENT: {
        if (in.a < 0 || in.a >= nevents) return fail(RT_ERR_BAD_ARG, "event slot out of range");
        // inside stream capture, an external record node really records the
        // event on every graph launch (a plain capture only orders nodes)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        int rc = cs == cudaStreamCaptureStatusActive
                     ? cuda_check(cudaEventRecordWithFlags((cudaEvent_t)events[in.a], s,
                                                           cudaEventRecordExternal),
                                  "cudaEventRecord(external)")
                     : cuda_check(cudaEventRecord((cudaEvent_t)events[in.a], s), "cudaEventRecord");
        if (rc) return rc;
        ++pc;
        break;
      }
      case RT_OP_ENVMOD: {
        if (in.a < 0 || in.a >= nenv || in.b < 0 || in.b >= nenv || in.c <= 0)
          return fail(RT_ERR_BAD_ARG, "bad envmod");
        env[in.a] = env[in.b] % in.c;
        ++pc;
        break;
      }
      case RT_OP_ENVADD: {
        if (in.a < 0 || in.a >= nenv) return fail(RT_ERR_BAD_ARG, "bad envadd");
        env[in.a] += in.b;
        ++pc;
        break;
      }
      case RT_OP_COLL: {
        int rc = rt_coll_exec(in.a, env, nenv, stream);
        if (rc) return rc;
        ++pc;
        break;
      }
      case RT_OP_HOOK:
        return fail(RT_ERR_BAD_ARG, "program has host hooks: use rt_run_segment");
      default:
        return fail(RT_ERR_BAD_ARG, "bad program instruction");
    }
  }
  return RT_OK;
}

extern "C" int rt_run_segment(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs,
                              int32_t nrec, int64_t* env, int32_t nenv, uint64_t stream,
                              int32_t* pc_io, int32_t* hook_out) {
  cudaStream_t s = (cudaStream_t)stream;
  int pc = *pc_io;
  while (pc < nprog) {
    const rt_instr& in = prog[pc];
    switch (in.op) {
      case RT_OP_LAUNCH: {
        int rc = launch_one(&recs[in.a], env, nenv, s);
        if (rc) return rc;
        ++pc;
        break;
      }
      case RT_OP_FOR: {
        bool empty = in.d > 0 ? (in.b >= in.c) : (in.b <= in.c);
        if (empty) pc = in.e; else { env[in.a] = in.b; ++pc; }
        break;
      }
      case RT_OP_END: {
        const rt_instr& f = prog[in.a];
        int64_t v = env[f.a] + f.d;
        bool more = f.d > 0 ? (v < f.c) : (v > f.c);
        if (more) { env[f.a] = v; pc = in.a + 1; } else ++pc;
        break;
      }
      case RT_OP_ENVMOD:
        if (in.a < 0 || in.a >= nenv || in.b < 0 || in.b >= nenv || in.c <= 0)
          return fail(RT_ERR_BAD_ARG, "bad envmod");
        env[in.a] = env[in.b] % in.c;
        ++pc;
        break;
      case RT_OP_ENVADD:
        if (in.a < 0 || in.a >= nenv) return fail(RT_ERR_BAD_ARG, "bad envadd");
        env[in.a] += in.b;
        ++pc;
        break;
      case RT_OP_COLL: {
        int rc = rt_coll_exec(in.a, env, nenv, stream);
        if (rc) return rc;
        ++pc;
        break;
      }
      case RT_OP_HOOK:
        *pc_io = pc + 1;
        *hook_out = in.a;
        return RT_HOOK;
      default:
        ++pc;
        break;
    }
  }
  *pc_io = nprog;
  return RT_OK;
}

// ------------------------------------------------------------ status word

extern "C" int rt_status_alloc(uint64_t* dev_ptr) {
  void* p = nullptr;
  int rc = cuda_check(cudaMalloc(&p, 4 * sizeof(int)), "cudaMalloc(status)");
  if (rc) return rc;
  rc = cuda_check(cudaMemset(p, 0, 4 * sizeof(int)), "cudaMemset(status)");
  *dev_ptr = (uint64_t)p;
  return rc;
}

extern "C" int rt_status_read(uint64_t dev_ptr, int32_t* host4, uint64_t stream) {
  int rc = cuda_check(cudaMemcpyAsync(host4, (void*)dev_ptr, 4 * sizeof(int), cudaMemcpyDeviceToHost,
                                      (cudaStream_t)stream), "status read");
  if (rc) return rc;
  return cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "status sync");
}

extern "C" int rt_status_clear(uint64_t dev_ptr, uint64_t stream) {
  return cuda_check(cudaMemsetAsync((void*)dev_ptr, 0, 4 * sizeof(int), (cudaStream_t)stream),
                    "status clear");
}

extern "C" int rt_status_free(uint64_t dev_ptr) {
  return cuda_check(cudaFree((void*)dev_ptr), "status free");
}

// ------------------------------------------------------------ tier moves

extern "C" int rt_memcpy_d2h_async(void* host_pinned, uint64_t dev, uint64_t bytes, uint64_t stream) {
  return cuda_check(cudaMemcpyAsync(host_pinned, (void*)dev, bytes, cudaMemcpyDeviceToHost,
                                    (cudaStream_t)stream), "d2h");
}

extern "C" int rt_memcpy_h2d_async(uint64_t dev, const void* host_pinned, uint64_t bytes, uint64_t stream) {
  return cuda_check(cudaMemcpyAsync((void*)dev, host_pinned, bytes, cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream), "h2d");
}

extern "C" int rt_memcpy2d_d2h_async(void* host_pinned, uint64_t hpitch, uint64_t dev,
                                     uint64_t dpitch, uint64_t width, uint64_t height,
                                     uint64_t stream) {
  return cuda_check(cudaMemcpy2DAsync(host_pinned, hpitch, (const void*)dev, dpitch, width, height,
                                      cudaMemcpyDeviceToHost, (cudaStream_t)stream), "d2h 2d");
}

extern "C" int rt_memcpy2d_h2d_async(uint64_t dev, uint64_t dpitch, const void* host_pinned,
                                     uint64_t hpitch, uint64_t width, uint64_t height,
                                     uint64_t stream) {
  return cuda_check(cudaMemcpy2DAsync((void*)dev, dpitch, host_pinned, hpitch, width, height,
                                      cudaMemcpyHostToDevice, (cudaStream_t)stream), "h2d 2d");
}

// ------------------------------------------------------------ rng fill

extern "C" int rt_rng_fill(uint64_t dev_out, const uint32_t* prefix, int32_t nprefix,
                           const int64_t* coords, int32_t ncoord, int64_t rows, int32_t count,
                           int32_t dist, uint64_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* dpre = nullptr;
  int64_t* dco = nullptr;
  int rc = cuda_check(cudaMalloc(&dpre, 8 * sizeof(uint32_t)), "malloc");
  if (rc) return rc;
  size_t cb = (size_t)(rows * (ncoord > 0 ? ncoord : 1)) * sizeof(int64_t);
  rc = cuda_check(cudaMalloc(&dco, cb), "malloc");
  if (rc) return rc;
  cudaMemcpyAsync(dpre, prefix, nprefix * sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  if (ncoord > 0) cudaMemcpyAsync(dco, coords, rows * ncoord * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  void* fn = rt_kernel_rng_fill();
  void* args[] = {&dev_out, &dpre, &nprefix, &dco, &ncoord, &rows, &count, &dist};
  int blocks = (int)((rows + 127) / 128);
  if (blocks > 65535) blocks = 65535;
  if (blocks < 1) blocks = 1;
  rc = cuda_check(cudaLaunchKernel(fn, dim3(blocks), dim3(128), args, 0, s), "rng_fill");
  cudaStreamSynchronize(s);
  cudaFree(dpre);
  cudaFree(dco);
  return rc;
}

// ------------------------------------------------------------ CUDA graphs
// Capture a whole lowered program (every loop iteration unrolled into the
// graph, each launch with its env already folded) and replay it with one
// cudaGraphLaunch: the per-step launch cost of the T-long acting loop goes
// from ~2 us of host work per kernel to the GPU's own inter-node gap.

extern "C" int rt_graph_capture(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs,
                                int32_t nrec, int64_t* env, int32_t nenv, uint64_t stream,
                                uint64_t* graph_exec_out) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaGraph_t graph = nullptr;
  int rc = cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
  if (rc) return rc;
  int rrc = rt_run(prog, nprog, recs, nrec, env, nenv, stream, nullptr, 0);
  rc = cuda_check(cudaStreamEndCapture(s, &graph), "end capture");
  if (rrc) { if (graph) cudaGraphDestroy(graph); return rrc; }
  if (rc) return rc;
  cudaGraphExec_t ex = nullptr;
  rc = cuda_check(cudaGraphInstantiate(&ex, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
  if (rc) return rc;
  *graph_exec_out = (uint64_t)ex;
  return RT_OK;
}

extern "C" int rt_graph_capture_ev(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs,
                                   int32_t nrec, int64_t* env, int32_t nenv, uint64_t stream,
                                   const uint64_t* events, int32_t nevents,
                                   uint64_t* graph_exec_out) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaGraph_t graph = nullptr;
  int rc = cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
  if (rc) return rc;
  int rrc = rt_run(prog, nprog, recs, nrec, env, nenv, stream, events, nevents);
  rc = cuda_check(cudaStreamEndCapture(s, &graph), "end capture");
  if (rrc) { if (graph) cudaGraphDestroy(graph); return rrc; }
  if (rc) return rc;
  cudaGraphExec_t ex = nullptr;
  rc = cuda_check(cudaGraphInstantiate(&ex, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
  if (rc) return rc;
  *graph_exec_out = (uint64_t)ex;
  return RT_OK;
}

extern "C" int rt_graph_launch(uint64_t graph_exec, uint64_t stream) {
  return cuda_check(cudaGraphLaunch((cudaGraphExec_t)graph_exec, (cudaStream_t)stream),
                    "graph launch");
}

extern "C" int rt_graph_destroy(uint64_t graph_exec) {
  return cuda_check(cudaGraphExecDestroy((cudaGraphExec_t)graph_exec), "graph destroy");
}

// ------------------------------------------------------------ profiling
// Run a program with a CUDA event pair around every launch instance and
// accumulate the device time per launch record (ms) and the instance count.
// Used by bench.py for the per-kernel breakdown and the live roofline.

extern "C" int rt_profile(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs,
                          int32_t nrec, int64_t* env, int32_t nenv, uint64_t stream,
                          double* rec_ms, int64_t* rec_count) {
  cudaStream_t s = (cudaStream_t)stream;
  static std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, int>> inst;  // (record, event pair index)
  size_t used = 0;
  int pc = 0;
  while (pc < nprog) {
    const rt_instr& in = prog[pc];
    if (in.op == RT_OP_LAUNCH) {
      while (pool.size() < used + 2) {
        cudaEvent_t e;
        int rc = cuda_check(cudaEventCreate(&e), "event create");
        if (rc) return rc;
        pool.push_back(e);
      }
      cudaEventRecord(pool[used], s);
      int rc = launch_one(&recs[in.a], env, nenv, s);
      if (rc) return rc;
      cudaEventRecord(pool[used + 1], s);
      inst.push_back({in.a, (int)used});
      used += 2;
      ++pc;
    } else if (in.op == RT_OP_FOR) {
      bool empty = in.d > 0 ? (in.b >= in.c) : (in.b <= in.c);
      if (empty) pc = in.e; else { env[in.a] = in.b; ++pc; }
    } else if (in.op == RT_OP_END) {
      const rt_instr& f = prog[in.a];
      int64_t v = env[f.a] + f.d;
      bool more = f.d > 0 ? (v < f.c) : (v > f.c);
      if (more) { env[f.a] = v; pc = in.a + 1; } else ++pc;
    } else if (in.op == RT_OP_ENVMOD) {
      if (in.c > 0 && in.a >= 0 && in.a < nenv && in.b >= 0 && in.b < nenv)
        env[in.a] = env[in.b] % in.c;
      ++pc;
    } else if (in.op == RT_OP_ENVADD) {
      if (in.a >= 0 && in.a < nenv) env[in.a] += in.b;
      ++pc;
    } else if (in.op == RT_OP_COLL) {
      int rc = rt_coll_exec(in.a, env, nenv, stream);
      if (rc) return rc;
      ++pc;
    } else {
      ++pc;
    }
  }
  int rc = cuda_check(cudaStreamSynchronize(s), "profile sync");
  if (rc) return rc;
  for (int r = 0; r < nrec; ++r) { rec_ms[r] = 0.0; rec_count[r] = 0; }
  for (auto& x : inst) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pool[x.second], pool[x.second + 1]);
    rec_ms[x.first] += ms;
    rec_count[x.first] += 1;
  }
  return RT_OK;
}

// ------------------------------------------------------------ JIT
// Fused elementwise programs and persistent loop bodies are compiled to
// straight-line CUDA at executable-build time (the interpreter VM stays as
// the reference semantics and the fallback for the library kernels).

static std::vector<std::string> split_opts(const char* opts, int nopt) {
  std::vector<std::string> v;
  const char* p = opts;
  for (int i = 0; i < nopt; ++i) {
    v.emplace_back(p);
    p += v.back().size() + 1;
  }
  return v;
}

static int nvrtc_build(const char* src, const char* opts, int nopt, std::string& image) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src, "rtb200_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail(RT_ERR_CUDA, "nvrtcCreateProgram failed");
  std::vector<std::string> o = split_opts(opts, nopt);
  std::vector<const char*> po;
  for (auto& x : o) po.push_back(x.c_str());
  nvrtcResult r = nvrtcCompileProgram(prog, (int)po.size(), po.data());
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    g_err = "nvrtc: " + log;
    return RT_ERR_CUDA;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  image.resize(n);
  nvrtcGetCUBIN(prog, &image[0]);
  nvrtcDestroyProgram(&prog);
  return RT_OK;
}

extern "C" int rt_jit_load(const void* image, const char* name, uint64_t* fn_out) {
  cudaFree(0);  // make sure the primary context is current
  DriverApi& D = drv();
  if (!D.ok) return fail(RT_ERR_CUDA, "driver API unavailable");
  CUmodule mod;
  CUresult r = D.moduleLoadData(&mod, image);
  if (r != CUDA_SUCCESS) {
    const char* m = nullptr;
    D.getErrorString(r, &m);
    return fail(RT_ERR_CUDA, m ? m : "cuModuleLoadData failed");
  }
  CUfunction f;
  r = D.moduleGetFunction(&f, mod, name);
  if (r != CUDA_SUCCESS) return fail(RT_ERR_CUDA, "cuModuleGetFunction failed");
  *fn_out = (uint64_t)f;
  return RT_OK;
}

extern "C" int rt_jit_cubin(const char* src, const char* opts, int32_t nopt, void* out,
                            uint64_t* size) {
  std::string image;
  int rc = nvrtc_build(src, opts, nopt, image);
  if (rc) return rc;
  if (out && *size >= image.size()) memcpy(out, image.data(), image.size());
  *size = image.size();
  return RT_OK;
}

extern "C" int rt_jit_compile(const char* src, const char* name, const char* opts, int32_t nopt,
                              uint64_t* fn_out) {
  std::string image;
  int rc = nvrtc_build(src, opts, nopt, image);
  if (rc) return rc;
  return rt_jit_load(image.data(), name, fn_out);
}
