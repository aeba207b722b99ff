"""ctypes binding to the C ABI in include/rtb200.h (librtb200.so).

Structures here mirror the header field for field; `check_layout()` compares
their sizes against the C side at load time.  There is no fallback: if the
library is missing or fails to load, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "librtb200.so")

RT_MAXD = 10
RT_MAXENV = 8
RT_MAXIN = 8
RT_MAXCHK = 3
RT_CODE = 256
RT_KONST = 32

RT_F64, RT_F32, RT_I64, RT_BOOL = 0, 1, 2, 3
DTYPE_CODE = {"f64": RT_F64, "f32": RT_F32, "i64": RT_I64, "bool": RT_BOOL}

RT_K_EW, RT_K_REDUCE, RT_K_SCAN, RT_K_GEMM, RT_K_RNG, RT_K_UDF, RT_K_SPLITK, RT_K_MEMCPY = \
    1, 2, 3, 4, 5, 6, 7, 8
RT_K_LOOP = 9
RT_K_GEMM_TC = 10
RT_K_THIN = 11
RT_K_GEMM_TMA = 12
TMA_SMEM = 2 * 48 * 1024 + 1024
TMA_SMEM_DRAIN = 4 * 48 * 1024 + 1024   # k_gemm_tma_drain: 4 stages, one CTA per SM
TMA_DRAIN_K = 256                        # K per TMEM accumulation chunk
TMA_SMEM_P = 4 * 48 * 1024 + 1024 + 8 * 4096   # k_gemm_tmap: persistent, 4 stages + epilogue C chunks
TMA_THREADS_P = 128 + 64 + 256
TC_SMEM = 2 * (2 * 128 * 32 * 4 + 2 * 256 * 32 * 4)

RT_OP_LAUNCH, RT_OP_FOR, RT_OP_END, RT_OP_EVENT, RT_OP_HOOK, RT_OP_ENVMOD = 1, 2, 3, 4, 6, 7
RT_OP_ENVADD = 9
RT_OP_COLL = 8
RT_HOOK = 100

RT_ERR_ROW_RANGE, RT_ERR_SLICE_RANGE = 1, 2
RT_ERR_DIV_ZERO = 6
RT_ERR_OVERFLOW = 7

i32, i64, u64, u32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_uint32, C.c_double


class rt_box(C.Structure):
    _fields_ = [("nd", i32), ("_pad", i32), ("ext", i64 * RT_MAXD)]


class rt_view(C.Structure):
    _fields_ = [("ptr", u64), ("dtype", i32), ("nchk", i32), ("off", i64),
                ("off_env", i64 * RT_MAXENV), ("stride", i64 * RT_MAXD),
                ("chk_c0", i64 * RT_MAXCHK), ("chk_hi", i64 * RT_MAXCHK),
                ("chk_env", (i32 * RT_MAXENV) * RT_MAXCHK),
                ("chk_a", (i32 * RT_MAXD) * RT_MAXCHK)]


class rt_hdr(C.Structure):
    _fields_ = [("env", i64 * RT_MAXENV), ("node", i32), ("status_slot", i32), ("status", u64)]


class rt_ew_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("box", rt_box), ("total", i64), ("nin", i32), ("f64", i32),
                ("out", rt_view), ("in_", rt_view * RT_MAXIN), ("code", i32 * RT_CODE),
                ("konst", f64 * RT_KONST)]


class rt_reduce_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("box", rt_box), ("total", i64), ("nred", i32), ("op", i32),
                ("gamma", f64), ("reverse", i32), ("f64", i32), ("len_prog", i32 * 4),
                ("len0", i64 * 4), ("len_env", (i64 * RT_MAXENV) * 4),
                ("len_a", (i64 * RT_MAXD) * 4), ("red_stride", i64 * 4), ("lo_prog", i32 * 4),
                ("threads_per_out", i32), ("splits", i32), ("part", u64), ("in_", rt_view),
                ("out", rt_view),
                ("code", i32 * RT_CODE), ("konst", f64 * RT_KONST)]


class rt_scan_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("box", rt_box), ("total_lines", i64), ("sdim", i32),
                ("reverse", i32), ("gamma", f64), ("f64", i32), ("chunk", i32),
                ("in_", rt_view), ("out", rt_view), ("win", i32), ("tile", i32),
                ("gae", i32), ("stages", i32), ("gae_c", f64), ("gae_vb", f64),
                ("in2", rt_view)]


class rt_memcpy_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("dst", u64), ("src", u64), ("bytes", i64), ("dir", i32),
                ("_pad", i32)]


class rt_gbox(C.Structure):
    _fields_ = [("nd", i32), ("_pad", i32), ("ext", i64 * 4)]


class rt_gop(C.Structure):
    _fields_ = [("ptr", u64), ("dtype", i32), ("_pad", i32), ("off", i64),
                ("off_env", i64 * RT_MAXENV), ("sz", i64 * 4), ("s1", i64 * 4), ("s2", i64 * 4)]


class rt_gemm_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("Z", rt_gbox), ("M", rt_gbox), ("N", rt_gbox), ("K", rt_gbox),
                ("z", i64), ("m", i64), ("n", i64), ("k", i64), ("f64", i32), ("splits", i32),
                ("accumulate", i32), ("epilogue", i32), ("A", rt_gop), ("B", rt_gop),
                ("C", rt_gop), ("part", u64), ("bias", rt_gop)]


class rt_splitk_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("Z", rt_gbox), ("M", rt_gbox), ("N", rt_gbox),
                ("z", i64), ("m", i64), ("n", i64), ("splits", i32), ("f64", i32),
                ("accumulate", i32), ("epilogue", i32), ("part", u64), ("C", rt_gop),
                ("bias", rt_gop)]


class rt_thin_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("variant", i32), ("f64", i32), ("w", i64), ("r", i64), ("k", i64),
                ("splits", i32), ("accumulate", i32), ("epilogue", i32), ("vec", i32),
                ("part_w", i64), ("part_r", i64), ("part", u64), ("X", rt_gop), ("Y", rt_gop),
                ("C", rt_gop), ("bias", rt_gop), ("W", rt_gbox), ("k2", i64), ("X2", rt_gop),
                ("Y2", rt_gop), ("ones", i32), ("colsum", i32), ("part2", u64), ("dw", i32),
                ("dw2", i32), ("part3", u64), ("part4", u64), ("r2", i64),
                ("C2", rt_gop), ("bias2", rt_gop)]


class rt_rng_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("box", rt_box), ("total", i64), ("nprefix", i32),
                ("ncoord", i32), ("prefix", u32 * 8), ("coord_src", i32 * RT_MAXD),
                ("coord_add", i64 * RT_MAXD), ("dist", i32), ("count", i32), ("out", rt_view)]


class rt_udf_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("box", rt_box), ("total", i64), ("nprefix", i32),
                ("ncoord", i32), ("prefix", u32 * 8), ("coord_src", i32 * RT_MAXD),
                ("coord_add", i64 * RT_MAXD), ("salt", f64), ("nin", i32), ("nout", i32), ("in_count", i32 * 4),
                ("out_count", i32 * 4), ("out_kind", i32 * 4), ("in_", rt_view * 4),
                ("out", rt_view * 4)]


class rt_loop_op(C.Structure):
    _fields_ = [("kernel", i32), ("f64", i32), ("params", u64), ("row_elems", i64),
                ("noise", u64), ("noise_off", i64), ("noise_row", i64), ("noise_step", i64),
                ("param_bytes", i32), ("smem_off", i32)]


class rt_loop_params(C.Structure):
    _fields_ = [("h", rt_hdr), ("slot", i32), ("nops", i32), ("start", i64), ("stop", i64),
                ("step", i64), ("rows", i64), ("rows_per_cta", i32), ("smem_bytes", i32),
                ("ring_off", i32), ("a_off", i32), ("ops", u64), ("prof", u64),
                ("blk_slot", i32), ("red_off", i32), ("blk_len", i64)]


class rt_launch_rec(C.Structure):
    _fields_ = [("kernel", i32), ("param_bytes", i32), ("params", u64), ("grid", i32 * 3),
                ("block", i32 * 3), ("smem", i32), ("cluster", i32), ("jit_fn", u64)]


class rt_instr(C.Structure):
    _fields_ = [("op", i32), ("a", i32), ("b", i64), ("c", i64), ("d", i64), ("e", i32),
                ("_pad", i32)]


class rt_coll(C.Structure):
    _fields_ = [("ptr", u64), ("off0", i64), ("off_env", i64 * RT_MAXENV), ("count", i64),
                ("dtype", i32), ("flush", i32)]


class NativeError(RuntimeError):
    pass


_lib = None


def lib():
    """Load librtb200.so; raise (never fall back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(
            f"native backend not built: {LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = C.CDLL(LIB_PATH)
    L.rt_version.restype = i32
    L.rt_last_error.restype = C.c_char_p
    L.rt_launch.argtypes = [C.POINTER(rt_launch_rec), C.POINTER(i64), i32, u64]
    L.rt_run.argtypes = [C.POINTER(rt_instr), i32, C.POINTER(rt_launch_rec), i32,
                         C.POINTER(i64), i32, u64, C.POINTER(u64), i32]
    L.rt_run_segment.argtypes = [C.POINTER(rt_instr), i32, C.POINTER(rt_launch_rec), i32,
                                 C.POINTER(i64), i32, u64, C.POINTER(i32), C.POINTER(i32)]
    L.rt_graph_capture.argtypes = [C.POINTER(rt_instr), i32, C.POINTER(rt_launch_rec), i32,
                                   C.POINTER(i64), i32, u64, C.POINTER(u64)]
    L.rt_graph_launch.argtypes = [u64, u64]
    L.rt_graph_capture_ev.argtypes = [C.POINTER(rt_instr), i32, C.POINTER(rt_launch_rec), i32,
                                      C.POINTER(i64), i32, u64, C.POINTER(u64), i32,
                                      C.POINTER(u64)]
    L.rt_profile.argtypes = [C.POINTER(rt_instr), i32, C.POINTER(rt_launch_rec), i32,
                             C.POINTER(i64), i32, u64, C.POINTER(f64), C.POINTER(i64)]
    L.rt_graph_destroy.argtypes = [u64]
    L.rt_jit_compile.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, i32, C.POINTER(u64)]
    L.rt_jit_load.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(u64)]
    L.rt_jit_cubin.argtypes = [C.c_char_p, C.c_char_p, i32, C.c_void_p, C.POINTER(u64)]
    L.rt_status_alloc.argtypes = [C.POINTER(u64)]
    L.rt_status_read.argtypes = [u64, C.POINTER(i32), u64]
    L.rt_status_clear.argtypes = [u64, u64]
    L.rt_status_free.argtypes = [u64]
    L.rt_rng_fill.argtypes = [u64, C.POINTER(u32), i32, C.POINTER(i64), i32, i64, i32, i32, u64]
    L.rt_memcpy_d2h_async.argtypes = [C.c_void_p, u64, u64, u64]
    L.rt_memcpy_h2d_async.argtypes = [u64, C.c_void_p, u64, u64]
    L.rt_memcpy2d_d2h_async.argtypes = [C.c_void_p, u64, u64, u64, u64, u64, u64]
    L.rt_memcpy2d_h2d_async.argtypes = [u64, u64, C.c_void_p, u64, u64, u64, u64]
    L.rt_pool_create.argtypes = [i32, u64, C.POINTER(u64)]
    L.rt_pool_destroy.argtypes = [u64]
    L.rt_pool_alloc.argtypes = [u64, u64, u64, C.POINTER(u64)]
    L.rt_pool_free.argtypes = [u64, u64, u64]
    L.rt_pool_host.argtypes = [u64, i64]
    L.rt_pool_stats.argtypes = [u64, C.POINTER(u64)]
    L.rt_offload.argtypes = [u64, C.c_void_p, u64, u64, u64, u64, u64, u64, u64, u64]
    L.rt_fetch.argtypes = [u64, u64, u64, C.c_void_p, u64, u64, u64, u64, u64, u64]
    L.rt_block_update.argtypes = [u64, i64, u64, u64, u64]
    L.rt_stack.argtypes = [u64, C.POINTER(u64), i32, u64, u64]
    L.rt_set_error.argtypes = [i32, C.c_char_p]
    L.rt_nccl_unique_id.argtypes = [C.c_char_p]
    L.rt_nccl_comm_init.argtypes = [i32, i32, C.c_char_p, C.POINTER(u64)]
    L.rt_nccl_comm_destroy.argtypes = [u64]
    L.rt_nccl_allreduce.argtypes = [u64, u64, u64, i32, u64]
    L.rt_set_collectives.argtypes = [u64, C.POINTER(rt_coll), i32]
    L.rt_coll_exec.argtypes = [i32, C.POINTER(i64), i32, u64]
    if L.rt_version() != 1:
        raise NativeError("librtb200 ABI version mismatch")
    _lib = L
    return L


EXPORTS = ("rt_version", "rt_launch", "rt_run", "rt_status_alloc", "rt_status_read",
           "rt_status_clear", "rt_status_free", "rt_memcpy_d2h_async", "rt_memcpy_h2d_async",
           "rt_rng_fill", "rt_last_error", "rt_graph_capture", "rt_graph_launch",
           "rt_graph_destroy", "rt_profile", "rt_graph_capture_ev", "rt_run_segment",
           "rt_jit_compile", "rt_jit_load", "rt_jit_cubin", "rt_memcpy2d_d2h_async",
           "rt_memcpy2d_h2d_async", "rt_pool_create", "rt_pool_destroy", "rt_pool_alloc",
           "rt_pool_free", "rt_pool_host", "rt_pool_stats", "rt_offload", "rt_fetch",
           "rt_block_update", "rt_stack", "rt_set_error", "rt_nccl_unique_id",
           "rt_nccl_comm_init", "rt_nccl_comm_destroy", "rt_nccl_allreduce",
           "rt_set_collectives", "rt_coll_exec")


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = lib().rt_last_error().decode(errors="replace")
        raise NativeError(f"{what}: rt error {rc}: {msg}")
