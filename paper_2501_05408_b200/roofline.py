"""Algorithmic cost of one launch record (SURVEY §8(d) cost model):
bytes that must cross HBM at least once, and flops.  Used by bench.py to
turn measured kernel times into roofline fractions."""

from __future__ import annotations

from . import native as N

ITEM = {N.RT_F64: 8, N.RT_F32: 4, N.RT_I64: 8, N.RT_BOOL: 1}
FAMILY = {N.RT_K_EW: "ew", N.RT_K_REDUCE: "reduce", N.RT_K_SCAN: "scan", N.RT_K_GEMM: "gemm",
          N.RT_K_RNG: "rng", N.RT_K_UDF: "udf", N.RT_K_SPLITK: "splitk",
          N.RT_K_MEMCPY: "memcpy", N.RT_K_LOOP: "loop", N.RT_K_GEMM_TC: "gemm_tc",
          N.RT_K_THIN: "thin", N.RT_K_GEMM_TMA: "gemm_tma"}


def _prod(xs):
    out = 1
    for x in xs:
        out *= x
    return out


def _view_bytes(v, box):
    """Distinct elements a view touches over the box (dims with stride 0 are
    broadcast) times the item size."""
    n = _prod(box[d] for d in range(len(box)) if v.stride[d] != 0)
    return n * ITEM.get(v.dtype, 4)


def _gop_elems(o, Z, M, N_, role):
    zs = _prod(Z.ext[i] for i in range(Z.nd) if o.sz[i] != 0)
    a = _prod(M.ext[i] for i in range(M.nd) if o.s1[i] != 0)
    b = _prod(N_.ext[i] for i in range(N_.nd) if o.s2[i] != 0)
    return zs * a * b


def cost(kernel, p, loop_info=None):
    """(bytes, flops) for one launch of record params p."""
    if kernel == N.RT_K_MEMCPY:
        return int(p.bytes), 0
    if kernel == N.RT_K_LOOP:
        if not loop_info:
            return 0, 0
        b = f = 0
        rows = p.rows
        for k, q, re, f64, noise, *_ in loop_info["ops"]:
            b2, f2 = cost(k, q)
            b += b2
            f += f2
        n = loop_info.get("trips_per_launch", loop_info["trips"])
        return b * n, f * n
    if kernel == N.RT_K_EW:
        box = [p.box.ext[i] for i in range(p.box.nd)]
        b = p.total * ITEM.get(p.out.dtype, 4)
        for i in range(p.nin):
            b += _view_bytes(p.in_[i], box)
        return b, 0
    if kernel == N.RT_K_REDUCE:
        box = [p.box.ext[i] for i in range(p.box.nd)]
        red = 1
        for j in range(p.nred):
            red *= max(1, p.len0[j]) if p.len_prog[j] < 0 and not any(
                p.len_a[j][d] for d in range(p.box.nd)) else 1
        b = p.total * ITEM.get(p.out.dtype, 4) + p.total * red * ITEM.get(p.in_.dtype, 4)
        return b, p.total * red
    if kernel == N.RT_K_SCAN:
        box = [p.box.ext[i] for i in range(p.box.nd)]
        tot = _prod(box)
        return tot * (ITEM.get(p.in_.dtype, 4) + ITEM.get(p.out.dtype, 4)), 2 * tot
    if kernel in (N.RT_K_GEMM, N.RT_K_GEMM_TC, N.RT_K_GEMM_TMA):
        fl = 2 * p.z * p.m * p.n * p.k
        ea = _gop_elems(p.A, p.Z, p.M, p.K, 0) * ITEM.get(p.A.dtype, 4)
        eb = _gop_elems(p.B, p.Z, p.K, p.N, 1) * ITEM.get(p.B.dtype, 4)
        ec = p.z * p.m * p.n * ITEM.get(p.C.dtype, 4)
        if kernel == N.RT_K_GEMM_TMA and p.epilogue == 2:   # tanh-VJP gate operand (m x n)
            ec += p.z * p.m * p.n * ITEM.get(p.bias.dtype, 4)
        return ea + eb + ec, fl
    if kernel == N.RT_K_THIN:
        it = 8 if p.f64 else 4
        if p.variant == 1:   # stream X[k, w], Y[k, r]; partials out
            return (p.k * (p.w + p.r) + p.splits * p.w * p.r) * it, 2 * p.w * p.r * p.k
        gate = p.w * p.r if (p.variant == 2 and p.epilogue == 2) else 0   # gate operand read
        return (p.w * p.k + p.k * p.r + p.w * p.r * (2 if p.accumulate else 1) + gate) * it, \
            2 * p.w * p.r * p.k
    if kernel == N.RT_K_RNG:
        return p.total * p.count * ITEM.get(p.out.dtype, 4), 0
    if kernel == N.RT_K_UDF:
        b = 0
        for i in range(p.nin):
            b += p.total * p.in_count[i] * ITEM.get(p.in_[i].dtype, 4)
        for j in range(p.nout):
            b += p.total * p.out_count[j] * ITEM.get(p.out[j].dtype, 4)
        return b, 0
    if kernel == N.RT_K_SPLITK:
        it = 8 if p.f64 else 4
        return p.z * p.m * p.n * it * (p.splits + 1), p.z * p.m * p.n * p.splits
    return 0, 0


# per-family compute ceilings for the whole-step roofline (TFLOP/s): the
# tcgen05 GEMMs run 3xTF32 (three tf32 MMAs per fp32 product: the dense bf16
# peak / 2 / 3), everything else computes on the FP32 SIMT pipes
def compute_peak_tflops(family, bf16_tflops, fp32_simt_tflops):
    if family in ("gemm_tma", "gemm_tc"):
        return bf16_tflops / 2.0 / 3.0
    return fp32_simt_tflops


def floor_ms(kernel, p, loop_info, hbm_gbs, bf16_tflops, fp32_simt_tflops):
    """Roofline time of one launch: max(algorithmic bytes / HBM, flops /
    the family's compute ceiling), in ms."""
    b, f = cost(kernel, p, loop_info)
    t_mem = b / (hbm_gbs * 1e9)
    t_cmp = f / (compute_peak_tflops(FAMILY.get(kernel, ""), bf16_tflops, fp32_simt_tflops) * 1e12)
    return 1e3 * max(t_mem, t_cmp)
