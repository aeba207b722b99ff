"""JIT specialisation of elementwise launches.

A lowered RT_K_EW record carries a small VM program (csrc/common.cuh) whose
interpretation costs ~100 instructions per element.  For large launches the
program is translated into straight-line CUDA — one C statement per VM
instruction on named registers, jumps as gotos — with the box extents,
strides and range-check coefficients baked in as literals, compiled with
NVRTC for sm_100a and launched in place of the library kernel (same
parameter block, so env folding and CUDA-graph capture are unchanged).
Compiled cubins are cached on disk by source hash.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os

from . import native as N

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.environ.get("RTB200_JIT_CACHE", os.path.join(os.path.expanduser("~"), ".cache",
                                                        "rtb200_jit"))
JIT_MIN_ELEMS = int(os.environ.get("RTB200_JIT_MIN", str(1 << 18)))
ENABLED = os.environ.get("RTB200_JIT", "1") != "0"

CT = {N.RT_F64: "double", N.RT_F32: "float", N.RT_I64: "long long", N.RT_BOOL: "unsigned char"}

OPS = {v: k for k, v in {
    "ICOORD": 1, "IENV": 2, "ICONST": 3, "IADD": 4, "ISUB": 5, "IMUL": 6, "IFDIV": 7,
    "IMOD": 8, "IMIN": 9, "IMAX": 10, "INEG": 11, "IEQ": 12, "ILT": 13, "ILE": 14,
    "IGT": 15, "IGE": 16, "INE": 17, "IAND": 18, "IOR": 19, "INOT": 20, "JZ": 21,
    "JMP": 22, "LOAD": 30, "LOADX": 31, "VCONST": 32, "VITOF": 33, "VADD": 34,
    "VSUB": 35, "VMUL": 36, "VDIV": 37, "VNEG": 38, "VEXP": 39, "VLOG": 40,
    "VTANH": 41, "VSQRT": 42, "VPOW": 43, "VEQ": 44, "VNE": 45, "VLT": 46, "VLE": 47,
    "VGT": 48, "VGE": 49, "VWHERE": 50, "VCAST": 51, "VMOV": 52, "VTOI": 53,
    "VALID": 54, "STORE": 60, "ERROR": 62, "ISTORE": 63}.items()}


def _lit(x):
    return f"{int(x)}LL"


def _flit(x, T):
    r = repr(float(x))
    if r in ("inf", "-inf", "nan"):
        return {"inf": "(1.0/0.0)", "-inf": "(-1.0/0.0)", "nan": "(0.0/0.0)"}[r]
    return f"(({T}){r})"


def _offset_expr(base, v, nd):
    terms = [base]
    for d in range(nd):
        s = v.stride[d]
        if s:
            terms.append(f"i{d}*{_lit(s)}")
    return " + ".join(terms)


def _valid_expr(pfx, v, nd):
    conds = []
    for c in range(v.nchk):
        terms = [f"{pfx}.chk_c0[{c}]"]
        for d in range(nd):
            a = v.chk_a[c][d]
            if a:
                terms.append(f"i{d}*{_lit(a)}")
        x = " + ".join(terms)
        conds.append(f"((unsigned long long)({x}) < {int(v.chk_hi[c])}ULL)")
    return " && ".join(conds) if conds else "true"


def ew_source(p, name):
    """CUDA source of a kernel equivalent to k_ew<T> on parameter block p."""
    nd = p.box.nd
    ext = [p.box.ext[i] for i in range(nd)]
    T = "double" if p.f64 else "float"
    code = [p.code[i] for i in range(N.RT_CODE)]
    # find the program end and jump targets
    targets = set()
    pc, end = 0, 0
    while pc < N.RT_CODE:
        op = code[pc] & 0xFF
        if op in (21, 22):
            targets.add(code[pc + 1])
        end = pc + 2
        if op in (0, 60, 63) and not any(t > pc for t in targets):
            break
        pc += 2
    lines = []
    w = lines.append
    pc = 0
    while pc < end:
        w0, imm = code[pc], code[pc + 1]
        op = w0 & 0xFF
        d, a, b, c = (w0 >> 8) & 15, (w0 >> 12) & 15, (w0 >> 16) & 15, (w0 >> 20) & 15
        if pc in targets:
            w(f"L{pc}:;")
        o = OPS.get(op)
        if op == 0:
            w("goto Lend;")
        elif o == "ICOORD":
            w(f"n{d} = i{imm};")
        elif o == "IENV":
            w(f"n{d} = p.h.env[{imm}];")
        elif o == "ICONST":
            w(f"n{d} = {_lit(imm)};")
        elif o in ("IADD", "ISUB", "IMUL"):
            w(f"n{d} = n{a} {'+-*'[['IADD', 'ISUB', 'IMUL'].index(o)]} n{b};")
        elif o == "IFDIV":
            w(f"n{d} = euclid_div(n{a}, n{b});")
        elif o == "IMOD":
            w(f"n{d} = euclid_mod(n{a}, n{b});")
        elif o in ("IMIN", "IMAX"):
            w(f"n{d} = n{a} {'<' if o == 'IMIN' else '>'} n{b} ? n{a} : n{b};")
        elif o == "INEG":
            w(f"n{d} = -n{a};")
        elif o in ("IEQ", "ILT", "ILE", "IGT", "IGE", "INE"):
            sym = {"IEQ": "==", "ILT": "<", "ILE": "<=", "IGT": ">", "IGE": ">=", "INE": "!="}[o]
            w(f"n{d} = n{a} {sym} n{b};")
        elif o == "IAND":
            w(f"n{d} = (n{a} != 0) && (n{b} != 0);")
        elif o == "IOR":
            w(f"n{d} = (n{a} != 0) || (n{b} != 0);")
        elif o == "INOT":
            w(f"n{d} = n{a} == 0;")
        elif o == "JZ":
            w(f"if (n{a} == 0) goto L{imm};")
        elif o == "JMP":
            w(f"goto L{imm};")
        elif o in ("LOAD", "LOADX"):
            v = p.in_[imm]
            pfx = f"p.in[{imm}]"
            off = _offset_expr(f"{pfx}.off", v, nd)
            valid = _valid_expr(pfx, v, nd)
            if o == "LOADX":
                off = f"{off} + n{a}"
                valid = f"(n{b} != 0) && {valid}"
            ct = CT[v.dtype]
            load = f"(({T})((const {ct}*){pfx}.ptr)[{off}])"
            if v.dtype == N.RT_BOOL:
                load = f"(((const unsigned char*){pfx}.ptr)[{off}] ? ({T})1 : ({T})0)"
            w(f"v{d} = ({valid}) ? {load} : ({T})0;" if valid != "true" else f"v{d} = {load};")
        elif o == "VCONST":
            w(f"v{d} = {_flit(p.konst[imm], T)};")
        elif o == "VITOF":
            w(f"v{d} = ({T})n{a};")
        elif o in ("VADD", "VSUB", "VMUL", "VDIV"):
            w(f"v{d} = v{a} {'+-*/'[['VADD', 'VSUB', 'VMUL', 'VDIV'].index(o)]} v{b};")
        elif o == "VNEG":
            w(f"v{d} = -v{a};")
        elif o in ("VEXP", "VLOG", "VTANH", "VSQRT"):
            w(f"v{d} = vm_{o[1:].lower()}<{T}>(v{a});")
        elif o == "VPOW":
            w(f"v{d} = vm_pow<{T}>(v{a}, {_flit(p.konst[imm], T)});")
        elif o in ("VEQ", "VNE", "VLT", "VLE", "VGT", "VGE"):
            sym = {"VEQ": "==", "VNE": "!=", "VLT": "<", "VLE": "<=", "VGT": ">", "VGE": ">="}[o]
            w(f"v{d} = ({T})(v{a} {sym} v{b});")
        elif o == "VWHERE":
            w(f"v{d} = v{a} != ({T})0 ? v{b} : v{c};")
        elif o == "VCAST":
            w(f"v{d} = vm_round<{T}>(v{a}, {imm});")
        elif o == "VMOV":
            w(f"v{d} = v{a};")
        elif o == "VTOI":
            w(f"n{d} = v{a} != ({T})0;")
        elif o == "VALID":
            w(f"n{d} = {_valid_expr(f'p.in[{imm}]', p.in_[imm], nd)};")
        elif o == "STORE":
            w(f"res = v{a}; goto Lend;")
        elif o == "ERROR":
            w(f"report(p.h, {imm}, n{a}, n{b});")
        else:
            raise ValueError(f"cannot translate VM op {op}")
        pc += 2
    body = "\n      ".join(lines)
    total = 1
    for e in ext:
        total *= e
    small = total < (1 << 31)
    dec = []
    idx_t = "unsigned int" if small else "long long"
    dec.append(f"{idx_t} r = ({idx_t})flat;")
    for dd in reversed(range(nd)):
        if dd == 0:
            dec.append(f"const long long i0 = (long long)r;")
        else:
            dec.append(f"const long long i{dd} = (long long)(r % {ext[dd]}u); r /= {ext[dd]}u;"
                       if small else
                       f"const long long i{dd} = r % {ext[dd]}LL; r /= {ext[dd]}LL;")
    dec_s = "\n      ".join(dec)
    ov = p.out
    out_off = _offset_expr("p.out.off", ov, nd)
    oct_ = CT[ov.dtype]
    store = (f"((unsigned char*)p.out.ptr)[{out_off}] = res != ({T})0;" if ov.dtype == N.RT_BOOL
             else f"(({oct_}*)p.out.ptr)[{out_off}] = ({oct_})res;")
    regs = ", ".join(f"v{i}" for i in range(8))
    iregs = ", ".join(f"n{i}" for i in range(8))
    return f"""#include "common.cuh"
extern "C" __global__ void __launch_bounds__(256) {name}(const __grid_constant__ rt_ew_params p) {{
  for (long long flat = (long long)blockIdx.x * 256 + threadIdx.x; flat < {total}LL;
       flat += (long long)gridDim.x * 256) {{
      {dec_s}
      {T} {regs};
      long long {iregs};
      {T} res = ({T})0;
      (void)n0;
      {body}
    Lend:
      {store}
  }}
}}
"""


_FN_CACHE: dict = {}


def _opts():
    # -fmad=false: each elementwise op rounds like the reference's numpy ops
    # (no contraction of a*b+c across program statements)
    return [b"-arch=sm_100a", b"-std=c++17", b"-lineinfo", b"-fmad=false",
            b"-I" + os.path.join(HERE, "csrc").encode()]


def compile_kernel(src: str, name: str) -> int:
    """CUfunction handle for `name` in `src` (process + on-disk cubin cache)."""
    key = hashlib.sha256((src + name).encode()).hexdigest()
    if key in _FN_CACHE:
        return _FN_CACHE[key]
    lib = N.lib()
    fn = N.u64(0)
    path = os.path.join(CACHE, key + ".cubin")
    image = None
    if os.path.exists(path):
        with open(path, "rb") as fh:
            image = fh.read()
    if image is None:
        opts = _opts()
        blob = b"\0".join(opts) + b"\0"
        size = N.u64(0)
        N.check(lib.rt_jit_cubin(src.encode(), blob, len(opts), None, C.byref(size)), "nvrtc")
        buf = C.create_string_buffer(size.value)
        N.check(lib.rt_jit_cubin(src.encode(), blob, len(opts), buf, C.byref(size)), "nvrtc")
        image = buf.raw[:size.value]
        try:
            os.makedirs(CACHE, exist_ok=True)
            tmp = path + f".{os.getpid()}"
            with open(tmp, "wb") as fh:
                fh.write(image)
            os.replace(tmp, path)
        except OSError:
            pass
    N.check(lib.rt_jit_load(image, name.encode(), C.byref(fn)), "jit load")
    _FN_CACHE[key] = fn.value
    return fn.value


def specialise(recs, kernels, params, labels):
    """Attach JIT kernels to large EW records (in place)."""
    if not ENABLED:
        return 0
    n = 0
    for i, (k, p) in enumerate(zip(kernels, params)):
        if k != N.RT_K_EW or p.total < JIT_MIN_ELEMS:
            continue
        src = ew_source(p, "ew_jit")
        recs[i].jit_fn = compile_kernel(src, "ew_jit")
        n += 1
    return n
