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
EW_UNROLL = int(os.environ.get("RTB200_EW_UNROLL", "4"))
JIT_LOOP_MIN = int(os.environ.get("RTB200_JIT_LOOP_MIN", str(1 << 16)))   # rows x trips
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


def _offset_expr(base, v, nd, var="i"):
    terms = [base]
    for d in range(nd):
        s = v.stride[d]
        if s:
            terms.append(f"{var}{d}*{_lit(s)}")
    return " + ".join(terms)


def _valid_expr(pfx, v, nd, c0=None):
    conds = []
    for c in range(v.nchk):
        terms = [c0(c) if c0 else f"{pfx}.chk_c0[{c}]"]
        for d in range(nd):
            a = v.chk_a[c][d]
            if a:
                terms.append(f"i{d}*{_lit(a)}")
        x = " + ".join(terms)
        conds.append(f"((unsigned long long)({x}) < {int(v.chk_hi[c])}ULL)")
    return " && ".join(conds) if conds else "true"


def _program_lines(p, T, nd, base=None, chk=None, env="p.h.env", load_override=None):
    """Straight-line C statements for the VM program of EW params p
    (load_override: {input k: expression} for unchecked LOADs of input k)."""
    code = [p.code[i] for i in range(N.RT_CODE)]
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
            w(f"n{d} = {env}[{imm}];")
        elif o == "ICONST":
            w(f"n{d} = {_lit(imm)};")
        elif o in ("IADD", "ISUB", "IMUL"):
            w(f"n{d} = n{a} {'+-*'[['IADD', 'ISUB', 'IMUL'].index(o)]} n{b};")
        elif o == "IFDIV":
            w(f"if (n{b} == 0) report(p.h, {N.RT_ERR_DIV_ZERO}, n{a}, 0);")
            w(f"n{d} = euclid_div(n{a}, n{b});")
        elif o == "IMOD":
            w(f"if (n{b} == 0) report(p.h, {N.RT_ERR_DIV_ZERO}, n{a}, 1);")
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
            off = _offset_expr(base(imm) if base else f"{pfx}.off", v, nd)
            valid = _valid_expr(pfx, v, nd, (lambda cc, k=imm: chk(k, cc)) if chk else None)
            if o == "LOADX":
                off = f"{off} + n{a}"
                valid = f"(n{b} != 0) && {valid}"
            ct = CT[v.dtype]
            if o == "LOAD" and load_override and imm in load_override:
                w(f"v{d} = {load_override[imm]};" if valid == "true" else
                  f"v{d} = ({valid}) ? ({T})({load_override[imm]}) : ({T})0;")
                pc += 2
                continue
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
    return lines


def _decompose(nd, ext, flat="flat", small=True):
    dec = []
    idx_t = "unsigned int" if small else "long long"
    dec.append(f"{idx_t} r = ({idx_t}){flat};")
    for dd in reversed(range(nd)):
        if dd == 0:
            dec.append("const long long i0 = (long long)r;")
        else:
            dec.append(f"const long long i{dd} = (long long)(r % {ext[dd]}u); r /= {ext[dd]}u;"
                       if small else
                       f"const long long i{dd} = r % {ext[dd]}LL; r /= {ext[dd]}LL;")
    return dec


def _store(p, T, nd, base):
    ov = p.out
    out_off = _offset_expr(base, ov, nd)
    oct_ = CT[ov.dtype]
    return (f"((unsigned char*)p.out.ptr)[{out_off}] = res != ({T})0;" if ov.dtype == N.RT_BOOL
            else f"(({oct_}*)p.out.ptr)[{out_off}] = ({oct_})res;")


def ew_source(p, name):
    """CUDA source of a kernel equivalent to k_ew<T> on parameter block p."""
    nd = p.box.nd
    ext = [p.box.ext[i] for i in range(nd)]
    T = "double" if p.f64 else "float"
    lines = _program_lines(p, T, nd)
    body = "\n      ".join(lines)
    total = 1
    for e in ext:
        total *= e
    dec_s = "\n      ".join(_decompose(nd, ext, small=total < (1 << 31)))
    store = _store(p, T, nd, "p.out.off")
    regs = ", ".join(f"v{i}" for i in range(8))
    iregs = ", ".join(f"n{i}" for i in range(8))
    # EW_UNROLL elements per thread, blockDim apart (coalescing unchanged):
    # every element's loads and arithmetic are issued before any store, so
    # EW_UNROLL independent load streams per thread are in flight
    U = EW_UNROLL if p.nin <= 2 else 1     # (measured: wider bodies lose to register pressure)
    out_off = _offset_expr("p.out.off", p.out, nd)
    oct_ = CT[p.out.dtype]
    st = (f"((unsigned char*)p.out.ptr)[oo[q]] = rr[q] != ({T})0;" if p.out.dtype == N.RT_BOOL
          else f"(({oct_}*)p.out.ptr)[oo[q]] = ({oct_})rr[q];")
    del store
    return f"""#include "common.cuh"
extern "C" __global__ void __launch_bounds__(256) {name}(const __grid_constant__ rt_ew_params p) {{
  for (long long b0 = (long long)blockIdx.x * {256 * U} + threadIdx.x; b0 < {total}LL;
       b0 += (long long)gridDim.x * {256 * U}) {{
    {T} rr[{U}];
    long long oo[{U}];
#pragma unroll
    for (int q = 0; q < {U}; ++q) {{
      const long long flat = b0 + q * 256LL;
      oo[q] = -1;
      if (flat >= {total}LL) continue;
      {dec_s}
      {T} {regs};
      long long {iregs};
      {T} res = ({T})0;
      (void)n0;
      {body}
    Lend:
      rr[q] = res;
      oo[q] = {out_off};
    }}
#pragma unroll
    for (int q = 0; q < {U}; ++q)
      if (oo[q] >= 0) {st}
  }}
}}
"""


def _env_fold(base, coefs):
    terms = [base] + [f"env[{e}]*{_lit(c)}" for e, c in enumerate(coefs) if c]
    return " + ".join(terms)


def loop_source(lp, ops, name, info=None):
    """A persistent loop kernel with the op sequence specialised: EW bodies
    straight-line, GEMM/UDF/RNG as single template instantiations.  With
    info["pair"] the kernel runs as 2-CTA clusters and that GEMM keeps its
    weights resident (one K-half per CTA, _gemm_pair_literal)."""
    pair = (info or {}).get("pair")
    fwd = _forward_pairs(lp, ops, info) if FORWARD_ENABLED and pair is None else set()
    ew_fwd = _ew_forward_pairs(lp, ops) if FORWARD_ENABLED and pair is None else set()
    fwd |= ew_fwd
    xfwd = _gemm_ew_forwards(lp, ops, info) if pair is None else {}
    xu = _ew_udf_forwards(lp, ops, info) if pair is None else {}
    xc = _udf_ew_carries(lp, ops, info) if pair is None else {}
    xc_src = {}
    for e_, (k_, u_, j_, off_) in xc.items():
        xc_src.setdefault(u_, {})[j_] = off_
    xu_src = {}
    for u_, m_ in xu.items():
        for k_, (e_, off_) in m_.items():
            xu_src.setdefault(e_, []).append(off_)
    xfwd_src = {g: e for e, (_k, g) in xfwd.items()}
    parts, step_pre, pair_pre_bias = [], [], []
    n_gemm = n_xpf = 0
    for i, (kernel, p, re, f64, noise, soff) in enumerate(ops):
        if pair is not None and i == pair["op"]:
            parts.append(_gemm_pair_literal(lp, p, soff, pair))
            parts.append("    __syncthreads();")
            parts.append(f"    if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) {{ long long c1 = clock64(); "
                         f"((long long*)p.prof)[{i}] += c1 - c0; c0 = c1; }}")
            continue
        if kernel == N.RT_K_EW:
            nd = p.box.nd
            ext = [p.box.ext[j] for j in range(nd)]
            T = "double" if p.f64 else "float"
            bases = []
            for k in range(p.nin):
                v = p.in_[k]
                bases.append(f"const long long b{k} = " + _env_fold(
                    f"p.in[{k}].off", [v.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
                for c in range(v.nchk):
                    bases.append(f"const long long c{k}_{c} = " + _env_fold(
                        f"p.in[{k}].chk_c0[{c}]", [v.chk_env[c][e] for e in range(N.RT_MAXENV)]) + ";")
            bases.append("const long long bo = " + _env_fold(
                "p.out.off", [p.out.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
            ov = None
            if i in xfwd and not p.f64:
                kx = xfwd[i][0]
                ov = {kx: f"lds1(smem_u32(smem + {info['xfwd_off']}) + (uint32_t)((int)(flat - r0 * {re}LL) * 4), 0.f)"}
            if i in xc and not p.f64:
                kc_, _u, _j, off_c = xc[i]
                ov = dict(ov or {})
                offc = _offset_expr(f"b{kc_}", p.in_[kc_], nd)
                ov[kc_] = (f"(t == T0_ ? ((const float*)p.in[{kc_}].ptr)[{offc}] : lds1(smem_u32(smem + {off_c}) + "
                           f"(uint32_t)((int)(flat - r0 * {re}LL) * 4), 0.f))")
            # operands no loop op writes (pre-drawn normals): staged one step
            # ahead by cp.async; the first step reads them from global
            pf_pre, pf_post = "", ""
            # (time-varying ones only; each (op, operand) its own slot row)
            xpf = [k for k in ((info or {}).get("ext_in") or {}).get(i, [])
                   if EW_PREFETCH and not p.f64 and p.in_[k].dtype == N.RT_F32 and not p.in_[k].nchk
                   and p.in_[k].off_env[lp.slot] != 0 and (ov is None or k not in ov)]
            xpf = xpf[:max(0, XPF_SLOTS - n_xpf)]
            if xpf and (info or {}).get("xpf_off") and lp.rows_per_cta * re <= 256 and pair is None:
                ov = dict(ov or {})
                t_first, t_stop = "T0_", "T1_"   # (the op's own `p` shadows the loop's)
                cmp_ = "<" if lp.step > 0 else ">"
                for si0, k in enumerate(xpf):
                    si = n_xpf + si0
                    v = p.in_[k]
                    off = _offset_expr(f"b{k}", v, nd)
                    slot = (f"smem_u32(smem + {info['xpf_off']}) + (uint32_t)(({si * 256} + "
                            f"(int)(flat - r0 * {re}LL)) * 4)")
                    ov[k] = f"(t == {t_first} ? ((const float*)p.in[{k}].ptr)[{off}] : lds1({slot}, 0.f))"
                    step_off = v.off_env[lp.slot] * lp.step
                    pf_post += (f"\n        if (t + {lp.step}LL {cmp_} {t_stop}) cp_async4({slot}, "
                                f"(const float*)p.in[{k}].ptr + ({off} + {step_off}LL));")
                n_xpf += len(xpf)
                pf_pre = f"if (t != {t_first}) cp_async_wait_all();"
                pf_post += "\n        cp_async_commit();"
            lines = _program_lines(p, T, nd, base=lambda k: f"b{k}",
                                   chk=lambda k, c: f"c{k}_{c}", env="env", load_override=ov)
            regs = ", ".join(f"v{j}" for j in range(8))
            iregs = ", ".join(f"n{j}" for j in range(8))
            body = "\n        ".join(lines)
            fwd_st = ""
            for off_ in xu_src.get(i, []):
                fwd_st += (f"\n        sts1(smem_u32(smem + {off_}) + (uint32_t)((int)(flat - r0 * {re}LL) * 4), "
                           f"(float)res);")
            if (i, i + 1) in ew_fwd:
                mrp_n = (lp.rows_per_cta * ops[i + 1][2] + 3) // 4 * 4
                fwd_st += (f"\n        {{ const int lf = (int)(flat - r0 * {re}LL); "
                          f"sts1(sA32 + (uint32_t)(((lf % {re}) * {mrp_n} + lf / {re}) * 4), (float)res); }}")
            dec = "\n        ".join(_decompose(nd, ext))
            bl = "\n      ".join(bases)
            parts.append(f"""    {{  // op {i}: elementwise
      const rt_ew_params& p = *(const rt_ew_params*)(smem + {soff});
      {bl}
      for (long long flat = r0 * {re}LL + threadIdx.x; flat < r1 * {re}LL; flat += blockDim.x) {{
        {pf_pre}
        {dec}
        {T} {regs};
        long long {iregs};
        {T} res = ({T})0;
        (void)n0;
        {body}
      Lend{i}:
        {_store(p, T, nd, "bo")}{fwd_st}{pf_post}
      }}
    }}""".replace("goto Lend;", f"goto Lend{i};").replace("L", "L") .replace(
                "goto L", f"goto X{i}L").replace(f"goto X{i}Lend{i}", f"goto Lend{i}"))
            # labels of this op are renamed to keep them unique per op
            parts[-1] = _rename_labels(parts[-1], i)
        elif kernel == N.RT_K_GEMM:
            nparts = len(parts)
            hy = (info or {}).get("hybrid")
            if hy is not None and hy["op"] == i:
                parts.append(_gemm_literal(lp, p, re, f64, soff, False, 0, (i - 1, i) in fwd,
                                           (i, i + 1) in fwd, hybrid=hy))
            else:
                parts.append(_gemm_call(lp, p, re, f64, soff, fwd_in=(i - 1, i) in fwd,
                                        fwd_out=(i, i + 1) in fwd,
                                        resident=((info or {}).get("resident") or {}).get(i),
                                        split_red=None if hy is None or hy["ncol"] != 2 else hy["red"],
                                        ew_fwd=(info or {}).get("xfwd_off") if i in xfwd_src else None))
            if GEMM_PHASES and n_gemm < 5:
                for mk, j in (("/*PHASE_A*/", 0), ("/*PHASE_C*/", 1)):
                    parts[-1] = parts[-1].replace(
                        mk, f"if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) {{ long long c1 = clock64(); "
                            f"((long long*)p.prof)[{len(ops)} + {3 * n_gemm + j}] += c1 - c0; c0 = c1; }}")
            n_gemm += 1
            boff_s = ((info or {}).get("bias_smem") or {}).get(i)
            if boff_s is not None and len(parts) == nparts + 1:
                bn = _gbox_off(p.N, [p.bias.s2[d] for d in range(4)], "n")
                T_ = "double" if f64 else "float"
                parts[-1] = parts[-1].replace(
                    f"Bp_[boff + {bn}]",
                    f"lds1(smem_u32(smem + {boff_s}) + (uint32_t)(n) * {8 if f64 else 4}u, ({T_})0)")
                env_bias = _env_terms([p.bias.off_env[e] for e in range(N.RT_MAXENV)])
                pair_pre_bias.append(f"""
  {{  // loop-invariant bias of op {i}
    const rt_gemm_params& q = *(const rt_gemm_params*)(smem + {soff});
    const {T_}* Bp_ = (const {T_}*)q.bias.ptr; const long long boff = q.bias.off{env_bias};
    for (long long n = threadIdx.x; n < {p.n}; n += blockDim.x) sts1(smem_u32(smem + {boff_s}) + (uint32_t)(n) * {8 if f64 else 4}u, Bp_[boff + {bn}]);
  }}""")
        elif kernel == N.RT_K_UDF:
            if noise:
                nz_off = (info or {}).get("nz_off")
                pf = _udf_prefetch(lp, p, i, nz_off) if UDF_PREFETCH and nz_off and \
                    _nz_row(p) * 8 * 8 <= (info or {}).get("nz_bytes", 0) else None
                if pf is not None:
                    step_pre.append("    " + pf[0])
                t1s = "T1_"
                parts.append(_udf_literal(p, i, soff, noise, prefetched=None if pf is None else
                                          (nz_off, pf[1], lp.step, t1s), staged=xu.get(i),
                                          carry=xc_src.get(i)))
            else:
                parts.append(f"""    udf_op(*(const rt_udf_params*)(smem + {soff}), ops[{i}], env, r0, r1, t);""")
        elif kernel == N.RT_K_RNG:
            parts.append(f"""    rng_op(*(const rt_rng_params*)(smem + {soff}), env, r0, r1);""")
        else:
            raise ValueError("unsupported op in loop JIT")
        parts.append("    __syncthreads();")
        parts.append(f"    if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) {{ long long c1 = clock64(); "
                     f"((long long*)p.prof)[{i}] += c1 - c0; c0 = c1; }}")
    body = "\n".join(parts)
    cmp = "<" if lp.step > 0 else ">"
    # a time-blocked loop takes its range from the launch (prepare() folds
    # the block index from env); otherwise the range is a literal
    t0, t1 = ("p.start", "p.stop") if lp.blk_len else (f"{lp.start}LL", f"{lp.stop}LL")
    early, pair_pro = "  if (r0 >= r1) return;", ""
    for ri_op, roff in ((info or {}).get("resident") or {}).items():
        q = ops[ri_op][1]
        env_b = _env_terms([q.B.off_env[e] for e in range(N.RT_MAXENV)])
        pair_pro += f"""
  {{  // resident weights of op {ri_op}
    const rt_gemm_params& q = *(const rt_gemm_params*)(smem + {ops[ri_op][5]});
    const float4* Bg = reinterpret_cast<const float4*>((const float*)q.B.ptr + (q.B.off{env_b}));
    const uint32_t sB = smem_u32(smem + {roff});
    for (int i = threadIdx.x; i < {q.k * q.n // 4}; i += blockDim.x) sts4(sB + 16u * (uint32_t)i, __ldg(Bg + i));
  }}
  __syncthreads();"""
    bias_pro = "".join(pair_pre_bias) + "\n  __syncthreads();" if pair_pre_bias else ""
    hy = (info or {}).get("hybrid")
    if hy is not None:
        q = ops[hy["op"]][1]
        kr = hy["kr"]
        env_b = _env_terms([q.B.off_env[e] for e in range(N.RT_MAXENV)])
        nc, n_ = hy["ncol"], q.n
        kp = q.k // nc
        krp, ks = kr // nc, q.k // nc - kr // nc
        pair_pro += f"""
  // on-chip weights of op {hy["op"]}: part p = tid / {n_ // nc} owns k rows [p*{kp}, (p+1)*{kp}),
  // the first {krp} of them in registers (NCOL = {nc} columns per thread), the rest in smem
  float wreg[{nc}][{krp}];
  {{
    const rt_gemm_params& q = *(const rt_gemm_params*)(smem + {ops[hy["op"]][5]});
    const float* Bg = (const float*)q.B.ptr + (q.B.off{env_b});
    const int part = threadIdx.x / {n_ // nc}, c0 = {nc} * (threadIdx.x % {n_ // nc});
    #pragma unroll
    for (int k = 0; k < {krp}; ++k)
      #pragma unroll
      for (int j = 0; j < {nc}; ++j)   // (an opaque load: the compiler may not re-load it per step)
        asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(wreg[j][k]) : "l"(Bg + (part * {kp} + k) * {n_} + c0 + j));
    const uint32_t sB = smem_u32(smem + {hy["off"]});
    for (int i = threadIdx.x; i < {nc * ks * n_ // 4}; i += blockDim.x) {{
      const int row = i / {n_ // 4}, p2 = row / {max(ks, 1)}, kk = row % {max(ks, 1)};
      sts4(sB + 16u * (uint32_t)i, __ldg(reinterpret_cast<const float4*>(Bg + (p2 * {kp} + {krp} + kk) * {n_}) + i % {n_ // 4}));
    }}
  }}
  __syncthreads();"""
    if pair is not None:
        # both CTAs of a pair take part in every cluster barrier, even one
        # without rows (the grid is padded to an even CTA count)
        early = "  const long long r1c = r1 > r0 ? r1 : r0; (void)r1c;"
        pair_pro = _pair_prologue(lp, ops[pair["op"]][1], ops[pair["op"]][5], pair)
    per_sm = (info or {}).get("ctas_per_sm", 1)
    return f"""#include "loop_lib.cuh"
extern "C" __global__ void __launch_bounds__(256, {per_sm}) {name}(const __grid_constant__ rt_loop_params p) {{
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[RING];
  long long env[RT_MAXENV];
  for (int e = 0; e < RT_MAXENV; ++e) env[e] = p.h.env[e];
  const long long r0 = (long long)blockIdx.x * {lp.rows_per_cta}LL;
  const long long r1 = r0 + {lp.rows_per_cta}LL < {lp.rows}LL ? r0 + {lp.rows_per_cta}LL : {lp.rows}LL;
{early}
  const rt_loop_op* ops = (const rt_loop_op*)p.ops;
  unsigned char* sA = smem + p.a_off;
  const uint32_t sA32 = smem_u32(sA);
  loop_ring ring;
  loop_prologue(p, smem, bars, ring);
  (void)sA32;
{bias_pro}
{pair_pro}
  long long c0 = clock64();
  const long long T0_ = {t0}, T1_ = {t1};   // loop range (ops name their own params `p`)
  (void)T0_; (void)T1_;
  for (long long t = {t0}; t {cmp} {t1}; t += {lp.step}LL) {{
    env[{lp.slot}] = t;
{chr(10).join(step_pre)}
{body}
  }}
}}
"""


def _pair_prologue(lp, q, soff, pair):
    """Load this CTA's K-half of the pair GEMM's weights into shared memory
    (once: the weights do not move with the loop dim)."""
    kh, n = pair["kh"], q.n
    env_b = _env_terms([q.B.off_env[e] for e in range(N.RT_MAXENV)])
    return f"""  {{  // pair GEMM: resident K-half of B
    const rt_gemm_params& q = *(const rt_gemm_params*)(smem + {soff});
    const float* Bg = (const float*)q.B.ptr + (q.B.off{env_b}) + (long long)cluster_rank() * {kh * n}LL;
    const uint32_t pB = smem_u32(smem + {pair["b_off"]});
    for (int i = threadIdx.x; i < {kh * n // 4}; i += blockDim.x)
      sts4(pB + 16u * (uint32_t)i, __ldg(reinterpret_cast<const float4*>(Bg) + i));
  }}
  __syncthreads();"""


def _gemm_pair_literal(lp, q, soff, pair):
    """One in-loop GEMM C = act(A B + bias) on a 2-CTA cluster: each CTA holds
    B[k-half] in shared memory, computes partial sums over its half for its
    own rows AND its partner's rows (the partner's A k-half is read through
    DSMEM), hands the partner's partials over, and finishes its own rows."""
    K, Nn, kh = q.k, q.n, pair["kh"]
    mrp = (lp.rows_per_cta + 3) // 4 * 4
    env_a = _env_terms([q.A.off_env[e] for e in range(N.RT_MAXENV)])
    env_c = _env_terms([q.C.off_env[e] for e in range(N.RT_MAXENV)])
    env_bias = _env_terms([q.bias.off_env[e] for e in range(N.RT_MAXENV)])
    a_m = _gbox_off(q.M, [q.A.s1[d] for d in range(4)], "m")
    c_m = _gbox_off(q.M, [q.C.s1[d] for d in range(4)], "m")
    a_k = _gbox_off(q.K, [q.A.s2[d] for d in range(4)], "k")
    c_n = _gbox_off(q.N, [q.C.s2[d] for d in range(4)], "n")
    bias_n = _gbox_off(q.N, [q.bias.s2[d] for d in range(4)], "n")
    has_bias = bool(q.bias.ptr)
    tanh = q.epilogue == 1
    bias = f"Bp_[boff + {bias_n}]" if has_bias else "0.f"
    act = "v = vm_tanh<float>(v);" if tanh else ""
    lines = [
        f"const rt_gemm_params& q = *(const rt_gemm_params*)(smem + {soff});",
        f"const float* Ap = (const float*)q.A.ptr; const long long aoff = q.A.off{env_a};",
        f"float* Cp = (float*)q.C.ptr; const long long coff = q.C.off{env_c};",
        "const long long m0 = r0; const int mr = (int)(r1 > r0 ? r1 - r0 : 0);",
        (f"const float* Bp_ = (const float*)q.bias.ptr; const long long boff = q.bias.off{env_bias};"
         if has_bias else ""),
        f"for (int i = threadIdx.x; i < {mrp * K}; i += blockDim.x) {{ const int r = i / {K}; "
        f"const long long k = i - r * {K}; const long long m = m0 + r; "
        f"sts1(sA32 + (uint32_t)((k * {mrp} + r) * 4), r < mr ? Ap[aoff + {a_m} + {a_k}] : 0.f); }}",
        "__syncthreads();",
        "PHASE(0);",
        "cluster_sync_all();                     // partner's rows are staged",
        "PHASE(1);",
        "const uint32_t me = cluster_rank(), pr = me ^ 1u;",
        f"const uint32_t kb = me * {kh}u;",
        f"const uint32_t pA = smem_u32(smem + {pair['pa_off']}), pB = smem_u32(smem + {pair['b_off']}), "
        f"pP = smem_u32(smem + {pair['p_off']});",
        "const uint32_t rA = dsmem_map(sA32, pr);",
        f"for (int i = threadIdx.x; i < {kh * mrp // 4}; i += blockDim.x) "
        f"sts4(pA + 16u * (uint32_t)i, dsmem_ld4(rA + kb * {mrp * 4}u + 16u * (uint32_t)i));",
        "__syncthreads();",
        f"float ao[{mrp}], ap[{mrp}];",
        f"#pragma unroll\nfor (int r = 0; r < {mrp}; ++r) {{ ao[r] = 0.f; ap[r] = 0.f; }}",
        f"const int col = threadIdx.x < {Nn} ? (int)threadIdx.x : {Nn - 1};",
        "PHASE(2);",
        f"pair_core<{mrp}, {kh}, {Nn}>(sA32 + kb * {mrp * 4}u, pA, pB, col, ao, ap);",
        "__syncthreads(); PHASE(3);",
        f"if (threadIdx.x < {Nn}) {{\n#pragma unroll\n  for (int r = 0; r < {mrp}; ++r) "
        f"sts1(pP + (uint32_t)((r * {Nn} + col) * 4), ap[r]); }}",
        "__syncthreads();",
        "PHASE(4);",
        "cluster_sync_all();                     // partner's partials for my rows",
        "PHASE(5);",
        "const uint32_t rP = dsmem_map(pP, pr);",
        f"if (threadIdx.x < {Nn}) {{ const long long n = threadIdx.x; const float bias = {bias};",
        f"  #pragma unroll\n  for (int r = 0; r < {mrp}; ++r) {{ if (r >= mr) break; const long long m = m0 + r;",
        f"    float v = (ao[r] + dsmem_ld(rP + (uint32_t)((r * {Nn} + col) * 4))) + bias; {act}",
        f"    Cp[coff + {c_m} + {c_n}] = v; }}",
        "}",
    ]
    ph = ("#define PHASE(k) if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) "
          f"{{ long long c1 = clock64(); ((long long*)p.prof)[{pair['nops']} + (k)] += c1 - c0; c0 = c1; }}"
          if PHASES else "#define PHASE(k)")
    lines.insert(0, ph)
    lines.append("#undef PHASE")
    return "    {  // gemm (CTA pair, resident weights)\n      " + "\n      ".join(
        x for x in lines if x) + "\n    }"


def _env_terms(coefs):
    return "".join(f" + env[{e}]*{_lit(c)}" for e, c in enumerate(coefs) if c)


def _gbox_off(gb, strides, var):
    """Offset expression of flat index `var` decomposed over gbox gb."""
    nd = gb.nd
    if nd == 0:
        return "0LL"
    terms, rem = [], var
    for d in reversed(range(nd)):
        e, st = gb.ext[d], strides[d]
        if d == 0:
            if st:
                terms.append(f"({rem})*{_lit(st)}")
        else:
            if st:
                terms.append(f"(({rem}) % {e}LL)*{_lit(st)}")
            rem = f"(({rem}) / {e}LL)"
    return " + ".join(terms) if terms else "0LL"


def _epi_rows(mrp, tanh):
    """v[r] = act(acc[j][r] + bias) for the padded rows of a loop GEMM
    epilogue; rows >= mr are zeroed by a select (no branch around the
    activation, so the rows' tanh chains interleave)."""
    if tanh and FAST_TANH:
        return (f"  #pragma unroll\n  for (int r = 0; r < {mrp}; ++r) {{ const float x_ = tanh_fast(acc[j][r] + bias); "
                "v[r] = r < mr ? x_ : 0.f; }")
    act = " v[r] = vm_tanh<float>(v[r]);" if tanh else ""
    return (f"  #pragma unroll\n  for (int r = 0; r < {mrp}; ++r) {{ v[r] = 0.f; if (r < mr) {{ v[r] = acc[j][r] + bias;"
            + act + " } }")


def _split_epilogue(mrp, tanh, has_bias, bias_n, c_m, c_n, fwd_out):
    """Epilogue after hyb_core<..., SPLIT>: thread t of part p = t / 128
    holds columns 2 (t % 128) + {0, 1} of rows [4p, 4p + 4) in acc[j][0..3]."""
    act = "tanh_fast(acc[j][rr] + bias)" if tanh and FAST_TANH else \
        ("vm_tanh<float>(acc[j][rr] + bias)" if tanh else "acc[j][rr] + bias")
    lines = ["{ const int part_ = (int)threadIdx.x / 128; const int rlo = part_ * 4;",
             "#pragma unroll\nfor (int j = 0; j < 2; ++j) {",
             "  const long long n = 2 * (long long)(threadIdx.x % 128) + j;",
             "  const float bias = " + (f"Bp_[boff + {bias_n}];" if has_bias else "0.f;"),
             "  float v[4];",
             f"  #pragma unroll\n  for (int rr = 0; rr < 4; ++rr) {{ const float x_ = {act}; v[rr] = rlo + rr < mr ? x_ : 0.f; }}",
             "  #pragma unroll\n  for (int rr = 0; rr < 4; ++rr) { if (rlo + rr >= mr) break; const long long m = m0 + rlo + rr;",
             f"    Cp[coff + {c_m} + {c_n}] = v[rr]; }}"]
    if fwd_out:
        lines.append(f"  sts4(sA32 + (uint32_t)((n * {mrp} + rlo) * 4), make_float4(v[0], v[1], v[2], v[3]));")
    lines.append("} }")
    return lines


def _gemm_literal(lp, q, re, f64, soff, tma, kc=0, fwd_in=False, fwd_out=False, resident=None,
                  hybrid=None, split_red=None, ew_fwd=None):
    """Fully specialised loop GEMM: shapes, strides and decompositions baked,
    descriptor pointers read once into registers."""
    T = "double" if f64 else "float"
    mrp = (lp.rows_per_cta * re + 3) // 4 * 4
    K, Nn = q.k, q.n
    nc = (Nn + 255) // 256
    env_a = _env_terms([q.A.off_env[e] for e in range(N.RT_MAXENV)])
    env_b = _env_terms([q.B.off_env[e] for e in range(N.RT_MAXENV)])
    env_c = _env_terms([q.C.off_env[e] for e in range(N.RT_MAXENV)])
    env_bias = _env_terms([q.bias.off_env[e] for e in range(N.RT_MAXENV)])
    a_m = _gbox_off(q.M, [q.A.s1[d] for d in range(4)], "m")
    c_m = _gbox_off(q.M, [q.C.s1[d] for d in range(4)], "m")
    a_k = _gbox_off(q.K, [q.A.s2[d] for d in range(4)], "k")
    c_n = _gbox_off(q.N, [q.C.s2[d] for d in range(4)], "n")
    bias_n = _gbox_off(q.N, [q.bias.s2[d] for d in range(4)], "n")
    has_bias = bool(q.bias.ptr)
    tanh = q.epilogue == 1
    lines = [f"const rt_gemm_params& q = *(const rt_gemm_params*)(smem + {soff});",
             f"const {T}* Ap = (const {T}*)q.A.ptr; const long long aoff = q.A.off{env_a};",
             f"{T}* Cp = ({T}*)q.C.ptr; const long long coff = q.C.off{env_c};",
             f"const long long m0 = r0 * {re}LL; const int mr = (int)((r1 - r0) * {re}LL);"]
    if has_bias:
        lines.append(f"const {T}* Bp_ = (const {T}*)q.bias.ptr; const long long boff = q.bias.off{env_bias};")
    if hybrid is not None:
        lines.append(f"const uint32_t sB = smem_u32(smem + {hybrid['off']});   // on-chip weights (rows >= KR)")
    elif resident is not None:
        lines.append(f"const uint32_t sB = smem_u32(smem + {resident});   // resident weights")
    elif tma:
        lines.append(f"const {T}* Bg = (const {T}*)q.B.ptr + (q.B.off{env_b});")
        lines.append(f"tma_prefetch<{T}, {K}, {Nn}, {kc}>(Bg, ring);")
    else:
        b_k = _gbox_off(q.K, [q.B.s1[d] for d in range(4)], "k")
        b_n = _gbox_off(q.N, [q.B.s2[d] for d in range(4)], "n")
        lines.append(f"const {T}* Bq = (const {T}*)q.B.ptr; const long long bqo = q.B.off{env_b};")
        lines.append(f"const uint32_t sB = smem_u32(ring.buf);")
        lines.append(f"for (int i = threadIdx.x; i < {K * Nn}; i += blockDim.x) {{ const long long k = i / {Nn}, n = i % {Nn}; "
                     f"sts1(sB + (uint32_t)(i * sizeof({T})), Bq[bqo + {b_k} + {b_n}]); }}")
    if not fwd_in:
        lines.append(f"for (int i = threadIdx.x; i < {mrp * K}; i += blockDim.x) {{ const int r = i / {K}; "
                     f"const long long k = i - r * {K}; const long long m = m0 + r; "
                     f"sts1(sA32 + (uint32_t)((k * {mrp} + r) * sizeof({T})), r < mr ? Ap[aoff + {a_m} + {a_k}] : ({T})0); }}")
        lines.append("__syncthreads();")
    else:
        # A rows forwarded in shared memory by the previous op's epilogue (the
        # barrier still orders this op's own shared-memory weight loads)
        lines.append("__syncthreads();")
    fwd_store = (f" sts1(sA32 + (uint32_t)((n * {mrp} + r) * sizeof({T})), v);" if fwd_out else "")
    if hybrid is not None:
        kr, nc = hybrid["kr"], hybrid["ncol"]
        red = f"smem_u32(smem + {hybrid['red']})" if nc > 1 else "0u"
        lines.append(f"float acc[{nc}][{mrp}];")
        lines.append(f"#pragma unroll\nfor (int j = 0; j < {nc}; ++j) {{\n#pragma unroll\nfor (int r = 0; r < {mrp}; ++r) acc[j][r] = 0.f; }}")
        if SPLIT_EPI and nc == 2 and mrp == 8 and Nn == 256:
            lines.append("/*PHASE_A*/")
            lines.append(f"hyb_core<{mrp}, {K}, {Nn}, {nc}, {kr // nc}, true>(wreg, sB, sA32, {red}, acc);")
            lines.append("/*PHASE_C*/")
            lines += _split_epilogue(mrp, tanh, has_bias, bias_n, c_m, c_n, fwd_out)
            return "    {  // gemm (specialised)\n      " + "\n      ".join(lines) + "\n    }"
        lines.append("/*PHASE_A*/")
        lines.append(f"hyb_core<{mrp}, {K}, {Nn}, {nc}, {kr // nc}>(wreg, sB, sA32, {red}, acc);")
        lines.append("/*PHASE_C*/")
        if fwd_out:
            lines.append("__syncthreads();   // every thread is done reading A before it is overwritten")
        lines += [f"if ((int)threadIdx.x < {Nn // nc}) {{",
                  f"#pragma unroll\nfor (int j = 0; j < {nc}; ++j) {{",
                  f"  const long long n = {nc} * (long long)threadIdx.x + j;",
                  f"  const float bias = " + (f"Bp_[boff + {bias_n}];" if has_bias else "0.f;"),
                  f"  float v[{mrp}];",
                  _epi_rows(mrp, tanh),
                  f"  #pragma unroll\n  for (int r = 0; r < {mrp}; ++r) {{ if (r >= mr) break; const long long m = m0 + r;",
                  f"    Cp[coff + {c_m} + {c_n}] = v[r]; }}"]
        if fwd_out:
            lines.append(f"  #pragma unroll\n  for (int r = 0; r < {mrp}; r += 4) sts4(sA32 + (uint32_t)((n * {mrp} + r) * 4), "
                         f"make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]));")
        lines.append("} }")
    elif resident is not None and split_red is not None and SPLIT_EPI and not f64 and Nn == 256 \
            and mrp == 8 and K % 2 == 0:
        lines.append("float acc[2][8];")
        lines.append("#pragma unroll\nfor (int j = 0; j < 2; ++j) {\n#pragma unroll\nfor (int r = 0; r < 8; ++r) acc[j][r] = 0.f; }")
        lines.append("float wdum_[2][1];")
        lines.append("/*PHASE_A*/")
        lines.append(f"hyb_core<8, {K}, 256, 2, 0, true>(wdum_, sB, sA32, smem_u32(smem + {split_red}), acc);")
        lines.append("/*PHASE_C*/")
        lines += _split_epilogue(mrp, tanh, has_bias, bias_n, c_m, c_n, fwd_out)
    elif resident is not None and Nn >= 16:
        nc2 = 2 if Nn % 2 == 0 and Nn <= 512 else 1
        lines.append(f"float acc[{nc2}][{mrp}];")
        lines.append(f"#pragma unroll\nfor (int j = 0; j < {nc2}; ++j) {{\n#pragma unroll\nfor (int r = 0; r < {mrp}; ++r) acc[j][r] = 0.f; }}")
        lines.append("/*PHASE_A*/")
        lines.append(f"res_core<{mrp}, {K}, {Nn}, {nc2}>(sB, sA32, acc);")
        lines.append("/*PHASE_C*/")
        lines += [f"if ((int)threadIdx.x < {-(-Nn // nc2)}) {{",
                  f"#pragma unroll\nfor (int j = 0; j < {nc2}; ++j) {{",
                  f"  const long long n = {nc2} * (long long)threadIdx.x + j; if (n >= {Nn}) break;",
                  f"  const float bias = " + (f"Bp_[boff + {bias_n}];" if has_bias else "0.f;"),
                  f"  float v[{mrp}];",
                  _epi_rows(mrp, tanh),
                  f"  #pragma unroll\n  for (int r = 0; r < {mrp}; ++r) {{ if (r >= mr) break; const long long m = m0 + r;",
                  f"    Cp[coff + {c_m} + {c_n}] = v[r]; }}"]
        if fwd_out:
            lines.append(f"  #pragma unroll\n  for (int r = 0; r < {mrp}; r += 4) sts4(sA32 + (uint32_t)((n * {mrp} + r) * 4), "
                         f"make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]));")
        lines.append("} }")
    elif tma and lp.red_off and KS_ENABLED and ks_eligible(lp.rows_per_cta, re, q, f64):
        opt = mrp * Nn // 256
        lines.append(f"{T} o[{opt}];")
        lines.append(f"tma_core_ks<{T}, {mrp}, {K}, {Nn}, {kc}>(Bg, sA32, ring, smem_u32(smem + {lp.red_off}), o);")
        lines += [f"const int o0 = threadIdx.x * {opt}; const int r = o0 / {Nn};",
                  f"if (r < mr) {{ const long long m = m0 + r;",
                  f"  #pragma unroll\n  for (int q = 0; q < {opt}; ++q) {{ const long long n = (o0 % {Nn}) + q;",
                  f"    const {T} bias = " + (f"Bp_[boff + {bias_n}];" if has_bias else f"({T})0;"),
                  f"    {T} v = o[q] + bias;" + (f" v = vm_tanh<{T}>(v);" if tanh else ""),
                  f"    Cp[coff + {c_m} + {c_n}] = v; }}",
                  "}"]
    elif tma and MMA_ENABLED and not f64 and mrp == 8 and Nn % 64 == 0 and K % 8 == 0 \
            and kc % 8 == 0:
        nt = Nn // 64
        lines.append(f"float acc[{nt}][4];")
        lines.append(f"mma_core<{mrp}, {K}, {Nn}, {kc}>(Bg, sA32, ring, acc);")
        lines += ["const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;",
                  f"const int nw0 = (int)(threadIdx.x >> 5) * {Nn // 8};",
                  "if (g < mr) { const long long m = m0 + g;",
                  f"  #pragma unroll\n  for (int j = 0; j < {nt}; ++j) {{",
                  "    #pragma unroll\n    for (int h = 0; h < 2; ++h) {",
                  "      const long long n = nw0 + j * 8 + 2 * t4 + h;",
                  f"      const float bias = " + (f"Bp_[boff + {bias_n}];" if has_bias else "0.f;"),
                  "      float v = acc[j][h] + bias;" + (" v = vm_tanh<float>(v);" if tanh else ""),
                  f"      Cp[coff + {c_m} + {c_n}] = v;"
                  + (f" sts1(sA32 + (uint32_t)((n * {mrp} + g) * 4), v);" if fwd_out else "")
                  + " } }",
                  "}"]
    elif tma and CORE2_NCOL > 1 and not f64 and Nn % CORE2_NCOL == 0 and \
            Nn <= 256 * CORE2_NCOL and kc % 4 == 0 and K >= 64:
        nc2 = CORE2_NCOL
        lines.append(f"float acc[{nc2}][{mrp}];")
        lines.append(f"#pragma unroll\nfor (int j = 0; j < {nc2}; ++j) {{\n#pragma unroll\nfor (int r = 0; r < {mrp}; ++r) acc[j][r] = 0.f; }}")
        if lp.red_off and k2_eligible(lp.rows_per_cta, re, q, f64) and kc % 8 == 0:
            lines.append(f"tma_core2k<{mrp}, {K}, {Nn}, {kc}, {nc2}>(Bg, sA32, ring, "
                         f"smem_u32(smem + {lp.red_off}), acc);")
        else:
            lines.append(f"tma_core2<{mrp}, {K}, {Nn}, {kc}, {nc2}>(Bg, sA32, ring, acc);")
        # forwarded A rows: this thread's column n is A row k = n, MRP
        # contiguous floats (k-major staging), so store them as float4s
        # (scalar stores at a 2 x MRP x 4 B lane stride were 16-way conflicts)
        fwd_vec = (f"  #pragma unroll\n  for (int r = 0; r < {mrp}; r += 4) sts4(sA32 + (uint32_t)((n * {mrp} + r) * 4), "
                   f"make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]));" if fwd_out else "")
        lines += [f"if ((int)threadIdx.x < {Nn // nc2}) {{",
                  f"#pragma unroll\nfor (int j = 0; j < {nc2}; ++j) {{",
                  f"  const long long n = {nc2} * (long long)threadIdx.x + j;",
                  f"  const float bias = " + (f"Bp_[boff + {bias_n}];" if has_bias else "0.f;"),
                  f"  float v[{mrp}];",
                  _epi_rows(mrp, tanh),
                  f"  #pragma unroll\n  for (int r = 0; r < {mrp}; ++r) {{ if (r >= mr) break; const long long m = m0 + r;",
                  f"    Cp[coff + {c_m} + {c_n}] = v[r]; }}",
                  fwd_vec,
                  "} }"]
    elif tma:
        lines.append(f"{T} acc[{nc}][{mrp}];")
        lines.append(f"#pragma unroll\nfor (int j = 0; j < {nc}; ++j) {{\n#pragma unroll\nfor (int r = 0; r < {mrp}; ++r) acc[j][r] = ({T})0; }}")
        lines.append(f"tma_core<{T}, {mrp}, {nc}, {K}, {Nn}, {kc}>(Bg, sA32, ring, acc);")
        epi = [f"#pragma unroll\nfor (int j = 0; j < {nc}; ++j) {{",
               f"  const long long n = threadIdx.x + j * 256LL; if (n >= {Nn}) break;",
               f"  const {T} bias = " + (f"Bp_[boff + {bias_n}];" if has_bias else f"({T})0;"),
               f"  #pragma unroll\n  for (int r = 0; r < {mrp}; ++r) {{ if (r >= mr) break; const long long m = m0 + r;",
               f"    {T} v = acc[j][r] + bias;" + (f" v = vm_tanh<{T}>(v);" if tanh else ""),
               f"    Cp[coff + {c_m} + {c_n}] = v;{fwd_store} }}",
               "}"]
        lines += epi
    else:
        outs = mrp * Nn
        g0 = 256 // outs
        G = max(x for x in (1, 2, 4, 8, 16, 32) if x <= max(1, g0))
        lines += [f"const int lane_in = threadIdx.x % {G};",
                  f"for (int base = 0; base < {outs}; base += {256 // G}) {{",
                  f"  const int o = base + (int)threadIdx.x / {G};",
                  f"  const bool act = o < {outs} && (o / {Nn}) < mr;",
                  f"  const int r = act ? o / {Nn} : 0; const long long n = act ? o % {Nn} : 0;",
                  f"  {T} a = ({T})0;",
                  (f"  if (act) {{\n#pragma unroll 4\n    for (int k = lane_in; k < {K}; k += {G}) a = fma(lds1(sA32 + (uint32_t)((k * {mrp} + r) * sizeof({T})), ({T})0), lds1(sB + (uint32_t)((k * {Nn} + n) * sizeof({T})), ({T})0), a); }}"
                   if K % (4 * G) or not HEAD_ILP else
                   # four partial sums: a 4x shorter dependent FMA chain
                   f"  if (act) {{ {T} a1 = ({T})0, a2 = ({T})0, a3 = ({T})0;\n#pragma unroll 2\n    for (int k = lane_in; k < {K}; k += {4 * G}) {{"
                   f" a = fma(lds1(sA32 + (uint32_t)((k * {mrp} + r) * sizeof({T})), ({T})0), lds1(sB + (uint32_t)((k * {Nn} + n) * sizeof({T})), ({T})0), a);"
                   f" a1 = fma(lds1(sA32 + (uint32_t)(((k + {G}) * {mrp} + r) * sizeof({T})), ({T})0), lds1(sB + (uint32_t)(((k + {G}) * {Nn} + n) * sizeof({T})), ({T})0), a1);"
                   f" a2 = fma(lds1(sA32 + (uint32_t)(((k + {2 * G}) * {mrp} + r) * sizeof({T})), ({T})0), lds1(sB + (uint32_t)(((k + {2 * G}) * {Nn} + n) * sizeof({T})), ({T})0), a2);"
                   f" a3 = fma(lds1(sA32 + (uint32_t)(((k + {3 * G}) * {mrp} + r) * sizeof({T})), ({T})0), lds1(sB + (uint32_t)(((k + {3 * G}) * {Nn} + n) * sizeof({T})), ({T})0), a3); }}"
                   " a = (a + a1) + (a2 + a3); }"),
                  f"  #pragma unroll\n  for (int s = {G // 2}; s > 0; s >>= 1) a += __shfl_down_sync(0xffffffffu, a, s, {G});",
                  f"  if (act && lane_in == 0) {{ const long long m = m0 + r; {T} v = a" + (f" + Bp_[boff + {bias_n}]" if has_bias else "") + ";"
                  + (f" v = vm_tanh<{T}>(v);" if tanh else "") + f" Cp[coff + {c_m} + {c_n}] = v;"
                  + (f" sts1(smem_u32(smem + {ew_fwd}) + (uint32_t)((r * {Nn} + n) * sizeof({T})), v);" if ew_fwd is not None else "")
                  + " }",
                  "}"]
    return "    {  // gemm (specialised)\n      " + "\n      ".join(lines) + "\n    }"


def _udf_prefetch(lp, p, op_index, soff_nz):
    """Pre-drawn normals of a loop env op copied to shared memory one step
    ahead (cp.async, one row per warp, one output element per lane): the
    HBM latency of step t+1's normals overlaps step t's remaining work and
    t+1's MLP, and no register scoreboard is shared with the step's other
    loads (register prefetches made unrelated loads wait on them).  Returns
    (code run at the first step, code issuing step tn's copies) or None
    when a warp has several rows or a row has more than 32 values."""
    if lp.rows_per_cta > 8 or any(p.out_count[j] > 32 for j in range(p.nout)):
        return None
    def issue(tv):
        lines = ["{ const int lane_ = threadIdx.x & 31, w_ = threadIdx.x >> 5; const long long row_ = r0 + w_;",
                 f"  const double* nzb = (const double*)ops[{op_index}].noise + ops[{op_index}].noise_off"
                 f" + row_ * ops[{op_index}].noise_row + ({tv}) * ops[{op_index}].noise_step;"]
        e0 = 0
        for j in range(p.nout):
            c = p.out_count[j]
            lines.append(f"  if (row_ < r1 && lane_ < {c}) cp_async8(smem_u32(smem + {soff_nz}) + "
                         f"(uint32_t)((w_ * {_nz_row(p)} + {e0} + lane_) * 8), nzb + {e0} + lane_);")
            e0 += c
        lines.append("  cp_async_commit(); }")
        return "\n    ".join(lines)
    first = f"if (t == T0_) {{\n    {issue('t')}\n    }}"
    return first, issue


def _nz_row(p):
    return sum(p.out_count[j] for j in range(p.nout))


def _udf_literal(p, op_index, soff, noise, prefetched=False, staged=None, carry=None):
    """Synthetic env body with counts, strides and the row decomposition baked."""
    nd = p.box.nd
    ext = [p.box.ext[j] for j in range(nd)]
    lines = [f"const rt_udf_params& q = *(const rt_udf_params*)(smem + {soff});",
             f"const double* noise = (const double*)ops[{op_index}].noise;",
             f"const long long nz0 = ops[{op_index}].noise_off; const long long nzr = ops[{op_index}].noise_row; const long long nzs = ops[{op_index}].noise_step;"]
    for k in range(p.nin):
        v = p.in_[k]
        ct = CT[v.dtype]
        lines.append(f"const {ct}* in{k} = (const {ct}*)q.in[{k}].ptr; const long long io{k} = q.in[{k}].off"
                     + _env_terms([v.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
    for j in range(p.nout):
        v = p.out[j]
        ct = CT[v.dtype]
        lines.append(f"{ct}* out{j} = ({ct}*)q.out[{j}].ptr; const long long oo{j} = q.out[{j}].off"
                     + _env_terms([v.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
    lines.append("const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;")
    lines.append("for (long long row = r0 + warp; row < r1; row += nwarps) {")
    dec = ["  unsigned int rr = (unsigned int)row;"]
    for dd in reversed(range(nd)):
        if dd == 0:
            dec.append("  const long long i0 = (long long)rr;")
        else:
            dec.append(f"  const long long i{dd} = (long long)(rr % {ext[dd]}u); rr /= {ext[dd]}u;")
    lines += dec
    lines.append(f"  double base = {repr(float(p.salt))};")
    for k in range(p.nin):
        v = p.in_[k]
        off = _offset_expr(f"io{k}", v, nd)
        if staged and k in staged:
            lines.append(f"  base = base + warp_pairwise_sum_s(smem_u32(smem + {staged[k][1]}) + (uint32_t)((row - r0) * "
                         f"{p.in_count[k] * 4}), {p.in_count[k]}, lane) / {float(p.in_count[k])!r};")
        else:
            lines.append(f"  base = base + warp_pairwise_sum((const void*)in{k}, {v.dtype}, {off}, {p.in_count[k]}LL, lane) / {float(p.in_count[k])!r};")
    lines.append("  long long nz = nz0 + row * nzr + t * nzs; (void)nz;")
    if prefetched:
        lines.append("  cp_async_wait_all();")
    for j in range(p.nout):
        v = p.out[j]
        off = _offset_expr(f"oo{j}", v, nd)
        kind = p.out_kind[j]
        if kind == N.RT_BOOL:
            expr = "((tb + z > 0.8) ? 1.0 : 0.0)"
            pre = "  const double tb = tanh(base);"
        elif kind == N.RT_I64:
            expr, pre = "floor(3.0 * tanh(base + z))", ""
        else:
            expr, pre = "tanh(base + 0.3 * z)", ""
        ct = CT[v.dtype]
        if pre:
            lines.append(pre)
        store = (f"out{j}[{off} + e] = ({expr}) != 0.0;" if v.dtype == N.RT_BOOL
                 else f"out{j}[{off} + e] = ({ct})({expr});")
        if carry and j in carry and v.dtype == N.RT_F32:
            # (the value is recomputed: numpy's double -> float32 cast, same rounding)
            store = (f"{{ const float cv_ = (float)({expr}); out{j}[{off} + e] = cv_; "
                     f"sts1(smem_u32(smem + {carry[j]}) + (uint32_t)(((row - r0) * {p.out_count[j]} + e) * 4), cv_); }}")
        if prefetched:
            e0 = sum(p.out_count[jj] for jj in range(j))
            lines.append(f"  if (lane < {p.out_count[j]}) {{ const int e = lane; const double z = lds1(smem_u32(smem + "
                         f"{prefetched[0]}) + (uint32_t)((warp * {_nz_row(p)} + {e0} + lane) * 8), 0.0); {store} }}")
        else:
            lines.append(f"  for (int e = lane; e < {p.out_count[j]}; e += 32) {{ const double z = __ldg(noise + nz + e); {store} }}")
        lines.append(f"  nz += {p.out_count[j]};")
    lines.append("}")
    if prefetched:
        # each lane re-fills only the slots it read itself, so no barrier is needed
        tn, stop = ("t + " + str(prefetched[2]) + "LL"), prefetched[3]
        lines.append(f"if ({tn} {'<' if prefetched[2] > 0 else '>'} {stop}) {prefetched[1](tn)}")
    return "    {  // env (specialised)\n      " + "\n      ".join(lines) + "\n    }"


def ks_eligible(rows_per_cta, re, q, f64):
    """In-loop GEMMs that take the K-split core (loop_lib.cuh tma_core_ks):
    fp32, N = 256 (or 128 with 8 rows), dense row-major B."""
    mrp = (rows_per_cta * re + 3) // 4 * 4
    dense_1d = q.N.nd == 1 and q.K.nd == 1 and q.Z.nd <= 1 and q.z == 1
    return (not f64 and dense_1d and mrp <= 8 and q.n in (128, 256) and q.k >= 128
            and (mrp * q.n // 256) % 4 == 0
            and q.B.s2[0] == 1 and q.B.s1[0] == q.n and q.B.dtype == N.RT_F32)


DUAL_ENABLED = os.environ.get("RTB200_LOOP_DUAL", "1") != "0"   # two loop CTAs per SM
CORE2_NCOL = int(os.environ.get("RTB200_LOOP_NCOL", "2"))   # columns per thread in-loop (1: one)
MMA_ENABLED = os.environ.get("RTB200_LOOP_MMA", "0") == "1"     # 3xTF32 mma.sync in-loop GEMMs (measured slower: 18.5k vs 15.6k cycles for h2)
PAIR_ENABLED = os.environ.get("RTB200_LOOP_PAIR", "0") == "1"   # measured: no gain at E=1024 (profiles/README.md)
PHASES = os.environ.get("RTB200_LOOP_PHASES", "0") == "1"   # clock probes inside the pair GEMM
SPLIT_EPI = os.environ.get("RTB200_LOOP_SPLIT_EPI", "1") != "0"   # 2-part cores finalise half the rows each
HEAD_ILP = os.environ.get("RTB200_LOOP_HEAD_ILP", "0") == "1"   # 4 partial sums in narrow-N loop GEMMs (measured slower)
XPF_SLOTS = 2   # staged operand rows (lower.py reserves 2 x 256 floats)
EW_PREFETCH = os.environ.get("RTB200_LOOP_EW_PREFETCH", "1") != "0"   # loop-external EW operands one step ahead
FAST_TANH = os.environ.get("RTB200_LOOP_FAST_TANH", "1") != "0"   # branch-free tanh in loop epilogues
GEMM_PHASES = os.environ.get("RTB200_LOOP_GEMM_PHASES", "0") == "1"   # staging / core / epilogue probes
KS_ENABLED = os.environ.get("RTB200_LOOP_KSPLIT", "0") == "1"   # measured slower (profiles/README.md)
K2_ENABLED = os.environ.get("RTB200_LOOP_K2", "0") == "1"   # both thread halves on N=256 layers (measured: no gain)
WIDE_RESIDENT = os.environ.get("RTB200_LOOP_WIDE_RESIDENT", "1") != "0"   # small wide layers resident when hybrid
BIAS_SMEM = os.environ.get("RTB200_LOOP_BIAS_SMEM", "1") != "0"   # loop-invariant biases in shared memory
UDF_PREFETCH = os.environ.get("RTB200_LOOP_UDF_PREFETCH", "1") != "0"   # env normals loaded at step start
HYBRID_ENABLED = os.environ.get("RTB200_LOOP_HYBRID", "1") != "0"   # widest layer's weights on chip
HYBRID_KR = int(os.environ.get("RTB200_LOOP_HYBRID_KR", "128"))   # of its K rows, in registers
HYBRID_NCOL = int(os.environ.get("RTB200_LOOP_HYBRID_NCOL", "2"))   # columns per thread = K parts


def k2_eligible(rows_per_cta, re, q, f64):
    """In-loop GEMMs that take tma_core2k (2 columns per thread, the two
    thread halves splitting every chunk's k rows): fp32, N = 256 (= 2 x 128
    threads), dense row-major B, <= 8 rows."""
    mrp = (rows_per_cta * re + 3) // 4 * 4
    dense_1d = q.N.nd == 1 and q.K.nd == 1 and q.Z.nd <= 1 and q.z == 1
    return (K2_ENABLED and CORE2_NCOL == 2 and not f64 and dense_1d and mrp <= 8 and q.n == 256
            and q.k >= 64 and q.B.s2[0] == 1 and q.B.s1[0] == q.n and q.B.dtype == N.RT_F32)


def _same_gop(a, b):
    return (a.ptr == b.ptr and a.off == b.off and a.dtype == b.dtype
            and all(a.off_env[e] == b.off_env[e] for e in range(N.RT_MAXENV)))


def _forward_pairs(lp, ops, info=None):
    """(i, i+1): GEMM op i+1 reads as its A exactly the rows GEMM op i just
    wrote as its C (h1 -> h2 -> mu of an MLP).  Op i's epilogue then also
    leaves its output in the A staging area, k-major, and op i+1 skips the
    global round trip.  Only for TMA-streamed producers (their core ends
    with a CTA barrier, so nobody still reads the producer's own A)."""
    out = set()
    for i in range(len(ops) - 1):
        (k1, p1, re1, f1, _n1, _s1), (k2, p2, re2, f2, _n2, _s2) = ops[i][:6], ops[i + 1][:6]
        if k1 != N.RT_K_GEMM or k2 != N.RT_K_GEMM or re1 != 1 or re2 != 1 or f1 or f2:
            continue
        # producers whose core ends with a CTA barrier: TMA-streamed, resident
        # (res_core) and on-chip (hybrid: barrier added before a forward)
        hy = (info or {}).get("hybrid")
        on_chip = i in ((info or {}).get("resident") or {}) or (hy is not None and hy["op"] == i)
        if (_gemm_kind(lp, p1, re1, f1) != "tma" and not on_chip) or (KS_ENABLED and lp.red_off):
            continue
        if not _same_gop(p1.C, p2.A):
            continue
        if [p1.M.ext[d] for d in range(p1.M.nd)] != [p2.M.ext[d] for d in range(p2.M.nd)] or \
                p1.M.nd != p2.M.nd or p1.n != p2.k or p1.N.nd != 1 or p2.K.nd != 1:
            continue
        if any(p1.C.s1[d] != p2.A.s1[d] for d in range(p1.M.nd)) or p1.C.s2[0] != p2.A.s2[0]:
            continue
        out.add((i, i + 1))
    return out


def _gbox_eval(gb, strides, x):
    """Python twin of _gbox_off: offset of flat index x over gbox gb."""
    off = 0
    for d in reversed(range(gb.nd)):
        e = gb.ext[d]
        if d == 0:
            off += x * strides[d]
        else:
            off += (x % e) * strides[d]
            x //= e
    return off


def _ew_forward_pairs(lp, ops):
    """(i, i+1): elementwise op i writes exactly the A rows of GEMM op i+1
    (same buffer view; element e of slab row r is A[r][e]).  Op i then also
    leaves its output in the A staging area (k-major) and the GEMM skips
    the global round trip (the observation copy feeding the first layer)."""
    out = set()
    for i in range(len(ops) - 1):
        (k1, p1, re1, f1, _n1, _s1), (k2, p2, re2, f2, _n2, _s2) = ops[i][:6], ops[i + 1][:6]
        if k1 != N.RT_K_EW or k2 != N.RT_K_GEMM or p1.f64 or f2 or re2 != 1:
            continue
        if p1.out.dtype != N.RT_F32 or p2.A.dtype != N.RT_F32 or re1 != p2.k or p2.K.nd != 1:
            continue
        if p1.out.ptr != p2.A.ptr or p1.out.off != p2.A.off or \
                any(p1.out.off_env[e] != p2.A.off_env[e] for e in range(N.RT_MAXENV)):
            continue
        nd = p1.box.nd
        ext = [p1.box.ext[d] for d in range(nd)]
        rows = lp.rows

        def ew_off(f):
            o = 0
            for d in reversed(range(nd)):
                o += (f % ext[d]) * p1.out.stride[d]
                f //= ext[d]
            return o
        s1 = [p2.A.s1[d] for d in range(4)]
        s2 = [p2.A.s2[d] for d in range(4)]
        ok = all(ew_off(r * re1 + e) == _gbox_eval(p2.M, s1, r) + _gbox_eval(p2.K, s2, e)
                 for r in sorted({0, 1, rows // 2, rows - 1}) if 0 <= r < rows
                 for e in sorted({0, 1, re1 - 1}) if 0 <= e < re1)
        if ok:
            out.add((i, i + 1))
    return out


def _gemm_ew_forwards(lp, ops, info):
    """{i + 1: (k, i)}: narrow in-loop GEMM op i (resident weights, N < 16:
    the policy head) whose output is input k of elementwise op i + 1 at the
    same (row, column) points; op i also leaves its rows in shared memory
    (info["xfwd_off"], [rows][N]) and op i + 1 reads them there instead of
    waiting on an L2 round trip."""
    out = {}
    res = (info or {}).get("resident") or {}
    if not (info or {}).get("xfwd_off") or not FORWARD_ENABLED:
        return out
    for i in range(len(ops) - 1):
        (k1, q, re1, f1, _n1, _s1), (k2, p2, re2, _f2, _n2, _s2) = ops[i][:6], ops[i + 1][:6]
        if k1 != N.RT_K_GEMM or k2 != N.RT_K_EW or f1 or p2.f64 or i not in res or q.n >= 16:
            continue
        mrp = (lp.rows_per_cta * re1 + 3) // 4 * 4
        if re1 != 1 or mrp > 8 or re2 != q.n or q.n * mrp > 8 * 32 or q.C.dtype != N.RT_F32 or \
                q.A.dtype != N.RT_F32 or (q.bias.ptr and q.bias.dtype != N.RT_F32) or q.N.nd != 1:
            continue
        nd = p2.box.nd
        ext = [p2.box.ext[d] for d in range(nd)]
        for kk in range(p2.nin):
            v = p2.in_[kk]
            if v.dtype != N.RT_F32 or v.nchk or v.ptr != q.C.ptr or v.off != q.C.off or \
                    any(v.off_env[e] != q.C.off_env[e] for e in range(N.RT_MAXENV)):
                continue

            def ew_off(f):
                o = 0
                for d in reversed(range(nd)):
                    o += (f % ext[d]) * v.stride[d]
                    f //= ext[d]
                return o
            s1 = [q.C.s1[d] for d in range(4)]
            s2 = [q.C.s2[d] for d in range(4)]
            rows = lp.rows
            if all(ew_off(r * re2 + e) == _gbox_eval(q.M, s1, r) + _gbox_eval(q.N, s2, e)
                   for r in sorted({0, 1, rows // 2, rows - 1}) if 0 <= r < rows
                   for e in range(re2)):
                out[i + 1] = (kk, i)
                break
    return out


def _ew_udf_forwards(lp, ops, info):
    """{udf op u: {input k: (ew op e, smem offset)}}: elementwise op e < u
    writes exactly env op u's input k (element j of slab row r at the
    input's row offset + j); op e also stages its rows in shared memory
    ([rows][count] floats) and the env op sums them there (the observation
    and action the synthetic env reads)."""
    out = {}
    base = (info or {}).get("xu_off")
    if not base or not FORWARD_ENABLED or lp.rows_per_cta > 8:
        return out
    cur = 0
    for u, (ku, pu, *_r) in enumerate(ops):
        if ku != N.RT_K_UDF:
            continue
        ndu = pu.box.nd
        extu = [pu.box.ext[d] for d in range(ndu)]

        def row_off(v, r):
            o = 0
            for d in reversed(range(ndu)):
                o += (r % extu[d]) * v.stride[d]
                r //= extu[d]
            return o
        for k in range(pu.nin):
            v = pu.in_[k]
            cnt = pu.in_count[k]
            if v.dtype != N.RT_F32 or cnt > 128 or cur + 8 * cnt > 512:
                continue
            for e in range(u - 1, -1, -1):
                ke, pe, re, _f, *_s = ops[e]
                if ke != N.RT_K_EW or pe.f64 or re != cnt or pe.out.dtype != N.RT_F32:
                    continue
                o = pe.out
                if o.ptr != v.ptr or o.off != v.off or \
                        any(o.off_env[x] != v.off_env[x] for x in range(N.RT_MAXENV)):
                    continue
                nd = pe.box.nd
                ext = [pe.box.ext[d] for d in range(nd)]

                def ew_off(f):
                    oo = 0
                    for d in reversed(range(nd)):
                        oo += (f % ext[d]) * o.stride[d]
                        f //= ext[d]
                    return oo
                rows = lp.rows
                if all(ew_off(r * re + j) == row_off(v, r) + j
                       for r in sorted({0, 1, rows // 2, rows - 1}) if 0 <= r < rows
                       for j in range(cnt)):
                    out.setdefault(u, {})[k] = (e, base + cur * 4)
                    cur += 8 * cnt
                    break
    return out


def _udf_ew_carries(lp, ops, info):
    """{ew op e: (input k, udf op u, output j, smem offset)}: elementwise op e
    reads at step t exactly what env op u wrote as output j at step t - step
    (the observation carried into the next step's merge).  Op u also stages
    its fp32 rows in shared memory and op e reads them there (from the second
    step of a launch on; the first reads global)."""
    out = {}
    base = (info or {}).get("xc_off")
    if not base or not FORWARD_ENABLED or lp.rows_per_cta > 8:
        return out
    slot = lp.slot
    used = 0
    for u, (ku, pu, *_r) in enumerate(ops):
        if ku != N.RT_K_UDF:
            continue
        ndu = pu.box.nd
        extu = [pu.box.ext[d] for d in range(ndu)]
        for j in range(pu.nout):
            vo = pu.out[j]
            cnt = pu.out_count[j]
            if vo.dtype != N.RT_F32 or cnt > 32 or used + 8 * cnt > 256:
                continue
            coef = vo.off_env[slot] * lp.step
            for e in range(len(ops)):
                ke, pe, re, _f, *_s = ops[e]
                if ke != N.RT_K_EW or pe.f64 or re != cnt or e >= u:
                    continue
                nd = pe.box.nd
                ext = [pe.box.ext[d] for d in range(nd)]
                for k in range(pe.nin):
                    v = pe.in_[k]
                    if v.dtype != N.RT_F32 or v.ptr != vo.ptr or v.off != vo.off - coef or \
                            any(v.off_env[x] != vo.off_env[x] for x in range(N.RT_MAXENV)):
                        continue

                    def ew_off(f, v=v, nd=nd, ext=ext):
                        oo = 0
                        for d in reversed(range(nd)):
                            oo += (f % ext[d]) * v.stride[d]
                            f //= ext[d]
                        return oo

                    def u_off(r):
                        oo = 0
                        for d in reversed(range(ndu)):
                            oo += (r % extu[d]) * vo.stride[d]
                            r //= extu[d]
                        return oo
                    rows = lp.rows
                    if all(ew_off(r * re + q) == u_off(r) + q
                           for r in sorted({0, 1, rows // 2, rows - 1}) if 0 <= r < rows
                           for q in range(cnt)):
                        out[e] = (k, u, j, base + used * 4)
                        used += 8 * cnt
                        break
                if e in out:
                    break
    return out


def _gemm_kind(lp, q, re, f64):
    it = 8 if f64 else 4
    mrp = (lp.rows_per_cta * re + 3) // 4 * 4
    stage = ((lp.smem_bytes - lp.ring_off) // 4) & ~127
    dense_1d = q.N.nd == 1 and q.K.nd == 1 and q.Z.nd <= 1 and q.z == 1
    b_dt = q.B.dtype == (N.RT_F64 if f64 else N.RT_F32)
    aligned = q.B.off % 4 == 0 and all(q.B.off_env[e] % 4 == 0 for e in range(N.RT_MAXENV))
    tdt = N.RT_F64 if f64 else N.RT_F32
    same_dt = q.A.dtype == tdt and q.C.dtype == tdt and (not q.bias.ptr or q.bias.dtype == tdt)
    if dense_1d and b_dt and mrp <= 8 and 64 <= q.n <= (256 if f64 else 512) and stage and \
            q.B.s2[0] == 1 and q.B.s1[0] == q.n and aligned and (q.n * it) % 16 == 0 and same_dt:
        return "tma"
    return "other"


FORWARD_ENABLED = os.environ.get("RTB200_LOOP_FORWARD", "1") != "0"
RESIDENT_ENABLED = os.environ.get("RTB200_LOOP_RESIDENT", "1") != "0"


def _gemm_call(lp, q, re, f64, soff, fwd_in=False, fwd_out=False, resident=None, split_red=None,
               ew_fwd=None):
    """Pick a shape-specialised GEMM body for a persistent-loop op."""
    T = "double" if f64 else "float"
    it = 8 if f64 else 4
    mrp = (lp.rows_per_cta * re + 3) // 4 * 4
    K, Nn = q.k, q.n
    stage = ((lp.smem_bytes - lp.ring_off) // 4) & ~127
    dense_1d = q.N.nd == 1 and q.K.nd == 1 and q.Z.nd <= 1 and q.z == 1
    b_dt = q.B.dtype == (N.RT_F64 if f64 else N.RT_F32)
    aligned = q.B.off % 4 == 0 and all(q.B.off_env[e] % 4 == 0 for e in range(N.RT_MAXENV))
    q_ref = f"*(const rt_gemm_params*)(smem + {soff})"
    tdt = N.RT_F64 if f64 else N.RT_F32
    same_dt = q.A.dtype == tdt and q.C.dtype == tdt and (not q.bias.ptr or q.bias.dtype == tdt)
    if resident is not None and same_dt and mrp <= 8:
        return _gemm_literal(lp, q, re, f64, soff, False, 0, fwd_in, fwd_out, resident,
                             split_red=split_red, ew_fwd=ew_fwd)
    if dense_1d and b_dt and mrp <= 8 and 64 <= Nn <= (256 if f64 else 512) and stage and \
            q.B.s2[0] == 1 and q.B.s1[0] == Nn and aligned and (Nn * it) % 16 == 0:
        kc = max(1, min(K, stage // (Nn * it)))
        if same_dt:
            return _gemm_literal(lp, q, re, f64, soff, True, kc, fwd_in, fwd_out)
        nc = 1 if Nn <= 256 else 2
        return (f"    gemm_tma_fixed<{T}, {mrp}, {nc}, {K}, {Nn}, {kc}>({q_ref}, env, r0 * {re}LL, "
                f"r1 * {re}LL, sA32, ring);")
    if dense_1d and mrp <= 8 and Nn < 64 and K * Nn * it <= 4 * stage and K * mrp * it <= 64 * 1024:
        if same_dt and q.B.dtype == q.A.dtype:
            return _gemm_literal(lp, q, re, f64, soff, False, 0, fwd_in, False)
        return (f"    gemm_small_fixed<{T}, {mrp}, {K}, {Nn}>({q_ref}, env, r0 * {re}LL, r1 * {re}LL, "
                f"sA32, smem_u32(ring.buf));")
    return f"    gemm_op<{T}>({q_ref}, env, r0 * {re}LL, r1 * {re}LL, sA, ring);"


def _rename_labels(src, i):
    import re
    src = re.sub(r"\bL(\d+):;", lambda m: f"X{i}L{m.group(1)}:;", src)
    return src


_FN_CACHE: dict = {}


def _opts():
    # -fmad=false: each elementwise op rounds like the reference's numpy ops
    # (no contraction of a*b+c across program statements)
    return [b"-arch=sm_100a", b"-std=c++17", b"-lineinfo", b"-fmad=false", b"--device-int128",
            b"-I" + os.path.join(HERE, "csrc").encode()]


def _headers_key():
    """Digest of the csrc headers JIT sources include (a header edit must not
    reuse a cubin cached for the same source text)."""
    h = hashlib.sha256()
    d = os.path.join(HERE, "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cuh", ".h")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + fh.read())
    return h.hexdigest()


_HDR_KEY = _headers_key()


def compile_kernel(src: str, name: str) -> int:
    """CUfunction handle for `name` in `src` (process + on-disk cubin cache)."""
    key = hashlib.sha256((src + name + _HDR_KEY).encode()).hexdigest()
    # cuModuleLoadData binds the function to the CURRENT context: one handle
    # per (kernel, device); callers load under torch.cuda.device(dev)
    import torch
    dkey = (key, torch.cuda.current_device())
    if dkey in _FN_CACHE:
        return _FN_CACHE[dkey]
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
    _FN_CACHE[dkey] = fn.value
    return fn.value


JIT_REPEAT = int(os.environ.get("RTB200_JIT_REPEAT", "4"))


def specialise(recs, kernels, params, labels, loop_info=None, mult=None):
    """Attach JIT kernels to persistent loops and to EW records that are
    large (>= JIT_MIN_ELEMS elements) or launched JIT_REPEAT+ times per run
    (e.g. a PPO minibatch's small elementwise ops: the interpreting kernel's
    fixed cost dominates them; C3 59.6 -> 57.2 ms/step with all of them
    specialised) -- in place."""
    if not ENABLED:
        return 0
    n = 0
    from . import jit_mlp
    for ri, info in (loop_info or {}).items():
        if params[ri].rows * info["trips"] < JIT_LOOP_MIN:
            continue
        m = None if (info.get("pair") or MMA_ENABLED or KS_ENABLED) else \
            jit_mlp.match(params[ri], info["ops"], info)
        sm = jit_mlp.smem_bytes(params[ri], m) if m is not None else 0
        if m is not None and sm <= 227 * 1024:
            # the six-op MLP acting step: one fused 512-thread kernel (loop_mlp.cuh)
            src = jit_mlp.source(params[ri], info["ops"], info, m)
            recs[ri].jit_fn = compile_kernel(src, "loop_mlp")
            recs[ri].block[0] = jit_mlp.THREADS
            recs[ri].smem = sm
            info["mlp"] = dict(m, smem=sm)
            n += 1
            continue
        src = loop_source(params[ri], info["ops"], "loop_jit", info)
        recs[ri].jit_fn = compile_kernel(src, "loop_jit")
        n += 1
    for i, (k, p) in enumerate(zip(kernels, params)):
        if k != N.RT_K_EW:
            continue
        if p.total < JIT_MIN_ELEMS and (mult is None or mult[i] < JIT_REPEAT):
            continue
        src = ew_source(p, "ew_jit")
        recs[i].jit_fn = compile_kernel(src, "ew_jit")
        n += 1
    return n
