"""The fused MLP acting step (csrc/loop_mlp.cuh): pattern match and kernel
source for the persistent acting loop of an MLP policy.

The loop body the planner hands over is six ops (lower._loop_persistent):

    0  EW    o[t]  = merge(t == 0: z0, onext[t-1])        (reference merge)
    1  GEMM  h1    = tanh(o @ W1 + b1)       K = d_obs <= 32, N = 256
    2  GEMM  h2    = tanh(h1 @ W2 + b2)      K = N = 256
    3  GEMM  mu    = h2 @ W3 + b3            N = d_act <= 4
    4  EW    a     = mu + eps                 (eps pre-drawn, loop-external)
    5  UDF   onext = env(o, a)               (dsl.py:288-307 synthetic env)

(reference frontend ops matmul/tanh/add, runtime.py:58-80, 153-158, 249).
The op-by-op JIT loop (jit.loop_source) runs them with a CTA barrier after
each; this generator emits one 512-thread kernel that keeps the ops' own
parameter blocks (every address comes from them, as in jit.loop_source) but
restructures the step: h1 without a K split, h2 on the on-chip-weight core
(mlp_h2q: four columns per thread), and ops 3-5 as one warp per row
(loop_mlp.cuh).  The generic
path stays the fallback for every loop this does not match.
"""

from __future__ import annotations

import os

from . import native as N
from .jit import (_decompose, _env_fold, _env_terms, _ew_udf_forwards, _forward_pairs,
                  _gbox_off, _gemm_ew_forwards, _offset_expr, _program_lines, _rename_labels,
                  _store, _udf_ew_carries, FAST_TANH)

ENABLED = os.environ.get("RTB200_LOOP_MLP", "1") != "0"
THREADS = 256
KR = 32   # W2 rows per K quarter (and column) held in registers (mlp_h2q)
# op 0 (observation merge) of step t + 1 computed by the env step's lanes
# instead of a separate phase behind its own CTA barrier
FOLD_OBS = os.environ.get("RTB200_MLP_FOLD_OBS", "1") != "0"
# h1 computed per K quarter of the h2 core: the 64 threads of part p produce
# the h1 columns [64p, 64p + 64) their own core reads, so h1 -> core is a
# 64-thread named barrier per part instead of a CTA barrier
PART_BAR = os.environ.get("RTB200_MLP_PART_BAR", "1") != "0"


def match(lp, ops, info):
    """The fields the generator needs, or None when the loop is not the
    six-op MLP acting step (then jit.loop_source runs it)."""
    if not ENABLED or info is None or len(ops) != 6 or lp.step != 1:
        return None
    kinds = [o[0] for o in ops]
    if kinds != [N.RT_K_EW, N.RT_K_GEMM, N.RT_K_GEMM, N.RT_K_GEMM, N.RT_K_EW, N.RT_K_UDF]:
        return None
    if any(o[3] for o in ops):                    # f64
        return None
    e0, g1, g2, g3, e4, u5 = (o[1] for o in ops)
    R = lp.rows_per_cta
    if R > 8 or R < 1 or any(o[2] != 1 for o in ops[1:4]):
        return None
    if not (g1.k <= 32 and g1.n == 256 and g2.k == 256 and g2.n == 256 and g3.k == 256
            and g3.n <= 4 and g1.epilogue == 1 and g2.epilogue == 1 and g3.epilogue == 0):
        return None
    for g in (g1, g2, g3):
        if g.z != 1 or g.splits != 1 or g.N.nd != 1 or g.K.nd != 1 or g.C.dtype != N.RT_F32 \
                or g.A.dtype != N.RT_F32 or g.B.dtype != N.RT_F32:
            return None
        if g.bias.ptr and (g.bias.dtype != N.RT_F32 or g.bias.off_env[lp.slot] != 0):
            return None
        if g.B.off_env[lp.slot] != 0:             # weights must not move with t
            return None
        # weights dense row-major [K][N]
        if g.B.s1[0] != g.n or g.B.s2[0] != 1:
            return None
    DO, DA = g1.k, g3.n
    if ops[0][2] != DO or ops[4][2] != DA:
        return None
    if u5.nin != 2 or u5.nout != 1 or list(u5.in_count[:2]) != [DO, DA] or \
            u5.out_count[0] != DO or u5.out_kind[0] != N.RT_F32 or u5.out[0].dtype != N.RT_F32:
        return None
    if not ops[5][4]:                             # normals pre-drawn (lower: op[4] = noise)
        return None
    # dataflow: 0 -> 1 (A rows), 1 -> 2 -> 3 (A rows), 3 -> 4 (mu), 0 and 4 -> 5, 5 -> 0 (carry)
    from .jit import _ew_forward_pairs
    fake = dict(info, resident={1: 0, 3: 0}, hybrid={"op": 2})
    fw = _forward_pairs(lp, ops, fake) | _ew_forward_pairs(lp, ops)
    if not {(0, 1), (1, 2), (2, 3)} <= fw:
        return None
    xf = _gemm_ew_forwards(lp, ops, dict(fake, xfwd_off=1))
    if xf.get(4, (None, None))[1] != 3:
        return None
    k_mu = xf[4][0]
    if e4.nin != 2:
        return None
    k_eps = 1 - k_mu
    v_eps = e4.in_[k_eps]
    if v_eps.dtype != N.RT_F32 or v_eps.nchk:
        return None
    xu = _ew_udf_forwards(lp, ops, dict(info, xu_off=1)).get(5, {})
    if xu.get(0, (None,))[0] != 0 or xu.get(1, (None,))[0] != 4:
        return None
    xc = _udf_ew_carries(lp, ops, dict(info, xc_off=1)).get(0)
    if xc is None or xc[1] != 5 or xc[2] != 0:
        return None
    if THREADS // 32 < R:
        return None
    return {"R": R, "MRP": 8, "DO": DO, "DA": DA, "k_mu": k_mu, "k_eps": k_eps, "k_carry": xc[0]}


def _layout(lp, m):
    """Shared-memory offsets (bytes) after the op descriptors."""
    MRP, DO, DA, H = m["MRP"], m["DO"], m["DA"], 256
    cur = (lp.a_off + 127) // 128 * 128
    lay = {}

    def put(name, nbytes):
        nonlocal cur
        lay[name] = cur
        cur = (cur + nbytes + 127) // 128 * 128
    put("w2", 4 * (64 - KR) * H * 4)         # W2 rows [64p + KR, 64p + 64), p < 4 (mlp_h2q)
    put("w1", DO * H * 4)
    put("w3t", DA * H * 4)
    put("b1", H * 4)
    put("b2", H * 4)
    put("b3", 16)
    put("so", DO * MRP * 4)                  # observation, k-major
    put("x1", H * MRP * 4)                   # h1, k-major
    put("red", 4 * MRP * H * 4)              # h2 K-quarter exchange (mlp_h2q red[p][r][n])
    put("h2", MRP * H * 4)                   # h2, row-major
    put("obs", MRP * DO * 4)                 # observation, row-major (env input)
    put("act", MRP * DA * 4)                 # action, row-major (env input)
    put("eps", MRP * DA * 4)                 # eps of the next step (cp.async)
    put("nz", MRP * DO * 8)                  # env normals of the next step (cp.async)
    put("carry", MRP * DO * 4)               # env output -> next step's observation
    put("prof", 64)                          # phase probe accumulators (profiling runs)
    lay["total"] = cur
    return lay


def smem_bytes(lp, m):
    return _layout(lp, m)["total"]


def _vec_ok(q, lp, w):
    """Loop GEMM q's output rows take w-float vector stores: one contiguous
    column dim and every offset term (base, row strides, per-step env
    offsets) a multiple of w floats on a 16-byte aligned buffer."""
    if q.N.nd != 1 or q.C.s2[0] != 1 or q.C.dtype != N.RT_F32 or q.C.ptr % 16:
        return False
    terms = [q.C.off] + [q.C.s1[d] for d in range(q.M.nd)] + [q.C.off_env[e] for e in range(N.RT_MAXENV)]
    return all(t % w == 0 for t in terms)


def _gemm_io(q, soff, name):
    """Pointer/offset lines and C/bias index expressions of loop GEMM q."""
    env_c = _env_terms([q.C.off_env[e] for e in range(N.RT_MAXENV)])
    env_b = _env_terms([q.B.off_env[e] for e in range(N.RT_MAXENV)])
    env_bias = _env_terms([q.bias.off_env[e] for e in range(N.RT_MAXENV)])
    lines = [f"const rt_gemm_params& q{name} = *(const rt_gemm_params*)(smem + {soff});",
             f"float* C{name} = (float*)q{name}.C.ptr; const long long co{name} = q{name}.C.off{env_c};"]
    pro = [f"const rt_gemm_params& q{name} = *(const rt_gemm_params*)(smem + {soff});",
           f"const float* B{name} = (const float*)q{name}.B.ptr + (q{name}.B.off{env_b});"]
    if q.bias.ptr:
        pro.append(f"const float* Bias{name} = (const float*)q{name}.bias.ptr + (q{name}.bias.off{env_bias});")
    c_m = _gbox_off(q.M, [q.C.s1[d] for d in range(4)], "m")
    c_n = _gbox_off(q.N, [q.C.s2[d] for d in range(4)], "n")
    bias_n = _gbox_off(q.N, [q.bias.s2[d] for d in range(4)], "n") if q.bias.ptr else None
    return lines, pro, c_m, c_n, bias_n


def source(lp, ops, info, m, name="loop_mlp"):
    lay = _layout(lp, m)
    R, MRP, DO, DA, H = m["R"], m["MRP"], m["DO"], m["DA"], 256
    HR = MRP // 2
    e0, g1, g2, g3, e4, u5 = (o[1] for o in ops)
    soff = [o[5] for o in ops]
    S = {k: f"smem_u32(smem + {v})" for k, v in lay.items() if k != "total"}
    t0, t1 = ("p.start", "p.stop") if lp.blk_len else (f"{lp.start}LL", f"{lp.stop}LL")
    tanh = "tanh_fast" if FAST_TANH else "vm_tanh<float>"

    # ---- weights / biases into shared memory and registers (once) ----------
    _l1, pro1, _c1m, _c1n, bn1 = _gemm_io(g1, soff[1], "1")
    _l2, pro2, _c2m, _c2n, bn2 = _gemm_io(g2, soff[2], "2")
    _l3, pro3, _c3m, _c3n, bn3 = _gemm_io(g3, soff[3], "3")
    KS = 64 - KR
    prologue = "\n    ".join(pro1 + pro2 + pro3)
    bias_loads = []
    for nm, q, bn, key, cnt in (("1", g1, bn1, "b1", H), ("2", g2, bn2, "b2", H), ("3", g3, bn3, "b3", DA)):
        if q.bias.ptr:
            bias_loads.append(f"for (int n = tid; n < {cnt}; n += {THREADS}) sts1({S[key]} + 4u * n, Bias{nm}[{bn}]);")
        else:
            bias_loads.append(f"for (int n = tid; n < {cnt}; n += {THREADS}) sts1({S[key]} + 4u * n, 0.f);")
    bias_loads = "\n    ".join(bias_loads)

    # ---- op 0: the observation merge (generic EW body) ----------------------
    nd0 = e0.box.nd
    ext0 = [e0.box.ext[j] for j in range(nd0)]
    bases = []
    for k in range(e0.nin):
        v = e0.in_[k]
        bases.append(f"const long long b{k} = " + _env_fold(
            f"p.in[{k}].off", [v.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
        for c in range(v.nchk):
            bases.append(f"const long long c{k}_{c} = " + _env_fold(
                f"p.in[{k}].chk_c0[{c}]", [v.chk_env[c][e] for e in range(N.RT_MAXENV)]) + ";")
    bases.append("const long long bo = " + _env_fold(
        "p.out.off", [e0.out.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
    kc = m["k_carry"]
    offc = _offset_expr(f"b{kc}", e0.in_[kc], nd0)

    def op0_src(tag, fold):
        """op 0's generic body: over the CTA's (row, e) elements (flat loop),
        or folded into the env step (fold: lane e of the row's warp computes
        observation t + 1 from the env output cv_ in its register)."""
        if fold:
            ov = {kc: "cv_"}
        else:
            ov = {kc: (f"(t == T0_ ? ((const float*)p.in[{kc}].ptr)[{offc}] : "
                       f"lds1({S['carry']} + (uint32_t)(lf * 4), 0.f))")}
        lines0 = _program_lines(e0, "float", nd0, base=lambda k: f"b{k}", chk=lambda k, c: f"c{k}_{c}",
                                env="env", load_override=ov)
        head = (f"{{ const long long flat = row * {DO}LL + e; const int lf = r * {DO} + e;" if fold else
                f"for (long long flat = r0 * {DO}LL + tid; flat < r1 * {DO}LL; flat += {THREADS}) {{\n"
                f"        const int lf = (int)(flat - r0 * {DO}LL);")
        src = f"""    {{  // op 0: observation (elementwise, generic body)
      const rt_ew_params& p = *(const rt_ew_params*)(smem + {soff[0]});
      {chr(10).join('      ' + b for b in bases).strip()}
      {head}
        {chr(10).join('        ' + x for x in _decompose(nd0, ext0)).strip()}
        float v0, v1, v2, v3, v4, v5, v6, v7;
        long long n0, n1, n2, n3, n4, n5, n6, n7;
        float res = 0.f;
        (void)n0;
        {chr(10).join('        ' + x for x in lines0).strip()}
      Lend:
        {_store(e0, "float", nd0, "bo")}
        sts1({S['obs']} + (uint32_t)(lf * 4), res);
        sts1({S['so']} + (uint32_t)((((lf % {DO}) * {MRP}) + lf / {DO}) * 4), res);
      }}
    }}"""
        src = src.replace("goto Lend;", f"goto Lend{tag};").replace("Lend:", f"Lend{tag}:")
        return _rename_labels(src.replace("goto L", f"goto X{tag}L").replace(f"goto X{tag}Lend{tag}", f"goto Lend{tag}"), tag)
    op0 = op0_src(0, False)
    op0f = op0_src(9, True).replace("\n", "\n    ") if FOLD_OBS else ""

    # ---- op 4 (action) body: mu and eps from registers ----------------------
    nd4 = e4.box.nd
    ext4 = [e4.box.ext[j] for j in range(nd4)]
    lines4 = _program_lines(e4, "float", nd4, base=lambda k: f"d{k}", chk=lambda k, c: f"e{k}_{c}",
                            env="env", load_override={m["k_mu"]: "muv", m["k_eps"]: "epsv"})
    bases4 = []
    for k in range(e4.nin):
        v = e4.in_[k]
        bases4.append(f"const long long d{k} = " + _env_fold(
            f"p4.in[{k}].off", [v.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
    bases4.append("const long long do4 = " + _env_fold(
        "p4.out.off", [e4.out.off_env[e] for e in range(N.RT_MAXENV)]) + ";")
    ke = m["k_eps"]
    eps_off = _offset_expr(f"d{ke}", e4.in_[ke], nd4)
    eps_step = e4.in_[ke].off_env[lp.slot] * lp.step
    st4 = _store(e4, "float", nd4, "do4").replace("p.out", "p4.out")
    body4 = "\n          ".join(lines4).replace("p.in[", "p4.in[").replace("goto Lend;", "goto Lend4;")
    body4 = _rename_labels(body4.replace("goto L", "goto X4L").replace("goto X4Lend4", "goto Lend4"), 4)

    # ---- op 5 (env) addressing ----------------------------------------------
    nd5 = u5.box.nd
    ext5 = [u5.box.ext[j] for j in range(nd5)]
    env_o = _env_terms([u5.out[0].off_env[e] for e in range(N.RT_MAXENV)])
    out5 = _offset_expr("oo5", u5.out[0], nd5)
    dec5 = "\n          ".join(x.replace("rr", "ur").replace("unsigned int r =", "unsigned int ur =")
                               .replace("(r %", "(ur %").replace("r /=", "ur /=").replace("(long long)r;", "(long long)ur;")
                               for x in _decompose(nd5, ext5, flat="row"))
    dec4 = "\n          ".join(x.replace("unsigned int r =", "unsigned int ar =").replace("(r %", "(ar %")
                               .replace("r /=", "ar /=").replace("(long long)r;", "(long long)ar;")
                               for x in _decompose(nd4, ext4, flat="f4"))

    # h1 / h2 rows to global: 8- / 16-byte stores when the columns are
    # contiguous and every row start is aligned (else one store per element)
    if _vec_ok(g1, lp, 2):
        h1_store = (f"#pragma unroll\n      for (int rr = 0; rr < {HR}; ++rr) {{ if (hh * {HR} + rr < mr) {{ "
                    f"const long long m = r0 + hh * {HR} + rr, n = c0; "
                    f"*reinterpret_cast<float2*>(C1 + co1 + {_c1m} + {_c1n}) = make_float2(v[0][rr], v[1][rr]); }} }}")
    else:
        h1_store = (f"#pragma unroll\n      for (int j = 0; j < 2; ++j)\n      #pragma unroll\n"
                    f"      for (int rr = 0; rr < {HR}; ++rr) {{ if (hh * {HR} + rr < mr) {{ "
                    f"const long long m = r0 + hh * {HR} + rr, n = c0 + j; C1[co1 + {_c1m} + {_c1n}] = v[j][rr]; }} }}")
    if _vec_ok(g2, lp, 4):
        h2_store = (f"{{ const long long n = qc; *reinterpret_cast<float4*>(C2 + co2 + {_c2m} + {_c2n}) = "
                    f"make_float4(v[0], v[1], v[2], v[3]); }}")
    else:
        h2_store = (f"#pragma unroll\n          for (int j = 0; j < 4; ++j) {{ const long long n = qc + j; "
                    f"C2[co2 + {_c2m} + {_c2n}] = v[j]; }}")

    if FOLD_OBS:
        # op 0 of step T0_ before the loop, op 0 of step t + 1 in the env step
        prologue_op0 = (f"  if (T0_ < T1_) {{\n    const long long t = T0_;\n    env[{lp.slot}] = t;\n"
                        f"{op0}\n  }}\n  __syncthreads();\n")
        loop_op0 = ""
        carry_or_fold = (f"if (t + 1LL < T1_) {{\n            env[{lp.slot}] = t + 1LL;\n"
                         + op0f.replace("\n", "\n        ") + "\n          }")
    else:
        prologue_op0 = ""
        loop_op0 = op0 + "\n    __syncthreads();\n    MLP_PROF(0)"
        carry_or_fold = f"sts1({S['carry']} + (uint32_t)((r * {DO} + e) * 4), cv_);"

    # ---- the kernel ---------------------------------------------------------
    src = f"""#include "loop_mlp.cuh"
// fused MLP acting step (jit_mlp.py): R={R} rows per CTA, obs {DO}, hidden {H}, act {DA}
extern "C" __global__ void __launch_bounds__({THREADS}, 1) {name}(const __grid_constant__ rt_loop_params p) {{
  extern __shared__ __align__(128) unsigned char smem[];
  long long env[RT_MAXENV];
  for (int e = 0; e < RT_MAXENV; ++e) env[e] = p.h.env[e];
  const long long r0 = (long long)blockIdx.x * {R}LL;
  const long long r1 = r0 + {R}LL < {lp.rows}LL ? r0 + {R}LL : {lp.rows}LL;
  if (r0 >= r1) return;
  const int tid = (int)threadIdx.x, {"hh = (tid >> 5) & 1, c0 = 64 * (tid >> 6) + 2 * (tid & 31)" if PART_BAR else "hh = tid >> 7, c0 = 2 * (tid & 127)"}, warp = tid >> 5, lane = tid & 31;
  const int mr = (int)(r1 - r0);
  const rt_loop_op* ops = (const rt_loop_op*)p.ops;
  for (int i = 0; i < p.nops; ++i) {{
    const int4* src = (const int4*)ops[i].params;
    int4* dst = (int4*)(smem + ops[i].smem_off);
    for (int w = tid; w < (ops[i].param_bytes + 15) / 16; w += {THREADS}) dst[w] = src[w];
  }}
  __syncthreads();
  float wreg[4][{KR}];
  {{  // loop-invariant weights: W1, W3^T, biases in shared memory; W2: part
      // tid / 64 owns k rows [64p, 64p + 64) of columns 4 (tid % 64) .. +4,
      // the first {KR} in registers, the rest in shared memory (mlp_h2q)
    {prologue}
    for (int i = tid; i < {DO * H}; i += {THREADS}) sts1({S['w1']} + 4u * i, B1[i]);
    for (int i = tid; i < {DA * H}; i += {THREADS}) {{ const int n = i / {H}, k = i % {H}; sts1({S['w3t']} + 4u * i, B3[k * {DA} + n]); }}
    {bias_loads}
    {{
      const int qp = tid >> 6, qc = 4 * (tid & 63);
      #pragma unroll
      for (int k = 0; k < {KR}; ++k)
        #pragma unroll
        for (int j = 0; j < 4; ++j)   // (an opaque load: not re-loaded per step)
          asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(wreg[j][k]) : "l"(B2 + (qp * 64 + k) * {H} + qc + j));
    }}
    for (int i = tid; i < {4 * KS * H // 4}; i += {THREADS}) {{
      const int row = i / {H // 4}, pp = row / {KS}, kk = row % {KS};
      sts4({S['w2']} + 16u * i, __ldg(reinterpret_cast<const float4*>(B2 + (pp * 64 + {KR} + kk) * {H}) + i % {H // 4}));
    }}
  }}
  __syncthreads();
  const long long T0_ = {t0}, T1_ = {t1};
  const double* nz_base = (const double*)ops[5].noise + ops[5].noise_off;
  const long long nz_row = ops[5].noise_row, nz_step = ops[5].noise_step;
  // phase probes (tools/loop_profile.py): CTA 0 / thread 0 accumulates the
  // clock deltas in shared memory (a global read-modify-write per probe put a
  // memory round trip on warp 0's path) and writes them out at the end
  const bool prof_on = p.prof && blockIdx.x == 0 && tid == 0;
  if (prof_on)
    for (int i = 0; i < 8; ++i) sts1({S['prof']} + 8u * i, 0.0);
  long long c0_ = clock64();
#define MLP_PROF(i) if (prof_on) {{ const long long c1_ = clock64(); \
    sts1({S['prof']} + 8u * (i), lds1({S['prof']} + 8u * (i), 0.0) + (double)(c1_ - c0_)); c0_ = c1_; }}
{prologue_op0}  for (long long t = T0_; t < T1_; t += 1LL) {{
    env[{lp.slot}] = t;
{loop_op0}
    {{  // op 1: h1 = tanh(o W1 + b1): rows [hh*{HR}, +{HR}) of columns c0, c0+1
      {chr(10).join('      ' + x for x in _l1).strip()}
      float acc[2][{HR}];
      mlp_h1<{MRP}, {DO}, {H}>({S['so']}, {S['w1']}, c0, hh, acc);
      float v[2][{HR}];
      #pragma unroll
      for (int j = 0; j < 2; ++j) {{
        const float bias = lds1({S['b1']} + 4u * (c0 + j), 0.f);
        #pragma unroll
        for (int rr = 0; rr < {HR}; ++rr) {{ const float x_ = {tanh}(acc[j][rr] + bias); v[j][rr] = hh * {HR} + rr < mr ? x_ : 0.f; }}
        sts4({S['x1']} + (uint32_t)(((c0 + j) * {MRP} + hh * {HR}) * 4), make_float4(v[j][0], v[j][1], v[j][2], v[j][3]));
      }}
      {h1_store}
    }}
    {"asm volatile(\"bar.sync %0, 64;\" :: \"r\"(1 + (tid >> 6)) : \"memory\");" if PART_BAR else "__syncthreads();"}
    MLP_PROF(1)
    {{  // op 2: h2 = tanh(h1 W2 + b2): K quarters, 4 columns per thread (mlp_h2q)
      {chr(10).join('      ' + x for x in _l2).strip()}
      float acc[4][{MRP // 4}];
      mlp_h2q<{MRP}, {R if R < MRP else MRP}, {KR}, {H}>(wreg, {S['w2']}, {S['x1']}, {S['red']}, acc);
      MLP_PROF(6)
      const int qp = tid >> 6, qc = 4 * (tid & 63);
      #pragma unroll
      for (int q = 0; q < {MRP // 4}; ++q) {{
        const int r = qp * {MRP // 4} + q;
        float v[4];
        #pragma unroll
        for (int j = 0; j < 4; ++j) {{
          const float x_ = {tanh}(acc[j][q] + lds1({S['b2']} + 4u * (qc + j), 0.f));
          v[j] = r < mr ? x_ : 0.f;
        }}
        sts4({S['h2']} + (uint32_t)((r * {H} + qc) * 4), make_float4(v[0], v[1], v[2], v[3]));
        if (r < mr) {{
          const long long m = r0 + r;
          {h2_store}
        }}
      }}
    }}
    __syncthreads();
    MLP_PROF(2)
    if (warp < mr) {{  // ops 3-5: one warp per row: head, action, env
      const int r = warp;
      const long long row = r0 + r;
      {chr(10).join('      ' + x for x in _l3).strip()}
      // the env's observation mean depends only on step t's observation:
      // issued ahead of the head so its loads / shuffles overlap the head's
      const double sobs_ = warp_pairwise_sum_s({S['obs']} + (uint32_t)(r * {DO * 4}), {DO}, lane);
      float actv_ = 0.f;
      float mu[{DA}];
      mlp_head<{DA}, {H}>({S['h2']} + (uint32_t)(r * {H} * 4), {S['w3t']}, lane, mu);
      MLP_PROF(4)
      const rt_ew_params& p4 = *(const rt_ew_params*)(smem + {soff[4]});
      {chr(10).join('      ' + b for b in bases4).strip()}
      if (t != T0_) cp_async_wait_all();     // this lane's eps / normals of step t
      if (lane < {DA}) {{
        float muv = 0.f;
        #pragma unroll
        for (int n_ = 0; n_ < {DA}; ++n_) muv = lane == n_ ? mu[n_] : muv;
        muv += lds1({S['b3']} + 4u * lane, 0.f);
        {{ const long long m = row, n = lane; C3[co3 + {_c3m} + {_c3n}] = muv; }}
        const long long f4 = row * {DA}LL + lane;
        {dec4}
        const float epsv = t == T0_ ? ((const float*)p4.in[{ke}].ptr)[{eps_off}]
                                    : lds1({S['eps']} + (uint32_t)((r * {DA} + lane) * 4), 0.f);
        float v0, v1, v2, v3, v4, v5, v6, v7;
        long long n0, n1, n2, n3, n4, n5, n6, n7;
        float res = 0.f;
        (void)n0; (void)epsv; (void)muv;
        {body4}
      Lend4:
        {st4}
        actv_ = res;
        if (t + 1LL < T1_) cp_async4({S['eps']} + (uint32_t)((r * {DA} + lane) * 4),
                                     (const float*)p4.in[{ke}].ptr + ({eps_off} + {eps_step}LL));
      }}
      __syncwarp();
      MLP_PROF(5)
      {{  // op 5: env (make_udf_fn body: numpy pairwise means in fp64)
        const rt_udf_params& q5 = *(const rt_udf_params*)(smem + {soff[5]});
        float* out5 = (float*)q5.out[0].ptr; const long long oo5 = q5.out[0].off{env_o};
        {dec5}
        double base = {repr(float(u5.salt))};
        base = base + sobs_ / {float(DO)!r};
        // the action mean: lane 0's serial fp64 sum of warp_pairwise_sum_s
        // (n < 8), read from the action lanes' registers by every lane
        double sact_ = 0.0;
        #pragma unroll
        for (int i_ = 0; i_ < {DA}; ++i_) sact_ += (double)__shfl_sync(0xffffffffu, actv_, i_);
        base = base + sact_ / {float(DA)!r};
        if (lane < {DO}) {{
          const int e = lane;
          const double z = t == T0_ ? nz_base[row * nz_row + t * nz_step + e]
                                    : lds1({S['nz']} + (uint32_t)((r * {DO} + e) * 8), 0.0);
          const float cv_ = (float)tanh(base + 0.3 * z);
          out5[{out5} + e] = cv_;
          {carry_or_fold}
          if (t + 1LL < T1_) cp_async8({S['nz']} + (uint32_t)((r * {DO} + e) * 8),
                                       nz_base + row * nz_row + (t + 1LL) * nz_step + e);
        }}
        cp_async_commit();
      }}
    }}
    __syncthreads();
    MLP_PROF(3)
  }}
  if (prof_on)
    for (int i = 0; i < 8; ++i) ((long long*)p.prof)[i] += (long long)lds1({S['prof']} + 8u * i, 0.0);
}}
"""
    return src
