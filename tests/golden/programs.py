"""Program builders for the parity corpus and the benchmark workloads.

These use the REFERENCE front end (`recten`, imported from
/root/reference/pkg/src), so they run only in the build container.  Their
products — serialised dependence graphs — are committed under
`tests/golden/graphs/` and are what the GPU-side tests, smoke() and bench.py
load.  Run `python tests/golden/make_golden.py` to regenerate.
"""

from __future__ import annotations

import os
import sys

REF_SRC = "/root/reference/pkg/src"
REF_PROGRAMS = "/root/reference/pkg/programs"


def recten():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import recten  # noqa: F401
    from recten import dsl, frontend, pdg, transforms, runtime, polysched
    return dsl, frontend, pdg, transforms, runtime, polysched


# reference pkg/tests/test_dsl.py:16-28
CORPUS_BINDS = {
    "running_total": ({"T": 6}, {"x": ("arange", 6)}),
    "reinforce": ({"I": 2, "B": 2, "T": 4}, {"winit": 0.1}),
    "nstep2": ({"T": 8}, None),
    "nstep4": ({"T": 8}, None),
    "mc_value": ({"T": 6}, {"x": ("linspace", -0.5, 0.5, 6)}),
    "gated_value": ({"T": 6}, {"x": ("linspace", 0.1, 0.6, 6)}),
    "checkpoint": ({"T": 8}, None),
    "epoch_minibatch": ({"E": 2, "K": 2, "T": 8}, None),
    "early_stop": ({}, None),
    "pixels": ({"B": 2, "T": 3}, None),
    "stream_window": ({"B": 2, "T": 6}, None),
}


def corpus_text(name):
    with open(os.path.join(REF_PROGRAMS, f"{name}.rtl")) as fh:
        return fh.read()


# ---------------------------------------------------------------------------
# KAT programs from the reference tests (pkg/tests/test_dsl.py:106-188)

KAT_TEXTS = {
    "kat_head_shift": ("""
        dims t: T;
        bounds T = 5;
        rec y[t] : f64[];
        y[0] = 1.0;
        y[t+1] = y[t] + 1.0;
        out y;
    """, None, None),
    "kat_reverse_head": ("""
        dims t: T;
        bounds T = 4;
        rec y[t] : f64[];
        y[T-1] = 10.0;
        y[t] = y[t+1] * 0.5 if t < T - 1;
        out y;
    """, None, None),
    "kat_if_order": ("""
        dims t: T;
        bounds T = 6;
        rec y[t] : f64[];
        y[0] = 0.0;
        y[t] = y[t-1] + 10.0 if t >= 1 and t % 3 == 0;
        y[t] = y[t-1] + 1.0;
        out y;
    """, None, None),
    "kat_slice_dsum": ("""
        dims t: T;
        bounds T = 3;
        input r[t] : f64[];
        g[t] = dsum(r[t:T], 0.5);
        tot[t] = sum(r[t:T]);
        out g; out tot;
    """, None, {"r": ("ones", 3)}),
    "kat_flag": ("""
        dims t: T;
        bounds T = 4;
        f[t] = flag(t % 2 == 0);
        out f;
    """, None, None),
    "kat_sumall": ("""
        dims t: T;
        bounds T = 3;
        input x[t] : f64[2];
        s = sumall(x);
        out s;
    """, None, {"x": ("arange_reshape", 6, (3, 2))}),
    "kat_udf": ("""
        dims t: T;
        bounds T = 3;
        rng e[t] : f64[2];
        udf step(f64[2]) -> f64[2];
        y[t] = step(e[t]);
        out y;
    """, None, None),
    "kat_dyn": ("""
        dims t: T;
        bounds T = dyn(stop);
        rec y[t] : f64[];
        y[0] = 1.0;
        y[t+1] = y[t] + 1.0;
        stop[t] = ge(y[t], 3.0);
        out y;
    """, None, None),
    # GAE in the liftable form
    "gae_liftable": ("""
        dims b: B, t: T;
        bounds B = 3, T = 6;
        input r[b,t] : f64[];
        input Vn[b,t] : f64[];
        input V[b,t] : f64[];
        dd[b,t] = r[b,t] + 0.99 * Vn[b,t] - V[b,t];
        rec A[b,t] : f64[];
        A[b,T-1] = dd[b,t];
        A[b,t] = dd[b,t] + A[b,t+1] * 0.9405;
        out A;
    """, None, {"r": ("normal", (3, 6), 1), "Vn": ("normal", (3, 6), 2),
                "V": ("normal", (3, 6), 3)}),
    # SURVEY Appendix B, with the training dim (reference reinforce.rtl:15-16)
    "mlp_reinforce_f64": ("""
        dims i: I, b: B, t: T;
        bounds I = 2, B = 3, T = 5;
        input W1i[] : f64[4,8];
        input W2i[] : f64[8,1];
        udf envstep(f64[1,4], f64[1,1]) -> f64[1,4];
        rng eps[i,b,t] : f64[1,1] normal;
        rec W1[i] : f64[4,8];
        rec gW1[i] : f64[4,8];
        rec o[i,b,t] : f64[1,4];
        const z0 : f64[1,4] = 0.1;
        W1[0] = W1i;
        W1[i+1] = detach(W1[i]) - 0.01 * detach(gW1[i]);
        o[i,b,0] = z0;
        h[i,b,t] = tanh(o[i,b,t] @ W1[i]);
        mu[i,b,t] = h[i,b,t] @ W2i;
        a[i,b,t] = detach(mu[i,b,t]) + eps[i,b,t];
        o[i,b,t+1] = envstep(o[i,b,t], a[i,b,t]);
        r[i,b,t] = sum(sum(o[i,b,t], 1), 0);
        G[i,b,t] = dsum(r[i,b,t:T], 0.99);
        lp[i,b,t] = sum(sum(-(a[i,b,t] - mu[i,b,t]) ** 2.0, 1), 0);
        score[i,b,t] = detach(G[i,b,t]) * lp[i,b,t];
        ep[i,b] = sum(score[i,b,0:T]);
        it[i] = sum(ep[i,0:B]);
        loss = sum(it[0:I]);
        grad loss wrt W1 into gW1;
        out G;
        out W1;
    """, None, {"W1i": ("normal_scaled", (4, 8), 11, 0.3),
                "W2i": ("full", (8, 1), 0.1)}),
}


def make_input(spec):
    import numpy as np
    if not isinstance(spec, tuple):
        return spec
    kind = spec[0]
    if kind == "arange":
        return np.arange(float(spec[1]))
    if kind == "linspace":
        return np.linspace(spec[1], spec[2], spec[3])
    if kind == "ones":
        return np.ones(spec[1])
    if kind == "arange_reshape":
        return np.arange(float(spec[1])).reshape(spec[2])
    if kind == "normal":
        return np.random.default_rng(spec[2]).standard_normal(spec[1])
    if kind == "normal_scaled":
        return np.random.default_rng(spec[2]).standard_normal(spec[1]) * spec[3]
    if kind == "full":
        return np.full(spec[1], spec[2])
    raise ValueError(spec)


# ---------------------------------------------------------------------------
# Context-API programs from the reference transform tests
# (pkg/tests/test_transforms.py:52-64, 96-110, 362-373)


def ctx_gated(gamma=0.9, T=7):
    dsl, fe, pdg, tr, rt, ps = recten()
    import recten.symexpr as se
    ctx = fe.Context()
    t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Tb, T)
    x = ctx.rng("x", (4,), domain=(t,))
    y = ctx.recurrent("y", (4,), domain=(t,))
    y.define([(se.eq(se.sym(t), se.cint(0)), x),
              (None, y["t-1"] * gamma + x["t"])])
    ctx.mark_output(y, "y")
    return ctx


def ctx_reverse_scan():
    dsl, fe, pdg, tr, rt, ps = recten()
    import recten.symexpr as se
    ctx = fe.Context()
    t, T = ctx.declare_dim("t", "T")
    ctx.bind(T, 6)
    x = ctx.rng("x", (), domain=(t,))
    G = ctx.recurrent("G", (), domain=(t,))
    last = se.eq(se.sym(t), se.sub(se.sym(T), se.cint(1)))
    G.define([(last, x), (None, x["t"] + G["t+1"] * 0.95)])
    ctx.mark_output(G, "G")
    return ctx


def ctx_widesum(T=3, payload=(40, 8)):
    dsl, fe, pdg, tr, rt, ps = recten()
    ctx = fe.Context()
    t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Tb, T)
    x = ctx.rng("x", payload, domain=(t,))
    h = ctx.op("tanh", [x])
    z = h * 2.0
    s = ctx.sum(z, 0)
    out = ctx.sum(s, 0) * 0.1
    ctx.mark_output(out, "out")
    return ctx


# ---------------------------------------------------------------------------
# The benchmark workload: REINFORCE with a 2-hidden-layer tanh MLP policy
# (BASELINE.json configs[1]), f32 via the Context API.


def ctx_reinforce_mlp(B=1024, T=1000, I=1, d_o=16, H=256, d_a=4,
                      gamma=0.99, lr=None, dtype="f32"):
    """One training iteration per point of `i`: roll out B envs for T steps
    under a Gaussian policy mu = MLP(o), score each step by its discounted
    return-to-go (a suffix dsum over t:T, reference runtime.py:115-122),
    backpropagate the surrogate through the MLP and emit updated weights.

    Env = the reference's synthetic UDF body (dsl.py:288-307)."""
    dsl, fe, pdg, tr, rt, ps = recten()
    import recten.symexpr as se
    if lr is None:
        lr = 0.01 / (B * T)
    ctx = fe.Context()
    i, Ib = ctx.declare_dim("i", "I")
    b, Bb = ctx.declare_dim("b", "B")
    t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Ib, I)
    ctx.bind(Bb, B)
    ctx.bind(Tb, T)
    shapes = {"W1": (d_o, H), "b1": (1, H), "W2": (H, H), "b2": (1, H),
              "W3": (H, d_a), "b3": (1, d_a)}
    init = {k: ctx.input(f"{k}_0", s, dtype) for k, s in shapes.items()}
    par = {k: ctx.recurrent(k, s, dtype, (i,)) for k, s in shapes.items()}
    grad = {k: ctx.recurrent(f"g{k}", s, dtype, (i,)) for k, s in shapes.items()}
    i0 = se.eq(se.sym(i), se.cint(0))
    for k in shapes:
        upd = ctx.detach(par[k]["i-1"]) - ctx.detach(grad[k]["i-1"]) * lr
        par[k].define([(i0, init[k]), (None, upd)])
    spec = ctx.register_udf("envstep", dsl.make_udf_fn("envstep", [(1, d_o)], [dtype]),
                            [(1, d_o)], [dtype])
    del spec
    eps = ctx.rng("eps", (1, d_a), dtype, (i, b, t), "normal")
    o = ctx.recurrent("o", (1, d_o), dtype, (i, b, t))
    z0 = ctx.constant(0.1, dtype, (1, d_o), name="z0")
    h1 = ctx.op("tanh", [o @ par["W1"] + par["b1"]], name="h1")
    h2 = ctx.op("tanh", [h1 @ par["W2"] + par["b2"]], name="h2")
    mu = ctx.op("add", [h2 @ par["W3"], par["b3"]], name="mu")
    a = ctx.op("add", [ctx.detach(mu), eps], name="a")
    (onext,) = ctx.udf("envstep", [o, a])
    o.define([(se.eq(se.sym(t), se.cint(0)), z0), (None, onext["i,b,t-1"])])
    r = ctx.sum(ctx.sum(o, 1), 0)
    G = ctx.discounted_sum(r["i,b,t:T"], gamma, dim=0)
    d = a - mu
    lp = ctx.sum(ctx.sum(-(d * d), 1), 0)
    score = ctx.detach(G) * lp
    ep = ctx.sum(score["i,b,0:T"], 0)
    it = ctx.sum(ep["i,0:B"], 0)
    loss = ctx.sum(it["0:I"], 0)
    gr = ctx.backward(loss, [par[k] for k in shapes])
    for k in shapes:
        grad[k].define([(None, gr[par[k]])])
    nxt = {k: ctx.op("sub", [ctx.detach(par[k]), ctx.detach(grad[k]) * lr], name=f"{k}_next")
           for k in shapes}
    for k in shapes:
        ctx.mark_output(nxt[k], f"{k}_next")
    ctx.mark_output(it, "objective")
    ctx.mark_output(G, "G")
    return ctx


def mlp_inputs(d_o=16, H=256, d_a=4, dtype="f32", seed=1234):
    """Weights ~ N(0, 1/fan_in) from default_rng(1234)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    from paper_2501_05408_b200.workloads import mlp_inputs as mk
    return mk(d_o=d_o, H=H, d_a=d_a, dtype=dtype, seed=seed)
