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
# the reference installed by `pip install --target baseline/_ref` (git-ignored;
# travels to the GPU box, where /root/reference does not exist)
REF_INSTALLED = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))), "baseline", "_ref")


def recten():
    if "recten" not in sys.modules:
        src = REF_SRC if os.path.isdir(REF_SRC) else REF_INSTALLED
        if src not in sys.path:
            sys.path.insert(0, src)
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


def ctx_opset(T=5, dtype="f64"):
    """Every remaining elementwise / layout / control kind of the reference
    KERNELS table (runtime.py:58-93, 149-150, 239-259) in one program:
    div, log, sqrt, exp, cmp, where, cast (both ways), reshape, squeeze,
    unsqueeze, identity, eval_symbol of a loop dim and of a bound, cumsum
    forward and reverse on a payload axis."""
    dsl, fe, pdg, tr, rt, ps = recten()
    ctx = fe.Context()
    t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Tb, T)
    other = "f32" if dtype == "f64" else "f64"
    x = ctx.rng("x", (3, 2), dtype, (t,))
    u = ctx.rng("u", (3, 2), dtype, (t,), dist="uniform")
    one = ctx.constant(1.0, dtype, (), name="one")
    half = ctx.constant(0.5, dtype, (), name="half")
    zero = ctx.constant(0.0, dtype, (), name="zero")
    lg = ctx.op("log", [ctx.op("exp", [x]) + one], name="lg")
    sq = ctx.op("sqrt", [u + half], name="sq")
    q = ctx.op("div", [lg, sq], name="q")
    pos = ctx.cmp("gt", x, zero)
    w = ctx.where(pos, x, -x)
    c1 = ctx.op("cast", [w], {"dtype": other}, name="c1")
    back = ctx.op("cast", [c1 * ctx.constant(3.0, other, (), name="three")],
                  {"dtype": dtype}, name="back")
    rs = ctx.reshape(q, (6,))
    rs2 = ctx.reshape(rs, (2, 3))
    uq = ctx.unsqueeze(rs2, 0)
    sqz = ctx.squeeze(uq, 0)
    idn = ctx.op("identity", [sqz], name="idn")
    ev = ctx.eval_symbol(t)
    evf = ctx.op("cast", [ev], {"dtype": dtype}, name="evf")
    y = ctx.op("mul", [idn, evf + one], name="y")
    nT = ctx.op("cast", [ctx.eval_symbol(Tb)], {"dtype": dtype}, name="nT")
    tot = ctx.sum(y["0:T"], 0)
    mean = ctx.op("div", [tot, nT], name="mean")
    csf = ctx.cumsum(back, 0)
    csr = ctx.cumsum(back, 1, reverse=True)
    for name, v in (("q", q), ("w", w), ("pos", pos), ("back", back), ("idn", idn),
                    ("ev", ev), ("y", y), ("mean", mean), ("csf", csf), ("csr", csr)):
        ctx.mark_output(v, name)
    return ctx


def ctx_unit_cumsum(T=6):
    """reference pkg/tests/test_transforms.py:223-237: a unit-gamma scan that
    vectorize_all lifts to a `cumsum` over the time axis."""
    dsl, fe, pdg, tr, rt, ps = recten()
    import recten.symexpr as se
    ctx = fe.Context()
    t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Tb, T)
    x = ctx.rng("x", (2,), domain=(t,))
    y = ctx.recurrent("y", (2,), domain=(t,))
    y.define([(se.eq(se.sym(t), se.cint(0)), x), (None, y["t-1"] + x["t"])])
    ctx.mark_output(y, "y")
    return ctx


def ctx_euclid(T=9):
    """Euclidean // and % with negative operands inside device index
    expressions (reference symexpr.py:491-506; KATs test_symexpr.py:34-49:
    -t % 4 with t=3 -> 1, -7 // 2 -> -4): y[t] = x[(t - 5) % 4] + x[(t - 7) // 2 + 4]."""
    dsl, fe, pdg, tr, rt, ps = recten()
    ctx = fe.Context()
    t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Tb, T)
    x = ctx.input("x", (), "f64", (t,))
    y = ctx.op("add", [x["(t - 5) % 4"], x["(t - 7) // 2 + 4"] * 100.0], name="y")
    z = ctx.op("mul", [x["(-t) % 4"], x["(8 - t) // 3"]], name="z")
    ctx.mark_output(y, "y")
    ctx.mark_output(z, "z")
    return ctx


def ctx_divzero(T=5):
    """An index expression that divides by zero at t = 2: the reference
    raises EvaluationError (symexpr.py:491-506)."""
    dsl, fe, pdg, tr, rt, ps = recten()
    ctx = fe.Context()
    t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Tb, T)
    x = ctx.input("x", (), "f64", (t,))
    y = ctx.op("mul", [x["t % (t - 2)"], ctx.constant(2.0, "f64", (), name="two")], name="y")
    ctx.mark_output(y, "y")
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


# ---------------------------------------------------------------------------
# C3/C5: PPO with GAE(lambda) and epochs x minibatches over a shared
# policy/value MLP (BASELINE.json configs[2], configs[4]).


def ctx_ppo_mlp(B=4096, T=512, I=1, epochs=4, minibatches=4, d_o=16, H=256, d_a=4,
                gamma=0.99, lam=0.95, lr=None, beta=0.5, cv=0.5, dtype="f32"):
    """One PPO iteration per point of `i`.

    Rollout over (i,b,t) at the iteration's entry weights theta[i,0,0]:
    shared tanh trunk h1,h2, policy head mu (d_a) and value head V (1);
    Gaussian actions a = mu + eps; the reference's synthetic env
    (dsl.py:288-307).  Advantages by GAE(lambda) written as the suffix
    discounted sum A = dsum(delta[t:T], gamma*lam) (the lifted form of
    SURVEY Appendix C), delta = r + gamma*V[t+1] - V (bootstrap 0 at T-1);
    returns R = A + V.

    Updates over epochs e and minibatches j (the two-level carry of the
    reference's epoch_minibatch.rtl: w[e,k+1] from w[e,k], w[e+1,0] from
    w[e,K-1]): minibatch j is the fixed env set {u*M + j : u < B/M} (an
    interleaved partition, so that an env shard [r*B/G, (r+1)*B/G) holds an
    equal slice of every minibatch and the sharded run is the same
    program); the policy/value are re-evaluated at theta[i,e,j] on the
    stored rollout and theta advances by -lr * grad.

    Loss per (e,j,u,t): -ratio*A + cv*(V_new - R)^2 + beta*(lp_new - lp_old)^2
    with ratio = exp(lp_new - lp_old).  The front end has no differentiable
    clip/min (`where`/`cmp` are gradient barriers, frontend.py:238-243), so
    the clipped surrogate is replaced by this quadratic trust-region penalty
    (SURVEY H9)."""
    dsl, fe, pdg, tr, rt, ps = recten()
    import recten.symexpr as se
    M, E = minibatches, epochs
    assert B % M == 0
    Bm = B // M
    if lr is None:
        # 0.01 / (Bm * T) made the importance ratio exp(lp_new - lp_old)
        # overflow in the second epoch at full width (weights ~1e14 in the
        # reference's own run); 1e-3 keeps every epoch finite
        lr = 1e-3 / (Bm * T)
    ctx = fe.Context()
    i, Ib = ctx.declare_dim("i", "I")
    e, Eb = ctx.declare_dim("e", "E")
    j, Mb = ctx.declare_dim("j", "M")
    u, Ub = ctx.declare_dim("u", "U")
    b, Bb = ctx.declare_dim("b", "B")
    t, Tb = ctx.declare_dim("t", "T")
    for s, v in ((Ib, I), (Eb, E), (Mb, M), (Ub, Bm), (Bb, B), (Tb, T)):
        ctx.bind(s, v)
    shapes = {"W1": (d_o, H), "b1": (1, H), "W2": (H, H), "b2": (1, H),
              "W3": (H, d_a), "b3": (1, d_a), "Wv": (H, 1), "bv": (1, 1)}
    init = {n: ctx.input(f"{n}_0", s, dtype) for n, s in shapes.items()}
    par = {n: ctx.recurrent(n, s, dtype, (i, e, j)) for n, s in shapes.items()}
    grad = {n: ctx.recurrent(f"g{n}", s, dtype, (i, e, j)) for n, s in shapes.items()}
    cond = {c: se.parse(c, ctx.resolve_symbol) for c in
            ("i == 0 and e == 0 and j == 0", "i >= 1 and e == 0 and j == 0",
             "e >= 1 and j == 0")}
    last = "E - 1,M - 1"

    def sgd(p, g_, at):
        return ctx.detach(p[at]) - ctx.detach(g_[at]) * lr

    for n in shapes:
        par[n].define([(cond["i == 0 and e == 0 and j == 0"], init[n]),
                       (cond["i >= 1 and e == 0 and j == 0"], sgd(par[n], grad[n], f"i-1,{last}")),
                       (cond["e >= 1 and j == 0"], sgd(par[n], grad[n], "i,e-1,M - 1")),
                       (None, sgd(par[n], grad[n], "i,e,j-1"))])
    ctx.register_udf("envstep", dsl.make_udf_fn("envstep", [(1, d_o)], [dtype]),
                     [(1, d_o)], [dtype])

    def trunk(o, p, tag):
        h1 = ctx.op("tanh", [o @ p["W1"] + p["b1"]], name=f"h1{tag}")
        h2 = ctx.op("tanh", [h1 @ p["W2"] + p["b2"]], name=f"h2{tag}")
        mu = ctx.op("add", [h2 @ p["W3"], p["b3"]], name=f"mu{tag}")
        v = ctx.op("add", [h2 @ p["Wv"], p["bv"]], name=f"V{tag}")
        return mu, ctx.sum(ctx.sum(v, 1), 0)

    # rollout at theta[i,0,0]
    p0 = {n: par[n]["i,0,0"] for n in shapes}
    eps = ctx.rng("eps", (1, d_a), dtype, (i, b, t), "normal")
    o = ctx.recurrent("o", (1, d_o), dtype, (i, b, t))
    z0 = ctx.constant(0.1, dtype, (1, d_o), name="z0")
    mu, V = trunk(o, p0, "")
    a = ctx.op("add", [ctx.detach(mu), eps], name="a")
    (onext,) = ctx.udf("envstep", [o, a])
    o.define([(se.eq(se.sym(t), se.cint(0)), z0), (None, onext["i,b,t-1"])])
    r = ctx.sum(ctx.sum(o, 1), 0)
    Vd = ctx.detach(V)
    zero = ctx.constant(0.0, dtype, (), name="vboot")
    Vn = ctx.recurrent("Vn", (), dtype, (i, b, t))
    Vn.define([(se.parse("t == T - 1", ctx.resolve_symbol), zero), (None, Vd["i,b,t+1"])])
    delta = ctx.op("sub", [r + Vn * gamma, Vd], name="delta")
    A = ctx.discounted_sum(delta["i,b,t:T"], gamma * lam, dim=0)
    Rt = ctx.op("add", [A, Vd], name="R")
    d0 = a - ctx.detach(mu)
    lp_old = ctx.sum(ctx.sum(-(d0 * d0) * 0.5, 1), 0)

    # updates at (e, j) on minibatch j: env b = u * M + j
    idx = "i,u * M + j,t"
    mu_n, V_n = trunk(o[idx], par, "_n")
    dn = a[idx] - mu_n
    lp_new = ctx.sum(ctx.sum(-(dn * dn) * 0.5, 1), 0)
    diff = lp_new - ctx.detach(lp_old)[idx]
    ratio = ctx.op("exp", [diff], name="ratio")
    verr = V_n - ctx.detach(Rt)[idx]
    L = ctx.op("add", [-(ratio * ctx.detach(A)[idx]) + verr * verr * cv, diff * diff * beta],
               name="L")
    Lu = ctx.sum(L["i,e,j,u,0:T"], 0)
    Lj = ctx.sum(Lu["i,e,j,0:U"], 0)
    Le = ctx.sum(Lj["i,e,0:M"], 0)
    Li = ctx.sum(Le["i,0:E"], 0)
    loss = ctx.sum(Li["0:I"], 0)
    gr = ctx.backward(loss, [par[n] for n in shapes])
    for n in shapes:
        grad[n].define([(None, gr[par[n]])])
    nxt = {n: ctx.op("sub", [ctx.detach(par[n][f"i,{last}"]),
                             ctx.detach(grad[n][f"i,{last}"]) * lr], name=f"{n}_next")
           for n in shapes}
    for n in shapes:
        ctx.mark_output(nxt[n], f"{n}_next")
    ctx.mark_output(Lj, "loss")
    ctx.mark_output(A, "A")
    return ctx


PPO_PARAMS = ("W1", "b1", "W2", "b2", "W3", "b3", "Wv", "bv")


# ---------------------------------------------------------------------------
# Single-kernel f32 programs for bench_kernels.py (scan / gather rooflines)


def ctx_kernel(name, B=4, T=5, M=2):
    dsl, fe, pdg, tr, rt, ps = recten()
    import recten.symexpr as se
    ctx = fe.Context()
    if name == "k_returns_tb":
        t, Tb = ctx.declare_dim("t", "T")
        b, Bb = ctx.declare_dim("b", "B")
    else:
        if name == "k_gather_mb":
            j, Mb = ctx.declare_dim("j", "M")
            u, Ub = ctx.declare_dim("u", "U")
            ctx.bind(Mb, M)
            ctx.bind(Ub, B // M)
        b, Bb = ctx.declare_dim("b", "B")
        t, Tb = ctx.declare_dim("t", "T")
    ctx.bind(Bb, B)
    ctx.bind(Tb, T)
    if name == "k_returns_bt":
        r = ctx.input("r", (), "f32", (b, t))
        G = ctx.discounted_sum(r["b,t:T"], 0.99, dim=0)
        ctx.mark_output(G, "G")
    elif name == "k_returns_tb":
        r = ctx.input("r", (), "f32", (t, b))
        G = ctx.discounted_sum(r["t:T,b"], 0.99, dim=0)
        ctx.mark_output(G, "G")
    elif name == "k_gae_bt":
        r = ctx.input("r", (), "f32", (b, t))
        V = ctx.input("V", (), "f32", (b, t))
        Vn = ctx.recurrent("Vn", (), "f32", (b, t))
        zero = ctx.constant(0.0, "f32", (), name="vboot")
        Vn.define([(se.parse("t == T - 1", ctx.resolve_symbol), zero), (None, V["b,t+1"])])
        d = ctx.op("sub", [r + Vn * 0.99, V], name="delta")
        A = ctx.discounted_sum(d["b,t:T"], 0.99 * 0.95, dim=0)
        ctx.mark_output(A, "A")
    elif name == "k_gather_mb":
        x = ctx.input("x", (16,), "f32", (b, t))
        y = ctx.op("mul", [x["u * M + j,t"], ctx.constant(1.0, "f32", (), name="one")],
                   name="y")
        ctx.mark_output(y, "y")
    else:
        raise KeyError(name)
    return ctx


KERNEL_NAMES = ("k_returns_bt", "k_returns_tb", "k_gae_bt", "k_gather_mb")
