"""Kernel-level parity at benchmark scale (sizes the per-point oracle cannot
reach): each test builds a small PDG directly in the executor IR and checks
the CUDA result against a numpy restatement of the reference kernel it
replaces.  fp32 tolerance 1e-5 relative (north_star)."""

import numpy as np
import pytest

from paper_2501_05408_b200 import execute, ir

pytestmark = pytest.mark.gpu


def S(n, k="loop"):
    return ("sym", n, k)


def graph(dims):
    return ir.Graph([d for d, _ in dims], {d: b for d, b in dims}, {b: v for (_, b), v in
                                                                     zip(dims, [None] * len(dims))})


def mm_graph(B, K, N, contract=False, dt="f32"):
    """y[b] = x[b] @ W  (rows GEMM, M = B)      or
       s = sum(permute(x[b]) @ g[b], b)        (contraction GEMM, K = B)."""
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    g.nodes[0] = ir.Node(0, "x", "input", ("b",), ((1, K),), (dt,))
    if not contract:
        g.nodes[1] = ir.Node(1, "W", "input", (), ((K, N),), (dt,))
        g.nodes[2] = ir.Node(2, "y", "matmul", ("b",), ((1, N),), (dt,), {}, 2)
        g.edges += [ir.Edge(2, 0, (S("b"),), None, 0, 0), ir.Edge(2, 1, (), None, 0, 1)]
        g.outputs = [("y", 2, 0)]
    else:
        g.nodes[1] = ir.Node(1, "gr", "input", ("b",), ((1, N),), (dt,))
        g.nodes[2] = ir.Node(2, "xt", "permute", ("b",), ((K, 1),), (dt,), {"order": (1, 0)}, 1)
        g.nodes[3] = ir.Node(3, "op", "matmul", ("b",), ((K, N),), (dt,), {}, 2)
        g.nodes[4] = ir.Node(4, "s", "sum", (), ((K, N),), (dt,), {"dims": (0,)}, 1)
        g.edges += [ir.Edge(2, 0, (S("b"),), None, 0, 0),
                    ir.Edge(3, 0, (S("b"),), None, 0, 2), ir.Edge(3, 1, (S("b"),), None, 0, 1),
                    ir.Edge(4, 0, (("slice", ("int", 0), S("B", "bound")),), None, 0, 3)]
        g.outputs = [("s", 4, 0)]
    return g


def test_tcgen05_rows_gemm_3xtf32():
    B, K, N = 8192, 256, 256
    rng = np.random.default_rng(0)
    x = rng.standard_normal((B, 1, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / 16).astype(np.float32)
    out = execute(mm_graph(B, K, N), inputs={"x": x, "W": W})["y"]
    want = (x.astype(np.float64) @ W.astype(np.float64)).astype(np.float32)
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-5)


def test_tcgen05_contraction_split_k():
    B, K, N = 16384, 256, 256
    rng = np.random.default_rng(1)
    x = rng.standard_normal((B, 1, K)).astype(np.float32)
    gr = rng.standard_normal((B, 1, N)).astype(np.float32)
    out = execute(mm_graph(B, K, N, contract=True), inputs={"x": x, "gr": gr})["s"]
    want = np.einsum("bk,bn->kn", x[:, 0].astype(np.float64), gr[:, 0].astype(np.float64))
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-4 * np.sqrt(B))


def test_suffix_dsum_scan_at_c2_scale():
    """G[b,t] = dsum(r[b,t:T], 0.99) at E=1024, T=1000 (reference
    runtime.py:115-122 per point) == reverse discounted cumsum."""
    Bn, T = 1024, 1000
    g = ir.Graph(["b", "t"], {"b": "B", "t": "T"}, {"B": Bn, "T": T})
    g.nodes[0] = ir.Node(0, "r", "input", ("b", "t"), ((),), ("f32",))
    g.nodes[1] = ir.Node(1, "G", "discounted_sum", ("b", "t"), ((),), ("f32",),
                         {"dim": 0, "gamma": 0.99, "reverse": False}, 1)
    g.edges.append(ir.Edge(1, 0, (S("b"), ("slice", S("t"), S("T", "bound"))), None, 0, 0))
    g.outputs = [("G", 1, 0)]
    r = np.random.default_rng(2).standard_normal((Bn, T)).astype(np.float32)
    out = execute(g, inputs={"r": r})["G"]
    want = np.zeros((Bn, T))
    acc = np.zeros(Bn)
    for t in reversed(range(T)):
        acc = r[:, t].astype(np.float64) + 0.99 * acc
        want[:, t] = acc
    np.testing.assert_allclose(out, want.astype(np.float32), rtol=1e-5, atol=1e-5)


def _kinds(g, inputs):
    from paper_2501_05408_b200 import get_executable
    exe, _ = get_executable(g, None, inputs, seed=0)
    return {r.kernel for r in exe.recs}


@pytest.mark.parametrize("K,N,dt", [(256, 4, "f32"), (16, 256, "f32"), (256, 4, "f64"),
                                    (16, 200, "f32"), (3, 256, "f32")])
def test_thin_contraction(K, N, dt):
    """dW of a narrow layer over all points (frontend.py:766-776 backward):
    RT_K_THIN variant 1 + split-K partial sum."""
    from paper_2501_05408_b200 import native as NN
    B = 20000
    npdt = np.float64 if dt == "f64" else np.float32
    rng = np.random.default_rng(K * 1000 + N)
    x = rng.standard_normal((B, 1, K)).astype(npdt)
    gr = rng.standard_normal((B, 1, N)).astype(npdt)
    g = mm_graph(B, K, N, contract=True, dt=dt)
    assert NN.RT_K_THIN in _kinds(g, {"x": x, "gr": gr})
    out = execute(g, inputs={"x": x, "gr": gr})["s"]
    want = np.einsum("bk,bn->kn", x[:, 0].astype(np.float64), gr[:, 0].astype(np.float64))
    tol = 1e-12 if dt == "f64" else 1e-5
    np.testing.assert_allclose(out, want.astype(npdt), rtol=tol, atol=tol * np.sqrt(B) * 10)


@pytest.mark.parametrize("K,N,B", [(16, 600, 30011), (8, 1000, 4099), (16, 256, 70001), (4, 64, 4100)])
def test_thin_contraction_bulk(K, N, B):
    """Variant 1 streamed by cp.async.bulk (k_thin_contract_bulk): column
    slices of several CTAs (N > 256, ragged last slice), per-row and whole-
    stage copies, a ragged last stage, fewer rows than stages; fp64 numpy."""
    from paper_2501_05408_b200 import get_executable, native as NN
    rng = np.random.default_rng(K * 7 + N + B)
    x = rng.standard_normal((B, 1, K)).astype(np.float32)
    gr = rng.standard_normal((B, 1, N)).astype(np.float32)
    g = mm_graph(B, K, N, contract=True)
    exe, _ = get_executable(g, None, {"x": x, "gr": gr}, seed=0)
    assert any(k == NN.RT_K_THIN and p.variant == 1 and p.vec
               for k, p in zip(exe.kernels, exe._params)), "bulk contraction not lowered"
    out = execute(g, inputs={"x": x, "gr": gr})["s"]
    want = np.einsum("bk,bn->kn", x[:, 0].astype(np.float64), gr[:, 0].astype(np.float64))
    np.testing.assert_allclose(out, want.astype(np.float32), rtol=1e-5, atol=1e-5 * np.sqrt(B) * 10)


@pytest.mark.parametrize("K,N", [(4, 256), (16, 300), (1, 64)])
def test_thin_small_k_rows(K, N):
    """y[b] = x[b] @ W with K <= 32 (write-bound): RT_K_THIN variant 2."""
    from paper_2501_05408_b200 import native as NN
    B = 9000
    rng = np.random.default_rng(K + N)
    x = rng.standard_normal((B, 1, K)).astype(np.float32)
    W = rng.standard_normal((K, N)).astype(np.float32)
    g = mm_graph(B, K, N)
    assert NN.RT_K_THIN in _kinds(g, {"x": x, "W": W})
    out = execute(g, inputs={"x": x, "W": W})["y"]
    want = (x.astype(np.float64) @ W.astype(np.float64)).astype(np.float32)
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("N", [256, 4, 37])
def test_column_reduce(N):
    """bias gradient: s = sum(g[0:B]) over many points (runtime.py:95-96)."""
    B = 50000
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    g.nodes[0] = ir.Node(0, "gr", "input", ("b",), ((N,),), ("f32",))
    g.nodes[1] = ir.Node(1, "s", "sum", (), ((N,),), ("f32",), {"dims": (0,)}, 1)
    g.edges.append(ir.Edge(1, 0, (("slice", ("int", 0), S("B", "bound")),), None, 0, 0))
    g.outputs = [("s", 1, 0)]
    gr = np.random.default_rng(N).standard_normal((B, N)).astype(np.float32)
    out = execute(g, inputs={"gr": gr})["s"]
    want = gr.astype(np.float64).sum(0).astype(np.float32)
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("W", [256, 40])
def test_warp_reduce_per_point(W):
    """s[b] = sum(g[b]) over a W-wide payload axis for many points
    (runtime.py:95-96; warp-per-output mode)."""
    B = 70000
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    g.nodes[0] = ir.Node(0, "gr", "input", ("b",), ((W,),), ("f32",))
    g.nodes[1] = ir.Node(1, "s", "sum", ("b",), ((),), ("f32",), {"dims": (0,)}, 1)
    g.edges.append(ir.Edge(1, 0, (S("b"),), None, 0, 0))
    g.outputs = [("s", 1, 0)]
    gr = np.random.default_rng(W).standard_normal((B, W)).astype(np.float32)
    out = execute(g, inputs={"gr": gr})["s"]
    want = gr.astype(np.float64).sum(1).astype(np.float32)
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("B,K,N,contract", [(5000, 100, 200, False), (9000, 40, 256, False),
                                            (8192, 256, 256, False), (20000, 64, 96, True),
                                            (70000, 256, 256, True), (3001, 256, 520, False)])
def test_tma_gemm_pipeline(B, K, N, contract):
    """TMA-fed tcgen05 pipeline (RT_K_GEMM_TMA): K-major and MN-major
    operands, M/N/K tails, split-K."""
    from paper_2501_05408_b200 import native as NN
    rng = np.random.default_rng(B + K + N)
    x = rng.standard_normal((B, 1, K)).astype(np.float32)
    if contract:
        gr = rng.standard_normal((B, 1, N)).astype(np.float32)
        inp = {"x": x, "gr": gr}
        want = np.einsum("bk,bn->kn", x[:, 0].astype(np.float64), gr[:, 0].astype(np.float64))
        atol = 1e-4 * np.sqrt(B)
    else:
        W = (rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
        inp = {"x": x, "W": W}
        want = x.astype(np.float64) @ W.astype(np.float64)
        atol = 1e-5
    g = mm_graph(B, K, N, contract=contract)
    assert NN.RT_K_GEMM_TMA in _kinds(g, inp)
    out = execute(g, inputs=inp)["s" if contract else "y"]
    np.testing.assert_allclose(out, want.astype(np.float32), rtol=1e-5, atol=atol)


@pytest.mark.parametrize("N,K,dt", [(1, 256, "f32"), (4, 256, "f32"), (2, 100, "f32"),
                                    (4, 256, "f64"), (3, 64, "f64")])
def test_narrow_head_rows_gemm(N, K, dt):
    """Policy/value heads over all points (N <= 4): RT_K_THIN variant 3."""
    B = 20000
    npd = np.float32 if dt == "f32" else np.float64
    rng = np.random.default_rng(N * 100 + K)
    x = rng.standard_normal((B, 1, K)).astype(npd)
    W = (rng.standard_normal((K, N)) / 16).astype(npd)
    out = execute(mm_graph(B, K, N, dt=dt), inputs={"x": x, "W": W})["y"]
    want = (x.astype(np.float64) @ W.astype(np.float64))
    tol = 1e-5 if dt == "f32" else 1e-12
    np.testing.assert_allclose(out, want, rtol=tol, atol=tol)


@pytest.mark.parametrize("N,K,B", [(4, 256, 20011), (1, 128, 9001), (2, 100, 4099), (3, 256, 70003)])
def test_narrow_head_rows_bulk_bit_identical(N, K, B):
    """Variant 3 with rows streamed by cp.async.bulk (k_thin_rows_bulk) gives
    the bits of the register-load kernel (same fma order and reduction), on
    ragged row counts (CTA ranges not multiples of a stage), and matches
    fp64 numpy."""
    from paper_2501_05408_b200 import executor as X, get_executable, lower as L, native as NN
    rng = np.random.default_rng(N * 1000 + K + B)
    x = rng.standard_normal((B, 1, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / 16).astype(np.float32)
    g = mm_graph(B, K, N)
    outs = {}
    cls = [c for c in vars(L).values() if isinstance(c, type) and hasattr(c, "ROWS_BULK")][0]
    saved = cls.ROWS_BULK
    try:
        for bulk in (True, False):
            cls.ROWS_BULK = bulk
            X._CACHE.clear()
            exe, _ = get_executable(g, None, {"x": x, "W": W}, seed=0)
            thin = [p for k, p in zip(exe.kernels, exe._params) if k == NN.RT_K_THIN]
            assert thin and thin[0].variant == 3 and (thin[0].vec == 2) == bulk
            outs[bulk] = execute(g, inputs={"x": x, "W": W})["y"]
    finally:
        cls.ROWS_BULK = saved
        X._CACHE.clear()
    assert np.array_equal(outs[True], outs[False])
    want = x[:, 0].astype(np.float64) @ W.astype(np.float64)
    np.testing.assert_allclose(outs[True][:, 0], want, rtol=1e-5, atol=1e-5)


def _scan_graph(layout, n_env, T, dt, forward):
    """G = dsum over a suffix r[t:T] (reverse scan) or, forward, the
    reversed-weight prefix dsum r[0:t+1] (reference runtime.py:108-122),
    env-major (b,t) or time-major (t,b)."""
    dims = [("b", "B"), ("t", "T")] if layout == "bt" else [("t", "T"), ("b", "B")]
    g = ir.Graph([d for d, _ in dims], dict(dims), {"B": n_env, "T": T})
    dom = tuple(d for d, _ in dims)
    g.nodes[0] = ir.Node(0, "r", "input", dom, ((),), (dt,))
    g.nodes[1] = ir.Node(1, "G", "discounted_sum", dom, ((),), (dt,),
                         {"dim": 0, "gamma": 0.97, "reverse": forward}, 1)
    tsl = ("slice", ("int", 0), ("add", S("t"), ("int", 1))) if forward else \
        ("slice", S("t"), S("T", "bound"))
    phi = tuple(tsl if d == "t" else S(d) for d in dom)
    g.edges.append(ir.Edge(1, 0, phi, None, 0, 0))
    g.outputs = [("G", 1, 0)]
    return g


@pytest.mark.parametrize("layout", ["bt", "tb"])
@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("forward", [False, True])
@pytest.mark.parametrize("n_env,T", [(4096, 1000), (192, 37), (100, 64)])
def test_scan_kernels_layouts(layout, dt, forward, n_env, T):
    """Pipelined tiled scans (line-major / step-major) and their fallbacks
    (ragged lengths, line counts not a multiple of 64) vs a float64 scan."""
    npd = np.float32 if dt == "f32" else np.float64
    shape = (n_env, T) if layout == "bt" else (T, n_env)
    r = np.random.default_rng(T + n_env).standard_normal(shape).astype(npd)
    out = execute(_scan_graph(layout, n_env, T, dt, forward), inputs={"r": r})["G"]
    x = (r if layout == "bt" else r.T).astype(np.float64)
    want = np.zeros_like(x)
    acc = np.zeros(x.shape[0])
    order = range(T) if forward else reversed(range(T))
    for i, t in enumerate(order):
        acc = x[:, t] + (0.97 * acc if i else 0.0)
        want[:, t] = acc
    if layout == "tb":
        want = want.T
    tol = 1e-5 if dt == "f32" else 1e-12
    np.testing.assert_allclose(out, want, rtol=tol, atol=tol * 10)


def _scan_tiles(g, inputs, bounds=None):
    from paper_2501_05408_b200 import get_executable, native as N
    exe, _ = get_executable(g, bounds or {}, inputs, 0)
    return [(p.tile, p.stages) for k, p in zip(exe.kernels, exe._params) if k == N.RT_K_SCAN]


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("stages", [2, 3, 5, 8])
@pytest.mark.parametrize("forward", [False, True])
@pytest.mark.parametrize("n_env,T", [(300, 212), (32, 8), (1, 1000)])
def test_scan_tma_configs(dt, stages, forward, n_env, T, monkeypatch):
    """The TMA scan (k_scan_tma: 32-line x 128-byte boxes on a stage ring,
    TMA stores) at several stage counts, on line counts that are not a
    multiple of the 32-line CTA and lengths that are not a multiple of the
    box width (zero-filled loads, clipped stores), vs a float64 scan; the
    lowering must have picked it (tile 4)."""
    from paper_2501_05408_b200 import executor as X
    monkeypatch.setenv("RTB200_SCAN_STAGES", str(stages))
    X._CACHE.clear()
    npd = np.float32 if dt == "f32" else np.float64
    r = np.random.default_rng(T + stages).standard_normal((n_env, T)).astype(npd)
    g = _scan_graph("bt", n_env, T, dt, forward)
    assert _scan_tiles(g, {"r": r}) == [(4, stages)]
    out = execute(g, inputs={"r": r})["G"]
    x = r.astype(np.float64)
    want = np.zeros_like(x)
    acc = np.zeros(n_env)
    order = range(T) if forward else reversed(range(T))
    for i, t in enumerate(order):
        acc = x[:, t] + (0.97 * acc if i else 0.0)
        want[:, t] = acc
    tol = 1e-5 if dt == "f32" else 1e-12
    np.testing.assert_allclose(out, want, rtol=tol, atol=tol * 10)
    X._CACHE.clear()


@pytest.mark.parametrize("stages", [2, 3, 6])
@pytest.mark.parametrize("B,T", [(4096, 512), (33, 100), (7, 4)])
def test_gae_tma_scan(stages, B, T, monkeypatch):
    """GAE residual formed inside the TMA scan (r and V boxes on one stage
    barrier, V[t+1] carried across boxes in reverse order), ragged boxes."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import executor as X
    monkeypatch.setenv("RTB200_SCAN_STAGES", str(stages))
    X._CACHE.clear()
    rng = np.random.default_rng(B + T + stages)
    r = rng.standard_normal((B, T)).astype(np.float32)
    V = rng.standard_normal((B, T)).astype(np.float32)
    g = load_graph("k_gae_bt")
    assert _scan_tiles(g, {"r": r, "V": V}, {"B": B, "T": T}) == [(4, stages)]
    out = execute(g, bounds={"B": B, "T": T}, inputs={"r": r, "V": V})["A"]
    Vn = np.concatenate([V[:, 1:], np.zeros((B, 1), np.float32)], axis=1)
    delta = (r + Vn * np.float32(0.99)) - V
    want = np.zeros((B, T))
    acc = np.zeros(B)
    for t in reversed(range(T)):
        acc = delta[:, t].astype(np.float64) + (0.99 * 0.95 * acc if t < T - 1 else 0.0)
        want[:, t] = acc
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-5)
    X._CACHE.clear()


def test_scan_pipe_fallback_still_exact(monkeypatch):
    """RTB200_SCAN_TMA=0 keeps the cp.async ring (k_scan_pipe, tile 2)."""
    from paper_2501_05408_b200 import executor as X, lower
    monkeypatch.setattr(lower.Lowering, "SCAN_TMA", False)
    X._CACHE.clear()
    r = np.random.default_rng(5).standard_normal((256, 300)).astype(np.float32)
    g = _scan_graph("bt", 256, 300, "f32", False)
    assert [t for t, _ in _scan_tiles(g, {"r": r})] == [2]
    out = execute(g, inputs={"r": r})["G"]
    want = np.zeros((256, 300))
    acc = np.zeros(256)
    for i, t in enumerate(reversed(range(300))):
        acc = r[:, t] + (0.97 * acc if i else 0.0)
        want[:, t] = acc
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-4)
    X._CACHE.clear()


@pytest.mark.parametrize("K,N,dt", [(16, 256, "f32"), (16, 64, "f64"), (7, 33, "f32")])
def test_gathered_rows_small_k_gemm(K, N, dt):
    """y[j,u,t] = x[u*M + j, t] @ W: minibatch rows gathered by a symbolic
    index (a multi-dim row box, thin variant 2 with K <= 32)."""
    Mb, U, T = 4, 256, 24
    B = Mb * U
    npd = np.float32 if dt == "f32" else np.float64
    g = ir.Graph(["j", "u", "b", "t"], {"j": "M", "u": "U", "b": "B", "t": "T"},
                 {"M": Mb, "U": U, "B": B, "T": T})
    g.nodes[0] = ir.Node(0, "x", "input", ("b", "t"), ((1, K),), (dt,))
    g.nodes[1] = ir.Node(1, "W", "input", (), ((K, N),), (dt,))
    g.nodes[2] = ir.Node(2, "y", "matmul", ("j", "u", "t"), ((1, N),), (dt,), {}, 2)
    bidx = ("add", ("mul", S("u"), S("M", "bound")), S("j"))
    g.edges += [ir.Edge(2, 0, (bidx, S("t")), None, 0, 0), ir.Edge(2, 1, (), None, 0, 1)]
    g.outputs = [("y", 2, 0)]
    rng = np.random.default_rng(K * N)
    x = rng.standard_normal((B, T, 1, K)).astype(npd)
    W = rng.standard_normal((K, N)).astype(npd)
    out = execute(g, inputs={"x": x, "W": W})["y"]
    xs = x.reshape(U, Mb, T, 1, K).transpose(1, 0, 2, 3, 4).astype(np.float64)
    want = xs @ W.astype(np.float64)
    tol = 1e-5 if dt == "f32" else 1e-12
    np.testing.assert_allclose(out, want, rtol=tol, atol=tol)


@pytest.mark.parametrize("B,T", [(4096, 512), (100, 36), (64, 4)])
def test_gae_fused_scan(B, T):
    """A = dsum(delta[t:T], gamma*lam) with delta = r + 0.99*V[t+1] - V
    (bootstrap 0) formed inside the scan kernel (k_scan_gae) == numpy: the
    residual in float32 with numpy's operation order, the discounted sum
    in float64."""
    from golden_cases import load_graph
    rng = np.random.default_rng(B + T)
    r = rng.standard_normal((B, T)).astype(np.float32)
    V = rng.standard_normal((B, T)).astype(np.float32)
    out = execute(load_graph("k_gae_bt"), bounds={"B": B, "T": T}, inputs={"r": r, "V": V})["A"]
    Vn = np.concatenate([V[:, 1:], np.zeros((B, 1), np.float32)], axis=1)
    delta = (r + Vn * np.float32(0.99)) - V
    want = np.zeros((B, T))
    acc = np.zeros(B)
    for t in reversed(range(T)):
        acc = delta[:, t].astype(np.float64) + (0.99 * 0.95 * acc if t < T - 1 else 0.0)
        want[:, t] = acc
    np.testing.assert_allclose(out, want, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("B", [65536, 1 << 20])
def test_tcgen05_long_k_contraction_is_unbiased(B):
    """Long-K tcgen05 contractions drain their TMEM accumulator every 256 K
    into round-to-nearest fp32 registers (k_gemm_tma_drain): positive
    operands (no cancellation to hide it) show no systematic shrink.  Before
    the drain: -2.1e-5 (K=65536) and -7.9e-5 (K=2^20, the C2 dW2 shape)."""
    K, Nn = 256, 256
    rng = np.random.default_rng(B)
    x = rng.random((B, 1, K)).astype(np.float32)
    gr = rng.random((B, 1, Nn)).astype(np.float32)
    out = execute(mm_graph(B, K, Nn, contract=True), inputs={"x": x, "gr": gr})["s"]
    want = np.einsum("bk,bn->kn", x[:, 0].astype(np.float64), gr[:, 0].astype(np.float64))
    rel = (out.astype(np.float64) - want) / want
    assert abs(rel.mean()) < 4e-6, rel.mean()
    assert np.abs(rel).max() < 1e-5, np.abs(rel).max()


@pytest.mark.parametrize("dt,ka,kb", [("f32", 4, 1), ("f64", 4, 1), ("f32", 16, 4)])
def test_summed_gated_products_one_launch(dt, ka, kb):
    """y = (ga @ Wa + gb @ Wb) * (1 - h*h) -- the PPO trunk's d(h2) from the
    policy and value heads (reference frontend.py:961-963 tanh VJP,
    runtime.py:249 matmul) -- runs as ONE small-K thin launch with a second
    product (executor.find_gate_epilogues, k_thin_smallk KP2) and matches
    numpy evaluated in the reference's order (product, product, add, gate)."""
    from paper_2501_05408_b200 import executor as X, get_executable, native as N
    B, H = 8192, 256
    npd = np.float32 if dt == "f32" else np.float64
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    nodes = [("ga", "input", ("b",), (1, ka), 0), ("gb", "input", ("b",), (1, kb), 0),
             ("Wa", "input", (), (ka, H), 0), ("Wb", "input", (), (kb, H), 0),
             ("h", "input", ("b",), (1, H), 0), ("m1", "matmul", ("b",), (1, H), 2),
             ("m2", "matmul", ("b",), (1, H), 2), ("s", "add", ("b",), (1, H), 2),
             ("hh", "mul", ("b",), (1, H), 2), ("one", "const", (), (), 0),
             ("om", "sub", ("b",), (1, H), 2), ("y", "mul", ("b",), (1, H), 2)]
    ids = {}
    for i, (name, kind, dom, shp, nin) in enumerate(nodes):
        params = {"value": np.array(1.0, dtype=npd)} if kind == "const" else {}
        g.nodes[i] = ir.Node(i, name, kind, dom, (shp,), (dt,), params, nin)
        ids[name] = i
    b = (S("b"),)
    for snk, srcs in (("m1", [("ga", b), ("Wa", ())]), ("m2", [("gb", b), ("Wb", ())]),
                      ("s", [("m1", b), ("m2", b)]), ("hh", [("h", b), ("h", b)]),
                      ("om", [("one", ()), ("hh", b)]), ("y", [("s", b), ("om", b)])):
        for iid, (src, phi) in enumerate(srcs):
            g.edges.append(ir.Edge(ids[snk], iid, phi, None, 0, ids[src]))
    g.outputs = [("y", ids["y"], 0)]
    rng = np.random.default_rng(ka * 10 + kb)
    inp = {"ga": rng.standard_normal((B, 1, ka)).astype(npd),
           "gb": rng.standard_normal((B, 1, kb)).astype(npd),
           "Wa": rng.standard_normal((ka, H)).astype(npd),
           "Wb": rng.standard_normal((kb, H)).astype(npd),
           "h": np.tanh(rng.standard_normal((B, 1, H))).astype(npd)}
    X._CACHE.clear()
    exe, _ = get_executable(g, {}, inp, 0)
    thin = [p for k, p in zip(exe.kernels, exe._params) if k == N.RT_K_THIN]
    assert exe.launch_count == 1 and len(thin) == 1 and thin[0].k2 == kb and thin[0].epilogue == 2
    out = execute(g, inputs=inp)["y"]
    a = inp["ga"].astype(np.float64) @ inp["Wa"].astype(np.float64)
    c = inp["gb"].astype(np.float64) @ inp["Wb"].astype(np.float64)
    hv = inp["h"].astype(np.float64)
    want = (a + c) * (1 - hv * hv)
    tol = 1e-5 if dt == "f32" else 1e-12
    np.testing.assert_allclose(out, want, rtol=tol, atol=tol)
    X._CACHE.clear()


@pytest.mark.parametrize("K,Nc,dt,epi", [(16, 256, "f32", "tanh"), (8, 64, "f64", "plain"),
                                         (4, 256, "f32", "plain"), (8, 128, "f64", "tanh"),
                                         (3, 256, "f32", "tanh")])
def test_vectorised_small_k_is_bit_identical(K, Nc, dt, epi, monkeypatch):
    """k_thin_smallv (VW columns per thread, 16-byte stores) computes every
    output with the scalar kernel's operation sequence: bit-identical results
    on gathered minibatch rows, with and without the bias + tanh epilogue."""
    from paper_2501_05408_b200 import executor as X, get_executable, lower, native as N
    Mb, U, T = 4, 256, 24
    B = Mb * U
    npd = np.float32 if dt == "f32" else np.float64
    g = ir.Graph(["j", "u", "b", "t"], {"j": "M", "u": "U", "b": "B", "t": "T"},
                 {"M": Mb, "U": U, "B": B, "T": T})
    g.nodes[0] = ir.Node(0, "x", "input", ("b", "t"), ((1, K),), (dt,))
    g.nodes[1] = ir.Node(1, "W", "input", (), ((K, Nc),), (dt,))
    g.nodes[2] = ir.Node(2, "y", "matmul", ("j", "u", "t"), ((1, Nc),), (dt,), {}, 2)
    bidx = ("add", ("mul", S("u"), S("M", "bound")), S("j"))
    g.edges += [ir.Edge(2, 0, (bidx, S("t")), None, 0, 0), ir.Edge(2, 1, (), None, 0, 1)]
    out_id = 2
    if epi == "tanh":
        g.nodes[3] = ir.Node(3, "bb", "input", (), ((1, Nc),), (dt,))
        g.nodes[4] = ir.Node(4, "z", "add", ("j", "u", "t"), ((1, Nc),), (dt,), {}, 2)
        g.nodes[5] = ir.Node(5, "h", "tanh", ("j", "u", "t"), ((1, Nc),), (dt,), {}, 1)
        jut = (S("j"), S("u"), S("t"))
        g.edges += [ir.Edge(4, 0, jut, None, 0, 2), ir.Edge(4, 1, (), None, 0, 3),
                    ir.Edge(5, 0, jut, None, 0, 4)]
        out_id = 5
    g.outputs = [("out", out_id, 0)]
    rng = np.random.default_rng(K * Nc)
    inp = {"x": rng.standard_normal((B, T, 1, K)).astype(npd),
           "W": rng.standard_normal((K, Nc)).astype(npd)}
    if epi == "tanh":
        inp["bb"] = rng.standard_normal((1, Nc)).astype(npd)
    res = {}
    for vec in (False, True):
        monkeypatch.setattr(lower.Lowering, "THIN_VEC", vec)
        X._CACHE.clear()
        exe, _ = get_executable(g, {}, inp, 0)
        thin = [p for k, p in zip(exe.kernels, exe._params) if k == N.RT_K_THIN]
        assert len(thin) == 1 and thin[0].vec == int(vec), (vec, [t.vec for t in thin])
        res[vec] = execute(g, inputs=inp)["out"]
    np.testing.assert_array_equal(res[True], res[False])
    X._CACHE.clear()


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_bias_gradient_rides_the_weight_contraction(dt):
    """db = sum(dP over the points) and dW = sum(a^T dP) of one layer
    (reference frontend.py VJPs of `+ b` and matmul) in ONE pass over dP:
    the thin contraction carries a column of ones (find_ones_bias), the
    separate column reduction is gone; both match float64 numpy."""
    from paper_2501_05408_b200 import executor as X, get_executable, native as N
    B, K, Nc = 16384, 16, 256
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    g.nodes[0] = ir.Node(0, "a", "input", ("b",), ((1, K),), (dt,))
    g.nodes[1] = ir.Node(1, "P", "input", ("b",), ((1, Nc),), (dt,))
    g.nodes[2] = ir.Node(2, "at", "permute", ("b",), ((K, 1),), (dt,), {"order": (1, 0)}, 1)
    g.nodes[3] = ir.Node(3, "x", "matmul", ("b",), ((K, Nc),), (dt,), {}, 2)
    g.nodes[4] = ir.Node(4, "dW", "sum", (), ((K, Nc),), (dt,), {"dims": (0,)}, 1)
    g.nodes[5] = ir.Node(5, "db", "sum", (), ((1, Nc),), (dt,), {"dims": (0,)}, 1)
    full = (("slice", ("int", 0), S("B", "bound")),)
    g.edges += [ir.Edge(2, 0, (S("b"),), None, 0, 0),
                ir.Edge(3, 0, (S("b"),), None, 0, 2), ir.Edge(3, 1, (S("b"),), None, 0, 1),
                ir.Edge(4, 0, full, None, 0, 3), ir.Edge(5, 0, full, None, 0, 1)]
    g.outputs = [("dW", 4, 0), ("db", 5, 0)]
    npd = np.float32 if dt == "f32" else np.float64
    rng = np.random.default_rng(7)
    inp = {"a": rng.standard_normal((B, 1, K)).astype(npd),
           "P": rng.standard_normal((B, 1, Nc)).astype(npd)}
    X._CACHE.clear()
    exe, _ = get_executable(g, {}, inp, 0)
    thin = [p for k, p in zip(exe.kernels, exe._params) if k == N.RT_K_THIN]
    assert len(thin) == 1 and thin[0].ones == 1
    assert N.RT_K_REDUCE not in exe.kernels
    out = execute(g, inputs=inp)
    a64, p64 = inp["a"][:, 0].astype(np.float64), inp["P"][:, 0].astype(np.float64)
    # fp32 sums of 16 k terms of size ~1: absolute error ~1e-4 where they cancel
    tol = dict(rtol=1e-5, atol=2e-3) if dt == "f32" else dict(rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(out["dW"], a64.T @ p64, **tol)
    np.testing.assert_allclose(out["db"], p64.sum(axis=0, keepdims=True), **tol)
    X._CACHE.clear()


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_bias_gradient_summed_by_the_gate_launch(dt):
    """d(hidden) = (g @ W) * (1 - h*h), its bias gradient sum(d(hidden)) and
    the head's weight gradient sum(h^T g) over the points from ONE launch: the vectorised gate kernel accumulates
    fp64 column sums per CTA (colsum), a split-K pass finishes them; no
    separate column reduction; both match float64 numpy."""
    from paper_2501_05408_b200 import executor as X, get_executable, native as N
    B, K, H = 16384, 4, 256
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    nodes = [("gz", "input", ("b",), (1, K), 0), ("W", "input", (), (K, H), 0),
             ("h", "input", ("b",), (1, H), 0), ("m", "matmul", ("b",), (1, H), 2),
             ("hh", "mul", ("b",), (1, H), 2), ("one", "const", (), (), 0),
             ("om", "sub", ("b",), (1, H), 2), ("y", "mul", ("b",), (1, H), 2),
             ("db", "sum", (), (1, H), 1), ("ht", "permute", ("b",), (H, 1), 1),
             ("xw", "matmul", ("b",), (H, K), 2), ("dW", "sum", (), (H, K), 1)]
    ids = {}
    npd = np.float32 if dt == "f32" else np.float64
    for i, (name, kind, dom, shp, nin) in enumerate(nodes):
        params = {"value": np.array(1.0, dtype=npd)} if kind == "const" else \
            ({"dims": (0,)} if kind == "sum" else ({"order": (1, 0)} if kind == "permute" else {}))
        g.nodes[i] = ir.Node(i, name, kind, dom, (shp,), (dt,), params, nin)
        ids[name] = i
    b = (S("b"),)
    for snk, srcs in (("m", [("gz", b), ("W", ())]), ("hh", [("h", b), ("h", b)]),
                      ("om", [("one", ()), ("hh", b)]), ("y", [("m", b), ("om", b)]),
                      ("db", [("y", (("slice", ("int", 0), S("B", "bound")),))]),
                      ("ht", [("h", b)]), ("xw", [("ht", b), ("gz", b)]),
                      ("dW", [("xw", (("slice", ("int", 0), S("B", "bound")),))])):
        for iid, (src, phi) in enumerate(srcs):
            g.edges.append(ir.Edge(ids[snk], iid, phi, None, 0, ids[src]))
    g.outputs = [("y", ids["y"], 0), ("db", ids["db"], 0), ("dW", ids["dW"], 0)]
    rng = np.random.default_rng(3)
    inp = {"gz": rng.standard_normal((B, 1, K)).astype(npd),
           "W": rng.standard_normal((K, H)).astype(npd),
           "h": np.tanh(rng.standard_normal((B, 1, H))).astype(npd)}
    X._CACHE.clear()
    exe, _ = get_executable(g, {}, inp, 0)
    thin = [p for k, p in zip(exe.kernels, exe._params) if k == N.RT_K_THIN]
    # one launch: d(hidden), its bias gradient (colsum) and the head's weight
    # gradient h^T gz (dw); only split-K finishes after it
    assert len(thin) == 1 and thin[0].colsum == 1 and thin[0].vec == 1 and thin[0].dw == 1
    assert N.RT_K_REDUCE not in exe.kernels
    out = execute(g, inputs=inp)
    y = (inp["gz"][:, 0].astype(np.float64) @ inp["W"].astype(np.float64)) * \
        (1 - inp["h"][:, 0].astype(np.float64) ** 2)
    tol = dict(rtol=1e-5, atol=1e-4) if dt == "f32" else dict(rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(out["y"][:, 0], y, **tol)
    # db sums the kernel's own (rounded) y values in fp64
    np.testing.assert_allclose(out["db"], out["y"][:, 0].astype(np.float64).sum(0, keepdims=True),
                               rtol=1e-6 if dt == "f32" else 1e-13, atol=1e-6 if dt == "f32" else 1e-11)
    np.testing.assert_allclose(out["db"], y.sum(0, keepdims=True), **tol)
    dW = inp["h"][:, 0].astype(np.float64).T @ inp["gz"][:, 0].astype(np.float64)
    np.testing.assert_allclose(out["dW"], dW, **(dict(rtol=1e-5, atol=2e-3) if dt == "f32" else tol))
    X._CACHE.clear()


@pytest.mark.parametrize("dt,n1,n2", [("f32", 4, 1), ("f64", 4, 1), ("f32", 2, 2)])
def test_sibling_heads_share_one_row_stream(dt, n1, n2):
    """mu = h @ W3 + b3 and V = h @ Wv + bv over the same rows (the PPO
    policy and value heads, reference frontend.py matmul/add) from ONE
    row-stream launch that reads h once (find_sibling_rows), vs numpy."""
    from paper_2501_05408_b200 import executor as X, get_executable, native as N
    B, K = 20000, 256
    npd = np.float32 if dt == "f32" else np.float64
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    nodes = [("h", "input", ("b",), (1, K), 0), ("W3", "input", (), (K, n1), 0),
             ("b3", "input", (), (1, n1), 0), ("Wv", "input", (), (K, n2), 0),
             ("bv", "input", (), (1, n2), 0), ("m3", "matmul", ("b",), (1, n1), 2),
             ("mu", "add", ("b",), (1, n1), 2), ("mv", "matmul", ("b",), (1, n2), 2),
             ("V", "add", ("b",), (1, n2), 2)]
    ids = {}
    for i, (name, kind, dom, shp, nin) in enumerate(nodes):
        g.nodes[i] = ir.Node(i, name, kind, dom, (shp,), (dt,), {}, nin)
        ids[name] = i
    b = (S("b"),)
    for snk, srcs in (("m3", [("h", b), ("W3", ())]), ("mu", [("m3", b), ("b3", ())]),
                      ("mv", [("h", b), ("Wv", ())]), ("V", [("mv", b), ("bv", ())])):
        for iid, (src, phi) in enumerate(srcs):
            g.edges.append(ir.Edge(ids[snk], iid, phi, None, 0, ids[src]))
    g.outputs = [("mu", ids["mu"], 0), ("V", ids["V"], 0)]
    rng = np.random.default_rng(n1 * 10 + n2)
    inp = {"h": np.tanh(rng.standard_normal((B, 1, K))).astype(npd),
           "W3": (rng.standard_normal((K, n1)) / 16).astype(npd),
           "b3": rng.standard_normal((1, n1)).astype(npd),
           "Wv": (rng.standard_normal((K, n2)) / 16).astype(npd),
           "bv": rng.standard_normal((1, n2)).astype(npd)}
    X._CACHE.clear()
    exe, _ = get_executable(g, {}, inp, 0)
    thin = [p for k, p in zip(exe.kernels, exe._params) if k == N.RT_K_THIN]
    assert len(thin) == 1 and thin[0].variant == 3 and thin[0].r2 == n2 and exe.launch_count == 1
    out = execute(g, inputs=inp)
    h64 = inp["h"][:, 0].astype(np.float64)
    tol = 1e-5 if dt == "f32" else 1e-12
    np.testing.assert_allclose(out["mu"][:, 0], h64 @ inp["W3"] + inp["b3"], rtol=tol, atol=tol)
    np.testing.assert_allclose(out["V"][:, 0], h64 @ inp["Wv"] + inp["bv"], rtol=tol, atol=tol)
    X._CACHE.clear()


@pytest.mark.gpu
def test_tanh_fast_flush_to_zero_forms_are_bit_identical():
    """tanh_fast (common.cuh) uses ex2/rcp.approx.ftz; over EVERY fp32 bit
    pattern it returns the bits of the __expf/__fdividef formulation it
    replaced (tanh_fast_ref), compiled both with -fmad=false (the JIT loop
    kernels) and with contraction on (the nvcc-built kernels)."""
    import ctypes as C
    import torch
    from paper_2501_05408_b200 import jit
    src = r'''#include "common.cuh"
extern "C" __global__ void tanh_cmp(unsigned long long* bad, unsigned* first) {
  const unsigned long long n = 1ull << 32;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((unsigned)i);
    const unsigned a = __float_as_uint(tanh_fast(x)), b = __float_as_uint(tanh_fast_ref(x));
    const bool nan = x != x;
    if (!nan && a != b) { atomicAdd(bad, 1ull); atomicMin(first, (unsigned)i); }
  }
}'''
    cu = C.CDLL("libcuda.so.1")
    torch.zeros(1, device="cuda")
    for fmad in (False, True):
        opts = jit._opts
        try:
            if fmad:
                jit._opts = lambda: [o for o in opts() if o != b"-fmad=false"] + [b"-fmad=true"]
            fn = jit.compile_kernel(src + f"\n// fmad={fmad}\n", "tanh_cmp")
        finally:
            jit._opts = opts
        bad = torch.zeros(1, dtype=torch.int64, device="cuda")
        first = torch.full((1,), -1, dtype=torch.int32, device="cuda")
        args = [C.c_void_p(bad.data_ptr()), C.c_void_p(first.data_ptr())]
        ptrs = (C.c_void_p * 2)(*[C.cast(C.byref(a), C.c_void_p) for a in args])
        assert cu.cuLaunchKernel(C.c_void_p(fn), 148 * 8, 1, 1, 256, 1, 1, 0, None, ptrs, None) == 0
        torch.cuda.synchronize()
        assert int(bad.item()) == 0, (fmad, int(bad.item()), hex(int(first.item()) & 0xffffffff))
