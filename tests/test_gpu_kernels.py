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


def mm_graph(B, K, N, contract=False):
    """y[b] = x[b] @ W  (rows GEMM, M = B)      or
       s = sum(permute(x[b]) @ g[b], b)        (contraction GEMM, K = B)."""
    g = ir.Graph(["b"], {"b": "B"}, {"B": B})
    g.nodes[0] = ir.Node(0, "x", "input", ("b",), ((1, K),), ("f32",))
    if not contract:
        g.nodes[1] = ir.Node(1, "W", "input", (), ((K, N),), ("f32",))
        g.nodes[2] = ir.Node(2, "y", "matmul", ("b",), ((1, N),), ("f32",), {}, 2)
        g.edges += [ir.Edge(2, 0, (S("b"),), None, 0, 0), ir.Edge(2, 1, (), None, 0, 1)]
        g.outputs = [("y", 2, 0)]
    else:
        g.nodes[1] = ir.Node(1, "gr", "input", ("b",), ((1, N),), ("f32",))
        g.nodes[2] = ir.Node(2, "xt", "permute", ("b",), ((K, 1),), ("f32",), {"order": (1, 0)}, 1)
        g.nodes[3] = ir.Node(3, "op", "matmul", ("b",), ((K, N),), ("f32",), {}, 2)
        g.nodes[4] = ir.Node(4, "s", "sum", (), ((K, N),), ("f32",), {"dims": (0,)}, 1)
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
