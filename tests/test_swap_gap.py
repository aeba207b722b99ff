"""General swapping across idle gaps (swap.plan_gap_swap; SURVEY §8 a22/a23,
polysched `_swap_managed` :876-877, `augment_memory_ops` :936-1105,
`schedule_memory` :1116-1137).

CPU: the program rewrite (top-level insertion with FOR/END remapping), the
gap finder and the greedy planner on synthetic programs.  GPU: a graph whose
first activation is read again only after a chain of GEMMs; with swap on it
is offloaded across the chain and fetched back, the arena shrinks, the
trace shows OFFLOAD/FETCH in stream order and the results are unchanged."""

import numpy as np
import pytest

from paper_2501_05408_b200 import memplan, native as N
from paper_2501_05408_b200.swap import (gap_candidates, insert_instrs, key_touches,
                                         plan_gap_swap)

L, F, E = N.RT_OP_LAUNCH, N.RT_OP_FOR, N.RT_OP_END


def test_insert_instrs_remaps_loops():
    prog = [(L, 0, 0, 0, 0, 0), (F, 1, 0, 4, 1, 4), (L, 1, 0, 0, 0, 0), (E, 1, 0, 0, 0, 0),
            (L, 2, 0, 0, 0, 0)]
    out = insert_instrs(prog, {1: [(L, 9, 0, 0, 0, 0)], 4: [(L, 8, 0, 0, 0, 0)],
                               5: [(L, 7, 0, 0, 0, 0)]})
    assert [x[:2] for x in out] == [(L, 0), (L, 9), (F, 1), (L, 1), (E, 2), (L, 8), (L, 2), (L, 7)]
    assert out[2][5] == 5          # FOR.e: the pc after its END
    assert out[4][1] == 2          # END.a: the pc of its FOR


def _toy():
    # rec r touches the keys in touch[r]; key A is read at pc 0 and pc 6,
    # B/C/D are gap temporaries; a loop (pcs 2..4) touches B only
    A, B, C, D = ("A", 0), ("B", 0), ("C", 0), ("D", 0)
    fake = {A: 1 << 44, B: 2 << 44, C: 3 << 44, D: 4 << 44}
    touch = [{A, B}, {B, C}, {C}, {C, D}, {D, A}]
    rec_ptrs = [{fake[k] for k in t} for t in touch]
    prog = [(L, 0, 0, 0, 0, 0), (L, 1, 0, 0, 0, 0), (F, 0, 0, 3, 1, 5), (L, 2, 0, 0, 0, 0),
            (E, 2, 0, 0, 0, 0), (L, 3, 0, 0, 0, 0), (L, 4, 0, 0, 0, 0)]
    key_of = {v: k for k, v in fake.items()}
    return prog, rec_ptrs, key_of, (A, B, C, D)


def test_gap_candidates_top_level_segments():
    prog, rec_ptrs, key_of, (A, B, C, D) = _toy()
    t = key_touches(prog, rec_ptrs, key_of)
    assert t[A] == [0, 6] and t[C] == [1, 3, 5]
    cands = gap_candidates(prog, t, [A, B, C, D])
    # A: idle from pc 1 to 5 (offload before pc 1, fetch before pc 6); C is
    # touched inside the loop, so its segment is the loop span: no gap left
    assert cands == [(A, 1, 6)]


def test_plan_gap_swap_lowers_the_arena():
    prog, rec_ptrs, key_of, (A, B, C, D) = _toy()
    sizes = {A: 1000, B: 1000, C: 1000, D: 1000}

    def lifetimes_of(p, ptrs):
        return memplan.lifetimes(p, ptrs, key_of, set())

    base = lifetimes_of(prog, rec_ptrs)
    _, arena0 = memplan.assign(sizes, base)
    chosen, p2, ptrs, life = plan_gap_swap(prog, rec_ptrs, key_of, [A], sizes, base,
                                           memplan.assign, lifetimes_of)
    assert [c[0] for c in chosen] == [A]
    _, arena1 = memplan.assign(sizes, life)
    assert arena1 < arena0
    # offload right after A's first reader, fetch right before its second
    kinds = [(x[0], x[1]) for x in p2]
    assert kinds[1] == (L, 5) and kinds[-2] == (L, 6) and kinds[-1] == (L, 4)
    lo_iv, hi_iv = life[A]
    assert lo_iv == (0, 1) and hi_iv == (len(p2) - 2, len(p2) - 1)


def test_assign_interval_lists_share_a_gap():
    sizes = {"a": 512, "b": 512}
    offs, top = memplan.assign(sizes, {"a": [(0, 1), (5, 6)], "b": (2, 4)})
    assert top == 512 and offs["a"] == offs["b"] == 0


def gap_graph(B, T, H, dt="f32"):
    """y = tanh(x) read by the first GEMM and again at the end, with a
    wider working set in between: m1 = y @ W; a1 = tanh(m1); m2 = a1 @ W;
    m2b = a1 @ W; a2 = tanh(m2 + m2b); m3 = a2 @ W; out = sum(y * m3)."""
    from paper_2501_05408_b200 import ir

    def S(n):
        return ("sym", n, "loop")
    g = ir.Graph(["b", "t"], {"b": "B", "t": "T"}, {"B": B, "T": T})
    dom, pt = ("b", "t"), (S("b"), S("t"))
    nd = [("x", "input", dom, (1, H), 0), ("W", "input", (), (H, H), 0),
          ("y", "tanh", dom, (1, H), 1), ("m1", "matmul", dom, (1, H), 2),
          ("a1", "tanh", dom, (1, H), 1), ("m2", "matmul", dom, (1, H), 2),
          ("m2b", "matmul", dom, (1, H), 2), ("q", "add", dom, (1, H), 2),
          ("a2", "tanh", dom, (1, H), 1), ("m3", "matmul", dom, (1, H), 2),
          ("w", "mul", dom, (1, H), 2), ("s", "sum", (), (1, H), 1)]
    ids = {}
    for i, (name, kind, d, shp, nin) in enumerate(nd):
        params = {"dims": (0, 1)} if kind == "sum" else {}
        g.nodes[i] = ir.Node(i, name, kind, d, (shp,), (dt,), params, nin)
        ids[name] = i
    full = (("slice", ("int", 0), ("sym", "B", "bound")), ("slice", ("int", 0), ("sym", "T", "bound")))
    for snk, srcs in (("y", ["x"]), ("m1", ["y", "W"]), ("a1", ["m1"]), ("m2", ["a1", "W"]),
                      ("m2b", ["a1", "W"]), ("q", ["m2", "m2b"]), ("a2", ["q"]),
                      ("m3", ["a2", "W"]), ("w", ["y", "m3"]), ("s", ["w"])):
        for iid, src in enumerate(srcs):
            phi = () if src == "W" else (full if snk == "s" else pt)
            g.edges.append(ir.Edge(ids[snk], iid, phi, None, 0, ids[src]))
    g.outputs = [("s", ids["s"], 0)]
    return g


@pytest.mark.gpu
def test_gap_swap_on_device():
    from paper_2501_05408_b200 import execute, executor as X, get_executable, trace
    B, T, H = 64, 256, 256
    rng = np.random.default_rng(0)
    x = rng.standard_normal((B, T, 1, H)).astype(np.float32)
    W = (rng.standard_normal((H, H)) / 16).astype(np.float32)
    g = gap_graph(B, T, H)
    X._CACHE.clear()
    plain, _ = get_executable(g, {}, {"x": x, "W": W}, 0)
    X._CACHE.clear()
    exe, _ = get_executable(g, {}, {"x": x, "W": W}, 0, swap=1 << 20)
    names = [exe.trace_names[k] for k, _, _ in exe.gap_swaps]
    assert "y" in names, names
    assert exe.arena_bytes < plain.arena_bytes
    lines = [ln.split()[0] + " " + ln.split()[1] for ln in trace.trace(exe)]
    off, fetch = lines.index("OFFLOAD y"), lines.index("FETCH y")
    # offloaded after its first reader, idle across the GEMM chain, fetched back
    assert lines.index("EXEC m1") < off < fetch
    assert any(ln.startswith("EXEC") for ln in lines[off + 1:fetch])
    assert any(ln.startswith("EXEC") for ln in lines[fetch + 1:])
    st = trace.stats(exe)
    assert st["offloads"] >= 1 and st["fetches"] >= 1 and "y" in st["gap_swaps"]
    out = execute(g, inputs={"x": x, "W": W}, swap=1 << 20)["s"]
    X._CACHE.clear()
    ref = execute(g, inputs={"x": x, "W": W})["s"]
    np.testing.assert_array_equal(out, ref)
    xd = x.astype(np.float64)
    y = np.tanh(xd)
    a1 = np.tanh(y @ W)
    m = np.tanh(a1 @ W + a1 @ W) @ W
    want = (y * m).sum(axis=(0, 1))
    np.testing.assert_allclose(out.astype(np.float64), want, rtol=1e-4, atol=1e-3)
