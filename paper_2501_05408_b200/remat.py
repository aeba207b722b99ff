"""Rematerialisation of acting-loop activations for the backward
(long horizons: SURVEY §8 a22, C4).

A time-blocked long-horizon program swaps the acting recurrence's outputs
that the backward reads (swap.py): at E = 256, T = 100k the two 256-wide
tanh layers are 26 GB each and their offload + fetch made C4 PCIe-bound
(106 GB over the bus per step).  Those layers are cheap functions of what
the backward keeps anyway -- the 16-wide observation o and the iteration's
weights:  h1 = tanh(o W1 + b1), h2 = tanh(h1 W2 + b2).  This pass gives the
backward its own copies of such chains (matmul -> + bias -> tanh rooted at
a recurrent state, the weights loop-invariant along the recurrence), so the
loop's layers are read only inside the loop (one slot of storage) and the
backward recomputes them block by block on the tensor cores.  The values
differ from the loop's by the GEMM's rounding (3xTF32 vs the loop's fp32
FMA chain; ~1e-7 relative), well inside the fp32 parity bound.
"""

from __future__ import annotations

from . import ir
from .ir import Graph


def _ident(e, src, snk):
    return e.psi is None and src.domain == snk.domain and \
        e.phi == tuple(("sym", d, "loop") for d in src.domain)


def _reach(g, start, fwd=True):
    seen, work = set(), [start]
    while work:
        v = work.pop()
        for e in (g.out_edges(v) if fwd else g.in_edges(v)):
            w = e.sink if fwd else e.src
            if w not in seen:
                seen.add(w)
                work.append(w)
    return seen


def remat_chains(g: Graph, dim: str):
    """Clone the tanh-layer chains of the recurrence over `dim` for their
    readers outside it.  Returns {original layer id: clone id}."""
    # the recurrence: nodes on a cycle through an edge that reads dim - 1
    rec = set()
    for e in g.edges:
        src = g.nodes[e.src]
        if dim in src.domain and e.phi and e.phi[src.domain.index(dim)] != ("sym", dim, "loop"):
            cyc = _reach(g, e.sink) & _reach(g, e.src, fwd=False)
            if e.src in cyc or e.src == e.sink:
                rec |= cyc | {e.src, e.sink}
    if not rec:
        return {}

    def layer(t):
        """(matmul, add, x edge, w edge, b edge) if t = tanh(add(matmul(x, w), b))."""
        if t.kind != "tanh" or len(g.in_edges(t.id)) != 1:
            return None
        ea = g.in_edges(t.id)[0]
        ad = g.nodes[ea.src]
        if ad.kind != "add" or not _ident(ea, ad, t) or len(g.in_edges(ad.id)) != 2:
            return None
        ins = sorted(g.in_edges(ad.id), key=lambda e: e.iid)
        mm_e = [e for e in ins if g.nodes[e.src].kind == "matmul" and _ident(e, g.nodes[e.src], ad)]
        if len(mm_e) != 1:
            return None
        be = [e for e in ins if e is not mm_e[0]][0]
        mm = g.nodes[mm_e[0].src]
        mins = sorted(g.in_edges(mm.id), key=lambda e: e.iid)
        if len(mins) != 2 or not _ident(mins[0], g.nodes[mins[0].src], mm):
            return None
        xe, we = mins
        # weights and bias: no dependence on the recurrence dim
        for e in (we, be):
            if dim in g.nodes[e.src].domain:
                return None
        return mm, ad, xe, we, be

    clones = {}
    nxt = max(g.nodes) + 1

    def clone_of(x_id):
        return clones.get(x_id, x_id)

    # in dependence order: a chain may feed the next (h1 -> h2)
    for t in g.sorted_nodes():
        if t.id not in rec:
            continue
        lay = layer(t)
        if lay is None:
            continue
        mm, ad, xe, we, be = lay
        if mm.id not in rec or ad.id not in rec:
            continue
        x_src = xe.src
        if g.nodes[x_src].kind == "tanh" and x_src in rec and x_src not in clones:
            continue      # its operand is a loop layer without a copy: keep the swap
        outside = [e for e in g.out_edges(t.id) if e.sink not in rec]
        if not outside:
            continue
        ids = {}
        for old in (mm, ad, t):
            n = ir.Node(nxt, f"{old.name}_re", old.kind, old.domain, old.out_shapes,
                        old.out_dtypes, dict(old.params), old.nin)
            g.nodes[nxt] = n
            ids[old.id] = nxt
            nxt += 1
        g.edges.append(ir.Edge(ids[mm.id], xe.iid, xe.phi, xe.psi, xe.oid, clone_of(x_src)))
        g.edges.append(ir.Edge(ids[mm.id], we.iid, we.phi, we.psi, we.oid, we.src))
        ea = [e for e in g.in_edges(ad.id) if e.src == mm.id][0]
        g.edges.append(ir.Edge(ids[ad.id], ea.iid, ea.phi, ea.psi, 0, ids[mm.id]))
        g.edges.append(ir.Edge(ids[ad.id], be.iid, be.phi, be.psi, be.oid, be.src))
        g.edges.append(ir.Edge(ids[t.id], 0, g.in_edges(t.id)[0].phi, None, 0, ids[ad.id]))
        for e in outside:
            e.src = ids[t.id]
        clones[t.id] = ids[t.id]
        g.invalidate()
    return clones
