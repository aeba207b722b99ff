"""Time blocking for long horizons: incrementalization over a DOMAIN dim.

The reference tiles an oversized reduction over a payload axis into DI
blocks along a fresh dim, re-indexes the producer chain by the block, and
adds a final sum over the DI partials (`transforms.incrementalize`,
pkg/src/recten/transforms.py:814-945).  Its per-point programs keep time in
the domain (`G[i,b,t]`), where `find_incrementalizable` (transforms.py:
783-811) finds nothing to tile, so a T=100k REINFORCE backward would keep
every per-step intermediate for every step alive at once.

`block_dim(g, benv, "t", bs)` applies the same rewrite to a domain dim:

  * the region R: top-level (not inside any recurrence) nodes over t whose
    every read along t is at their own t, and whose values are only read
    at the same t or by full-range sums over t (the backward chain of a
    policy-gradient program: per-step products, tanh', dH = dZ W^T ...);
  * t is split as t = kb*bs + tl over two fresh dims kb (DI = T/bs blocks)
    and tl (bs steps): R nodes move to (.., kb, tl), reads of outside
    tensors become `x[.., kb*bs + tl]`;
  * every full-range sum over t of an R node becomes a per-block partial
    over tl (a new kb axis on the sum) plus a `<name>_total` sum over the DI
    partials that takes over the sum's consumers (transforms.py:899-905).

The planner then loops over kb (planner.group_block_loops) and the
storage of every R intermediate folds to one block (executor.find_folds):
peak HBM scales with bs, not T.  Results are the reference's up to the
reassociation of the sums over t (partials per block), within the 1e-5
rel. tolerance of north_star — the same tolerance class as the reference's
own incrementalize tests (1e-12 in f64, pkg/tests/test_transforms.py:
393-459).
"""

from __future__ import annotations

from . import ir
from .planner import Bulk, Planner

BLOCK_KINDS_EXCLUDED = {"input", "const", "rng", "udf", "set_symbol", "eval_symbol", "scan",
                        "cumsum", "discounted_cumsum", "discounted_sum", "window_reduce",
                        "index_select", "slice_axis", "dataflow"}


class BlockError(Exception):
    pass


def _mentions(e, d):
    return (d, "loop") in ir.free_syms(e)


def region(g: ir.Graph, benv: dict, d: str):
    """(R, S): blockable node ids and the full-range sums over d fed by R."""
    T = benv[g.dim_bound[d]]
    full = ("slice", ("int", 0), ("sym", g.dim_bound[d], "bound"))
    plan = Planner(g, benv).plan()
    top = {s.nid for s in plan.steps if isinstance(s, Bulk)}
    out_ids = {nid for _, nid, _ in g.outputs}
    cand = set()
    for nid in top:
        n = g.nodes[nid]
        if d not in n.domain or n.kind in BLOCK_KINDS_EXCLUDED or nid in out_ids:
            continue
        if n.params.get("vec"):
            continue
        ok = True
        for e in g.in_edges(nid):
            src = g.nodes[e.src]
            if d in src.domain and e.phi[src.domain.index(d)] != ("sym", d, "loop"):
                ok = False
                break
        if ok:
            cand.add(nid)

    def reduction_consumer(e):
        s = g.nodes[e.sink]
        src = g.nodes[e.src]
        return (s.kind == "sum" and d not in s.domain and s.id in top
                and e.phi[src.domain.index(d)] in (full, ("slice", ("int", 0), ("int", T))))

    changed = True
    while changed:
        changed = False
        for nid in sorted(cand):
            for e in g.out_edges(nid):
                if e.sink in cand or reduction_consumer(e):
                    continue
                cand.discard(nid)
                changed = True
                break
    sums = set()
    for nid in cand:
        for e in g.out_edges(nid):
            if e.sink not in cand:
                sums.add(e.sink)
    # a partial sum must read R alone (one input) and not be an output
    for s in list(sums):
        if len(g.in_edges(s)) != 1 or s in out_ids:
            raise BlockError(f"{g.nodes[s].name}: reduction over {d} cannot be split")
    return cand, sums


def block_dim(g: ir.Graph, benv: dict, d: str, bs: int):
    """Rewrite g in place; returns the new bound env (adds KB/TL bounds)."""
    T = benv[g.dim_bound[d]]
    if bs <= 0 or T % bs or T // bs < 2:
        raise BlockError(f"block size {bs} must divide {d}'s extent {T} into >= 2 blocks")
    R, S = region(g, benv, d)
    if not R:
        raise BlockError(f"nothing to block along {d}")
    DI = T // bs
    kb, tl = f"{d}_blk", f"{d}_in"
    KB, TL = f"{g.dim_bound[d]}_BLK", f"{g.dim_bound[d]}_IN"
    pos = g.dim_order.index(d)
    g.dim_order = g.dim_order[:pos + 1] + (kb, tl) + g.dim_order[pos + 1:]
    g.dim_bound[kb], g.dim_bound[tl] = KB, TL
    g.bindings[KB], g.bindings[TL] = DI, bs
    benv = dict(benv, **{KB: DI, TL: bs})
    order = {x: i for i, x in enumerate(g.dim_order)}
    t_of = ("add", ("mul", ("sym", kb, "loop"), ("int", bs)), ("sym", tl, "loop"))
    sub = {(d, "loop"): t_of}

    def canon(dims):
        return tuple(sorted(dims, key=order.__getitem__))

    old_dom = {nid: g.nodes[nid].domain for nid in g.nodes}
    for nid in R:
        n = g.nodes[nid]
        n.domain = canon([x for x in n.domain if x != d] + [kb, tl])
        if n.kind == "merge":
            n.params["conds"] = tuple(ir.substitute(c, sub) for c in n.params["conds"])
    for sid in S:
        n = g.nodes[sid]
        n.domain = canon(list(n.domain) + [kb])

    def new_phi(e):
        """Components of e's read, in the (possibly new) source domain."""
        src_dom_old = old_dom[e.src]
        comps = list(e.phi)
        if e.src in R:
            # source moved to (.., kb, tl): its d component splits
            j = src_dom_old.index(d)
            c = comps[j]
            if e.sink in S:
                if c[0] != "slice":
                    raise BlockError("reduction read is not a full slice")
                kb_c, tl_c = ("sym", kb, "loop"), ("slice", ("int", 0), ("sym", TL, "bound"))
            else:
                kb_c, tl_c = ("sym", kb, "loop"), ("sym", tl, "loop")
            rest = {x: comps[i] for i, x in enumerate(src_dom_old) if x != d}
            rest[kb], rest[tl] = kb_c, tl_c
            comps = [rest[x] for x in g.nodes[e.src].domain]
        if e.sink in R:
            comps = [ir.substitute(c, sub) for c in comps]
        return tuple(comps)

    for e in g.edges:
        if e.src in R or e.sink in R:
            e.phi = new_phi(e)
            if e.psi is not None and e.sink in R:
                e.psi = ir.substitute(e.psi, sub)
    # totals over the DI partials take over each split sum's consumers
    nxt = max(g.nodes) + 1
    for sid in sorted(S):
        s = g.nodes[sid]
        dom_tot = old_dom[sid]
        tot = ir.Node(nxt, f"{s.name}_total", "sum", dom_tot, s.out_shapes, s.out_dtypes,
                      {"dims": (0,)}, 1)
        g.nodes[nxt] = tot
        for e in g.edges:
            if e.src == sid:
                e.src = nxt
        g.outputs = [(nm, nxt if nid == sid else nid, oid) for nm, nid, oid in g.outputs]
        phi = tuple(("slice", ("int", 0), ("sym", KB, "bound")) if x == kb else ("sym", x, "loop")
                    for x in s.domain)
        g.edges.append(ir.Edge(nxt, 0, phi, None, 0, sid))
        nxt += 1
    g.block_dims = tuple(getattr(g, "block_dims", ())) + (kb,)
    g.invalidate()
    return benv
