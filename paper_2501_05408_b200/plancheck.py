"""Check the executor's own plan against polysched's (the reference
scheduler's outputs, reference pkg/src/recten/polysched.py).

The B200 executor derives its loop nest and memory plan itself (planner.py,
memplan.py: lifetimes over the lowered launch program).  polysched computes
the reference's plan for the same graph: a ScheduleFn `theta` (affine
execution times, :92-143), producer -> consumer donations (:767-835) and a
MemOpSet of deallocate / offload / fetch ops anchored on the provably last
consumer (:842-859, :936-1105).  `execute(..., theta=, memops=)` hands them
over; this module checks, for every tensor the executor materialises:

  * deallocation safety: the executor's storage stays live at least until
    the launch that computes polysched's dealloc anchor (the last consumer)
    -- a violation raises PlanError;
  * agreement: the storage dies exactly at that launch ("same point") or
    later (loop-level lifetimes, arena folds);
  * swap: polysched's swap-managed set (`_swap_managed`, :876-877) against
    the executor's swapped buffers;
  * donation: each donated pair is realised when the consumer aliases or is
    fused with the producer, or the producer's storage dies at the
    consumer's launch (its range is free for reuse from there).
The report is kept on the executable (`exe.plan_report`).
"""

from __future__ import annotations


class PlanError(Exception):
    pass


def _node_launch_pcs(prog, labels, g, fused_into):
    """node id -> sorted pcs of the launch instructions that compute it
    (directly, or as a member of a fused group / epilogue)."""
    from . import native as N
    out = {}
    for pc, ins in enumerate(prog):
        if ins[0] != N.RT_OP_LAUNCH:
            continue
        nid = labels[ins[1]][0] if isinstance(labels[ins[1]], tuple) else None
        if nid is None:
            continue
        out.setdefault(nid, []).append(pc)
    for v, root in fused_into.items():
        if root in out and v not in out:
            out[v] = out[root]
    return out


def check(g, bufs, labels, prog, lifetimes, fused_into, theta=None, memops=None,
          swapped=()):
    """Report dict (see module doc); raises PlanError on an unsafe free."""
    names = {n.id: n.name for n in g.nodes.values()}
    pcs = _node_launch_pcs(prog, labels, g, fused_into)
    rep = {}
    if theta is not None:
        from .schedule import _levels, _rows, band_lags
        rep["theta_levels"] = [lev[0] if lev[0] != "band" else f"band({lev[1]})"
                               for lev in _levels(theta)]
        rep["theta_nodes"] = len(_rows(theta))
        sk = band_lags(theta, g)
        rep["theta_skew"] = {names.get(k, str(k)): c for k, c in sk[1] if c} if sk else {}
    if memops is None:
        return rep
    root = {}
    for k, b in bufs.items():
        r = k
        while bufs[r].alias is not None:
            r = bufs[r].alias
        root[k] = r
    d = {"checked": 0, "same_point": 0, "later": 0, "unmaterialized": 0, "unsafe": []}
    for op in memops.ops:
        if op.kind != "deallocate":
            continue
        key = (op.tensor, 0)
        if key not in bufs or root.get(key) not in lifetimes:
            d["unmaterialized"] += 1
            continue
        anchor = op.anchor if op.anchor in pcs else None
        if anchor is None:
            d["unmaterialized"] += 1
            continue
        lo, hi = lifetimes[root[key]]
        a_pc = max(pcs[anchor])
        d["checked"] += 1
        if hi < a_pc:
            d["unsafe"].append((names.get(op.tensor), names.get(anchor), hi, a_pc))
        elif hi == a_pc:
            d["same_point"] += 1
        else:
            d["later"] += 1
    rep["deallocate"] = d
    mgr = getattr(memops, "managed", {}) or {}
    rep["swap"] = {"reference_managed": sorted(names.get(k, str(k)) for k, v in mgr.items()
                                               if v.get("swap")),
                   "executor_swapped": sorted(names.get(k[0], str(k)) for k in swapped)}
    don = getattr(memops, "donations", None) or getattr(g, "_donations", None) or {}
    rep["donation"] = donation_report(don, bufs, root, lifetimes, pcs, fused_into, names)
    if d["unsafe"]:
        raise PlanError(f"executor frees storage before polysched's last consumer: {d['unsafe'][:3]}")
    return rep


def donation_report(donations, bufs, root, lifetimes, pcs, fused_into, names):
    out = {"pairs": len(donations), "aliased_or_fused": 0, "freed_at_consumer": 0, "other": 0}
    for prod, cons in donations.items():
        kp, kc = (prod, 0), (cons, 0)
        if fused_into.get(prod) in (cons, fused_into.get(cons)) or fused_into.get(cons) == prod or \
                (kp in root and kc in root and root[kp] == root[kc]) or kp not in bufs:
            out["aliased_or_fused"] += 1
        elif root.get(kp) in lifetimes and cons in pcs and \
                lifetimes[root[kp]][1] == max(pcs[cons]):
            out["freed_at_consumer"] += 1
        else:
            out["other"] += 1
    return out


def fused_map(exe_like):
    """virtual node -> the node whose launch computes it (fusions, GEMM
    epilogues, contractions, absorbed layouts, GAE)."""
    out = {}
    for v, root in (getattr(exe_like, "fuse_src", None) or {}).items():
        out[v] = root if isinstance(root, int) else getattr(root, "id", root)
    for f, info in (getattr(exe_like, "gemm_epi", None) or {}).items():
        x = info[0]
        out[x] = f
        extra = info[2]
        if isinstance(extra, tuple):
            for m in extra[1:3] + extra[4:6]:
                if isinstance(m, int):
                    out[m] = f
    for s, x in (getattr(exe_like, "contract", None) or {}).items():
        out[x] = s
    plan = getattr(exe_like, "plan", None)
    for s, r in (getattr(plan, "ones_bias", None) or {}).items():
        out[r] = s        # the bias sum computed by its contraction's launch
    # chains (a fused producer of a fused producer) end at a launched node
    for v in list(out):
        seen, r = {v}, out[v]
        while r in out and r not in seen:
            seen.add(r)
            r = out[r]
        out[v] = r
    return out
