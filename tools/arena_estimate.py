"""Static HBM plan of a benchmark graph at given bounds, on the CPU (no GPU):
naive bytes (every buffer), arena bytes (the executor's peak), largest
buffers.   python tools/arena_estimate.py reinforce_mlp_c2 '{"I":1,"B":256,"T":100000}'"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from golden_cases import load_graph  # noqa: E402
from paper_2501_05408_b200 import executor as X, memplan, lower as L  # noqa: E402


def plan(g, benv):
    """(prepared graph, bufs, lowering, lifetimes, analysis) of the executor's
    plan at bounds benv, with fake device pointers (no GPU)."""
    h = X.copy_graph(g)
    X.prepare(h, benv)
    an = X.analyze(h, benv, X.payload_shapes(h, benv))
    bufs, virtual = an["bufs"], an["virtual"]
    roots = [k for k, b in bufs.items() if b.alias is None and k[0] not in virtual]
    fake = {k: (i + 1) << 44 for i, k in enumerate(roots)}
    for k, p in fake.items():
        bufs[k].ptr = p
    for k, b in bufs.items():
        r = b
        while r.alias is not None:
            r = bufs[r.alias]
        b.ptr = r.ptr
    low = L.Lowering(an["plan"], bufs, 0, 0, lambda nb: 0, an["contract"], an["fuse_src"],
                     an["gemm_epi"], absorbed=an["absorbed"]).lower()
    key_of = {v: k for k, v in fake.items()}
    rec_ptrs = []
    for ri, (_, p, *_r) in enumerate(low.recs):
        ptrs = memplan.touched_ptrs(p)
        for op in low.loop_subs.get(ri, {}).get("ops", ()):
            ptrs |= memplan.touched_ptrs(op[1])
        rec_ptrs.append({(q >> 44) << 44 for q in ptrs if q >> 44})
    out_keys = {(nid, oid) for _, nid, oid in h.outputs}
    pinned = {k for k in roots if h.nodes[k[0]].kind in ("const", "input")}
    for k in out_keys:
        r = k
        while bufs[r].alias is not None:
            r = bufs[r].alias
        pinned.add(r)
    folds = X.fold_slots(bufs, low.slot)
    life = memplan.lifetimes(low.prog, rec_ptrs, key_of, pinned, folds,
                             hook_ptrs=memplan.hook_touches(low.prog, low.hooks))
    return h, bufs, low, life, an


def estimate(g, benv):
    h = X.copy_graph(g)
    X.prepare(h, benv)
    an = X.analyze(h, benv, X.payload_shapes(h, benv))
    bufs, virtual = an["bufs"], an["virtual"]
    roots = [k for k, b in bufs.items() if b.alias is None and k[0] not in virtual]
    fake = {k: (i + 1) << 44 for i, k in enumerate(roots)}
    for k, p in fake.items():
        bufs[k].ptr = p
    for k, b in bufs.items():
        r = b
        while r.alias is not None:
            r = bufs[r.alias]
        b.ptr = r.ptr
    low = L.Lowering(an["plan"], bufs, 0, 0, lambda nb: 0, an["contract"], an["fuse_src"],
                     an["gemm_epi"], absorbed=an["absorbed"]).lower()
    key_of = {v: k for k, v in fake.items()}
    rec_ptrs = []
    for ri, (_, p, *_r) in enumerate(low.recs):
        ptrs = memplan.touched_ptrs(p)
        for op in low.loop_subs.get(ri, {}).get("ops", ()):
            ptrs |= memplan.touched_ptrs(op[1])
        rec_ptrs.append({(q >> 44) << 44 for q in ptrs if q >> 44})
    out_keys = {(nid, oid) for _, nid, oid in h.outputs}
    pinned = {k for k in roots if h.nodes[k[0]].kind in ("const", "input")}
    for k in out_keys:
        r = k
        while bufs[r].alias is not None:
            r = bufs[r].alias
        pinned.add(r)
    folds = X.fold_slots(bufs, low.slot)
    life = memplan.lifetimes(low.prog, rec_ptrs, key_of, pinned, folds)
    for k in roots:
        life.setdefault(k, (-1, -1))
    sizes = {k: max(1, bufs[k].nbytes) for k in roots}
    offs, arena = memplan.assign(sizes, life)
    top = sorted(roots, key=lambda k: -sizes[k])[:12]
    return {"naive_gb": sum(sizes.values()) / 1e9, "arena_gb": arena / 1e9,
            "largest": [(h.nodes[k[0]].name, round(sizes[k] / 1e9, 3), life[k]) for k in top]}


if __name__ == "__main__":
    g = load_graph(sys.argv[1])
    print(json.dumps(estimate(g, json.loads(sys.argv[2])), indent=1))
