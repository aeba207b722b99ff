"""Print graph nodes (kind, domain, payload, inputs) of a bench workload's
program, recursively to a depth: python tools/show_nodes.py c3 v357 v409 --depth 2"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from golden_cases import load_graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("names", nargs="+")
ap.add_argument("--depth", type=int, default=1)
a = ap.parse_args()
g = load_graph(bench.WORKLOADS[a.workload].graph)
byname = {n.name: n for n in g.nodes.values()}


def show(n, d, seen):
    ins = sorted(g.in_edges(n.id), key=lambda e: e.iid)
    desc = ", ".join(f"{g.nodes[e.src].name}{list(e.phi) if any(not (isinstance(c, tuple) and c[0] == 'sym') for c in e.phi) else ''}" for e in ins)
    extra = {k: v for k, v in n.params.items() if k != "graph"}
    print("  " * (a.depth - d) + f"{n.name}: {n.kind} {n.domain} {n.out_shapes} {extra or ''} <- {desc}")
    if d > 1:
        for e in ins:
            s = g.nodes[e.src]
            if s.id not in seen:
                seen.add(s.id)
                show(s, d - 1, seen)


for nm in a.names:
    show(byname[nm], a.depth, set())
