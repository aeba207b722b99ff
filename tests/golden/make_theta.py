"""Fixtures of polysched's schedule (the reference's ScheduleFn, pkg/src/
recten/polysched.py:92-143, 546-612) for the corpus programs whose band
schedule is skewed, in schedule.theta_json form, so GPU tests can hand the
reference's schedule to execute(..., theta=) without the reference.
Run in the build container: python tests/golden/make_theta.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [HERE, os.path.dirname(os.path.dirname(HERE))]
import programs as P  # noqa: E402
from paper_2501_05408_b200.schedule import theta_json  # noqa: E402

dsl, fe, pdg, tr, rt, ps = P.recten()
os.makedirs(os.path.join(HERE, "theta"), exist_ok=True)
for name in ("nstep2", "nstep4", "stream_window"):
    g = pdg.build(dsl.load_text(P.corpus_text(name)))
    for d, b in g.dim_bound.items():
        g.bindings[b] = 8
    domains, deps, prox = ps.extract(g)
    theta = ps.schedule(domains, deps, prox)
    with open(os.path.join(HERE, "theta", f"{name}.json"), "w") as fh:
        json.dump(theta_json(theta), fh, indent=1, sort_keys=True)
    print(name, theta.levels)
