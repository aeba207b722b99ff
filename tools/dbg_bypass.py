import os, sys
sys.path[:0] = [".", "tests"]
import numpy as np
from golden_cases import load_case
from paper_2501_05408_b200 import execute, executor as X, planner
c = load_case(sys.argv[1] if len(sys.argv) > 1 else "corpus_running_total_lift_s0")
got = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed)
print(os.environ.get("KNOB"), {k: bool(np.allclose(got[k], c.outputs[k])) for k in c.outputs})
exe, _ = X.get_executable(c.graph(), c.bounds, c.inputs, c.seed)
print(planner.describe(exe.plan.steps, exe.g))
print("labels", exe.labels)
print("fold", {exe.g.nodes[k[0]].name: tuple(b.folded) for k, b in exe.bufs.items() if b.folded})
print("alias", {exe.g.nodes[k[0]].name: exe.g.nodes[b.alias[0]].name for k, b in exe.bufs.items() if b.alias})
