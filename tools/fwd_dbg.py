import sys, os
sys.path[:0]=['.', 'tests']
import numpy as np
from golden_cases import load_graph
from paper_2501_05408_b200 import execute, jit
from paper_2501_05408_b200.workloads import mlp_inputs
bounds = {"I": 1, "B": int(sys.argv[1]), "T": 48}
jit.JIT_LOOP_MIN = 1 << 40
ref = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=1)
for fw in (False, True):
    jit.JIT_LOOP_MIN = 0
    jit.FORWARD_ENABLED = fw
    got = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=1)
    print("forward", fw, {k: float(np.max(np.abs(got[k] - ref[k]) / (np.abs(ref[k]) + 1e-6))) for k in ref})
