"""Run one golden case through the executor and print per-output errors
against the reference's own outputs (GPU debugging aid).

    python tools/debug_case.py <case> [env knobs via RTB200_NOFUSE/NOFOLD/...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from golden_cases import load_case  # noqa: E402
from paper_2501_05408_b200 import execute  # noqa: E402

c = load_case(sys.argv[1])
got = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed)
for k, want in c.outputs.items():
    g = np.asarray(got[k], np.float64)
    w = np.asarray(want, np.float64)
    err = np.abs(g - w) / (np.abs(w) + 1e-6)
    bad = np.argwhere(err > 1e-5)
    print(f"{k:10s} shape={w.shape} max_rel={err.max():.3e} nbad={len(bad)} first={bad[:3].tolist()}")
