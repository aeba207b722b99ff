"""Debug helper: run one TMA GEMM small enough to inspect."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2501_05408_b200 import execute, lower as L  # noqa
from test_gpu_kernels import mm_graph  # noqa
L.Lowering.TC_MIN_MACS = 0
B, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
contract = len(sys.argv) > 4
rng = np.random.default_rng(0)
x = rng.standard_normal((B, 1, K)).astype(np.float32)
if contract:
    gr = rng.standard_normal((B, 1, N)).astype(np.float32)
    inp = {"x": x, "gr": gr}
    want = np.einsum("bk,bn->kn", x[:, 0].astype(np.float64), gr[:, 0].astype(np.float64))
else:
    W = rng.standard_normal((K, N)).astype(np.float32)
    inp = {"x": x, "W": W}
    want = x[:, 0].astype(np.float64) @ W.astype(np.float64)
    print("x[0,:4]", x[0, 0, :4], "W[0,:4]", W[0, :4])
out = execute(mm_graph(B, K, N, contract=contract), inputs=inp)["s" if contract else "y"]
out = out.reshape(want.shape)
print("out[0,:4]", out[0, :4], "want", want[0, :4])
err = np.abs(out - want) / (np.abs(want) + 1e-3)
print("max rel err", err.max(), "frac bad", (err > 1e-4).mean())
