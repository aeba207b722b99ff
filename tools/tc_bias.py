"""Signed error of the tcgen05 3xTF32 GEMMs vs float64, by accumulation
length: positive operands (no cancellation) expose a systematic bias of the
tensor-core accumulation (round-toward-zero) that random-sign data hides."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from test_gpu_kernels import mm_graph  # noqa: E402
from paper_2501_05408_b200 import execute, executor as X  # noqa: E402

for gem in ("", "simt"):
    os.environ["RTB200_GEMM"] = gem
    for B in (2048, 8192, 65536, 1 << 20):
        X._CACHE.clear()
        rng = np.random.default_rng(B)
        K, Nn = 256, 256
        x = rng.random((B, 1, K)).astype(np.float32)
        gr = rng.random((B, 1, Nn)).astype(np.float32)
        out = execute(mm_graph(B, K, Nn, contract=True), inputs={"x": x, "gr": gr})["s"]
        want = np.einsum("bk,bn->kn", x[:, 0].astype(np.float64), gr[:, 0].astype(np.float64))
        rel = (out.astype(np.float64) - want) / want
        print(f"gemm={gem or 'tma':5s} contraction K={B:8d}: mean signed rel {rel.mean():+.2e}  max |rel| {np.abs(rel).max():.2e}",
              flush=True)
    for K in (256, 1024):
        X._CACHE.clear()
        rng = np.random.default_rng(K)
        Bn = 8192
        x = rng.random((Bn, 1, K)).astype(np.float32)
        W = rng.random((K, 256)).astype(np.float32)
        out = execute(mm_graph(Bn, K, 256), inputs={"x": x, "W": W})["y"]
        want = x[:, 0].astype(np.float64) @ W.astype(np.float64)
        rel = (out[:, 0].astype(np.float64) - want) / want
        print(f"gemm={gem or 'tma':5s} rows M={Bn} K={K:5d}: mean signed rel {rel.mean():+.2e}  max |rel| {np.abs(rel).max():.2e}",
              flush=True)
