"""Kernel-level HBM roofline checks for the scan and gather kernels
(north star: returns/GAE scans and symbolic-index gathers at >= 60% of
HBM bandwidth), each at full HBM scale through the executor's public
path (one program per kernel, inputs already resident in HBM).

  returns_bt : G = dsum(r[b, t:T], 0.99), env-major lines  (8 B/step)
  returns_tb : the same, time-major (lines strided by E)   (8 B/step)
  gae_bt     : delta = r + g V[t+1] - V; A = dsum(delta[t:T], g l) (12 B/step)
  gather_mb  : y[j,u,t] = x[u*M + j, t]  (16 floats/row; 2 x row bytes)

Prints one JSON line per program: per-launch device time (event pairs,
median of --reps profiled runs), algorithmic bytes, GB/s and the fraction
of the HBM peak (MEASURED_PEAKS.json, else the profiling guide's fallback).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

E, T = 32768, 1000
CASES = {
    "returns_bt": ("k_returns_bt", {"B": E, "T": T}, 8 * E * T),
    "returns_tb": ("k_returns_tb", {"B": E, "T": T}, 8 * E * T),
    "gae_bt": ("k_gae_bt", {"B": E, "T": T}, 12 * E * T),
    "gather_mb": ("k_gather_mb", {"M": 4, "U": 4096, "B": 16384, "T": 512},
                  2 * 16384 * 512 * 16 * 4),
}


def cpu_numpy_ms(name, bounds):
    """The reference's numpy kernel for the same op on the host (one core):
    `_k_discounted_cumsum` (reference runtime.py:133-146: acc = x[j] + g*acc
    along the axis) for the scans, a fancy-index row gather for the
    minibatch gather (runtime.py:161-179 rows mode)."""
    import time
    rng = np.random.default_rng(0)
    if name.startswith("returns") or name.startswith("gae"):
        E, T = bounds["B"], bounds["T"]
        x = rng.standard_normal((E, T)).astype(np.float32)
        if name == "gae_bt":
            V = rng.standard_normal((E, T)).astype(np.float32)
        t0 = time.perf_counter()
        if name == "gae_bt":
            Vn = np.concatenate([V[:, 1:], np.zeros((E, 1), np.float32)], axis=1)
            x = x + np.float32(0.99) * Vn - V
        g = np.float32(0.9405 if name == "gae_bt" else 0.99)
        xt = np.moveaxis(x, 1, 0) if name != "returns_tb" else x.T
        out = np.empty_like(xt)
        acc = None
        for j in reversed(range(xt.shape[0])):
            acc = xt[j].copy() if acc is None else xt[j] + g * acc
            out[j] = acc
        return (time.perf_counter() - t0) * 1e3
    M, U, B, T = bounds["M"], bounds["U"], bounds["B"], bounds["T"]
    x = rng.standard_normal((B, T, 16)).astype(np.float32)
    t0 = time.perf_counter()
    idx = (np.arange(U)[None, :] * M + np.arange(M)[:, None])
    y = x[idx] * np.float32(1.0)
    del y
    return (time.perf_counter() - t0) * 1e3


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default=None)
    ap.add_argument("--envs", type=int, default=None, help="override E of the scan programs")
    args = ap.parse_args()
    import torch
    from golden_cases import load_graph
    from paper_2501_05408_b200 import get_executable, roofline as RF
    hbm, src = peak()
    for name, (graph, bounds, algo) in CASES.items():
        if args.only and name != args.only:
            continue
        if args.envs and "B" in bounds and name != "gather_mb":
            bounds = dict(bounds, B=args.envs)
            algo = algo // E * args.envs
        g = load_graph(graph)
        gen = torch.Generator(device="cuda").manual_seed(0)
        inputs = {}
        ext = {g.dim_bound[d]: bounds[g.dim_bound[d]] for d in g.dim_order}
        for n in g.sorted_nodes():
            if n.kind == "input":
                shp = tuple(ext[g.dim_bound[d]] for d in n.domain) + tuple(n.out_shapes[0])
                inputs[n.name] = torch.randn(shp, device="cuda", generator=gen)
        exe, _ = get_executable(g, bounds, inputs, seed=0)
        runs = []
        for _ in range(args.reps + 1):
            runs.append(exe.profile(inputs))
        runs = runs[1:]
        recs = []
        for i, r in enumerate(runs[0]):
            if r["count"] == 0:
                continue
            ms = float(np.median([run[i]["ms"] for run in runs]))
            recs.append({"kernel": RF.FAMILY.get(r["kernel"]), "node": r["label"][1],
                         "ms": round(ms, 4), "launches": r["count"]})
        tot = sum(r["ms"] for r in recs)
        gbs = algo / (tot / 1e3) / 1e9
        cpu_ms = cpu_numpy_ms(name, bounds)
        print(json.dumps({"program": name, "bounds": bounds, "algorithmic_bytes": algo,
                          "ms": round(tot, 4), "achieved_gbs": round(gbs, 1),
                          "peak_gbs": hbm, "peak_source": src, "frac": round(gbs / hbm, 3),
                          "kernels": recs,
                          "cpu_numpy": {"ms": round(cpu_ms, 2), "cores": 1,
                                        "gbs": round(algo / (cpu_ms / 1e3) / 1e9, 2)}}))
        del exe
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
