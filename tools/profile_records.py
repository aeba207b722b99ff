"""Per-launch-record device times of one step of a bench workload (event
pair around every launch), sorted, with kernel family, node and shape.
    python tools/profile_records.py c3"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from golden_cases import load_graph  # noqa: E402
from paper_2501_05408_b200 import get_executable, roofline as RF  # noqa: E402

WL = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
bench.WL = WL
B = WL.local_envs(1)
g = load_graph(WL.graph)
inp = {k: torch.from_numpy(v).cuda() for k, v in WL.inputs().items()}
exe, _ = get_executable(g, WL.bounds(B), inp, seed=0, block=WL.block, swap=WL.swap)
exe.profile(inp)
prof = exe.profile(inp)
tot = sum(r["ms"] for r in prof)
for r in sorted(prof, key=lambda r: -r["ms"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    b, f = RF.cost(r["kernel"], r["params"], exe.loop_info.get(r["rec"]))
    per = r["ms"] / max(1, r["count"])
    print(f"{r['ms']:8.3f} ms {100 * r['ms'] / tot:5.1f}% x{r['count']:<5d} {RF.FAMILY.get(r['kernel']):8s} "
          f"{r['label'][1]:14s} {b / 1e6 / max(1, 1):9.1f} MB/launch {b / (per / 1e3) / 1e9 if per else 0:7.0f} GB/s "
          f"{f / (per / 1e3) / 1e12 if f and per else 0:6.1f} TF/s grid={exe.recs[r['rec']].grid[0]}")
print(f"total {tot:.3f} ms")
