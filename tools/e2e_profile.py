"""Where the time of one e2e `execute()` call goes (host phases)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402

import bench  # noqa: E402
from golden_cases import load_graph  # noqa: E402
from paper_2501_05408_b200 import execute, get_executable  # noqa: E402
from paper_2501_05408_b200.workloads import next_inputs  # noqa: E402

WL = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
bench.WL = WL
g = load_graph(WL.graph)
bounds = WL.bounds(WL.local_envs(1))
hin = WL.inputs()
for _ in range(3):
    outs = execute(g, bounds=bounds, inputs=hin, seed=0)
    hin = next_inputs(outs, WL.params())
exe, _ = get_executable(g, bounds, hin, 0)
torch.cuda.synchronize()
T = {"upload": 0.0, "run": 0.0, "status": 0.0, "outputs": 0.0}
n = 5
for _ in range(n):
    t0 = time.perf_counter()
    s = torch.cuda.current_stream()
    exe.upload_inputs(hin, s)
    t1 = time.perf_counter()
    exe.run(hin)          # (uploads again inside run: measured separately above)
    t2 = time.perf_counter()
    t3 = time.perf_counter()
    outs = exe.fetch()
    t4 = time.perf_counter()
    hin = next_inputs(outs, WL.params())
    T["upload"] += t1 - t0
    T["run"] += t2 - t1
    T["status"] += t3 - t2
    T["outputs"] += t4 - t3
print({k: round(v / n * 1e3, 3) for k, v in T.items()}, "ms per call")
t0 = time.perf_counter()
for _ in range(n):
    outs = execute(g, bounds=bounds, inputs=hin, seed=0)
    hin = next_inputs(outs, WL.params())
print("execute():", round((time.perf_counter() - t0) / n * 1e3, 3), "ms per call")
