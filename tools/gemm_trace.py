"""Per-role stage timeline of the persistent tcgen05 GEMM (CTA 0), from a
build with -DTM_TRACE=1 (RTB200_NVCC_EXTRA): producer issue, converter sees
the stage, converter done, MMA start, MMA commit; epilogue accumulator-ready
per tile.  python tools/gemm_trace.py [rows]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from test_gpu_kernels import mm_graph  # noqa: E402
from paper_2501_05408_b200 import execute, native as N  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
TANH = "--tanh" in sys.argv
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((B, 1, 256)).astype(np.float32)).cuda()
W = torch.from_numpy((rng.standard_normal((256, 256)) / 16).astype(np.float32)).cuda()
inp = {"x": x, "W": W}
if TANH:
    # y = tanh(x @ W + b): the bias + tanh epilogue of the learner's forward
    from paper_2501_05408_b200 import ir
    g = mm_graph(B, 256, 256)
    S = ("sym", "b", "loop")
    g.nodes[3] = ir.Node(3, "bb", "input", (), ((1, 256),), ("f32",))
    g.nodes[4] = ir.Node(4, "z", "add", ("b",), ((1, 256),), ("f32",), {}, 2)
    g.nodes[5] = ir.Node(5, "h", "tanh", ("b",), ((1, 256),), ("f32",), {}, 1)
    g.edges += [ir.Edge(4, 0, (S,), None, 0, 2), ir.Edge(4, 1, (), None, 0, 3),
                ir.Edge(5, 0, (S,), None, 0, 4)]
    g.outputs = [("h", 5, 0)]
    inp["bb"] = torch.zeros((1, 256), device="cuda")
elif "--gate" in sys.argv:
    # y = (x @ W) * (1 - h*h): the gated dX GEMM of the backward
    from paper_2501_05408_b200 import ir
    g = mm_graph(B, 256, 256)
    S = ("sym", "b", "loop")
    g.nodes[3] = ir.Node(3, "hg", "input", ("b",), ((1, 256),), ("f32",))
    g.nodes[4] = ir.Node(4, "hh", "mul", ("b",), ((1, 256),), ("f32",), {}, 2)
    g.nodes[5] = ir.Node(5, "one", "const", (), ((),), ("f32",), {"value": np.array(1.0, np.float32)})
    g.nodes[6] = ir.Node(6, "om", "sub", ("b",), ((1, 256),), ("f32",), {}, 2)
    g.nodes[7] = ir.Node(7, "yg", "mul", ("b",), ((1, 256),), ("f32",), {}, 2)
    g.edges += [ir.Edge(4, 0, (S,), None, 0, 3), ir.Edge(4, 1, (S,), None, 0, 3),
                ir.Edge(6, 0, (), None, 0, 5), ir.Edge(6, 1, (S,), None, 0, 4),
                ir.Edge(7, 0, (S,), None, 0, 2), ir.Edge(7, 1, (S,), None, 0, 6)]
    g.outputs = [("yg", 7, 0)]
    inp["hg"] = torch.tanh(torch.randn((B, 1, 256), device="cuda"))
else:
    g = mm_graph(B, 256, 256)
for _ in range(3):
    execute(g, inputs=inp, device_outputs=True)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
execute(g, inputs=inp, device_outputs=True)
t1.record()
torch.cuda.synchronize()
print("call ms", t0.elapsed_time(t1))
buf = (C.c_longlong * (10 * 512))()
lib = N.lib()
assert lib.rt_gemm_tma_trace(buf, 10 * 512) == 0, "build with -DTM_TRACE=1"
tr = np.array(buf[:], dtype=np.int64).reshape(10, 512)
base = tr[0, 0]
names = ["issue", "conv_sees", "mma_start", "mma_commit", "conv_done"]
print("stage  " + "  ".join(f"{n:>10s}" for n in names))
for gidx in list(range(0, 20)) + list(range(200, 216)):
    print(f"{gidx:5d}  " + "  ".join(f"{(tr[r, gidx] - base) / 1e3:10.2f}" for r in range(5)))
acc = tr[5, :40]
print("epilogue acc ready (us):", [round((a - base) / 1e3, 1) for a in acc[:20] if a])
d = np.diff(tr[2, 16:400]) / 1e3
print("MMA start spacing us: median", np.median(d), "mean", d.mean())
lat = (tr[1, :400] - tr[0, :400]) / 1e3
print("issue -> converter sees (us): median", np.median(lat), "p90", np.percentile(lat, 90))
wait = (tr[0, 4:400] - tr[3, :396]) / 1e3
print("commit(g) -> issue(g+4) (us): median", np.median(wait))

ep0, ep1 = tr[6, :128], tr[7, :128]
print("epilogue warp 0, tiles 2-3: chunk LDTM-done / stored (us rel. to acc ready)")
for t in (2, 3):
    a0 = tr[5, t]
    print("  (compute done, store-buffer free) tile", t,
          [(round((tr[8, t * 16 + c] - a0) / 1e3, 2), round((tr[9, t * 16 + c] - a0) / 1e3, 2))
           for c in range(8)])
    print("  tile", t, [(round((ep0[t * 16 + c] - a0) / 1e3, 2), round((ep1[t * 16 + c] - a0) / 1e3, 2))
                        for c in range(8)])
