"""Per-op cycle breakdown of the persistent loop kernel on the C2 workload
(CTA 0's clock64 deltas, accumulated over all steps)."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_cases import load_graph  # noqa: E402
from paper_2501_05408_b200 import get_executable, native as N, roofline as RF  # noqa: E402

import bench  # noqa: E402

WL = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
bench.WL = WL
B = int(sys.argv[2]) if len(sys.argv) > 2 else WL.local_envs(1)
g = load_graph(WL.graph)
inp = {k: torch.from_numpy(v).cuda() for k, v in WL.inputs().items()}
exe, _ = get_executable(g, WL.bounds(B), inp, seed=0)
for ri, info in exe.loop_info.items():
    lp = exe.recs[ri]
    params = exe._params[ri]
    prof = torch.zeros(len(info["ops"]) + 16, dtype=torch.int64, device="cuda")
    params.prof = prof.data_ptr()
    exe.run(inp, graph=False)
    torch.cuda.synchronize()
    prof.zero_()
    exe.run(inp, graph=False)
    torch.cuda.synchronize()
    cyc = prof.cpu().tolist()
    tot = sum(cyc[:len(info["ops"])])
    print(f"loop record {ri}: rows={params.rows} rows_per_cta={params.rows_per_cta} "
          f"smem={params.smem_bytes} trips={info['trips']} hybrid={info.get('hybrid')}")
    fn = getattr(exe.recs[ri], "jit_fn", 0)
    if fn:
        cu = C.CDLL("libcuda.so.1")
        for name, attr in (("regs", 4), ("local_bytes", 3)):
            v = C.c_int(0)
            cu.cuFuncGetAttribute(C.byref(v), attr, C.c_void_p(fn))
            print(f"  jit {name}: {v.value}")
        from paper_2501_05408_b200 import jit as J
        os.makedirs("gpurun_out", exist_ok=True)
        with open(f"gpurun_out/loop_src_{ri}.cu", "w") as fh:
            if info.get("mlp"):
                from paper_2501_05408_b200 import jit_mlp as JM
                fh.write(JM.source(params, info["ops"], info, info["mlp"]))
            else:
                fh.write(J.loop_source(params, info["ops"], "loop_jit", info))
    if info.get("mlp"):
        # fused MLP step (jit_mlp.py): phase probes 0..3, h2 core alone in 6
        # (probe k charges the cycles since the previous probe: 6 = h2 core,
        # 2 = h2 epilogue, 4 = head, 5 = action, 3 = env (+ folded op 0))
        names = [(0, "obs (op 0; 0 when folded into the env step)"), (1, "h1 (op 1)"),
                 (6, "h2 core (mlp_h2q)"), (2, "h2 epilogue"), (4, "head (op 3)"),
                 (5, "action (op 4)"), (3, "env (op 5 [+ op 0 of t+1])")]
        tot = sum(cyc[k] for k, _ in names)
        for k, nm in names:
            print(f"  {nm:46s} cycles/step={cyc[k] / info['trips']:8.0f} share={100 * cyc[k] / max(1, tot):5.1f}%")
        print(f"  total cycles/step {tot / info['trips']:.0f}")
        params.prof = 0
        continue
    for (k, q, re, f64, noise, *_), c in zip(info["ops"], cyc):
        print(f"  {RF.FAMILY.get(k):6s} row_elems={re:5d} cycles/step={c / info['trips']:10.0f} "
              f"share={100 * c / max(1, tot):5.1f}%")
    print(f"  total cycles/step {tot / info['trips']:.0f}")
    extra = cyc[len(info["ops"]):]
    if os.environ.get("RTB200_LOOP_GEMM_PHASES") == "1":
        print("  gemm phases (cycles/step: op start..core start, core, [epilogue = the op line])",
              [round(c / info["trips"]) for c in extra[:15]])
    if any(extra):
        print("  pair GEMM phases (cycles/step):",
              [round(c / info["trips"]) for c in extra[:6]])
    params.prof = 0
prof = exe.profile(inp)
for r in sorted(prof, key=lambda r: -r["ms"])[:6]:
    print(RF.FAMILY.get(r["kernel"]), r["label"], round(r["ms"], 3), "ms")
