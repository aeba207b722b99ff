"""Debug the full-width parity: run a fw_* golden under lowering variants
and print, per output and per training iteration, the max relative error
against the reference fixture.  python tools/fw_debug.py fw_mlp_f32_I2B1024T8"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from golden_cases import load_case  # noqa: E402
from paper_2501_05408_b200 import execute, executor as X, jit  # noqa: E402


def err(got, want):
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    scale = np.abs(want.astype(np.float64)) + 1e-6
    return float((d / scale).max()), int((d > 1e-5 * np.abs(want) + 1e-6).sum())


def run(name, label, **knobs):
    saved = {}
    for mod, k, v in knobs.get("set", ()):
        saved[(mod, k)] = getattr(mod, k)
        setattr(mod, k, v)
    X._CACHE.clear()
    c = load_case(name)
    try:
        outs = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed)
    finally:
        for (mod, k), v in saved.items():
            setattr(mod, k, v)
    line = [f"{label:22s}"]
    for k, want in sorted(c.outputs.items()):
        got = outs[k]
        if want.ndim >= 1 and want.shape[0] > 1 and k != "loss":
            per = [err(got[i], want[i]) for i in range(want.shape[0])]
            line.append(f"{k}:" + "/".join(f"{e:.1e}({n})" for e, n in per))
        else:
            e, n = err(got, want)
            line.append(f"{k}:{e:.1e}({n})")
    print("  ".join(line), flush=True)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"dbg_{name}_{label}.npz"), **outs)


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for name in sys.argv[1:]:
        print("==", name)
        run(name, "default")
        run(name, "jit_forced", set=[(jit, "JIT_LOOP_MIN", 0), (jit, "JIT_MIN_ELEMS", 0)])
        run(name, "no_jit", set=[(jit, "ENABLED", False)])
        run(name, "no_gate", set=[(X, "GATE_ENABLED", False)])
        os.environ["RTB200_GEMM"] = "tc"
        run(name, "gemm_tc")
        os.environ["RTB200_GEMM"] = "simt"
        run(name, "gemm_simt")
        os.environ["RTB200_GEMM"] = ""
        run(name, "no_fuse", set=[(X, "OPTS", dict(X.OPTS, fuse=False))])
