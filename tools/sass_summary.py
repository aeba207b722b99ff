"""Per-kernel SASS mnemonic counts that prove the Blackwell paths (profiling
guide: UTC*MMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st, UTMALDG/UTMASTG/
UBLKCP = TMA / bulk copies, LDGSTS = cp.async, HMMA = legacy mma.sync,
FFMA2 = packed fp32 FMA).  Library kernels from the built .so; the C2 acting
loop from its NVRTC cubin (CPU only: cuobjdump + NVRTC, no GPU needed).

    python tools/sass_summary.py > profiles/r2_sass_summary.txt
"""
import ctypes as C
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

KEYS = ("UTCHMMA", "UTCQMMA", "UTCMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS",
        "HMMA", "FFMA2", "FFMA", "DFMA", "LDS", "STS", "BAR", "SYNCS")


def _demangle(fn):
    """cu++filt, with the anonymous-namespace and parameter noise removed."""
    try:
        out = subprocess.run(["cu++filt", fn], capture_output=True, text=True).stdout.strip()
    except OSError:
        return fn
    out = re.sub(r"\(anonymous namespace\)::", "", out or fn)
    return re.sub(r"\((rt_|tm_|scan_)\w+\)$", "", out)


def summarize(sass_text):
    out = OrderedDict()
    cur = None
    for line in sass_text.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out.setdefault(cur, Counter())
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(1).split(".")[0]
        for k in KEYS:
            if op == k or (k == "UTCHMMA" and op.startswith("UTC") and "MMA" in op):
                out[cur][k] += 1
                break
    return out


def emit(title, counts):
    print(f"== {title}")
    for fn, c in counts.items():
        if not any(c.values()):
            continue
        short = _demangle(fn)
        short = short if len(short) < 72 else short[:69] + "..."
        print(f"  {short:60s} " + " ".join(f"{k}={c[k]}" for k in KEYS if c[k]))


def main():
    so = os.path.join(ROOT, "paper_2501_05408_b200", "_lib", "librtb200.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    emit("librtb200.so (library kernels)", summarize(sass))
    from test_host_logic import dry_lower
    from golden_cases import load_graph
    from paper_2501_05408_b200 import jit, jit_mlp, native as N
    g = load_graph("reinforce_mlp_c2")
    _p, low, _c, _a = dry_lower(g, {"I": 1, "B": 1024, "T": 1000})
    (ri, info), = list(low.loop_subs.items())
    lp = low.recs[ri][1]
    m = jit_mlp.match(lp, info["ops"], info)
    src = jit_mlp.source(lp, info["ops"], info, m)
    lib = N.lib()
    opts = jit._opts()
    blob = b"\0".join(opts) + b"\0"
    size = C.c_uint64(0)
    assert lib.rt_jit_cubin(src.encode(), blob, len(opts), None, C.byref(size)) == 0
    buf = C.create_string_buffer(size.value)
    assert lib.rt_jit_cubin(src.encode(), blob, len(opts), buf, C.byref(size)) == 0
    with tempfile.NamedTemporaryFile(suffix=".cubin") as fh:
        fh.write(buf.raw[:size.value])
        fh.flush()
        sass = subprocess.run(["cuobjdump", "-sass", fh.name], capture_output=True, text=True).stdout
        res = subprocess.run(["cuobjdump", "--dump-resource-usage", fh.name], capture_output=True,
                             text=True).stdout
    emit("loop_mlp (C2 fused acting step, NVRTC)", summarize(sass))
    print("  resources:", " ".join(x for x in res.split() if ":" in x and x.split(":")[0] in
                                   ("REG", "STACK", "SHARED", "LOCAL")))


if __name__ == "__main__":
    main()
