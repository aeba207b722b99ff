"""Execution trace and statistics in the SPEC's reporting format.

The reference specifies (but does not implement) a stats report and a
golden-file trace for its compiled runtime ("peak
device/host bytes, transfer counts/bytes, Execute-event count ... and the
static memory estimate tensor-by-tensor using bytes = prod extents x
dtype-size"; "trace emitted as one event per line `EXEC op point` /
`DEALLOC tensor points` / `FETCH ...` / `OFFLOAD ...`").  Here both come from
the executor's own lowered program:

  * `trace(exe)` walks the program exactly as the C++ VM does
    (csrc/runtime.cu rt_run: FOR/END/ENVMOD/LAUNCH/HOOK) and emits one
    `EXEC` per launch (the node and the slab of points it covers, fixed dims
    at their loop values), `DEALLOC` after the launch that last touches a
    buffer (the memory plan's lifetime end, memplan.py), and `OFFLOAD` /
    `FETCH` for every swap hook (swap.py);
  * `stats(exe)` gives the report as a dict (also `key=value` lines).
"""

from __future__ import annotations

from math import prod

from . import native as N
from .ir import ITEMSIZE


def _slab_text(exe, nid, env):
    n = exe.g.nodes[nid]
    fixed = {d: int(env[exe.slot_of[d]]) for d in exe.fixed_of.get(nid, ()) if d in n.domain}
    parts = []
    for d in n.domain:
        if d in fixed:
            parts.append(f"{d}={fixed[d]}")
        else:
            parts.append(f"{d}=0:{exe.ext[d]}")
    return "[" + ", ".join(parts) + "]"


def trace(exe, max_lines=100000):
    """SPEC trace lines for one run of the executable's program."""
    prog = [(exe.prog[i].op, exe.prog[i].a, exe.prog[i].b, exe.prog[i].c, exe.prog[i].d,
             exe.prog[i].e) for i in range(exe.nprog)]
    ends = {}
    for k, (lo, hi) in exe.lifetimes.items():
        if 0 <= hi < len(prog) and k in exe.trace_names:
            ends.setdefault(hi, []).append(k)
    env = [0] * N.RT_MAXENV
    out = []
    pc = 0
    last_iter = {}
    while pc < len(prog) and len(out) < max_lines:
        op, a, b, c, d, e = prog[pc]
        if op == N.RT_OP_FOR:
            if (b >= c) if d > 0 else (b <= c):
                pc = e
                continue
            env[a] = b
            pc += 1
        elif op == N.RT_OP_END:
            f = prog[a]
            v = env[f[1]] + f[4]
            if (v < f[3]) if f[4] > 0 else (v > f[3]):
                env[f[1]] = v
                pc = a + 1
            else:
                # buffers live across a whole loop die when it finishes
                for k in ends.get(pc, ()):
                    out.append(f"DEALLOC {exe.trace_names[k]} {_full_points(exe, k)}")
                pc += 1
        elif op == N.RT_OP_ENVMOD:
            env[a] = env[b] % c
            pc += 1
        elif op == N.RT_OP_ENVADD:
            env[a] += b
            pc += 1
        elif op == N.RT_OP_LAUNCH and exe.kernels[a] == N.RT_K_MEMCPY:
            # a gap swap (swap.plan_gap_swap): the whole buffer moves
            name, what = exe.labels[a][1].rsplit(":", 1)
            k = next(k for k in exe.trace_names if exe.trace_names[k] == name)
            out.append(f"{'FETCH' if what == 'fetch' else 'OFFLOAD'} {name} {_full_points(exe, k)}")
            pc += 1
        elif op == N.RT_OP_LAUNCH:
            label = exe.labels[a]
            nid = label[0]
            name = label[1]
            slab = _slab_text(exe, nid, env) if nid in exe.g.nodes else ""
            if exe.kernels[a] == N.RT_K_LOOP:
                # a persistent loop launch runs its whole loop range (or one time block)
                lp = exe._params[a]
                dim = [d for d, sl in exe.slot_of.items() if sl == lp.slot][0]
                lo, hi = (env[lp.blk_slot] * lp.blk_len, (env[lp.blk_slot] + 1) * lp.blk_len) \
                    if lp.blk_len else (min(lp.start, lp.stop + 1), max(lp.stop, lp.start + 1))
                slab = slab.replace(f"{dim}=0]", f"{dim}={lo}:{hi}]").replace(
                    f"{dim}=0,", f"{dim}={lo}:{hi},")
            out.append(f"EXEC {name} {slab}")
            # a buffer dies after its last touching launch in its last loop trip
            for k in ends.get(pc, ()):
                key = (k, tuple(env))
                if key in last_iter:
                    continue
                last_iter[key] = True
                out.append(f"DEALLOC {exe.trace_names[k]} {_full_points(exe, k)}")
            pc += 1
        elif op == N.RT_OP_HOOK:
            h = exe.hooks[a]
            kind = h.get("kind", "allreduce")
            if kind == "swap_out":
                for k in exe.swap_plan.keys:
                    out.append(f"OFFLOAD {exe.trace_names[k]} [block {env[h['slot']]}]")
            elif kind == "swap_in":
                kb = env[h["slot"]]
                nxt = [kb] if kb == 0 else []
                if kb + 1 < exe.swap_plan.DI:
                    nxt.append(kb + 1)
                for blk in nxt:
                    for k in exe.swap_plan.keys:
                        out.append(f"FETCH {exe.trace_names[k]} [block {blk}]")
            elif kind == "allreduce":
                out.append(f"ALLREDUCE {h['node']} [{h['count']} values]")
            pc += 1
        else:
            pc += 1
    return out


def _full_points(exe, k):
    b = exe.bufs[k]
    return "[" + ", ".join(f"{d}=0:{x}" for d, x in zip(b.dims, b.dshape)) + "]"


def stats(exe):
    """SPEC collect_stats report."""
    lines = trace(exe, max_lines=1 << 62) if exe.launch_count < 200000 else []
    n_exec = exe.launch_count
    swap = exe.swap_rt
    gaps = getattr(exe, "gap_swaps", [])
    gap_host = getattr(exe, "gap_host_bytes", 0)
    rep = {
        "peak_device_bytes": int(exe.peak_bytes),
        "arena_bytes": int(exe.arena_bytes),
        "naive_device_bytes": int(exe.naive_bytes),
        "peak_host_bytes": (int(swap.host_bytes) if swap else 0) + int(gap_host),
        "offloads": (exe.swap_plan.DI * len(exe.swap_plan.keys) if swap else 0) + len(gaps),
        "fetches": (exe.swap_plan.DI * len(exe.swap_plan.keys) if swap else 0) + len(gaps),
        "bytes_moved": (2 * swap.host_bytes if swap else 0) + 2 * int(gap_host),
        "gap_swaps": [exe.trace_names[k] for k, _, _ in gaps],
        "execute_events": int(n_exec),
        "deallocations": sum(1 for x in lines if x.startswith("DEALLOC")),
        "static_estimate": static_estimate(exe),
    }
    return rep


def static_estimate(exe):
    """Eager footprint per tensor: prod(domain extents) x payload x dtype
    size (the reference's static_tensor_bytes, runtime.py:482-511)."""
    out = {}
    oname = {nid: name for name, nid, oid in exe.g.outputs if oid == 0}
    for n in exe.g.sorted_nodes():
        if n.kind in ("const",):
            continue
        key = (n.id, 0)
        if key not in exe.bufs:
            continue
        b = exe.bufs[key]
        out[oname.get(n.id, n.name)] = prod(b.dshape) * prod(b.pshape) * ITEMSIZE[b.dtype]
    return out


def stats_text(rep):
    """key=value lines."""
    return "\n".join(f"{k}={v}" for k, v in rep.items() if k != "static_estimate")
