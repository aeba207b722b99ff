"""Static HBM memory plan for a lowered program: lifetimes -> arena offsets.

The reference *plans* deallocation and donation (polysched.py:767-1137:
`donation_analysis`, `augment_memory_ops`, `schedule_memory`) but never
executes them.  Here they are realised for the executor's own
loop nest:

  * deallocation: a buffer's storage is released after its last touching
    launch (program order; a touch inside a loop with more than one trip
    keeps the buffer live for the whole outermost such loop, because full-
    domain buffers carry values across iterations);
  * donation: pass-through nodes alias their producer (executor.find_aliases)
    and fused producers never get storage at all;
  * reuse: released ranges are handed to later buffers by best-fit over an
    interval graph, so the arena size IS the peak HBM of a run.

Inputs and constants are live for the whole program (uploaded before it).
"""

from __future__ import annotations

from . import native as N

ALIGN = 256


def touched_ptrs(params) -> set:
    """Every u64 field named ptr/part found in a parameter block."""
    out = set()

    def walk(obj):
        for name, ctype in getattr(obj, "_fields_", ()):
            v = getattr(obj, name)
            if name in ("ptr", "part") and isinstance(v, int):
                if v:
                    out.add(v)
            elif hasattr(v, "_fields_"):
                walk(v)
            elif hasattr(v, "_length_") and hasattr(v, "_type_") and \
                    hasattr(v._type_, "_fields_"):
                for x in v:
                    walk(x)
    walk(params)
    return out


def loop_spans(prog):
    """[(for_pc, end_pc, trips, env slot)] for every loop of a lowered program."""
    spans, stack = [], []
    for pc, ins in enumerate(prog):
        if ins[0] == N.RT_OP_FOR:
            stack.append((pc, abs(ins[3] - ins[2]), ins[1]))
        elif ins[0] == N.RT_OP_END:
            a, trips, slot = stack.pop()
            spans.append((a, pc, trips, slot))
    return spans


def hook_touches(prog, hooks):
    """pc -> buffer pointers an all-reduce hook reads and writes there.  A
    bucketed hook (lower._bucket_allreduces) defers its collective to the
    flushing hook of its run, so its buffer is touched at that pc too."""
    out, pending = {}, set()
    for pc, ins in enumerate(prog):
        if ins[0] != N.RT_OP_HOOK:
            continue
        h = hooks[ins[1]]
        if h.get("kind", "allreduce") != "allreduce" or "ptr" not in h:
            continue
        pending.add(h["ptr"])
        out.setdefault(pc, set()).add(h["ptr"])
        if h.get("flush", True):
            out[pc] |= pending
            pending = set()
    return out


def lifetimes(prog, rec_ptrs, key_of_ptr, pinned, folds=None, hook_ptrs=None):
    """key -> (first pc, last pc).  A buffer folded along a loop's dim
    (executor.find_folds: produced and consumed within one iteration) is
    not kept live across that loop's iterations.  hook_ptrs (pc -> ptrs,
    hook_touches) extends buffers to the hooks that all-reduce them."""
    folds = folds or {}
    hook_ptrs = hook_ptrs or {}
    spans = [s for s in loop_spans(prog) if s[2] > 1]
    touch = {}
    for pc, ins in enumerate(prog):
        if ins[0] == N.RT_OP_HOOK:
            ptrs = {(q >> 44) << 44 for q in hook_ptrs.get(pc, ())}
        elif ins[0] == N.RT_OP_LAUNCH:
            ptrs = rec_ptrs[ins[1]]
        else:
            continue
        for p in ptrs:
            k = key_of_ptr.get(p)
            if k is None:
                continue
            lo, hi = touch.get(k, (pc, pc))
            touch[k] = (min(lo, pc), max(hi, pc))
    end = len(prog)
    out = {}
    for k, (lo, hi) in touch.items():
        # outermost multi-trip loop containing any touch
        fs = folds.get(k, ())
        for a, b, _, slot in spans:
            if slot in fs:
                continue
            if a <= lo <= b or a <= hi <= b:
                lo, hi = min(lo, a), max(hi, b)
        out[k] = (lo, hi)
    for k in pinned:
        out[k] = (-1, end + 1)
    return out


def _ivals(x):
    """A lifetime: (lo, hi), or a list of them (a buffer swapped out across
    an idle gap, swap.plan_gap_swap, is live in two intervals)."""
    return [x] if isinstance(x, tuple) else list(x)


def assign(sizes: dict, life: dict):
    """Best-fit offsets for interval lists; returns (offsets, arena bytes)."""
    order = sorted(sizes, key=lambda k: (-sizes[k], _ivals(life[k])[0][0]))
    placed = []   # (off, size, [(lo, hi)])
    offs = {}
    top = 0
    for k in order:
        sz = (sizes[k] + ALIGN - 1) // ALIGN * ALIGN
        mine = _ivals(life[k])
        busy = sorted((o, s) for (o, s, iv) in placed
                      if any(not (b < lo or hi < a) for lo, hi in mine for a, b in iv))
        best, cur = None, 0
        for o, s in busy:
            if o - cur >= sz and (best is None or (o - cur) < best[1]):
                best = (cur, o - cur)
            cur = max(cur, o + s)
        off = best[0] if best else cur
        offs[k] = off
        placed.append((off, sz, mine))
        top = max(top, off + sz)
    return offs, top
