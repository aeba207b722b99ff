"""GPU <-> host swapping of recurrent-tensor time blocks.

The reference plans offload/fetch memory ops but never executes them
(`polysched.augment_memory_ops`, pkg/src/recten/polysched.py:936-1105,
SURVEY F3): a tensor is swap-managed when its domain has more than one dim
and its bytes reach `DEFAULT_SWAP_THRESHOLD` = 64 MiB (polysched.py:28,
`_swap_managed` :876-877); it is offloaded after it is produced and fetched
before each consumer.

Here that plan is realised for long-horizon programs that are time-blocked
(`blocking.block_dim`): an activation written by the acting recurrence and
read only (a) by the recurrence at the same step and (b) by the backward
chain one time block at a time keeps just TWO time blocks in HBM (a ring
along t, slot = block mod 2; `lower.Buf.ring`).  The acting loop runs one
block per launch (`rt_loop_params.blk_*`); after each block its ring slot is
offloaded to pinned host memory by a 2-D cudaMemcpyAsync on a copy stream;
the backward's block loop fetches block kb+1 on the copy stream while block
kb computes.  Streams are ordered by events only (no host synchronisation).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import native as N
from .ir import ITEMSIZE
from .planner import Bulk, Loop

DEFAULT_SWAP_THRESHOLD = 64 << 20   # reference polysched.py:28


@dataclass
class SwapPlan:
    dim: str            # the blocked time dim (t)
    kb: str             # its block dim (blocking.block_dim)
    bs: int
    DI: int
    ring_slot: int      # env slot holding kb mod 2
    keys: list = field(default_factory=list)   # managed root buffer keys


def _nodes(st):
    if isinstance(st, Bulk):
        return {st.nid}
    out = set()
    for b in st.body:
        out |= _nodes(b)
    return out


def plan_swap(g, plan, bufs, virtual, benv, threshold=DEFAULT_SWAP_THRESHOLD):
    """Managed buffers of a time-blocked graph, or None if nothing qualifies."""
    kbs = getattr(g, "block_dims", ())
    if not kbs:
        return None
    kb = kbs[-1]
    d = kb[:-len("_blk")]
    bs = benv[g.dim_bound[f"{d}_in"]]
    DI = benv[g.dim_bound[kb]]
    acting = [st for st in plan.steps if isinstance(st, Loop) and st.dim == d and st.lo is None]
    blk = [st for st in plan.steps if isinstance(st, Loop) and st.dim == kb]
    if len(acting) != 1 or len(blk) != 1:
        return None
    loop_nodes, region_nodes = _nodes(acting[0]), _nodes(blk[0])
    t_read = ("add", ("mul", ("sym", kb, "loop"), ("int", bs)), ("sym", f"{d}_in", "loop"))
    out_keys = {(nid, oid) for _, nid, oid in g.outputs}
    members = {}
    for k, b in bufs.items():
        r = k
        while bufs[r].alias is not None:
            r = bufs[r].alias
        members.setdefault(r, []).append(k)

    def reads_ok(e, depth=0):
        src, snk = g.nodes[e.src], g.nodes[e.sink]
        c = e.phi[src.domain.index(d)] if d in src.domain else None
        if snk.id in loop_nodes:
            ok = c == ("sym", d, "loop")
        elif snk.id in region_nodes:
            ok = c == t_read
        else:
            return False
        if ok and snk.id in virtual and depth < 16:
            ok = all(_ok_through(f, depth + 1) for f in g.out_edges(snk.id))
        return ok

    def _ok_through(f, depth):
        return f.sink in loop_nodes or f.sink in region_nodes

    keys = []
    for r, mem in members.items():
        n = g.nodes[r[0]]
        b = bufs[r]
        if r[0] not in loop_nodes or r[0] in virtual or not n.domain or n.domain[-1] != d:
            continue
        if b.folded or any(m in out_keys for m in mem) or b.nbytes < threshold:
            continue
        if all(reads_ok(e) for m in mem for e in g.out_edges(m[0]) if e.oid == m[1]):
            keys.append(r)
    if not keys:
        return None
    return SwapPlan(d, kb, bs, DI, len(g.dim_order), sorted(keys))


def adjust_views(params_list, plan: SwapPlan, bufs, slot_of):
    """Ring addressing: every view of a managed buffer maps step t of block
    kb to ring row t - kb*bs + (kb mod 2)*bs (affine in env slots kb and
    ring), applied to the parameter blocks in place."""
    adj = {}
    for k in plan.keys:
        b = bufs[k]
        adj[b.ptr] = b.strides[b.dims.index(plan.dim)] * plan.bs
    kbs, rs = slot_of[plan.kb], plan.ring_slot

    def walk(obj):
        names = [f[0] for f in getattr(obj, "_fields_", ())]
        if "ptr" in names and "off_env" in names and getattr(obj, "ptr") in adj:
            a = adj[obj.ptr]
            obj.off_env[kbs] -= a
            obj.off_env[rs] += a
            return
        for name in names:
            v = getattr(obj, name)
            if hasattr(v, "_fields_"):
                walk(v)
            elif hasattr(v, "_length_") and hasattr(v, "_type_") and \
                    hasattr(v._type_, "_fields_"):
                for x in v:
                    walk(x)

    for p in params_list:
        walk(p)


class SwapRuntime:
    """Pinned host copies + copy stream + events for one executable."""

    def __init__(self, exe, plan: SwapPlan):
        torch = exe.torch
        self.torch, self.exe, self.plan = torch, exe, plan
        self.lib = exe.lib
        self.side = torch.cuda.Stream(exe.dev)
        self.ev_out = [torch.cuda.Event(), torch.cuda.Event()]
        self.ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        self.geo = []
        self.host = []
        for k in plan.keys:
            b = exe.bufs[k]
            row = N_prod(b.pshape) * ITEMSIZE[b.dtype]    # bytes per time step
            rows = N_prod(b.dshape[:-1])                  # (.., t) with t last
            T = b.dshape[-1]
            h = torch.empty(b.full_nbytes, dtype=torch.uint8, pin_memory=True)
            self.host.append(h)
            self.geo.append((b.ptr, h.data_ptr(), rows, plan.bs * row, 2 * plan.bs * row,
                             T * row))
        self.host_bytes = sum(h.numel() for h in self.host)
        # tier moves through the SPEC Backend (backend.py, csrc/backend.cu):
        # ordered by events, counted by its MemorySim
        from .backend import Backend
        dev = exe.dev
        self.backend = Backend(dev if isinstance(dev, int) else (dev.index or 0))
        self.backend.host_tier(self.host_bytes)

    def _issue_in(self, k, after=None):
        ev = self.ev_in[k % 2]
        for i, (dev, host, rows, width, dpitch, hpitch) in enumerate(self.geo):
            self.backend.fetch(dev + (k % 2) * width, host + k * width, width, rows, dpitch=dpitch,
                               hpitch=hpitch, stream=self.side.cuda_stream,
                               after_event=after.cuda_event if (after is not None and i == 0) else 0)
        ev.record(self.side)

    def hook(self, kind, kb, stream):
        torch = self.torch
        if kind == "swap_wait":
            if kb >= 2:
                stream.wait_event(self.ev_out[kb % 2])
        elif kind == "swap_out":
            ev = torch.cuda.Event()
            ev.record(stream)          # the block's producer is done with it
            for i, (dev, host, rows, width, dpitch, hpitch) in enumerate(self.geo):
                self.backend.offload(host + kb * width, dev + (kb % 2) * width, width, rows,
                                     hpitch=hpitch, dpitch=dpitch, stream=self.side.cuda_stream,
                                     after_event=ev.cuda_event if i == 0 else 0)
            self.ev_out[kb % 2].record(self.side)
        elif kind == "swap_in":
            if kb == 0:
                ev = torch.cuda.Event()
                ev.record(stream)
                self._issue_in(0, after=ev)
            stream.wait_event(self.ev_in[kb % 2])
            if kb + 1 < self.plan.DI:
                ev = torch.cuda.Event()
                ev.record(stream)      # block kb-1 is done with the other slot
                self._issue_in(kb + 1, after=ev)
        else:
            raise ValueError(kind)


def N_prod(xs):
    out = 1
    for x in xs:
        out *= int(x)
    return out


# ---------------------------------------------------------------------------
# General swapping across idle gaps (polysched
# `_swap_managed` :876-877, `augment_memory_ops` :936-1105).
#
# Any swap-managed buffer (a multi-dim domain and at least the threshold's
# bytes, not an input/output) whose touches in the lowered program leave an
# idle gap -- launches in between that neither read nor write it -- can be
# moved to pinned host memory after its last touch before the gap (OFFLOAD)
# and brought back before its next touch (FETCH).  Its arena range is then
# free for other buffers during the gap, so the memory plan (memplan.assign
# over interval LISTS) can place them there.  The copies are RT_K_MEMCPY
# launch records on the program's stream: stream order IS polysched's `mem`
# level (fetch < exec < offload < dealloc, `schedule_memory` :1116-1137), and
# the program still captures into one CUDA graph.  A gap swap is kept only
# if it lowers the arena (peak HBM); the cost is 2 x bytes over PCIe.


def _segments(prog, touches):
    """Top-level touch segments: a touch inside a loop counts as the whole
    span of its outermost loop (insertion points must be at depth 0)."""
    outer, stack = [], []
    for pc, ins in enumerate(prog):
        if ins[0] == N.RT_OP_FOR:
            stack.append(pc)
        elif ins[0] == N.RT_OP_END:
            a = stack.pop()
            if not stack:
                outer.append((a, pc))
    segs = set()
    for pc in touches:
        lo = hi = pc
        for a, b in outer:
            if a <= pc <= b:
                lo, hi = a, b
                break
        segs.add((lo, hi))
    out = []
    for lo, hi in sorted(segs):
        if out and lo <= out[-1][1] + 1:
            out[-1] = (out[-1][0], max(out[-1][1], hi))
        else:
            out.append((lo, hi))
    return out


def key_touches(prog, rec_ptrs, key_of, hook_ptrs=None):
    """key -> sorted pcs of the launches (and all-reduce hooks) touching it."""
    hook_ptrs = hook_ptrs or {}
    out = {}
    for pc, ins in enumerate(prog):
        if ins[0] == N.RT_OP_LAUNCH:
            ptrs = rec_ptrs[ins[1]]
        elif ins[0] == N.RT_OP_HOOK:
            ptrs = {(q >> 44) << 44 for q in hook_ptrs.get(pc, ())}
        else:
            continue
        for p in ptrs:
            k = key_of.get(p)
            if k is not None:
                out.setdefault(k, []).append(pc)
    return out


def gap_candidates(prog, touches, managed):
    """[(key, off_pos, fetch_pos)]: for each managed key, its largest idle
    gap between two top-level touch segments that contains a launch.
    off_pos / fetch_pos are instruction positions in `prog` (the offload is
    inserted before off_pos, i.e. right after the earlier segment; the fetch
    before fetch_pos, the start of the later one)."""
    launches = [pc for pc, ins in enumerate(prog) if ins[0] == N.RT_OP_LAUNCH]
    out = []
    for k in managed:
        segs = _segments(prog, touches.get(k, ()))
        best = None
        for (a0, a1), (b0, b1) in zip(segs, segs[1:]):
            inside = sum(1 for pc in launches if a1 < pc < b0)
            if inside and (best is None or b0 - a1 > best[1] - best[0]):
                best = (a1 + 1, b0)
        if best is not None:
            out.append((k, best[0], best[1]))
    return out


def insert_instrs(prog, inserts):
    """Insert instructions at top-level positions: inserts = {pos: [instr]}
    (before the instruction at old position pos; pos == len(prog) appends).
    FOR.e (pc after its END) and END.a (pc of its FOR) are remapped."""
    shift, acc = [], 0
    for pc in range(len(prog) + 1):
        acc += len(inserts.get(pc, ()))
        shift.append(acc)

    def new(pc):            # new position of old instruction pc
        return pc + shift[pc]

    def target(pc):         # jump target: the first instruction inserted at pc, if any
        return pc + (shift[pc - 1] if pc > 0 else 0)

    out = []
    for pc, ins in enumerate(prog):
        out.extend(inserts.get(pc, ()))
        ins = tuple(ins)
        if ins[0] == N.RT_OP_FOR:
            ins = ins[:5] + (target(ins[5]),)
        elif ins[0] == N.RT_OP_END:
            ins = (ins[0], new(ins[1])) + ins[2:]
        out.append(ins)
    out.extend(inserts.get(len(prog), ()))
    return out


def plan_gap_swap(prog, rec_ptrs, key_of, managed, sizes, base_life, assign, lifetimes_of):
    """Greedy choice of gap swaps that lower the arena.  `lifetimes_of(prog,
    rec_ptrs)` recomputes key -> (lo, hi) on a rewritten program; returns
    (chosen [(key, off_pos, fetch_pos)], program, rec_ptrs, lifetimes) with
    the chosen copies inserted as launch records numbered after the
    existing ones (offload, fetch per key, in `chosen` order)."""
    touches = key_touches(prog, rec_ptrs, key_of)
    cands = gap_candidates(prog, touches, managed)
    cands.sort(key=lambda c: -sizes[c[0]])
    fake = {v: k for k, v in key_of.items()}
    chosen = []

    def build(sel):
        inserts, ptrs = {}, list(rec_ptrs)
        for k, a, b in sel:
            ptrs.append({fake[k]})
            inserts.setdefault(a, []).append((N.RT_OP_LAUNCH, len(ptrs) - 1, 0, 0, 0, 0))
            ptrs.append({fake[k]})
            inserts.setdefault(b, []).append((N.RT_OP_LAUNCH, len(ptrs) - 1, 0, 0, 0, 0))
        p2 = insert_instrs(prog, inserts)
        life = lifetimes_of(p2, ptrs)
        # split lifetimes: live up to its offload, and again from its fetch
        tl = key_touches(p2, ptrs, key_of)
        for i, (k, a, b) in enumerate(sel):
            off_rec, fetch_rec = len(rec_ptrs) + 2 * i, len(rec_ptrs) + 2 * i + 1
            off_pc = [pc for pc, x in enumerate(p2) if x[0] == N.RT_OP_LAUNCH and x[1] == off_rec][0]
            fe_pc = [pc for pc, x in enumerate(p2) if x[0] == N.RT_OP_LAUNCH and x[1] == fetch_rec][0]
            lo, hi = life[k]
            assert min(tl[k]) <= off_pc < fe_pc <= max(tl[k])
            life[k] = [(lo, off_pc), (fe_pc, hi)]
        return p2, ptrs, life

    _, best = assign(sizes, base_life)
    cur = (prog, rec_ptrs, base_life)
    for c in cands:
        trial = chosen + [c]
        p2, ptrs, life = build(trial)
        _, arena = assign(sizes, life)
        if arena < best:
            chosen, best, cur = trial, arena, (p2, ptrs, life)
    return chosen, cur[0], cur[1], cur[2]
