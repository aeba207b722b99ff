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
