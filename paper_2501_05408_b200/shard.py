"""Env sharding across GPUs.

Within one training iteration every (b, t) node reads only its own env b;
the only cross-env dependences are full-range reductions over b (the
REINFORCE/PPO objective and gradient sums, e.g. reference
pkg/programs/reinforce.rtl:29-31 `it[i] = sum(ep[i,0:B])`).  So the env dim
shards into contiguous blocks of B/G per rank with:

  * per-point RNG keyed by the GLOBAL env index (rank * B_local + b), so the
    draws — and hence the results — do not depend on G;
  * a sum all-reduce (NCCL over NVLink on GPUs) of each reduction over b,
    right after the kernel that produced the local partial sum; everything
    downstream of those reductions (parameter updates) is replicated.

`check_shardable` proves the graph fits that shape or explains why not.
"""

from __future__ import annotations

import ctypes as C

from dataclasses import dataclass

from . import ir


class ShardError(Exception):
    pass


@dataclass(frozen=True)
class ShardSpec:
    dim: str             # the sharded loop dim (envs)
    rank: int
    world: int
    also: tuple = ()     # co-sharded dims indexing the same envs (e.g. the
    #                      minibatch-local env u of a PPO update, b = u*M + j)

    @property
    def dims(self):
        return (self.dim,) + tuple(self.also)

    def offset(self, local_extent: int) -> int:
        return self.rank * local_extent


def _mentions(e, d) -> bool:
    return (d, "loop") in ir.free_syms(e)


def check_shardable(g: ir.Graph, d: str, also=(), benv=None) -> set:
    """Node ids whose outputs are partial sums over d or a co-sharded dim
    (need an all-reduce).  Raises ShardError when some dependence crosses
    envs otherwise.  A co-sharded dim u may index d only as u*m + f with
    m = ext(d)/ext(u) and 0 <= f < m (each env shard holds the same slice
    of every u-block; needs the concrete bounds `benv`)."""
    reduce_nodes = set()
    for dd in (d,) + tuple(also):
        reduce_nodes |= _check_dim(g, dd, d, tuple(also), benv)
    return reduce_nodes


def _check_dim(g: ir.Graph, d: str, env_dim: str, also: tuple, benv) -> set:
    from .planner import interval, subst_bounds
    bound = g.dim_bound[d]
    reduce_nodes = set()
    for n in g.sorted_nodes():
        vec = [s.name for s in n.params.get("vec", ())]
        if d in vec:
            raise ShardError(f"{n.name}: dim {d} is folded into a payload axis")
        if n.kind == "merge" and any(_mentions(c, d) for c in n.params["conds"]):
            raise ShardError(f"{n.name}: branch condition depends on {d}")
        if n.kind == "eval_symbol" and n.params["symbol"].name in (d, bound):
            # the bound too: a shard sees the per-rank extent, so e.g.
            # sum(x[0:B]) / B would divide the all-reduced sum by the local B
            raise ShardError(f"{n.name}: reads the value of {n.params['symbol'].name}")
        if n.kind in ("index_select", "window_reduce", "slice_axis", "scan") and \
                getattr(n.params.get("dim"), "name", None) == d:
            raise ShardError(f"{n.name}: {n.kind} along {d}")
    for e in g.edges:
        src, snk = g.nodes[e.src], g.nodes[e.sink]
        if e.psi is not None and _mentions(e.psi, d):
            raise ShardError(f"{snk.name}: edge condition depends on {d}")
        if d not in src.domain:
            continue
        c = e.phi[src.domain.index(d)]
        if d in snk.domain:
            if c != ("sym", d, "loop"):
                raise ShardError(f"{snk.name} reads {src.name} at {ir.expr_text(c)} along {d}")
            continue
        co = [u for u in also if u in snk.domain and (u, "loop") in ir.free_syms(c)]
        if d == env_dim and co:
            u = co[0]
            ok = False
            if benv is not None:
                aff = ir.as_affine(subst_bounds(c, benv))
                ext = {x: benv[g.dim_bound[x]] for x in g.dim_order if g.dim_bound[x] in benv}
                if aff is not None and ext.get(u) and ext[d] % ext[u] == 0:
                    coef, k0 = aff
                    m = ext[d] // ext[u]
                    rest = ("int", k0)
                    for (name, kind), cc in coef.items():
                        if (name, kind) != (u, "loop"):
                            rest = ("add", rest, ("mul", ("int", cc), ("sym", name, kind)))
                    box = {x: (0, ext[x] - 1) for x in snk.domain if x in ext}
                    lo, hi = interval(rest, box)
                    ok = coef.get((u, "loop")) == m and lo >= 0 and hi < m
            if not ok:
                raise ShardError(f"{snk.name} reads {src.name}[{ir.expr_text(c)}] across envs")
            continue
        full = c == ("slice", ("int", 0), ("sym", bound, "bound"))
        if not full:
            raise ShardError(f"{snk.name} reads {src.name}[{ir.expr_text(c)}] across envs")
        if snk.kind != "sum":
            raise ShardError(f"{snk.name}: {snk.kind} over all envs is not a sum")
        slice_axes = [j for j, cc in enumerate(e.phi) if cc[0] == "slice"]
        ax = slice_axes.index(src.domain.index(d))
        if ax not in tuple(snk.params["dims"]):
            raise ShardError(f"{snk.name}: gathers {src.name} over envs without reducing")
        reduce_nodes.add(snk.id)
    return reduce_nodes


class TorchComm:
    """Sum all-reduce through torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def allreduce_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t


class NcclComm:
    """The library's own NCCL communicator (csrc/coll.cu): the sharded
    program's gradient all-reduces become in-program collectives (RT_OP_COLL)
    issued by the interpreter on the program's stream, so a whole step --
    rollout, backward, all-reduces, updates -- is one CUDA graph.  The unique
    id travels through torch.distributed (any backend) once at setup."""

    native = True

    def __init__(self, rank=None, world=None, group=None):
        import torch
        import torch.distributed as dist
        from . import native as N
        self.lib = N.lib()
        rank = dist.get_rank(group) if rank is None else rank
        world = dist.get_world_size(group) if world is None else world
        buf = bytearray(128)
        if rank == 0:
            cid = C.create_string_buffer(128)
            N.check(self.lib.rt_nccl_unique_id(cid), "nccl unique id")
            buf = bytearray(cid.raw[:128])
        t = torch.tensor(list(buf), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=group)
        idb = bytes(t.cpu().tolist())
        h = N.u64()
        N.check(self.lib.rt_nccl_comm_init(int(world), int(rank), idb, C.byref(h)), "nccl init")
        self.handle = h.value
        self.rank, self.world = rank, world

    def allreduce_(self, t):
        """(host-side fallback path: one tensor, on torch's current stream)"""
        import torch
        from . import native as N
        code = {torch.float64: N.RT_F64, torch.float32: N.RT_F32, torch.int64: N.RT_I64}[t.dtype]
        N.check(self.lib.rt_nccl_allreduce(self.handle, t.data_ptr(), t.numel(), code,
                                           torch.cuda.current_stream().cuda_stream), "allreduce")
        return t

    def close(self):
        if getattr(self, "handle", 0):
            from . import native as N
            N.check(self.lib.rt_nccl_comm_destroy(self.handle), "nccl destroy")
            self.handle = 0
