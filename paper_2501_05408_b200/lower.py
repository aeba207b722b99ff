"""Lowering: planned steps -> parameter blocks for the C-ABI kernel families
plus the loop program `rt_run` interprets.

Each bulk step of node n with enclosing loop dims F evaluates n over
box = (free dims of n's domain) x (payload).  Every in-edge becomes an
operand view: the edge's index expression phi (reference pdg.py:58-68,
evaluated per point by runtime.py:396-425) is folded at compile time into
element strides over the box, offsets linear in the loop variables, and
range checks for components that may leave the source domain; index
expressions that are not affine compile to small int programs (Euclidean
// and %, reference symexpr.py:491-506).  Slice components become value
axes: reduced in place by RT_K_REDUCE / RT_K_SCAN, or walked as payload
axes when their length is constant.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import zlib
from dataclasses import dataclass, field

import numpy as np

from . import ir
from . import native as N
from .planner import INF, Bulk, Loop, Shift, interval, subst_bounds


class LowerError(Exception):
    pass


def prod(xs):
    out = 1
    for x in xs:
        out *= x
    return out


def cstrides(shape):
    st, acc = [], 1
    for s in reversed(shape):
        st.append(acc)
        acc *= s
    return list(reversed(st))


# ---------------------------------------------------------------------------
# buffers


@dataclass
class Buf:
    key: tuple            # (nid, oid)
    dims: tuple           # domain dims
    dshape: tuple         # domain extents
    pshape: tuple         # payload shape
    dtype: str
    alias: tuple | None = None   # (nid, oid) whose storage this is
    host: np.ndarray | None = None  # constant/input contents
    ptr: int = 0
    folded: frozenset = frozenset()  # loop dims stored as one slot (stride 0)
    ring: tuple | None = None        # (dim, bs): swap-managed, 2 time blocks resident

    @property
    def shape(self):
        return tuple(self.dshape) + tuple(self.pshape)

    def storage_ext(self):
        ext = [1 if d in self.folded else x for d, x in zip(self.dims, self.dshape)]
        if self.ring:
            ext[self.dims.index(self.ring[0])] = 2 * self.ring[1]
        return ext

    @property
    def strides(self):
        if not self.folded and not self.ring:
            return cstrides(self.shape)
        st = list(cstrides(self.storage_ext() + list(self.pshape)))
        for j, d in enumerate(self.dims):
            if d in self.folded:
                st[j] = 0
        return tuple(st)

    def dim_stride(self, d):
        return self.strides[self.dims.index(d)]

    def payload_strides(self):
        return self.strides[len(self.dims):]

    @property
    def nbytes(self):
        return prod(self.storage_ext()) * prod(self.pshape) * ir.ITEMSIZE[self.dtype]

    @property
    def full_nbytes(self):
        """bytes of every value (the pinned host copy of a swap-managed buffer)"""
        return prod(self.dshape) * prod(self.pshape) * ir.ITEMSIZE[self.dtype]


# ---------------------------------------------------------------------------
# VM programs


OPC = {"ICOORD": 1, "IENV": 2, "ICONST": 3, "IADD": 4, "ISUB": 5, "IMUL": 6, "IFDIV": 7,
       "IMOD": 8, "IMIN": 9, "IMAX": 10, "INEG": 11, "IEQ": 12, "ILT": 13, "ILE": 14,
       "IGT": 15, "IGE": 16, "INE": 17, "IAND": 18, "IOR": 19, "INOT": 20, "JZ": 21,
       "JMP": 22, "LOAD": 30, "LOADX": 31, "VCONST": 32, "VITOF": 33, "VADD": 34,
       "VSUB": 35, "VMUL": 36, "VDIV": 37, "VNEG": 38, "VEXP": 39, "VLOG": 40,
       "VTANH": 41, "VSQRT": 42, "VPOW": 43, "VEQ": 44, "VNE": 45, "VLT": 46, "VLE": 47,
       "VGT": 48, "VGE": 49, "VWHERE": 50, "VCAST": 51, "VMOV": 52, "VTOI": 53,
       "VALID": 54, "STORE": 60, "ERROR": 62, "ISTORE": 63}

TMA_PERSIST = os.environ.get("RTB200_GEMM_PERSIST", "1") != "0"

IBIN = {"add": "IADD", "sub": "ISUB", "mul": "IMUL", "floordiv": "IFDIV", "mod": "IMOD",
        "eq": "IEQ", "lt": "ILT", "le": "ILE", "gt": "IGT", "ge": "IGE", "and": "IAND",
        "or": "IOR"}


class Prog:
    """Builder for the two-word VM code (csrc/common.cuh)."""

    def __init__(self):
        self.code: list[int] = []
        self.konst: list[float] = []
        self.ifree = list(range(8))
        self.vfree = list(range(8))

    def emit(self, op, d=0, a=0, b=0, c=0, imm=0):
        self.code += [OPC[op] | (d << 8) | (a << 12) | (b << 16) | (c << 20), int(imm)]
        if len(self.code) > N.RT_CODE:
            raise LowerError("program too long")
        return len(self.code) - 1  # index of the imm word (for patching jumps)

    def pc(self):
        return len(self.code)

    def ireg(self):
        if not self.ifree:
            raise LowerError("out of int registers")
        return self.ifree.pop(0)

    def vreg(self):
        if not self.vfree:
            raise LowerError("out of value registers")
        return self.vfree.pop(0)

    def ifree_(self, r):
        self.ifree.insert(0, r)

    def vfree_(self, r):
        self.vfree.insert(0, r)

    def k(self, v):
        v = float(v)
        for i, x in enumerate(self.konst):
            if x == v and math.copysign(1, x) == math.copysign(1, v):
                return i
        self.konst.append(v)
        if len(self.konst) > N.RT_KONST:
            raise LowerError("too many constants")
        return len(self.konst) - 1

    def int_expr(self, e, dimmap):
        """Compile an integer/bool expression; returns the result register.
        dimmap: (name, kind) -> ("coord", i) | ("env", slot) | ("const", v)."""
        k = e[0]
        if k in ("int", "bool"):
            r = self.ireg()
            v = int(e[1])
            if not -(1 << 31) <= v < (1 << 31):
                raise LowerError("integer constant out of range")
            self.emit("ICONST", d=r, imm=v)
            return r
        if k == "sym":
            m = dimmap.get((e[1], e[2]))
            if m is None:
                raise LowerError(f"unbound symbol {e[1]} in index expression")
            r = self.ireg()
            if m[0] == "coord":
                self.emit("ICOORD", d=r, imm=m[1])
            elif m[0] == "env":
                self.emit("IENV", d=r, imm=m[1])
            else:
                self.emit("ICONST", d=r, imm=m[1])
            return r
        if k == "neg":
            a = self.int_expr(e[1], dimmap)
            self.emit("INEG", d=a, a=a)
            return a
        if k == "not":
            a = self.int_expr(e[1], dimmap)
            self.emit("INOT", d=a, a=a)
            return a
        if k in ("min", "max"):
            a = self.int_expr(e[1], dimmap)
            for x in e[2:]:
                b = self.int_expr(x, dimmap)
                self.emit("IMIN" if k == "min" else "IMAX", d=a, a=a, b=b)
                self.ifree_(b)
            return a
        if k in IBIN:
            a = self.int_expr(e[1], dimmap)
            b = self.int_expr(e[2], dimmap)
            self.emit(IBIN[k], d=a, a=a, b=b)
            self.ifree_(b)
            return a
        raise LowerError(f"cannot compile index expression kind {k}")


# ---------------------------------------------------------------------------
# operand views


@dataclass
class Axis:
    ext: int | None        # None: ragged (length varies per point)
    stride: int
    len_expr: object = None  # ragged slice: hi - lo (bounds substituted)
    lo_expr: object = None   # slice lower endpoint (bounds substituted)


@dataclass
class EdgeVal:
    buf: Buf
    off: int = 0
    coef: dict = field(default_factory=dict)      # sink dim -> element stride
    checks: list = field(default_factory=list)    # (k, {sink dim: a}, hi)
    axes: list = field(default_factory=list)      # value axes (slices then payload)
    nslices: int = 0
    progs: list = field(default_factory=list)     # (expr, stride, hi) non-affine comps
    psi: object = None


class Ctx:
    """Per-bulk-step context: slab dims, loop slots, concrete bounds."""

    def __init__(self, low, node, fixed):
        self.low = low
        self.node = node
        self.fixed = tuple(fixed)
        self.slab = [d for d in node.domain if d not in fixed]
        self.slab_ext = [low.ext[d] for d in self.slab]

    def dimmap(self, payload_coords=None):
        m = {}
        for b, v in self.low.benv.items():
            m[(b, "bound")] = ("const", v)
        for d in self.node.domain:
            if d in self.fixed:
                m[(d, "loop")] = ("env", self.low.slot[d])
            else:
                m[(d, "loop")] = ("coord", self.slab.index(d))
        if payload_coords:
            m.update(payload_coords)
        return m

    def sink_box(self):
        return {d: (0, self.low.ext[d] - 1) for d in self.node.domain}


class Lowering:
    def __init__(self, plan, bufs: dict, status_ptr: int, seed: int, alloc, contract=None,
                 fuse_src=None, gemm_epi=None, persistent=True, use_tc=True, absorbed=None,
                 shard=None, shard_reduce=None, swap=None):
        self.plan = plan
        self.g = plan.graph
        self.benv = plan.benv
        self.ext = plan.ext
        self.bufs = bufs
        self.status = status_ptr
        self.seed = seed
        self.slot = {d: i for i, d in enumerate(self.g.dim_order)}
        if len(self.slot) > N.RT_MAXENV:
            raise LowerError("too many dims")
        self.recs: list = []       # (kernel, params ctypes obj, grid, block, smem, label)
        self.prog: list = []       # (op, a, b, c, d, e)
        self.alloc = alloc         # nbytes -> device pointer (scratch)
        self.contract = contract or {}   # sum nid -> virtual matmul nid
        self.virtual = set(self.contract.values())
        self.absorbed = set(absorbed or ())
        self.virtual |= self.absorbed
        self.persistent = persistent
        self.use_tc = use_tc and os.environ.get("RTB200_GEMM", "") != "simt"
        self.use_tma = os.environ.get("RTB200_GEMM", "") != "tc"
        self.shard = shard
        self.shard_reduce = set(shard_reduce or ())
        self.hooks = []                        # all-reduce hooks (sharded reductions)
        self.rec_cluster = {}                  # launch record -> cluster size (pair loops)
        self.swap = swap                       # swap.SwapPlan (time-blocked swapping)
        self._capture = None
        self._smallk_capture = None            # dual gate: the second product's thin params
        self._smallk_second = None
        self.loop_subs = {}                    # loop record -> sub-op descriptors
        self.fuse_src = dict(fuse_src or {})   # producer nid -> consumer nid (inlined)
        self.gemm_epi = dict(gemm_epi or {})   # final nid -> (matmul nid, bias edge, tanh)
        self.virtual |= set(self.fuse_src)
        for info in getattr(plan, "gae", {}).values():
            self.virtual |= info["nodes"]          # delta chain formed inside the scan
        self.ones_bias = dict(getattr(plan, "ones_bias", {}) or {})   # contraction -> bias sum
        self.ones_targets = {r: s_ for s_, r in self.ones_bias.items()}   # bias sum -> contraction
        self._ones_done = set()
        self.colsum = dict(getattr(plan, "colsum", {}) or {})   # gate product -> its row sum
        self._colsum_done = set()
        self._colsum_req = None
        self.dw_epi = dict(getattr(plan, "dw_epi", {}) or {})   # gate product -> [(dW sum, which)]
        self._dw_req = None
        self.sibling = dict(getattr(plan, "sibling", {}) or {})  # head -> sibling head
        self._rows_capture = None
        self._rows_second = None
        self._sibling_done = set()
        for f, (x, _b, t) in self.gemm_epi.items():
            self.virtual.add(x)
            if isinstance(t, tuple):           # tanh-VJP gate: (1 - h*h) chain
                self.virtual |= {t[1], t[2]} | set(t[4:6])   # (+ the summed second product)
            elif t:
                self.virtual.add(self.g.in_edges(f)[0].src)
        self.launches_per_kernel = {}

    # -- buffers -------------------------------------------------------------

    def storage(self, key):
        b = self.bufs[key]
        while b.alias is not None:
            b = self.bufs[b.alias]
        return b

    # -- edge views ----------------------------------------------------------

    def edge_val(self, ctx: Ctx, e) -> EdgeVal:
        if e.src in self.absorbed:
            return self._absorbed_val(ctx, e)
        src = self.g.nodes[e.src]
        sb = self.bufs[(e.src, e.oid)]
        st = self.storage((e.src, e.oid))
        dstr = sb.strides[:len(sb.dims)]
        ev = EdgeVal(buf=st)
        box = ctx.sink_box()
        if e.psi is not None:
            ev.psi = subst_bounds(e.psi, self.benv)
        slice_axes = []
        for j, c in enumerate(e.phi):
            c = subst_bounds(c, self.benv)
            S = dstr[j]
            hi_dom = sb.dshape[j]
            if c[0] == "slice":
                lo, hi = c[1], c[2]
                aff = ir.as_affine(lo)
                ln = ir.as_affine(("sub", hi, lo))
                if aff is None:
                    raise LowerError(f"{ctx.node.name}: non-affine slice start {ir.expr_text(lo)}")
                self._add_affine(ev, aff, S)
                L = None
                if ln is not None and not ln[0]:
                    L = max(0, ln[1])
                slice_axes.append(Axis(L, S, ("sub", hi, lo), lo))
                continue
            aff = ir.as_affine(c)
            if aff is None:
                ev.progs.append((c, S, hi_dom))
                continue
            self._add_affine(ev, aff, S)
            lo_, hi_ = interval(c, box)
            if lo_ < 0 or hi_ >= hi_dom:
                ev.checks.append((aff[1], {n: v for (n, k), v in aff[0].items()}, hi_dom))
        ev.axes = slice_axes + [Axis(p, s) for p, s in zip(sb.pshape, sb.payload_strides())]
        ev.nslices = len(slice_axes)
        return ev

    def _absorbed_val(self, ctx, e):
        """Edge into a layout node that was never materialised: read its
        source through the same point map, then apply the node's payload
        transform (permute/reshape/squeeze/unsqueeze/expand) to the axes."""
        L = self.g.nodes[e.src]
        (ein,) = self.g.in_edges(L.id)
        ev = self.edge_val(ctx, ir.Edge(e.sink, e.iid, e.phi, e.psi, ein.oid, ein.src))
        sl = ev.axes[:ev.nslices]
        pay = ev.axes[ev.nslices:]
        k = L.kind
        if k == "permute":
            pay = [pay[o] for o in L.params["order"]]
        elif k == "squeeze":
            dd = L.params["dim"]
            pay = pay[:dd] + pay[dd + 1:]
        elif k == "unsqueeze":
            dd = L.params["dim"]
            pay = pay[:dd] + [Axis(1, 0)] + pay[dd:]
        elif k == "reshape":
            if [a.stride for a in pay] != cstrides([a.ext for a in pay]):
                raise LowerError(f"{L.name}: reshape of a non-contiguous view")
            shape = list(self.bufs[(L.id, 0)].pshape)
            pay = [Axis(x, st) for x, st in zip(shape, cstrides(shape))]
        elif k == "expand":
            shape = list(self.bufs[(L.id, 0)].pshape)
            off = len(shape) - len(pay)
            new = []
            for j, x in enumerate(shape):
                vj = j - off
                if vj < 0 or pay[vj].ext == 1:
                    new.append(Axis(x, 0))
                else:
                    new.append(pay[vj])
            pay = new
        else:
            raise LowerError(f"cannot absorb {k}")
        ev.axes = list(sl) + list(pay)
        return ev

    def _add_affine(self, ev, aff, S):
        co, k = aff
        ev.off += k * S
        for (name, kind), a in co.items():
            if kind != "loop":
                raise LowerError(f"unbound symbol {name}")
            ev.coef[name] = ev.coef.get(name, 0) + a * S

    def make_view(self, ctx: Ctx, ev: EdgeVal, payload_strides: list, extra_off=0,
                  extra_checks=()) -> N.rt_view:
        """rt_view over box = slab dims + payload dims."""
        v = N.rt_view()
        v.ptr = ev.buf.ptr
        v.dtype = N.DTYPE_CODE[ev.buf.dtype]
        v.off = ev.off + extra_off
        nd = len(ctx.slab) + len(payload_strides)
        if nd > N.RT_MAXD:
            raise LowerError("box rank too large")
        for d, s in ev.coef.items():
            if d in ctx.fixed:
                v.off_env[self.slot[d]] += s
            elif d in ctx.slab:
                v.stride[ctx.slab.index(d)] += s
            else:
                raise LowerError(f"{ctx.node.name}: index uses dim {d} outside its domain")
        for i, s in enumerate(payload_strides):
            v.stride[len(ctx.slab) + i] = s
        checks = list(ev.checks) + list(extra_checks)
        if len(checks) > N.RT_MAXCHK:
            raise LowerError("too many range checks")
        v.nchk = len(checks)
        for ci, (k, co, hi) in enumerate(checks):
            v.chk_c0[ci] = k
            v.chk_hi[ci] = hi
            for d, a in co.items():
                if isinstance(d, int):           # payload box dim
                    v.chk_a[ci][len(ctx.slab) + d] = a
                elif d in ctx.fixed:
                    v.chk_env[ci][self.slot[d]] = a
                else:
                    v.chk_a[ci][ctx.slab.index(d)] = a
        return v

    def out_view(self, ctx: Ctx, key) -> N.rt_view:
        b = self.bufs[key]
        st = self.storage(key)
        v = N.rt_view()
        v.ptr = st.ptr
        v.dtype = N.DTYPE_CODE[st.dtype]
        strides = st.strides
        for j, d in enumerate(b.dims):
            if d in ctx.fixed:
                v.off_env[self.slot[d]] = strides[j]
            else:
                v.stride[ctx.slab.index(d)] = strides[j]
        for i, s in enumerate(strides[len(b.dims):]):
            v.stride[len(ctx.slab) + i] = s
        return v

    # -- payload maps -------------------------------------------------------

    @staticmethod
    def bcast(ev: EdgeVal, out_shape):
        """numpy broadcasting of the edge value onto out_shape."""
        V = ev.axes
        off = len(out_shape) - len(V)
        if off < 0:
            raise LowerError("cannot broadcast to a lower rank")
        out = []
        for j in range(len(out_shape)):
            vj = j - off
            if vj < 0:
                out.append(0)
            else:
                ax = V[vj]
                if ax.ext is None:
                    raise LowerError("ragged slice feeds an elementwise op")
                out.append(0 if ax.ext == 1 else ax.stride)
        return out

    # -- records -----------------------------------------------------------------

    def add_rec(self, kernel, params, grid, block, smem=0, label=""):
        params.h.node = int(label[0]) if isinstance(label, tuple) else 0
        params.h.status = self.status
        if self._capture is not None:
            self._capture.append((kernel, params, grid, block, smem, label))
            return -1
        self.recs.append((kernel, params, grid, block, smem, label))
        self.prog.append((N.RT_OP_LAUNCH, len(self.recs) - 1, 0, 0, 0, 0))
        return len(self.recs) - 1

    @staticmethod
    def grid1(total, block=256, cap=148 * 32):
        return [max(1, min(cap, (int(total) + block - 1) // block)), 1, 1]

    # -- program ----------------------------------------------------------------

    def lower(self):
        self.steps(self.plan.steps)
        if self.swap is not None:
            from .swap import adjust_views
            params = [p for (_, p, *_r) in self.recs]
            for info in self.loop_subs.values():
                params += [op[1] for op in info["ops"]]
            adjust_views(params, self.swap, self.bufs, self.slot)
        self._bucket_allreduces()
        return self

    def _bucket_allreduces(self):
        """Mark which all-reduce hooks flush.  A hook whose program continues,
        before any launch that reads an already-reduced buffer, with another
        all-reduce hook defers its collective; the last one of such a run
        all-reduces every pending buffer as ONE bucket (per dtype) — one
        collective per optimizer step, e.g. C2's six gradient
        sums and its objective.  Loop boundaries and other hooks flush."""
        from .memplan import touched_ptrs
        pending = set()
        for pc, ins in enumerate(self.prog):
            if ins[0] != N.RT_OP_HOOK:
                continue
            h = self.hooks[ins[1]]
            if h.get("kind", "allreduce") != "allreduce":
                continue
            pending.add(h["ptr"])
            flush = True
            for j in range(pc + 1, len(self.prog)):
                nxt = self.prog[j]
                if nxt[0] == N.RT_OP_LAUNCH:
                    if touched_ptrs(self.recs[nxt[1]][1]) & pending:
                        break
                    continue
                if nxt[0] == N.RT_OP_HOOK and \
                        self.hooks[nxt[1]].get("kind", "allreduce") == "allreduce":
                    flush = False
                break
            h["flush"] = flush
            if flush:
                pending = set()

    def steps(self, steps):
        for s in steps:
            if isinstance(s, Bulk):
                self.bulk(s)
            elif isinstance(s, Shift):
                self.shift(s)
            else:
                self.loop(s)

    def shift(self, s: Shift):
        """Lagged nodes of a skewed band (planner.skew_steps): the loop
        index minus k while they launch (launches fold env when issued)."""
        slot = self.slot[s.dim]
        self.prog.append((N.RT_OP_ENVADD, slot, -s.k, 0, 0, 0))
        self.steps(s.body)
        self.prog.append((N.RT_OP_ENVADD, slot, s.k, 0, 0, 0))

    # -- persistent loops ------------------------------------------------------

    def _persistent_ok(self, s: Loop):
        """Body = bulk steps over one common slab S whose internal dependences
        keep the S coordinates (row-local), so CTAs can own rows."""
        if not self.persistent or any(not isinstance(b, Bulk) for b in s.body):
            return None
        fixed = tuple(s.fixed) + (s.dim,)
        body = {b.nid for b in s.body}
        if body & self.shard_reduce:
            return None
        slabs = set()
        for b in s.body:
            n = self.g.nodes[b.nid]
            if n.kind in ("const", "input") or self.bufs[(n.id, 0)].alias is not None:
                continue
            slabs.add(tuple(d for d in n.domain if d not in fixed))
        if len(slabs) != 1:
            return None
        S = slabs.pop()
        if not S:
            return None
        for nid in body:
            for e in self.g.in_edges(nid):
                if e.src not in body:
                    continue
                src = self.g.nodes[e.src]
                for d in S:
                    if d in src.domain and e.phi[src.domain.index(d)] != ("sym", d, "loop"):
                        return None
        return S

    PAIR_MIN_BYTES = 64 * 1024
    RESIDENT_MAX_BYTES = 32 * 1024

    def _resident_ops(self, ops, rows, T, dim, base, wide=False, skip=None):
        """{op index: shared-memory offset} for in-loop GEMMs whose weights are
        fp32, dense row-major, <= 32 KB and do not move with the loop dim
        (wide layers only with `wide`: when the widest layer is on chip
        (hybrid), nothing else keeps the TMA ring busy)."""
        from . import jit
        if not (jit.ENABLED and jit.RESIDENT_ENABLED) or rows * T < jit.JIT_LOOP_MIN:
            return {}, 0
        out, cur = {}, 0
        for i, (kernel, p, re, f64, _) in enumerate(ops):
            if kernel != N.RT_K_GEMM or f64 or p.B.dtype != N.RT_F32 or i == skip:
                continue
            if not (p.N.nd == 1 and p.K.nd == 1 and p.z == 1 and p.B.s2[0] == 1
                    and p.B.s1[0] == p.n and p.n % 4 == 0):
                continue
            if p.B.off_env[self.slot[dim]] != 0 or (p.B.ptr + 4 * p.B.off) % 16 or \
                    any(p.B.off_env[e] % 4 for e in range(N.RT_MAXENV)):
                continue
            nb = p.k * p.n * 4
            if nb > self.RESIDENT_MAX_BYTES or (p.n >= 64 and not wide):
                continue   # (wide layers: the TMA-streamed core measured faster)
            out[i] = base + cur
            cur += (nb + 127) // 128 * 128
        return out, cur

    def _hybrid_op(self, ops, R, rows, T, dim, dual):  # noqa: C901
        """(op index, KR) for the in-loop GEMM whose weights stay on chip for
        the whole loop split between registers and shared memory
        (jit.py HYBRID_*: rows [0, KR) of B in KR registers per thread, one
        column per thread; rows [KR, K) resident in shared memory), or None.
        fp32, N = 256 = blockDim, dense row-major B that does not move with
        the loop dim, one CTA per SM (the register budget)."""
        from . import jit
        if not (jit.ENABLED and jit.HYBRID_ENABLED) or dual or rows * T < jit.JIT_LOOP_MIN:
            return None
        best = None
        for i, (kernel, p, re, f64, _) in enumerate(ops):
            if kernel != N.RT_K_GEMM or f64 or p.B.dtype != N.RT_F32 or p.A.dtype != N.RT_F32 \
                    or p.C.dtype != N.RT_F32 or (p.bias.ptr and p.bias.dtype != N.RT_F32):
                continue
            if not (p.N.nd == 1 and p.K.nd == 1 and p.z == 1 and p.B.s2[0] == 1
                    and p.B.s1[0] == p.n and p.n == 256 and p.k >= jit.HYBRID_KR + 16 and p.k % jit.HYBRID_NCOL == 0
                    and jit.HYBRID_NCOL in (1, 2, 4) and jit.HYBRID_KR % jit.HYBRID_NCOL == 0
                    and (R * re + 3) // 4 * 4 <= 8):
                continue
            if p.B.off_env[self.slot[dim]] != 0 or (p.B.ptr + 4 * p.B.off) % 16 or \
                    any(p.B.off_env[e] % 4 for e in range(N.RT_MAXENV)):
                continue
            if best is None or p.k > ops[best][1].k:
                best = i
        return None if best is None else (best, jit.HYBRID_KR, jit.HYBRID_NCOL)

    def _pair_op(self, ops, R, rows, T, dim):
        """Index of the in-loop GEMM to run in CTA-pair mode, or None: fp32,
        one row per point, dense row-major B of >= 64 KB that does not move
        with the loop dim, N <= 256, K even; the loop must be JIT-specialised
        (the pair code exists only there)."""
        from . import jit
        if not (jit.ENABLED and jit.PAIR_ENABLED) or rows * T < jit.JIT_LOOP_MIN or R > 8:
            return None
        best, size = None, 0
        for i, (kernel, p, re, f64, _) in enumerate(ops):
            if kernel != N.RT_K_GEMM or f64 or re != 1:
                continue
            if any(g.dtype != N.RT_F32 for g in (p.A, p.B, p.C)):
                continue
            if not (p.N.nd == 1 and p.K.nd == 1 and p.z == 1 and p.B.s2[0] == 1
                    and p.B.s1[0] == p.n and p.n <= 256 and p.k % 8 == 0):
                continue
            if p.B.off_env[self.slot[dim]] != 0 or (p.B.ptr + 4 * p.B.off) % 16:
                continue
            nb = p.k * p.n * 4
            if nb >= self.PAIR_MIN_BYTES and nb > size:
                best, size = i, nb
        return best

    def _loop_persistent(self, s: Loop, S, blk=None):
        self._capture = []
        try:
            self.steps(s.body)
        finally:
            subs, self._capture = self._capture, None
        Sext = [self.ext[d] for d in S]
        rows = prod(Sext)
        if s.lo not in (None, 0) or s.hi not in (None, self.ext[s.dim]):
            raise LowerError("persistent loops run a dim's full extent")
        T = self.ext[s.dim]
        ops = []
        max_m = 1
        for (kernel, p, grid, block, smem, label) in subs:
            if kernel == N.RT_K_EW:
                if p.total % rows:
                    raise LowerError("ew box is not row-major over the slab")
                ops.append([kernel, p, p.total // rows, p.f64, None])
            elif kernel == N.RT_K_GEMM:
                # M = slab rows x m, row-major; the index path may have
                # collapsed adjacent dims (m == 1 -> M is the slab itself)
                mext = [p.M.ext[i] for i in range(p.M.nd)]
                if p.z != 1 or p.splits != 1 or p.k > 4096 or prod(mext) % rows:
                    raise LowerError("gemm is not row-blocked over the slab")
                m = prod(mext) // rows
                if not (mext == Sext + [m] or (m == 1 and mext == Sext)
                        or (p.M.nd == 1 and mext[0] == rows * m)):
                    raise LowerError("gemm is not row-blocked over the slab")
                max_m = max(max_m, m)
                ops.append([kernel, p, m, p.f64, None])
            elif kernel in (N.RT_K_UDF, N.RT_K_RNG):
                if p.box.nd != len(S) or [p.box.ext[i] for i in range(len(S))] != Sext:
                    raise LowerError("per-point op box differs from the slab")
                ops.append([kernel, p, 1, 0, None])
            else:
                raise LowerError("op family not supported inside a persistent loop")
        # rows per CTA: the specialised in-loop GEMMs hold <= 8 rows (jit.py
        # _gemm_call); spread rows evenly over the waves that needs
        # JIT-specialised loops fit two CTAs per SM (<= 128 registers,
        # <= 112 KB shared memory): twice the resident row groups, and two
        # independent step chains interleaved on every SM
        from . import jit as _jit
        rmax = max(1, 8 // max_m)
        # (only when one CTA per SM would need several waves: a single wave of
        # 7-row CTAs is faster than two interleaved 4-row chains, C2 measured)
        dual = (_jit.ENABLED and _jit.DUAL_ENABLED and rows * T >= _jit.JIT_LOOP_MIN
                and rows > 148 * rmax)
        slots = 148 * (2 if dual else 1)
        waves = -(-rows // (slots * rmax))
        R = max(1, min(rmax, -(-rows // (slots * waves))))
        a_need, tma = 0, False
        for kernel, p, re, f64, _ in ops:
            if kernel == N.RT_K_GEMM:
                it = 8 if f64 else 4
                need = ((((R * re + 3) // 4 * 4) * p.k * it + 15) // 16) * 16 + p.k * 8
                a_need = max(a_need, need)
                tma = tma or p.n >= 64
        p_off, cur = [], 0
        for kernel, p, re, f64, _ in ops:
            p_off.append(cur)
            cur += (C.sizeof(p) + 127) // 128 * 128
        a_off = cur
        # K-split in-loop GEMMs (jit.ks_eligible) sum per-warp partial tiles
        # through a [8 warps][rows][N] area before the weight ring
        from .jit import KS_ENABLED, ks_eligible, k2_eligible as jit_k2

        def jit_wide():
            return _jit.WIDE_RESIDENT
        red_bytes = 0
        for kernel, p, re, f64, _ in ops:
            if KS_ENABLED and kernel == N.RT_K_GEMM and p.n >= 64 and p.k >= 128 and \
                    ks_eligible(R, re, p, f64):
                mrp = (R * re + 3) // 4 * 4
                red_bytes = max(red_bytes, 8 * mrp * p.n * 4)
            if kernel == N.RT_K_GEMM and jit_k2(R, re, p, f64):
                mrp = (R * re + 3) // 4 * 4
                red_bytes = max(red_bytes, mrp * p.n * 4)
        red_off = (a_off + a_need + 127) // 128 * 128
        # CTA-pair mode (jit._gemm_pair_literal): the largest in-loop weight
        # matrix stays resident, one K-half per SM of a 2-CTA cluster, instead
        # of streaming through the ring from L2 every step
        pair = None if dual else self._pair_op(ops, R, rows, T, s.dim)
        pair_info = None
        pair_bytes = 0
        if pair is not None:
            q = ops[pair][1]
            mrp = (R + 3) // 4 * 4
            kh = q.k // 2
            b_bytes, p_bytes, pa_bytes = kh * q.n * 4, mrp * q.n * 4, kh * mrp * 4
            base = (red_off + red_bytes + 127) // 128 * 128
            pair_info = {"op": pair, "kh": kh, "b_off": base, "p_off": base + b_bytes,
                         "pa_off": base + b_bytes + p_bytes, "nops": len(ops)}
            pair_bytes = b_bytes + p_bytes + pa_bytes
        # small loop-invariant weights stay resident in shared memory
        # (jit._gemm_literal resident=...): no per-step reload or stream
        resident, res_bytes = {}, 0
        res_base = (red_off + red_bytes + pair_bytes + 127) // 128 * 128
        hy = None if pair is not None else self._hybrid_op(ops, R, rows, T, s.dim, dual)
        if pair is None:
            resident, res_bytes = self._resident_ops(ops, rows, T, s.dim, res_base,
                                                     wide=hy is not None and jit_wide(),
                                                     skip=None if hy is None else hy[0])
        # the largest N=256 layer keeps its weights on chip: KR rows in
        # registers, the rest in shared memory (when that leaves room for a
        # small ring for the other streamed layers)
        hybrid = None
        if hy is not None:
            hi, kr, nc = hy
            q = ops[hi][1]
            h_off = (res_base + res_bytes + 127) // 128 * 128
            h_bytes = (q.k - kr) * q.n * 4
            mrp = (R * ops[hi][2] + 3) // 4 * 4
            r_bytes = (nc - 1) * mrp * q.n * 4
            if h_off + h_bytes + r_bytes + 4 * 4096 <= 210 * 1024:
                hybrid = {"op": hi, "kr": kr, "ncol": nc, "off": h_off, "red": h_off + h_bytes}
                res_bytes = h_off + h_bytes + r_bytes - res_base
        ring_off = (res_base + res_bytes + 127) // 128 * 128
        # env normals staged one step ahead (jit._udf_prefetch): 8 rows, in
        # front of the ring (jit derives the ring stage from smem - ring_off)
        nz_bytes = max([8 * 8 * sum(p.out_count[j] for j in range(p.nout))
                        for k, p, *_r in ops if k == N.RT_K_UDF] + [0])
        nz_off = 0
        if nz_bytes:
            nz_off = ring_off
            ring_off = (nz_off + nz_bytes + 127) // 128 * 128
        # EW operands read from buffers no op of this loop writes
        written = set()
        for (kernel, p, grid, block, smem_, label) in subs:
            nd_ = self.g.nodes.get(label[0]) if isinstance(label, tuple) else None
            for oid in range(len(nd_.out_shapes) if nd_ is not None else 0):
                try:
                    written.add(id(self.storage((label[0], oid))))
                except Exception:
                    pass
        ext_in = {}
        for i, (kernel, p, re, f64, _) in enumerate(ops):
            keys = p.__dict__.get("in_keys") if kernel == N.RT_K_EW else None
            if keys:
                try:
                    ext_in[i] = [k for k, key in enumerate(keys)
                                 if id(self.storage(key)) not in written]
                except Exception:
                    pass
        # narrow GEMM outputs forwarded to the next elementwise op (8 rows x
        # <= 32 columns) and loop-external elementwise inputs staged one step
        # ahead (256 threads x 4 inputs x 8 B): jit._ew_stage_plan
        xfwd_off = ring_off
        xpf_off = xfwd_off + 8 * 32 * 4
        xu_off = xpf_off + 256 * 4 * 2         # env-op inputs staged by their producers
        xc_off = xu_off + 512 * 4              # env-op outputs carried to the next step
        ring_off = (xc_off + 256 * 4 + 127) // 128 * 128
        # loop-invariant GEMM biases copied to shared memory once (their
        # per-step global loads sat on each layer's epilogue critical path)
        bias_smem = {}
        from . import jit as _jit2
        if _jit2.ENABLED and _jit2.BIAS_SMEM and rows * T >= _jit2.JIT_LOOP_MIN:
            for i, (k, p, re, f64, _) in enumerate(ops):
                if k != N.RT_K_GEMM or not p.bias.ptr or \
                        p.bias.dtype != (N.RT_F64 if f64 else N.RT_F32) or \
                        p.bias.off_env[self.slot[s.dim]] != 0:
                    continue
                bias_smem[i] = ring_off
                ring_off = (ring_off + p.n * (8 if f64 else 4) + 127) // 128 * 128
        if hybrid is not None:
            # the ring only feeds wide layers that are neither resident nor on chip
            tma = any(k == N.RT_K_GEMM and p.n >= 64 and i not in resident and i != hybrid["op"]
                      for i, (k, p, *_r) in enumerate(ops))
        stage = 0
        budget = (112 if dual else 210) * 1024
        if tma:
            stage = 32 * 1024
            while ring_off + 4 * stage > budget and stage > 4096:
                stage //= 2
        smem = ring_off + 4 * stage
        if dual and smem > budget:
            dual = False
        if smem > 220 * 1024:
            raise LowerError("persistent loop needs too much shared memory")
        # hoist the env's data-independent normals out of the loop
        for op in ops:
            if op[0] != N.RT_K_UDF:
                continue
            up = op[1]
            count = sum(up.out_count[j] for j in range(up.nout))
            buf = self.alloc(rows * T * count * 8)
            q = N.rt_rng_params()
            box = Sext + [T]
            q.box.nd = len(box)
            for i, x in enumerate(box):
                q.box.ext[i] = x
            q.total = prod(box)
            q.nprefix = up.nprefix
            for i in range(up.nprefix):
                q.prefix[i] = up.prefix[i]
            udf = self.g.nodes[[lab for (k2, p2, *_r, lab) in subs if p2 is up][0][0]]
            q.ncoord = len(udf.domain)
            for j, d in enumerate(udf.domain):
                if d == s.dim:
                    q.coord_src[j] = len(S)
                elif d in S:
                    q.coord_src[j] = S.index(d)
                else:
                    q.coord_src[j] = -1 - self.slot[d]
            self._coord_add(q, udf)
            q.dist = 0
            q.count = count
            q.out.ptr = buf
            q.out.dtype = N.RT_F64
            st = cstrides(Sext + [T, count])
            for i in range(len(S) + 1):
                q.out.stride[i] = st[i]
            self.add_rec(N.RT_K_RNG, q, self.grid1(q.total, 128), [128, 1, 1], 0,
                         (udf.id, udf.name + ":noise"))
            op[4] = (buf, 0, T * count, count)
        lp = N.rt_loop_params()
        lp.slot = self.slot[s.dim]
        lp.nops = len(ops)
        if blk is not None:
            lp.blk_slot, lp.blk_len = blk
        n = T
        lp.start, lp.stop, lp.step = (0, n, 1) if s.step > 0 else (n - 1, -1, -1)
        lp.rows = rows
        lp.rows_per_cta = R
        lp.smem_bytes = smem
        lp.ring_off = ring_off
        lp.a_off = a_off
        lp.red_off = red_off if red_bytes else 0
        for op, off in zip(ops, p_off):
            op.append(off)
        first = self.g.nodes[s.body[0].nid]
        nct = -(-rows // R)
        if pair_info is not None:
            nct += nct % 2
            if smem > 225 * 1024:
                raise LowerError("pair loop needs too much shared memory")
        idx = self.add_rec(N.RT_K_LOOP, lp, [nct, 1, 1], [256, 1, 1], smem,
                           (first.id, f"loop[{s.dim}]"))
        self.loop_subs[idx] = {"ops": ops, "trips": T, "pair": pair_info,
                               # a time-blocked loop runs one block per launch
                               "trips_per_launch": min(T, lp.blk_len) if lp.blk_len else T,
                               "ctas_per_sm": 2 if dual else 1, "resident": resident,
                               "hybrid": hybrid, "nz_off": nz_off, "nz_bytes": nz_bytes,
                               "bias_smem": bias_smem, "xfwd_off": xfwd_off, "xpf_off": xpf_off, "xu_off": xu_off, "xc_off": xc_off,
                               "ext_in": ext_in}
        if pair_info is not None:
            self.rec_cluster[idx] = 2

    def _swap_hook(self, kind):
        self.hooks.append({"kind": kind, "slot": self.slot[self.swap.kb]})
        self.prog.append((N.RT_OP_HOOK, len(self.hooks) - 1, 0, 0, 0, 0))

    def _swap_loop(self, s: Loop):
        """Time-blocked acting loop with swap-managed outputs: one persistent
        launch per time block inside a loop over blocks; the ring slot is set
        from the block index, the previous use of the slot is awaited, and
        the finished block is offloaded (swap.SwapRuntime)."""
        sw = self.swap
        S = self._persistent_ok(s)
        if not S:
            raise LowerError("swapping needs a persistent acting loop")
        mark = len(self.prog)
        self._loop_persistent(s, S, blk=(self.slot[sw.kb], sw.bs))
        launch = self.prog.pop()          # the loop record; hoisted draws stay before
        assert launch[0] == N.RT_OP_LAUNCH and len(self.prog) >= mark
        at = len(self.prog)
        self.prog.append([N.RT_OP_FOR, self.slot[sw.kb], 0, sw.DI, 1, 0])
        self.prog.append((N.RT_OP_ENVMOD, sw.ring_slot, self.slot[sw.kb], 2, 0, 0))
        self._swap_hook("swap_wait")
        self.prog.append(launch)
        self._swap_hook("swap_out")
        self.prog.append((N.RT_OP_END, at, 0, 0, 0, 0))
        self.prog[at][5] = len(self.prog)

    def loop(self, s: Loop):
        if self.swap is not None and s.dim == self.swap.dim and s.lo is None and not s.fixed:
            return self._swap_loop(s)
        if self.swap is not None and s.dim == self.swap.kb:
            at = len(self.prog)
            self.prog.append([N.RT_OP_FOR, self.slot[s.dim], 0, self.ext[s.dim], 1, 0])
            self.prog.append((N.RT_OP_ENVMOD, self.swap.ring_slot, self.slot[s.dim], 2, 0, 0))
            self._swap_hook("swap_in")
            self.steps(s.body)
            self.prog.append((N.RT_OP_END, at, 0, 0, 0, 0))
            self.prog[at][5] = len(self.prog)
            return
        S = self._persistent_ok(s)
        if S:
            mark = (len(self.recs), len(self.prog))
            try:
                return self._loop_persistent(s, S)
            except LowerError:
                del self.recs[mark[0]:]
                del self.prog[mark[1]:]
                self._capture = None
        lo = 0 if s.lo is None else s.lo
        hi = self.ext[s.dim] if s.hi is None else s.hi
        if s.step > 0:
            start, stop = lo, hi
        else:
            start, stop = hi - 1, lo - 1
        at = len(self.prog)
        self.prog.append([N.RT_OP_FOR, self.slot[s.dim], start, stop, s.step, 0])
        self.steps(s.body)
        self.prog.append((N.RT_OP_END, at, 0, 0, 0, 0))
        self.prog[at][5] = len(self.prog)

    # -- bulk steps ----------------------------------------------------------

    def bulk(self, s: Bulk):
        n = self.g.nodes[s.nid]
        if self.bufs[(n.id, 0)].alias is not None or n.kind in ("const", "input"):
            return  # aliases and leaves need no kernel
        if n.id in self.virtual:
            return  # fused into its consumer
        if n.id in self.ones_targets:
            return    # a bias sum written by its contraction's launch (ones column)
        if n.id in self._colsum_done:
            self._colsum_done.discard(n.id)   # (per plan instance: its producer ran just before)
            return    # summed by its producer's launch (k_thin_smallv colsum / dw)
        if n.id in self._sibling_done:
            self._sibling_done.discard(n.id)
            return    # written by its sibling head's launch
        ctx = Ctx(self, n, s.fixed)
        if n.id in self.sibling and self._capture is None:
            # the sibling head first, captured (its operands only)
            y2 = self.g.nodes[self.sibling[n.id]]
            x2, b2, _t2 = self.gemm_epi[y2.id]
            self._rows_capture = []
            try:
                self.k_matmul(Ctx(self, y2, s.fixed), self.g.nodes[x2], b2, 0)
                cap = self._rows_capture
            except LowerError:
                cap = []
            finally:
                self._rows_capture = None
            if len(cap) == 1:
                self._rows_second = (y2.id, cap[0])
        if n.id in self.dw_epi and self._capture is None:
            reqs = []
            for sid, which in self.dw_epi[n.id]:
                skey = (sid, 0)
                ss = self.storage(skey)
                sdst = {d: ss.strides[j] for j, d in enumerate(self.bufs[skey].dims)}
                g_ = N.rt_gop()
                g_.ptr, g_.dtype, g_.off = ss.ptr, N.DTYPE_CODE[ss.dtype], 0
                for d in ctx.fixed:
                    if d in sdst:
                        g_.off_env[self.slot[d]] += sdst[d]
                g_.s1[0], g_.s2[0] = ss.strides[-2], ss.strides[-1]
                reqs.append((sid, which, g_))
            self._dw_req = reqs
        if n.id in self.colsum and self._capture is None:
            rkey = (self.colsum[n.id], 0)
            sr = self.storage(rkey)
            rdst = {d: sr.strides[j] for j, d in enumerate(self.bufs[rkey].dims)}
            g_ = N.rt_gop()
            g_.ptr, g_.dtype, g_.off = sr.ptr, N.DTYPE_CODE[sr.dtype], 0
            for d in ctx.fixed:
                if d in rdst:
                    g_.off_env[self.slot[d]] += rdst[d]
            g_.s2[0] = sr.strides[-1]
            self._colsum_req = (rkey[0], g_)
        if any(e == 0 for e in ctx.slab_ext):
            return
        if n.id in self.gemm_epi:
            x, bias_e, tanh = self.gemm_epi[n.id]
            if isinstance(tanh, tuple) and len(tanh) > 4:
                # (X Y + X2 Y2) * (1 - h*h): lower the second product for its
                # operands only, then the first with it attached (one launch)
                self._smallk_capture = []
                try:
                    self.k_matmul(ctx, self.g.nodes[tanh[5]], None, 2, gate_edge=tanh[3])
                    if len(self._smallk_capture) != 1:
                        raise LowerError(f"{n.name}: second gated product is not small-K")
                    qb = self._smallk_capture[0]
                finally:
                    self._smallk_capture = None
                self._smallk_second = qb
                try:
                    self.k_matmul(ctx, self.g.nodes[x], None, 2, gate_edge=tanh[3])
                finally:
                    self._smallk_second = None
            elif isinstance(tanh, tuple):
                self.k_matmul(ctx, self.g.nodes[x], None, 2, gate_edge=tanh[3])
            else:
                self.k_matmul(ctx, self.g.nodes[x], bias_e, 1 if tanh else 0)
        else:
            fn = getattr(self, f"k_{n.kind}", None)
            if fn is None:
                if n.kind not in EW_KINDS:
                    raise LowerError(f"no kernel for op kind {n.kind!r}")
                fn = self.ew
            fn(ctx)
        self._colsum_req = None
        self._dw_req = None
        self._rows_second = None
        if n.id in self.shard_reduce:
            self._hook_allreduce(ctx, (n.id, 0))

    def _hook_allreduce(self, ctx, key):
        """Partial sums over the sharded env dim -> sum all-reduce of the
        slab this launch wrote (contiguous by construction of the layout)."""
        if self._capture is not None:
            raise LowerError("sharded reduction inside a persistent loop")
        v = self.out_view(ctx, key)
        box = list(ctx.slab_ext) + list(self.bufs[key].pshape)
        want = cstrides(box)
        if any(v.stride[i] != want[i] for i in range(len(box)) if box[i] > 1):
            raise LowerError("all-reduced slab is not contiguous")
        st = self.storage(key)
        self.hooks.append({"ptr": st.ptr, "dtype": st.dtype, "off0": v.off,
                           "off_env": {i: v.off_env[i] for i in range(N.RT_MAXENV)
                                       if v.off_env[i]},
                           "count": prod(box), "node": ctx.node.name})
        self.prog.append((N.RT_OP_HOOK, len(self.hooks) - 1, 0, 0, 0, 0))

    # ---- elementwise family

    def ew(self, ctx: Ctx):
        n = ctx.node
        key = (n.id, 0)
        out_p = list(self.bufs[key].pshape)
        P = Prog()
        views = []
        self._view_keys = []
        self._f64 = n.dtype == "f64"
        r = self._value(ctx, n, P, views, out_p, 0)
        P.emit("STORE", a=r)
        self._emit_ew(ctx, key, P, views, self._f64, out_p, (n.id, n.name))

    MAX_FUSE_DEPTH = 6

    def _fusable_operand(self, ctx, n, e, out_p, depth):
        p = self.fuse_src.get(e.src)
        if p is None or p != n.id or depth >= self.MAX_FUSE_DEPTH:
            return False
        src = self.g.nodes[e.src]
        return (e.psi is None and src.domain == n.domain
                and e.phi == tuple(("sym", d, "loop") for d in src.domain)
                and list(self.bufs[(src.id, e.oid)].pshape) == list(out_p))

    ROUND_KINDS = {"add", "sub", "mul", "div", "neg", "exp", "log", "tanh", "sqrt", "pow_const",
                   "scan"}

    def _value(self, ctx: Ctx, n, P: Prog, views: list, out_p, depth):
        """Compile node n's value at the current box element into a value
        register; single-consumer pointwise producers are inlined.  An
        inlined f32 result is rounded to f32 (a no-op unless the fused
        program computes in f64 because some other operand is f64: numpy
        rounds every f32 op, e.g. cast(x, f32) * 3 in an f64 program)."""
        r = self._value_raw(ctx, n, P, views, out_p, depth)
        if n.dtype == "f32" and n.kind in self.ROUND_KINDS and self._f64:
            P.emit("VCAST", d=r, a=r, imm=N.RT_F32)
        return r

    def _value_raw(self, ctx: Ctx, n, P: Prog, views: list, out_p, depth):
        ins = self.g.in_edges(n.id)
        if n.dtype == "f64":
            self._f64 = True

        def view_of(ev, pstrides, extra_off=0, extra_checks=()):
            if ev.progs:
                raise LowerError(f"{n.name}: non-affine index needs the gather path")
            views.append(self.make_view(ctx, ev, pstrides, extra_off, extra_checks))
            self._view_keys.append(ev.buf.key)
            if len(views) > N.RT_MAXIN:
                raise LowerError("too many operands")
            if ev.buf.dtype == "f64":
                self._f64 = True
            return len(views) - 1

        def operand(i, mapping="bcast"):
            e = ins[i]
            if mapping == "bcast" and self._fusable_operand(ctx, n, e, out_p, depth):
                src = self.g.nodes[e.src]
                return self._value(Ctx(self, src, ctx.fixed), src, P, views, out_p, depth + 1)
            ev = self.edge_val(ctx, e)
            if mapping == "bcast":
                pst = self.bcast(ev, out_p)
            else:
                pst = mapping(ev)
            if ev.progs:
                return gather(ev, pst)
            vi = view_of(ev, pst)
            r = P.vreg()
            P.emit("LOAD", d=r, imm=vi)
            return r

        def gather(ev, pst):
            """Non-affine φ components (floordiv/mod/min/max of dims,
            symexpr.py:521-570) evaluated per element on device (Euclidean
            // and %; a zero divisor sets RT_ERR_DIV_ZERO): row offset
            sum(c_j(point) * stride_j), the load masked when a component
            leaves the source's domain (like the affine checks)."""
            dm = ctx.dimmap()
            off = P.ireg()
            P.emit("ICONST", d=off, imm=0)
            ok = P.ireg()
            P.emit("ICONST", d=ok, imm=1)
            for c, S, hi_dom in ev.progs:
                r = P.int_expr(c, dm)
                t = P.ireg()
                P.emit("ICONST", d=t, imm=0)
                P.emit("IGE", d=t, a=r, b=t)
                P.emit("IAND", d=ok, a=ok, b=t)
                P.emit("ICONST", d=t, imm=hi_dom)
                P.emit("ILT", d=t, a=r, b=t)
                P.emit("IAND", d=ok, a=ok, b=t)
                P.emit("ICONST", d=t, imm=S)
                P.emit("IMUL", d=t, a=t, b=r)
                P.emit("IADD", d=off, a=off, b=t)
                P.ifree_(t)
                P.ifree_(r)
            plain = EdgeVal(buf=ev.buf, off=ev.off, coef=dict(ev.coef), checks=list(ev.checks),
                            axes=ev.axes, nslices=ev.nslices, psi=ev.psi)
            vi = view_of(plain, pst)
            v = P.vreg()
            P.emit("LOADX", d=v, a=off, b=ok, imm=vi)
            P.ifree_(ok)
            P.ifree_(off)
            return v

        k = n.kind
        if k in ("add", "sub", "mul", "div"):
            a = operand(0)
            b = operand(1)
            P.emit({"add": "VADD", "sub": "VSUB", "mul": "VMUL", "div": "VDIV"}[k], d=a, a=a, b=b)
            P.vfree_(b)
            return a
        if k in ("neg", "exp", "log", "tanh", "sqrt"):
            a = operand(0)
            P.emit("V" + k.upper(), d=a, a=a)
            return a
        if k == "pow_const":
            a = operand(0)
            P.emit("VPOW", d=a, a=a, imm=P.k(n.params["exponent"]))
            return a
        if k == "cmp":
            a = operand(0)
            b = operand(1)
            op = {"eq": "VEQ", "ne": "VNE", "lt": "VLT", "le": "VLE", "gt": "VGT",
                  "ge": "VGE"}[n.params["op"]]
            P.emit(op, d=a, a=a, b=b)
            P.vfree_(b)
            return a
        if k == "where":
            c = operand(0)
            a = operand(1)
            b = operand(2)
            P.emit("VWHERE", d=c, a=c, b=a, c=b)
            P.vfree_(a)
            P.vfree_(b)
            return c
        if k == "cast":
            a = operand(0)
            P.emit("VCAST", d=a, a=a, imm=N.DTYPE_CODE[n.params["dtype"]])
            return a
        if k in ("identity", "detach", "expand", "set_symbol"):
            return operand(0)
        if k == "reshape":
            def rs(ev):
                if ev.nslices and [a.stride for a in ev.axes] != cstrides([a.ext for a in ev.axes]):
                    raise LowerError("reshape of a non-contiguous gathered slice")
                return cstrides(out_p)
            return operand(0, rs)
        if k == "permute":
            order = n.params["order"]
            return operand(0, lambda ev: [ev.axes[o].stride for o in order])
        if k == "squeeze":
            dd = n.params["dim"]
            return operand(0, lambda ev: [ax.stride for i, ax in enumerate(ev.axes) if i != dd])
        if k == "unsqueeze":
            dd = n.params["dim"]

            def us(ev):
                pst = [ax.stride for ax in ev.axes]
                pst.insert(dd, 0)
                return pst
            return operand(0, us)
        if k == "eval_symbol":
            sym = n.params["symbol"]
            r = P.int_expr(("sym", sym.name, sym.kind), ctx.dimmap())
            v = P.vreg()
            P.emit("VITOF", d=v, a=r)
            P.ifree_(r)
            return v
        if k == "merge":
            dm = ctx.dimmap()
            conds = n.params["conds"]
            res = P.vreg()
            joins = []
            for bi, cond in enumerate(conds):
                if cond == ir.TRUE:
                    a = operand(bi)
                    P.emit("VMOV", d=res, a=a)
                    P.vfree_(a)
                    break
                r = P.int_expr(subst_bounds(cond, self.benv), dm)
                j = P.emit("JZ", a=r)
                P.ifree_(r)
                a = operand(bi)
                P.emit("VMOV", d=res, a=a)
                P.vfree_(a)
                joins.append(P.emit("JMP"))
                P.code[j] = P.pc()
            else:
                # no branch holds: the reference raises (runtime.py:369-370);
                # such points are never demanded by a valid program
                P.emit("VCONST", d=res, imm=P.k(0.0))
            for j in joins:
                P.code[j] = P.pc()
            return res
        if k == "scan":
            # y = x + gamma*prev; prev absent (edge condition false) at the head
            x = operand(0)
            psi = self.edge_val(ctx, ins[1]).psi
            j = None
            if psi is not None:
                r = P.int_expr(psi, ctx.dimmap())
                j = P.emit("JZ", a=r)
                P.ifree_(r)
            pv = operand(1)
            g = P.vreg()
            P.emit("VCONST", d=g, imm=P.k(n.params["gamma"]))
            P.emit("VMUL", d=g, a=g, b=pv)
            P.emit("VADD", d=x, a=x, b=g)
            P.vfree_(g)
            P.vfree_(pv)
            if j is not None:
                P.code[j] = P.pc()
            return x
        if k == "index_select":
            return self._index_select(ctx, P, self.edge_val(ctx, ins[0]), out_p, view_of)
        if k == "slice_axis":
            ev = self.edge_val(ctx, ins[0])
            ax = n.params["axis"]
            bs = n.params["block"]
            jd = n.params["dim"].name
            pst = [a.stride for a in ev.axes]
            if ev.axes[ax].ext is None:
                raise LowerError("slice_axis over a ragged axis")
            # source coordinate along ax = j*bs + k ; zero past the extent
            extra = [(0, {jd: bs, ax: 1}, ev.axes[ax].ext)]
            ev2 = EdgeVal(buf=ev.buf, off=ev.off, coef=dict(ev.coef), checks=list(ev.checks),
                          axes=ev.axes, nslices=ev.nslices)
            ev2.coef[jd] = ev2.coef.get(jd, 0) + bs * ev.axes[ax].stride
            vi = view_of(ev2, pst, extra_checks=extra)
            r = P.vreg()
            P.emit("LOAD", d=r, imm=vi)
            return r
        raise LowerError(f"no elementwise lowering for {k}")

    def _index_select(self, ctx, P, ev, out_p, view_of):
        n = ctx.node
        dname = n.params["dim"].name
        expr = subst_bounds(n.params["expr"], self.benv)
        D = ev.axes[0].ext
        S = ev.axes[0].stride
        rest = [a.stride for a in ev.axes[1:]]
        slab_n = len(ctx.slab)
        if n.params.get("rows"):
            # out[j, q] = x[expr(d := j), q]
            dm = ctx.dimmap({(dname, "loop"): ("coord", slab_n)})
            vi = view_of(ev, [0] + rest)
        elif expr[0] == "slice":
            dm = ctx.dimmap()
            lo = P.int_expr(expr[1], dm)
            hi = P.int_expr(expr[2], dm)
            ok = self._range_ok(P, lo, hi, D)
            j = P.emit("JZ", a=ok)
            skip = P.emit("JMP")
            P.code[j] = P.pc()
            P.emit("ERROR", a=lo, b=hi, imm=N.RT_ERR_SLICE_RANGE)
            P.code[skip] = P.pc()
            P.ifree_(ok)
            P.ifree_(hi)
            # offset = (lo + j) * S where j = payload coord 0
            vi = view_of(ev, [S] + rest)
            off = P.ireg()
            P.emit("ICONST", d=off, imm=S)
            P.emit("IMUL", d=off, a=off, b=lo)
            one = P.ireg()
            P.emit("ICONST", d=one, imm=1)
            v = P.vreg()
            P.emit("LOADX", d=v, a=off, b=one, imm=vi)
            return v
        else:
            dm = ctx.dimmap()
            vi = view_of(ev, rest)
        row = P.int_expr(expr, dm)
        zero = P.ireg()
        P.emit("ICONST", d=zero, imm=0)
        ok = P.ireg()
        P.emit("IGE", d=ok, a=row, b=zero)
        lim = P.ireg()
        P.emit("ICONST", d=lim, imm=D)
        t = P.ireg()
        P.emit("ILT", d=t, a=row, b=lim)
        P.emit("IAND", d=ok, a=ok, b=t)
        j = P.emit("JZ", a=ok)
        skip = P.emit("JMP")
        P.code[j] = P.pc()
        P.emit("ERROR", a=row, b=lim, imm=N.RT_ERR_ROW_RANGE)
        P.code[skip] = P.pc()
        off = P.ireg()
        P.emit("ICONST", d=off, imm=S)
        P.emit("IMUL", d=off, a=off, b=row)
        v = P.vreg()
        P.emit("LOADX", d=v, a=off, b=ok, imm=vi)
        return v

    def _range_ok(self, P, lo, hi, D):
        # 0 <= lo <= hi <= D
        z = P.ireg()
        P.emit("ICONST", d=z, imm=0)
        ok = P.ireg()
        P.emit("IGE", d=ok, a=lo, b=z)
        P.emit("ILE", d=z, a=lo, b=hi)
        P.emit("IAND", d=ok, a=ok, b=z)
        P.emit("ICONST", d=z, imm=D)
        P.emit("ILE", d=z, a=hi, b=z)
        P.emit("IAND", d=ok, a=ok, b=z)
        P.ifree_(z)
        return ok

    def _emit_ew(self, ctx, key, P, views, f64, out_p, label):
        p = N.rt_ew_params()
        box = list(ctx.slab_ext) + list(out_p)
        if len(box) > N.RT_MAXD:
            raise LowerError("box rank too large")
        allv = [self.out_view(ctx, key)] + list(views)
        code = list(P.code)
        box = collapse_box(box, allv, code)
        p.box.nd = len(box)
        for i, e in enumerate(box):
            p.box.ext[i] = e
        p.total = prod(box)
        p.nin = len(views)
        p.f64 = 1 if f64 else 0
        p.out = allv[0]
        for i, v in enumerate(allv[1:]):
            p.in_[i] = v
        for i, w in enumerate(code):
            p.code[i] = w
        for i, c in enumerate(P.konst):
            p.konst[i] = c
        if p.total == 0:
            return
        # source buffers of the operands (persistent loops stage the ones no
        # loop op writes one step ahead: jit._ew_prefetch_inputs)
        keys = list(getattr(self, "_view_keys", []))
        p.__dict__["in_keys"] = keys if len(keys) == len(views) else None
        self.add_rec(N.RT_K_EW, p, self.grid1(p.total), [256, 1, 1], 0, label)

    # ---- reductions

    def k_sum(self, ctx: Ctx):
        n = ctx.node
        if n.id in self.contract:
            return self.k_contract(ctx, self.g.nodes[self.contract[n.id]])
        (e,) = self.g.in_edges(n.id)
        ev = self.edge_val(ctx, e)
        dims = tuple(n.params["dims"])
        return self._reduce(ctx, ev, dims, op=0)

    def k_discounted_sum(self, ctx: Ctx):
        n = ctx.node
        gae = getattr(self.plan, "gae", {}).get(n.id)
        if gae is not None:
            return self._gae_scan(ctx, gae)
        (e,) = self.g.in_edges(n.id)
        ev = self.edge_val(ctx, e)
        ax = n.params["dim"]
        if self._try_scan_window(ctx, ev, ax, n.params["gamma"], n.params.get("reverse", False)):
            return
        return self._reduce(ctx, ev, (ax,), op=1, gamma=n.params["gamma"],
                            reverse=n.params.get("reverse", False))

    def _try_scan_window(self, ctx, ev, ax, gamma, reverse):
        """dsum/sum over r[..., t:T] (reverse scan) or r[..., 0:t+1] with
        reversed weights (forward scan): O(T) instead of O(T^2)."""
        n = ctx.node
        if ax != 0 or ev.nslices != 1 or ev.progs or ev.checks:
            return False
        (e,) = self.g.in_edges(n.id)
        if e.src in self.absorbed:
            return False
        src = self.g.nodes[e.src]
        slice_pos = [j for j, c in enumerate(e.phi) if c[0] == "slice"]
        (sj,) = slice_pos
        sd = src.domain[sj]
        if sd not in ctx.slab:
            return False
        # all other components must be the identity on the sink's dims
        for j, c in enumerate(e.phi):
            if j == sj:
                continue
            if c != ("sym", src.domain[j], "loop"):
                return False
        lo = subst_bounds(e.phi[sj][1], self.benv)
        hi = subst_bounds(e.phi[sj][2], self.benv)
        Tn = self.ext[sd]
        if lo == ("sym", sd, "loop") and hi == ("int", Tn) and not reverse:
            rev = True
        elif lo == ("int", 0) and ir.as_affine(hi) == ({(sd, "loop"): 1}, 1) and reverse:
            rev = False
        else:
            return False
        if list(src.domain) != [d for d in n.domain] or self.bufs[(e.src, e.oid)].pshape != \
                self.bufs[(n.id, 0)].pshape:
            return False
        # scan over the source buffer along sd, written to n's buffer
        sb = self.storage((e.src, e.oid))
        ob = self.storage((n.id, 0))
        p = N.rt_scan_params()
        slab = ctx.slab
        pay = list(self.bufs[(n.id, 0)].pshape)
        box = [self.ext[d] for d in slab] + pay
        p.box.nd = len(box)
        for i, x in enumerate(box):
            p.box.ext[i] = x
        p.sdim = slab.index(sd)
        p.reverse = 1 if rev else 0
        p.gamma = float(gamma) if gamma is not None else 1.0
        p.f64 = 1 if ob.dtype == "f64" else 0
        p.total_lines = prod(box) // box[p.sdim]
        for which, b in (("in_", sb), ("out", ob)):
            v = getattr(p, which)
            v.ptr = b.ptr
            v.dtype = N.DTYPE_CODE[b.dtype]
            st = b.strides
            for j, d in enumerate(n.domain):
                if d in ctx.fixed:
                    v.off_env[self.slot[d]] = st[j]
                else:
                    v.stride[slab.index(d)] = st[j]
            for i, s in enumerate(st[len(n.domain):]):
                v.stride[len(slab) + i] = s
        self._scan_launch(p, (n.id, n.name))
        return True

    def _reduce(self, ctx, ev: EdgeVal, red_axes, op, gamma=1.0, reverse=False):
        n = ctx.node
        key = (n.id, 0)
        if ev.progs:
            raise LowerError(f"{n.name}: non-affine index feeding a reduction")
        if op == 0 and len(red_axes) > 1:
            ev, red_axes = _merge_reduced(ev, red_axes)
        kept = [i for i in range(len(ev.axes)) if i not in red_axes]
        out_p = list(self.bufs[key].pshape)
        if [ev.axes[i].ext for i in kept] != out_p:
            raise LowerError(f"{n.name}: reduction shape mismatch")
        p = N.rt_reduce_params()
        box = list(ctx.slab_ext) + out_p
        p.box.nd = len(box)
        for i, x in enumerate(box):
            p.box.ext[i] = x
        p.total = prod(box)
        p.nred = len(red_axes)
        if p.nred > 4:
            raise LowerError("too many reduced axes")
        p.op = op
        p.gamma = float(gamma)
        p.reverse = 1 if reverse else 0
        out_dt = self.bufs[key].dtype
        p.f64 = 1 if (ev.buf.dtype == "f64" or out_dt == "f64") else 0
        pst = [ev.axes[i].stride for i in kept]
        p.in_ = self.make_view(ctx, ev, pst)
        p.out = self.out_view(ctx, key)
        maxlen = 1
        for j, ai in enumerate(red_axes):
            ax = ev.axes[ai]
            p.red_stride[j] = ax.stride
            p.len_prog[j] = -1
            p.lo_prog[j] = -1
            if ax.ext is not None:
                p.len0[j] = ax.ext
                maxlen *= max(1, ax.ext)
                continue
            aff = ir.as_affine(ax.len_expr)
            if aff is not None:
                co, k = aff
                p.len0[j] = k
                for (name, kind), a in co.items():
                    if name in ctx.fixed:
                        p.len_env[j][self.slot[name]] = a
                    elif name in ctx.slab:
                        p.len_a[j][ctx.slab.index(name)] = a
                    else:
                        raise LowerError("slice length uses a dim outside the domain")
                lo_, hi_ = interval(ax.len_expr, ctx.sink_box())
                maxlen *= max(1, int(hi_) if hi_ != INF else 1 << 20)
            else:
                P = Prog()
                r = P.int_expr(ax.len_expr, ctx.dimmap())
                P.emit("ISTORE", a=r)
                p.len_prog[j] = 0
                for i, w in enumerate(P.code):
                    p.code[i] = w
                lo_, hi_ = interval(ax.len_expr, ctx.sink_box())
                maxlen *= max(1, int(hi_) if hi_ != INF else 1 << 20)
        # column mode: outputs contiguous along the input's innermost box dim and
        # a long constant reduce range (bias gradients over all T*E points)
        const_lens = all(p.len_prog[j] < 0 and not any(p.len_a[j][d] for d in range(p.box.nd))
                         and not any(p.len_env[j][e] for e in range(N.RT_MAXENV))
                         for j in range(p.nred))
        if const_lens and p.box.nd >= 1 and p.in_.stride[p.box.nd - 1] == 1 and \
                maxlen >= 4096 and p.total * maxlen >= (1 << 20):
            ob = (p.total + 255) // 256
            splits = int(max(1, min(maxlen // 256, (148 * 8) // ob, 1024)))
            p.splits = splits
            p.part = self.alloc(splits * p.total * 8)
            self.add_rec(N.RT_K_REDUCE, p, [ob, splits, 1], [256, 1, 1], 0, (n.id, n.name))
            q = N.rt_reduce_params.from_buffer_copy(p)
            q.threads_per_out = -1     # k_reduce_cols_fin: a warp per output
            self.add_rec(N.RT_K_REDUCE, q, [min((p.total + 7) // 8, 148 * 8), 1, 1], [256, 1, 1], 0,
                         (n.id, n.name))
            return
        if const_lens and p.total <= 64 and maxlen >= 4096 and p.total * maxlen >= (1 << 18):
            # few outputs, long constant ranges (a head's bias gradient over all
            # points): split the range over CTAs (column kernel, lanes per output)
            splits = int(max(1, min(maxlen // 1024, 148 * 4, 1024)))
            p.splits = splits
            p.part = self.alloc(splits * p.total * 8)
            self.add_rec(N.RT_K_REDUCE, p, [1, splits, 1], [256, 1, 1], 0, (n.id, n.name))
            q = N.rt_reduce_params.from_buffer_copy(p)
            q.threads_per_out = -1     # k_reduce_cols_fin: a warp per output
            self.add_rec(N.RT_K_REDUCE, q, [min((p.total + 7) // 8, 148 * 8), 1, 1], [256, 1, 1], 0,
                         (n.id, n.name))
            return
        if maxlen >= 256 and p.total < 148 * 64:
            tpo = 1024 if maxlen >= 4096 else 256
            p.threads_per_out = tpo
            grid = [max(1, min(p.total, 148 * 16)), 1, 1]
            block = [tpo, 1, 1]
        elif maxlen >= 32 and p.nred == 1 and abs(p.red_stride[0]) == 1:
            p.threads_per_out = 32
            grid = [max(1, min((p.total + 7) // 8, 148 * 16)), 1, 1]
            block = [256, 1, 1]
        else:
            p.threads_per_out = 1
            grid = self.grid1(p.total)
            block = [256, 1, 1]
        self.add_rec(N.RT_K_REDUCE, p, grid, block, 0, (n.id, n.name))

    def k_window_reduce(self, ctx: Ctx):
        n = ctx.node
        (e,) = self.g.in_edges(n.id)
        ev = self.edge_val(ctx, e)
        if _ragged(ev):
            raise LowerError("window_reduce over a ragged slice")
        dname = n.params["dim"].name
        nb = self.benv[n.params["bound"].name]
        D = ev.axes[0].ext
        lo = subst_bounds(n.params["lo"], self.benv)
        hi = subst_bounds(n.params["hi"], self.benv)
        op = 0 if n.params["op"] == "sum" else 1
        gamma = n.params.get("gamma") or 1.0
        reverse = n.params.get("reverse", False)
        key = (n.id, 0)
        slab_n = len(ctx.slab)
        # payload coord 0 is the folded dim's row j
        dm = ctx.dimmap({(dname, "loop"): ("coord", slab_n)})
        # suffix form lo = d, hi = D: reverse scan of the value along axis 0
        if lo == ("sym", dname, "loop") and (hi == ("int", D) or hi == ("int", nb)) and D == nb \
                and not reverse and not ev.checks:
            return self._scan_value(ctx, ev, key, axis=0, gamma=gamma if op else 1.0, rev=True)
        lo_c = ("max", ("int", 0), lo)
        hi_c = ("min", ("int", D), hi)
        p = N.rt_reduce_params()
        out_p = list(self.bufs[key].pshape)
        box = list(ctx.slab_ext) + out_p
        p.box.nd = len(box)
        for i, x in enumerate(box):
            p.box.ext[i] = x
        p.total = prod(box)
        p.nred = 1
        p.op = op
        p.gamma = float(gamma)
        p.reverse = 1 if reverse else 0
        p.f64 = 1 if ev.buf.dtype == "f64" else 0
        pst = [0] + [a.stride for a in ev.axes[1:]]
        p.in_ = self.make_view(ctx, ev, pst)
        p.out = self.out_view(ctx, key)
        P = Prog()
        r = P.int_expr(lo_c, dm)
        P.emit("ISTORE", a=r)
        P.ifree_(r)
        lo_pc = 0
        len_pc = P.pc()
        a = P.int_expr(hi_c, dm)
        b = P.int_expr(lo_c, dm)
        P.emit("ISUB", d=a, a=a, b=b)
        P.emit("ISTORE", a=a)
        p.lo_prog[0] = lo_pc
        p.len_prog[0] = len_pc
        p.red_stride[0] = ev.axes[0].stride
        for i, w in enumerate(P.code):
            p.code[i] = w
        p.threads_per_out = 1
        self.add_rec(N.RT_K_REDUCE, p, self.grid1(p.total), [256, 1, 1], 0, (n.id, n.name))

    def _scan_value(self, ctx, ev, key, axis, gamma, rev):
        n = ctx.node
        p = N.rt_scan_params()
        out_p = list(self.bufs[key].pshape)
        box = list(ctx.slab_ext) + out_p
        p.box.nd = len(box)
        for i, x in enumerate(box):
            p.box.ext[i] = x
        p.sdim = len(ctx.slab) + axis
        p.reverse = 1 if rev else 0
        p.gamma = float(gamma)
        ob = self.storage(key)
        p.f64 = 1 if ob.dtype == "f64" else 0
        p.total_lines = prod(box) // box[p.sdim]
        p.in_ = self.make_view(ctx, ev, [a.stride for a in ev.axes])
        p.out = self.out_view(ctx, key)
        self._scan_launch(p, (n.id, n.name))

    SCAN_STAGES = 3

    def _gae_scan(self, ctx, info):
        """A = dsum(delta[t:T]) with delta = r + c*V[t+1] - V formed inside
        the scan (executor.find_gae_fusions, csrc/k_scan.cu k_scan_gae)."""
        n = ctx.node
        key = (n.id, 0)
        delta = self.g.nodes[info["x"].sink]
        dctx = Ctx(self, delta, ctx.fixed)
        p = N.rt_scan_params()
        box = list(ctx.slab_ext)
        p.box.nd = len(box)
        for i, x in enumerate(box):
            p.box.ext[i] = x
        p.sdim = len(ctx.slab) - 1
        if ctx.slab[-1] != n.domain[-1]:
            raise LowerError("GAE scan over a fixed dim")
        p.reverse = 1
        p.gamma = float(n.params["gamma"])
        ob = self.storage(key)
        p.f64 = 1 if ob.dtype == "f64" else 0
        p.total_lines = prod(box) // box[p.sdim]
        rx = self.edge_val(dctx, info["x"])
        vz = self.edge_val(dctx, info["z"])
        for ev in (rx, vz):
            if ev.progs or ev.checks or _ragged(ev) or ev.buf.dtype != ob.dtype:
                raise LowerError("GAE scan operand needs a gather")
        p.in_ = self.make_view(dctx, rx, [])
        p.in2 = self.make_view(dctx, vz, [])
        p.out = self.out_view(ctx, key)
        p.gae, p.gae_c, p.gae_vb = 1, info["c"], info["vb"]
        vw, esize = (2, 8) if p.f64 else (4, 4)
        for v in (p.in_, p.in2, p.out):
            if v.stride[p.sdim] != 1 or (v.ptr + esize * v.off) % 16 or \
                    any(v.off_env[e] % vw for e in range(N.RT_MAXENV)) or \
                    any(v.stride[d] % vw for d in range(p.box.nd) if d != p.sdim and box[d] > 1):
                raise LowerError("GAE scan operands are not line-major and 16-B aligned")
        if self._scan_bulk(p, 2, (n.id, n.name)):
            return
        smem = 2 * self.SCAN_STAGES * 64 * 8 * 16 + 3 * 64 * 8      # k_scan_gae: 8 vectors/line
        self.add_rec(N.RT_K_SCAN, p, [-(-p.total_lines // 64), 1, 1], [64, 1, 1], smem,
                     (n.id, n.name))

    SCAN_TMA = os.environ.get("RTB200_SCAN_TMA", "1") != "0"

    def _scan_bulk(self, p, nin, label):
        """TMA scan (csrc/k_scan_tma.cu, tile 4): one warp per 32 lines,
        128-byte x 32-line boxes per operand and stage.  Needs every
        operand 2-D: unit stride along the scan dim, the other dims
        collapsing to one line stride (a multiple of 16 bytes), 16-byte
        aligned bases.  The stage count is chosen so that every CTA of the
        launch is resident at once (no tail wave): one SM's shared memory
        (228 KB, 1 KB reserved per CTA) split over the CTAs it must hold,
        at most 4 (the r2t sweep: 2 -> 53%, 4 -> 75%, 8 -> 54% of HBM with
        a tail wave); RTB200_SCAN_STAGES overrides for measurements."""
        if not self.SCAN_TMA or p.total_lines >= (1 << 31):
            return False
        esize = 8 if p.f64 else 4
        nd, sd = p.box.nd, p.sdim
        L = p.box.ext[sd]
        if L >= (1 << 31) or L % (16 // esize):
            return False
        views = [p.in_, p.out] + ([p.in2] if nin == 2 else [])
        for v in views:
            if v.stride[sd] != 1 or (v.ptr + esize * v.off) % 16 or \
                    any(v.off_env[e] % (16 // esize) for e in range(N.RT_MAXENV)):
                return False
            st, span = None, 1
            for d in reversed(range(nd)):
                if d == sd or p.box.ext[d] <= 1:
                    continue
                if st is None:
                    st = v.stride[d]
                elif v.stride[d] != st * span:
                    return False
                span *= p.box.ext[d]
            if st is not None and p.total_lines > 1 and (st * esize) % 16:
                return False
        ctas = -(-p.total_lines // 32)
        per_sm = min(32, -(-ctas // 148))
        budget = (228 * 1024) // per_sm - 1024
        ns = min(4, (budget - 1024 - 64) // (nin * 4096))   # 4 measured best (r2t sweep)
        env_s = os.environ.get("RTB200_SCAN_STAGES")
        if env_s:
            ns = int(env_s)
        if ns < 2:
            return False
        smem = ns * nin * 4096 + 8 * ns + 1024
        if smem > 227 * 1024:
            return False
        p.tile, p.chunk, p.stages = 4, 128 // esize, ns
        self.add_rec(N.RT_K_SCAN, p, [ctas, 1, 1], [32, 1, 1], smem, label)
        return True

    def _scan_launch(self, p, label):
        """Pick the scan kernel (csrc/k_scan.cu): tiled 64-line CTAs with
        16-byte I/O for contiguous lines whose starts and length are
        vector-aligned; warp-per-line for other contiguous lines; one
        thread per line (64-thread CTAs, many in flight) for strided lines."""
        sd = p.sdim
        contig = p.in_.stride[sd] == 1 and p.out.stride[sd] == 1
        same_t = p.in_.dtype == p.out.dtype == (N.RT_F64 if p.f64 else N.RT_F32)
        vw = 2 if p.f64 else 4
        esize = 8 if p.f64 else 4

        def aligned(v, skip=(sd,)):
            if (v.ptr + esize * v.off) % 16:
                return False
            if any(v.off_env[e] % vw for e in range(N.RT_MAXENV)):
                return False
            return all(v.stride[d] % vw == 0 for d in range(p.box.nd)
                       if d not in skip and p.box.ext[d] > 1)

        L = p.box.ext[sd]
        smem = self.SCAN_STAGES * 64 * 16 * 16 + 2 * 64 * 8         # 16 vectors per line
        lines = [d for d in range(p.box.nd) if d != sd and p.box.ext[d] > 1]
        inner = lines[-1] if lines else None
        nblk = -(-p.total_lines // 64)
        if contig and same_t and L % vw == 0 and aligned(p.in_) and aligned(p.out) \
                and nblk < (1 << 31):
            if self._scan_bulk(p, 1, label):
                return
            p.tile = 2
            self.add_rec(N.RT_K_SCAN, p, [nblk, 1, 1], [64, 1, 1], smem, label)
        elif (same_t and inner is not None and p.in_.stride[inner] == 1
              and p.out.stride[inner] == 1 and p.box.ext[inner] % 64 == 0
              and aligned(p.in_, (inner,)) and aligned(p.out, (inner,))
              and nblk < (1 << 31)):
            p.tile = 3
            self.add_rec(N.RT_K_SCAN, p, [nblk, 1, 1], [64, 1, 1], smem, label)
        elif contig:
            self.add_rec(N.RT_K_SCAN, p, self.grid1(p.total_lines * 32), [256, 1, 1], 0, label)
        else:
            self.add_rec(N.RT_K_SCAN, p, self.grid1(p.total_lines, 64, 148 * 64), [64, 1, 1], 0,
                         label)

    def k_cumsum(self, ctx: Ctx):
        n = ctx.node
        (e,) = self.g.in_edges(n.id)
        ev = self.edge_val(ctx, e)
        if _ragged(ev) or ev.checks:
            raise LowerError("cumsum over a ragged slice")
        return self._scan_value(ctx, ev, (n.id, 0), n.params["dim"], 1.0,
                                bool(n.params.get("reverse")))

    def k_discounted_cumsum(self, ctx: Ctx):
        n = ctx.node
        (e,) = self.g.in_edges(n.id)
        ev = self.edge_val(ctx, e)
        if _ragged(ev) or ev.checks:
            raise LowerError("discounted_cumsum over a ragged slice")
        return self._scan_value(ctx, ev, (n.id, 0), n.params["dim"], n.params["gamma"],
                                bool(n.params.get("reverse")))

    # ---- matmul

    def k_matmul(self, ctx: Ctx, X=None, bias_edge=None, epilogue=0, gate_edge=None):
        """GEMM for matmul node X (default: ctx.node) written into ctx.node's
        buffer, optionally with a fused `+ bias` and `tanh` epilogue."""
        n = ctx.node
        X = X or n
        xctx = ctx if X is n else Ctx(self, X, ctx.fixed)
        ea, eb = self.g.in_edges(X.id)
        A, B = self.edge_val(xctx, ea), self.edge_val(xctx, eb)
        for ev in (A, B):
            if _ragged(ev) or ev.checks or ev.progs:
                raise LowerError(f"{n.name}: matmul operand needs a gather")
        key = (n.id, 0)
        st = self.storage(key)
        a_ax, b_ax, batch, m, nn, kk, c_log = self._mm_shapes(A, B, st.strides[len(st.dims):])
        cdst = {d: st.strides[j] for j, d in enumerate(self.bufs[key].dims)}
        Z, M, Nn, K = [], [], [], []
        nb = len(batch)
        for d in ctx.slab:
            a_s, b_s, c_s = A.coef.get(d, 0), B.coef.get(d, 0), cdst[d]
            if b_s != 0:
                Z.append((self.ext[d], a_s, b_s, c_s))
            else:
                M.append((self.ext[d], a_s, 0, c_s))
        for i, x in enumerate(batch):
            Z.append((x, self._bstride(a_ax, i, nb), self._bstride(b_ax, i, nb), c_log[i]))
        M.append((m, a_ax[-2].stride, 0, c_log[nb]))
        Nn.append((nn, 0, b_ax[-1].stride, c_log[nb + 1]))
        K.append((kk, a_ax[-1].stride, b_ax[-2].stride, 0))
        env_a = {self.slot[d]: s for d, s in A.coef.items() if d in ctx.fixed}
        env_b = {self.slot[d]: s for d, s in B.coef.items() if d in ctx.fixed}
        env_c = {self.slot[d]: cdst[d] for d in ctx.fixed if d in cdst}
        bias = None
        if bias_edge is not None:
            bv = self.edge_val(ctx, bias_edge)
            if any(d in ctx.slab and self.ext[d] != 1 for d in bv.coef) or bv.checks \
                    or bv.progs or _ragged(bv):
                raise LowerError(f"{n.name}: bias varies across the GEMM rows")
            bias = N.rt_gop()
            bias.ptr = bv.buf.ptr
            bias.dtype = N.DTYPE_CODE[bv.buf.dtype]
            bias.off = bv.off
            for d, sv in bv.coef.items():
                bias.off_env[self.slot[d]] += sv
            bias.s2[0] = bv.axes[-1].stride if bv.axes and bv.axes[-1].ext != 1 else 0
        gate = None
        if gate_edge is not None:
            # epilogue 2: C = acc * (1 - h*h) with h laid out exactly like C
            hv = self.edge_val(ctx, gate_edge)
            if hv.checks or hv.progs or _ragged(hv) or any(t[0] != 1 for t in Z) or len(hv.axes) != 2:
                raise LowerError(f"{n.name}: gate operand is not a plain view "
                                 f"({len(hv.checks)}, {len(hv.progs)}, {_ragged(hv)}, {Z}, {hv.axes})")
            same = all(hv.coef.get(d, 0) == cdst[d] for d in ctx.slab if self.ext[d] != 1) and \
                (m == 1 or hv.axes[-2].stride == c_log[nb]) and hv.axes[-1].stride == c_log[nb + 1]
            if not same:
                raise LowerError(f"{n.name}: gate operand layout differs from the output's")
            gate = N.rt_gop()
            gate.ptr = hv.buf.ptr if hasattr(hv.buf, "ptr") else self.storage(hv.buf.key).ptr
            gate.dtype = N.DTYPE_CODE[hv.buf.dtype]
            gate.off = hv.off
            for d, sv in hv.coef.items():
                if d in ctx.fixed:
                    gate.off_env[self.slot[d]] += sv
        self._gemm((A.buf, A.off, env_a), (B.buf, B.off, env_b), (st, 0, env_c),
                   Z, M, Nn, K, (n.id, n.name), epilogue=epilogue, bias=bias, gate=gate)

    @staticmethod
    def _bstride(axes, i, nb):
        off = nb - (len(axes) - 2)
        j = i - off
        if j < 0:
            return 0
        ax = axes[j]
        return 0 if ax.ext == 1 else ax.stride

    @staticmethod
    def _mm_shapes(A, B, c_pstr):
        """numpy matmul promotion (frontend.py:485-502): logical operands
        (batch..., m, k) @ (batch..., k, n); output strides for (batch, m, n)."""
        a_vec, b_vec = len(A.axes) == 1, len(B.axes) == 1
        a_ax = [Axis(1, 0)] + A.axes if a_vec else list(A.axes)
        b_ax = B.axes + [Axis(1, 0)] if b_vec else list(B.axes)
        m, kk = a_ax[-2].ext, a_ax[-1].ext
        k2, nn = b_ax[-2].ext, b_ax[-1].ext
        if kk != k2:
            raise LowerError("matmul inner dims differ")
        batch = list(np.broadcast_shapes(tuple(x.ext for x in a_ax[:-2]),
                                         tuple(x.ext for x in b_ax[:-2])))
        c = list(c_pstr)
        nb = len(batch)
        if a_vec and b_vec:
            c_log = c + [0, 0]
        elif a_vec:
            c_log = c[:nb] + [0] + c[nb:]
        elif b_vec:
            c_log = c + [0]
        else:
            c_log = c
        if len(c_log) != nb + 2:
            raise LowerError("matmul output layout mismatch")
        return a_ax, b_ax, batch, m, nn, kk, c_log

    def _gemm(self, A, B, Cc, Z, M, Nn, K, label, accumulate=0, epilogue=0, bias=None, gate=None,
              ones=None):
        """Z/M/N/K: lists of (extent, a_stride, b_stride, c_stride).
        A/B/C: (buf, element offset, {env slot: stride})."""
        p = N.rt_gemm_params()
        M, K = self._collapse_box(M), self._collapse_box(K)
        if bias is None:
            Nn = self._collapse_box(Nn)
        if not Z:
            Z = [(1, 0, 0, 0)]
        for gb, lst in ((p.Z, Z), (p.M, M), (p.N, Nn), (p.K, K)):
            if len(lst) > 4:
                raise LowerError("gemm decomposition too deep")
            gb.nd = len(lst)
            for i, t in enumerate(lst):
                gb.ext[i] = t[0]
        p.z, p.m, p.n, p.k = (prod(t[0] for t in Z), prod(t[0] for t in M),
                              prod(t[0] for t in Nn), prod(t[0] for t in K))
        for op, (buf, off, envs), role in ((p.A, A, 0), (p.B, B, 1), (p.C, Cc, 2)):
            op.ptr = buf.ptr
            op.dtype = N.DTYPE_CODE[buf.dtype]
            op.off = off
            for sl, s in envs.items():
                op.off_env[sl] += s
            col = 1 + role if role < 2 else 3
            for i, t in enumerate(Z):
                op.sz[i] = t[1 + role]
            if role == 0:
                for i, t in enumerate(M):
                    op.s1[i] = t[1]
                for i, t in enumerate(K):
                    op.s2[i] = t[1]
            elif role == 1:
                for i, t in enumerate(K):
                    op.s1[i] = t[2]
                for i, t in enumerate(Nn):
                    op.s2[i] = t[2]
            else:
                for i, t in enumerate(M):
                    op.s1[i] = t[3]
                for i, t in enumerate(Nn):
                    op.s2[i] = t[3]
            del col
        p.f64 = 1 if Cc[0].dtype == "f64" else 0
        p.splits = 1
        p.accumulate = accumulate
        p.epilogue = epilogue
        if bias is not None:
            p.bias = bias
        if gate is not None:
            # the tanh-VJP gate epilogue: the narrow-K thin kernel or the
            # tcgen05 TMA GEMM (executor.find_gate_epilogues fuses only there)
            if not self._capture_active() and self._gemm_thin(p, Z, M, Nn, K, label, accumulate,
                                                              epilogue, None, gate=gate):
                return
            if self._smallk_capture is not None or self._smallk_second is not None:
                raise LowerError(f"{label[1]}: summed gated products need the small-K kernel")
            if not self._capture_active() and self.use_tc and self._tc_ok(p, A, B, Cc) and \
                    self.use_tma and self._tma_ok(p) and p.k <= N.TMA_DRAIN_K and not accumulate:
                g = N.rt_gop()
                C.memmove(C.addressof(g), C.addressof(gate), C.sizeof(g))
                g.s1[0], g.s2[0] = p.C.s1[0], p.C.s2[0]     # laid out like C (k_matmul)
                p.bias = g
                p.epilogue = 2
                return self._gemm_tc(p, label, accumulate, 2, None)
            raise LowerError(f"{label[1]}: gate epilogue needs the thin or the TMA GEMM")
        if not self._capture_active() and self._gemm_thin(p, Z, M, Nn, K, label, accumulate,
                                                          epilogue, bias, ones=ones):
            return
        if ones is not None:
            raise LowerError(f"{label[1]}: the bias-gradient column needs the thin contraction")
        if self.use_tc and self._tc_ok(p, A, B, Cc):
            return self._gemm_tc(p, label, accumulate, epilogue, bias)
        tiles = ((p.m + 63) // 64) * ((p.n + 63) // 64) * p.z
        splits = 1
        if tiles < 148 and p.k >= 1024:
            splits = int(min(128, max(1, (148 * 4) // max(1, tiles)), max(1, p.k // 512)))
        if p.z * splits > 65535 or (p.n + 63) // 64 > 65535:
            raise LowerError("gemm grid too large")
        if splits > 1:
            p.splits = splits
            esize = 8 if p.f64 else 4
            p.part = self.alloc(splits * p.z * p.m * p.n * esize)
            grid = [(p.m + 63) // 64, (p.n + 63) // 64, p.z * splits]
            self.add_rec(N.RT_K_GEMM, p, grid, [256, 1, 1], 0, label)
            q = N.rt_splitk_params()
            q.Z, q.M, q.N = p.Z, p.M, p.N
            q.z, q.m, q.n = p.z, p.m, p.n
            q.splits = splits
            q.f64 = p.f64
            q.accumulate = accumulate
            q.epilogue = epilogue
            q.part = p.part
            q.C = p.C
            if bias is not None:
                q.bias = bias
            self.add_rec(N.RT_K_SPLITK, q, [int(min((p.z * p.m * p.n + 7) // 8, 148 * 16)), 1, 1], [256, 1, 1], 0,
                         label)   # k_splitk: a warp per output
        else:
            grid = [(p.m + 63) // 64, (p.n + 63) // 64, p.z]
            self.add_rec(N.RT_K_GEMM, p, grid, [256, 1, 1], 0, label)

    @staticmethod
    def _collapse(lst, cols):
        """Merge the (extent, strides...) dims of a GEMM box into one dim when
        every operand in `cols` walks them contiguously; None otherwise."""
        dims = [t for t in lst if t[0] != 1]
        if not dims:
            return 1, [0] * len(cols)
        ext, st = dims[-1][0], [dims[-1][c] for c in cols]
        for t in reversed(dims[:-1]):
            if any(t[c] != st[i] * ext for i, c in enumerate(cols)):
                return None
            ext *= t[0]
        return ext, st

    @staticmethod
    def _collapse_box(lst):
        """Merge adjacent (extent, a, b, c strides) GEMM box dims that every
        operand walks contiguously; extent-1 dims are dropped."""
        dims = [t for t in lst if t[0] != 1]
        if not dims:
            return [(1, 0, 0, 0)]
        out = [dims[-1]]
        for t in reversed(dims[:-1]):
            nxt = out[0]
            if all(t[c] == nxt[c] * nxt[0] for c in (1, 2, 3)):
                out[0] = (t[0] * nxt[0],) + tuple(nxt[1:])
            else:
                out.insert(0, t)
        return out

    THIN_MAX_R = 32
    THIN_MIN_K = 4096

    def ones_bias_label(self, label):
        return self.ones_bias.get(label[0], label[0])

    def ones_bias_name(self, label):
        r = self.ones_bias.get(label[0])
        return self.g.nodes[r].name if r is not None else label[1]

    def _gemm_thin(self, p, Z, M, Nn, K, label, accumulate, epilogue, bias, gate=None, ones=None):
        """Narrow GEMMs -> RT_K_THIN (csrc/k_gemm_thin.cu); False if not one."""
        if p.z != 1 or any(t[0] != 1 for t in Z):
            return False
        mc, nc, kc = self._collapse(M, (1, 3)), self._collapse(Nn, (2, 3)), self._collapse(K, (1, 2))
        dt = [self._gop_dtype(x) for x in (p.A, p.B, p.C)]
        f64 = dt == ["f64"] * 3
        if not (f64 or dt == ["f32"] * 3):
            return False
        if gate is not None:
            if nc is None or kc is None or self._gop_dtype(gate) != dt[0]:
                return False
            return self._gemm_smallk(p, M, nc, kc, f64, label, accumulate, epilogue, None, gate=gate)
        if nc is not None and kc is not None and self._gemm_rows(p, M, nc, kc, f64, label,
                                                                 accumulate, epilogue, bias):
            return True
        if nc is None or kc is None:
            return False
        if mc is None:
            # rows that do not collapse (e.g. gathered minibatch rows): only
            # the small-K variant walks a multi-dim row box
            return self._gemm_smallk(p, M, nc, kc, f64, label, accumulate, epilogue, bias)
        (m, (a_m, c_m)), (n, (b_n, c_n)), (k, (a_k, b_k)) = mc, nc, kc
        q = N.rt_thin_params()
        q.f64 = int(f64)
        esize = 8 if f64 else 4

        def gop(src, s1, s2):
            g = N.rt_gop()
            C.memmove(C.addressof(g), C.addressof(src), C.sizeof(g))
            for arr in (g.sz, g.s1, g.s2):
                for i in range(4):
                    arr[i] = 0
            g.s1[0], g.s2[0] = s1, s2
            return g

        if k >= self.THIN_MIN_K and (n <= self.THIN_MAX_R < m and a_m == 1
                                      or m <= self.THIN_MAX_R < n and b_n == 1):
            q.variant = 1
            if n <= self.THIN_MAX_R and a_m == 1:
                if ones is not None:
                    return False
                q.w, q.r = m, n
                q.X, q.Y = gop(p.A, a_k, a_m), gop(p.B, b_k, b_n)
                q.part_w, q.part_r = n, 1
            else:
                q.w, q.r = n, m
                q.X, q.Y = gop(p.B, b_k, b_n), gop(p.A, a_k, a_m)
                q.part_w, q.part_r = 1, n
            q.k = k
            gx = (q.w + 255) // 256
            smem = 0
            if self._thin_bulk_ok(q):
                # k_thin_contract_bulk: 2 CTAs per SM, the splits one wave
                q.vec = 1
                q.splits = int(max(1, min(296 // gx, -(-k // 32), 65535)))
                rp = 4 if q.r <= 4 else 8 if q.r <= 8 else 16
                smem = 3 * 32 * (256 + rp) * 4 + 3 * 8      # BK_ST x BK_SR rows + mbarriers
            else:
                q.splits = int(max(1, min(k // 256, (148 * 8) // gx, 65535)))
            q.part = self.alloc(q.splits * m * n * esize)
            self.add_rec(N.RT_K_THIN, q, [gx, q.splits, 1], [256, 1, 1], smem, label)
            r = N.rt_splitk_params()
            r.Z, r.M, r.N = p.Z, p.M, p.N
            r.z, r.m, r.n = p.z, p.m, p.n
            r.splits, r.f64, r.accumulate, r.epilogue = q.splits, q.f64, accumulate, epilogue
            r.part, r.C = q.part, p.C
            if bias is not None:
                r.bias = bias
            self.add_rec(N.RT_K_SPLITK, r, [int(min((p.m * p.n + 7) // 8, 148 * 16)), 1, 1], [256, 1, 1], 0,
                         label)   # k_splitk: a warp per output
            if ones is not None:
                # the ones column: sum_k X[k, w] per split -> part2 -> the bias sum
                q.ones, q.part2 = 1, self.alloc(q.splits * q.w * esize)
                r2 = N.rt_splitk_params()
                r2.Z.nd = r2.M.nd = 1
                r2.Z.ext[0] = r2.M.ext[0] = 1
                r2.N.nd = 1
                r2.N.ext[0] = q.w
                r2.z, r2.m, r2.n = 1, 1, q.w
                r2.splits, r2.f64 = q.splits, q.f64
                r2.part, r2.C = q.part2, ones
                self.add_rec(N.RT_K_SPLITK, r2, [int(min((q.w + 7) // 8, 148 * 16)), 1, 1],
                             [256, 1, 1], 0, (self.ones_bias_label(label), self.ones_bias_name(label)))
            return True
        return self._gemm_smallk(p, M, nc, kc, f64, label, accumulate, epilogue, bias)

    THIN_BULK = os.environ.get("RTB200_THIN_BULK", "1") != "0"

    def _thin_bulk_ok(self, q):
        """Variant 1 can stream its rows by cp.async.bulk (k_thin_contract_bulk):
        fp32, contiguous 16-byte-aligned X and Y rows at every env offset."""
        if not self.THIN_BULK or q.f64 or q.r > 16 or q.w % 4 or q.r % 4:
            return False
        for g in (q.X, q.Y):
            if g.s2[0] != 1 or g.s1[0] % 4 or g.off % 4 or (g.ptr + 4 * g.off) % 16:
                return False
            if any(g.off_env[e] % 4 for e in range(N.RT_MAXENV)):
                return False
        return True

    def _gemm_smallk(self, p, M, nc, kc, f64, label, accumulate, epilogue, bias, gate=None):
        """K <= 32 products over many rows (the observation layer, dX of a
        narrow head) -> RT_K_THIN variant 2; rows may be a multi-dim box
        (gathered minibatch rows)."""
        (n, (b_n, c_n)), (k, (a_k, b_k)) = nc, kc
        m = prod(t[0] for t in M)
        esize = 8 if f64 else 4
        kp = 4 if k <= 4 else 8 if k <= 8 else 16 if k <= 16 else 32
        smem = (kp * n + 64 * kp + n) * esize
        mdims = [t for t in M if t[0] != 1] or [(1, 0, 0, 0)]
        if not (k <= 32 and m >= 4096 and c_n == 1 and smem <= 48 * 1024 and len(mdims) <= 4):
            return False
        if bias is not None and p.N.nd > 1:
            return False
        q = N.rt_thin_params()
        q.f64 = int(f64)
        q.variant = 2
        q.w, q.r, q.k = m, n, k
        q.W.nd = len(mdims)
        for i, t in enumerate(mdims):
            q.W.ext[i] = t[0]

        def gop(src, s1, s2):
            g = N.rt_gop()
            C.memmove(C.addressof(g), C.addressof(src), C.sizeof(g))
            for arr in (g.sz, g.s1, g.s2):
                for i in range(4):
                    arr[i] = 0
            for i, v in enumerate(s1):
                g.s1[i] = v
            for i, v in enumerate(s2):
                g.s2[i] = v
            return g

        q.X = gop(p.A, [a_k], [t[1] for t in mdims])
        q.Y = gop(p.B, [b_k], [b_n])
        q.C = gop(p.C, [t[3] for t in mdims], [c_n])
        if bias is not None:
            q.bias = gop(bias, [0], [bias.s2[0]])
        if gate is not None:
            # epilogue 2: the gate operand walks C's strides (checked in k_matmul)
            q.bias = gop(gate, [t[3] for t in mdims], [c_n])
        q.accumulate, q.epilogue = accumulate, epilogue
        if self._smallk_capture is not None:
            self._smallk_capture.append(q)     # the second product of a dual gate
            return True
        qb = self._smallk_second
        if qb is not None:
            if gate is None or qb.w != q.w or qb.r != q.r or qb.k > 4 or \
                    kp > (8 if f64 else 16) or qb.W.nd != q.W.nd or \
                    any(qb.W.ext[i] != q.W.ext[i] for i in range(q.W.nd)):
                return False
            q.k2, q.X2, q.Y2 = qb.k, qb.X, qb.Y
            smem += (4 * n + 64 * 4) * esize
            if smem > 48 * 1024:
                return False
        if self.THIN_VEC and self._smallk_vec_ok(q, kp, f64, gate is not None):
            q.vec, smem = 1, 0           # k_thin_smallv: static shared memory
        grid = [int(min((m + 63) // 64, 148 * 8)), 1, 1]
        self._dw_recs = []
        req = self._colsum_req
        if req is not None and q.vec and gate is not None and not accumulate:
            # the row sum of this output (its bias gradient) from the same launch
            q.colsum, q.part2 = 1, self.alloc(grid[0] * q.r * 8)
        self.add_rec(N.RT_K_THIN, q, grid, [256, 1, 1], smem, label)
        for sid, which, gd in (self._dw_req or []) if (q.vec and gate is not None) else []:
            kk = q.k2 if which else q.k
            if which and not q.k2:
                continue
            part = self.alloc(grid[0] * q.r * kk * 8)
            if which:
                q.dw2, q.part4 = 1, part
            else:
                q.dw, q.part3 = 1, part
            r3 = N.rt_splitk_params()
            r3.Z.nd = r3.M.nd = r3.N.nd = 1
            r3.Z.ext[0] = 1
            r3.M.ext[0], r3.N.ext[0] = q.r, kk
            r3.z, r3.m, r3.n = 1, q.r, kk
            r3.splits, r3.f64 = grid[0], 1          # fp64 partials, stored in C's dtype
            r3.part, r3.C = part, gd
            self._dw_recs.append((r3, [int(min((q.r * kk + 7) // 8, 148 * 16)), 1, 1],
                                  (sid, self.g.nodes[sid].name)))
            self._colsum_done.add(sid)
        for r3, g3, lab in self._dw_recs:
            self.add_rec(N.RT_K_SPLITK, r3, g3, [256, 1, 1], 0, lab)
        self._dw_recs = []
        if q.colsum:
            rid, gc = req
            r2 = N.rt_splitk_params()
            r2.Z.nd = r2.M.nd = r2.N.nd = 1
            r2.Z.ext[0] = r2.M.ext[0] = 1
            r2.N.ext[0] = q.r
            r2.z, r2.m, r2.n = 1, 1, q.r
            r2.splits, r2.f64 = grid[0], 1          # fp64 partials, stored in C's dtype
            r2.part, r2.C = q.part2, gc
            self.add_rec(N.RT_K_SPLITK, r2, [int(min((q.r + 7) // 8, 148 * 16)), 1, 1],
                         [256, 1, 1], 0, (rid, self.g.nodes[rid].name))
            self._colsum_done.add(rid)
            self._colsum_req = None
        return True

    THIN_VEC = os.environ.get("RTB200_THIN_VEC", "1") != "0"

    @staticmethod
    def _smallk_vec_ok(q, kp, f64, gate):
        """k_thin_smallv: VW = 16 / itemsize output columns per thread with
        16-byte stores (and 16-byte gate loads): every C row start (base,
        row strides, env offsets) a multiple of VW elements, unit column
        stride, R a multiple of VW with R / VW dividing 256."""
        vw = 2 if f64 else 4
        es = 8 if f64 else 4
        R = q.r
        if kp > (8 if f64 else 16) or R % vw or R // vw > 256 or 256 % (R // vw) or \
                q.C.s2[0] != 1 or q.accumulate and q.epilogue == 2:
            return False
        ops = [q.C] + ([q.bias] if gate else [])
        for g in ops:
            if (g.ptr + es * g.off) % 16 or any(g.off_env[e] % vw for e in range(N.RT_MAXENV)):
                return False
            if any(g.s1[i] % vw for i in range(max(1, q.W.nd))):
                return False
        return True

    ROWS_MAX_R = 4

    def _gemm_rows(self, p, M, nc, kc, f64, label, accumulate, epilogue, bias):
        """Narrow-N products over many rows (policy/value heads, N <= 4,
        32 <= K <= 1024, contiguous K) -> RT_K_THIN variant 3: HBM-bound
        row streams instead of tensor-core tiles that would be 98% padding."""
        (n, (b_n, c_n)), (k, (a_k, b_k)) = nc, kc
        m = prod(t[0] for t in M)
        vw = 2 if f64 else 4
        ki = -(-k // (32 * vw))
        if not (n <= self.ROWS_MAX_R and 32 <= k and ki <= 8 and ki * vw * n <= 32
                and m >= 2048 and a_k == 1):
            return False
        mdims = [t for t in M if t[0] != 1] or [(1, 0, 0, 0)]
        if len(mdims) > 4:
            return False
        esize = 8 if f64 else 4
        q = N.rt_thin_params()
        q.variant, q.f64 = 3, int(f64)
        q.w, q.r, q.k = m, n, k
        q.W.nd = len(mdims)
        for i, t in enumerate(mdims):
            q.W.ext[i] = t[0]

        def gop(src, s1, s2):
            g = N.rt_gop()
            C.memmove(C.addressof(g), C.addressof(src), C.sizeof(g))
            for arr in (g.sz, g.s1, g.s2):
                for i in range(4):
                    arr[i] = 0
            for i, v in enumerate(s1):
                g.s1[i] = v
            for i, v in enumerate(s2):
                g.s2[i] = v
            return g

        q.X = gop(p.A, [1], [t[1] for t in mdims])
        q.Y = gop(p.B, [b_k], [b_n])
        q.C = gop(p.C, [t[3] for t in mdims], [c_n])
        if bias is not None:
            q.bias = gop(bias, [0], [bias.s2[0]])
        q.accumulate, q.epilogue = accumulate, epilogue
        A = p.A
        q.vec = int(k % vw == 0 and (A.ptr + esize * A.off) % 16 == 0
                    and all(t[1] % vw == 0 for t in mdims)
                    and all(A.off_env[e] % vw == 0 for e in range(N.RT_MAXENV)))
        if self._rows_capture is not None:
            self._rows_capture.append(q)        # a sibling head, merged by its partner
            return True
        sec = self._rows_second
        if sec is not None:
            sid, q2 = sec
            same_x = q2.X.ptr == q.X.ptr and q2.X.off == q.X.off and \
                all(q2.X.off_env[e] == q.X.off_env[e] for e in range(N.RT_MAXENV)) and \
                all(q2.X.s2[i] == q.X.s2[i] for i in range(4))
            if same_x and q2.w == q.w and q2.k == q.k and q2.f64 == q.f64 and \
                    q.r + q2.r <= 8 and ki * vw * 8 <= 64 and not accumulate and \
                    not q2.accumulate and q.epilogue == 0 and q2.epilogue == 0 and \
                    q2.W.nd == q.W.nd and all(q2.W.ext[i] == q.W.ext[i] for i in range(q.W.nd)):
                q.r2 = q2.r
                q.r = q.r + q2.r
                q.Y2, q.C2, q.bias2 = q2.Y, q2.C, q2.bias
                self._sibling_done.add(sid)
            self._rows_second = None
        rows_per_cta = 8 * 8
        grid = [int(max(1, min(-(-m // rows_per_cta), 148 * 16))), 1, 1]
        smem = 0
        rp = 1 if q.r <= 1 else 2 if q.r <= 2 else 4 if q.r <= 4 else 8
        kin = 1 if k <= 128 else 2
        rw = 4 if rp * kin * 4 >= 16 else 8
        # k_thin_rows_bulk: rows by cp.async.bulk, 2 CTAs per SM -- only when
        # its 3-stage ring fits twice in shared memory (8-row warps over
        # 256-wide rows would need 192 KB: one CTA per SM, two waves; the
        # register-load kernel streams those single-output rows at ~6.5 TB/s)
        if self.ROWS_BULK and q.vec and not f64 and k <= 256 and 3 * (8 * rw) * (kin * 128) * 4 <= 100 * 1024:
            q.vec = 2
            grid = [296, 1, 1]
            smem = 3 * (8 * rw) * (kin * 128) * 4 + 3 * 8    # BK_ST stages x SR rows x KP
        self.add_rec(N.RT_K_THIN, q, grid, [256, 1, 1], smem, label)
        return True

    ROWS_BULK = os.environ.get("RTB200_ROWS_BULK", "1") != "0"

    @staticmethod
    def _gop_dtype(g):
        return {v: k for k, v in N.DTYPE_CODE.items()}[g.dtype]

    TC_MIN_MACS = 1 << 26

    def _tc_ok(self, p, A, B, Cc):
        f32 = all(x[0].dtype == "f32" for x in (A, B, Cc))
        return (f32 and p.m * p.n * p.k >= self.TC_MIN_MACS and p.m >= 64
                and p.m < (1 << 31) and p.k < (1 << 31) and not self._capture_active())

    def _capture_active(self):
        return self._capture is not None

    @staticmethod
    def _tma_b_span(p):
        """Elements of B's storage a 2-D TMA view covers (k_gemm_tma.cu pack)."""
        b_k, b_n = p.B.s1[0], p.B.s2[0]
        if b_k == 1 or p.k == 1:
            return (p.n - 1) * b_n + p.k
        return (p.k - 1) * b_k + p.n

    @staticmethod
    def _tma_ok(p):
        """Plain 2-D f32 operands with a unit-stride dim and 16-byte aligned
        rows: eligible for the TMA-fed pipeline (csrc/k_gemm_tma.cu)."""
        if p.z != 1 or p.Z.nd > 1 or any(b.nd != 1 for b in (p.M, p.N, p.K)) or p.n < 16:
            return False
        if any(g.dtype != N.RT_F32 for g in (p.A, p.B, p.C)):
            return False
        for g, s_mn, s_k in ((p.A, p.A.s1[0], p.A.s2[0]), (p.B, p.B.s2[0], p.B.s1[0])):
            if (g.ptr + 4 * g.off) % 16 or any(g.off_env[e] % 4 for e in range(N.RT_MAXENV)):
                return False
            if not ((s_k == 1 and s_mn % 4 == 0 and s_mn > 0) or (s_mn == 1 and s_k % 4 == 0 and s_k > 0)):
                return False
        return max(p.m, p.n, p.k) < (1 << 31)

    def _gemm_tc(self, p, label, accumulate, epilogue, bias):
        """tcgen05 3xTF32 path (csrc/k_gemm_tc.cu): 128 x 256 CTA tiles."""
        tiles = ((p.m + 127) // 128) * ((p.n + 255) // 256) * p.z
        splits = 1
        if tiles < 148 and p.k >= 4096:
            # long-K contractions run the draining TMA variant, one CTA per SM
            splits = int(max(1, min(148 // max(1, tiles), p.k // 2048)))
        if p.z * splits > 65535 or (p.n + 255) // 256 > 65535:
            raise LowerError("gemm grid too large")
        p.splits = splits
        if splits > 1:
            p.part = self.alloc(splits * p.z * p.m * p.n * 4)
        # M tiles on grid.x (up to 2^31 - 1: E*T rows), N tiles on grid.y
        grid = [(p.m + 127) // 128, (p.n + 255) // 256, p.z * splits]
        if self.use_tma and self._tma_ok(p):
            # K per CTA beyond one TMEM accumulation chunk -> the draining
            # variant (csrc/k_gemm_tma.cu, rt_gemm_tma_pack: same rule);
            # one chunk, no split -> the persistent warp-specialised variant
            # (p.part = scratch for B's tf32 hi/lo split when B is a small
            # operand every M tile reads, else ~0)
            kper = (-(-p.k // splits) + 15) // 16 * 16
            if kper > N.TMA_DRAIN_K:
                self.add_rec(N.RT_K_GEMM_TMA, p, grid, [320, 1, 1], N.TMA_SMEM_DRAIN, label)
            elif splits == 1 and TMA_PERSIST:
                b_span = self._tma_b_span(p)
                mtiles = (p.m + 127) // 128
                if b_span * 4 <= (16 << 20) and mtiles >= 16:
                    p.part = self.alloc(2 * b_span * 4)
                else:
                    p.part = (1 << 64) - 1
                g = [int(min(tiles, 148)), 1, 1]
                self.add_rec(N.RT_K_GEMM_TMA, p, g, [N.TMA_THREADS_P, 1, 1], N.TMA_SMEM_P, label)
            else:
                self.add_rec(N.RT_K_GEMM_TMA, p, grid, [320, 1, 1], N.TMA_SMEM, label)
        else:
            self.add_rec(N.RT_K_GEMM_TC, p, grid, [256, 1, 1], N.TC_SMEM, label)
        if splits > 1:
            q = N.rt_splitk_params()
            q.Z, q.M, q.N = p.Z, p.M, p.N
            q.z, q.m, q.n = p.z, p.m, p.n
            q.splits = splits
            q.f64 = 0
            q.accumulate = accumulate
            q.epilogue = epilogue
            q.part = p.part
            q.C = p.C
            if bias is not None:
                q.bias = bias
            self.add_rec(N.RT_K_SPLITK, q, [int(min((p.z * p.m * p.n + 7) // 8, 148 * 16)), 1, 1], [256, 1, 1], 0,
                         label)   # k_splitk: a warp per output

    def k_contract(self, ctx: Ctx, X):
        """sum over full-range slices of a per-point matmul X, never
        materialising X: one GEMM whose K runs over the gathered points
        (the dW of the symbolic backward, frontend.py:766-776, 984-989)."""
        S = ctx.node
        (es,) = self.g.in_edges(S.id)
        xctx = Ctx(self, X, ctx.fixed)
        ea, eb = self.g.in_edges(X.id)
        A, B = self.edge_val(xctx, ea), self.edge_val(xctx, eb)
        for ev in (A, B):
            if ev.nslices or ev.checks or ev.progs:
                raise LowerError(f"{X.name}: contraction operand needs a gather")
        key = (S.id, 0)
        st = self.storage(key)
        a_ax, b_ax, batch, m, nn, kk, c_log = self._mm_shapes(A, B, st.strides[len(st.dims):])
        if batch:
            raise LowerError("batched contraction")
        cdst = {d: st.strides[j] for j, d in enumerate(self.bufs[key].dims)}
        red = [X.domain[j] for j, c in enumerate(es.phi) if c[0] == "slice"]
        Z, M, Nn, K = [], [], [], []
        for d in ctx.slab:              # kept dims of S (identity in X)
            a_s, b_s, c_s = A.coef.get(d, 0), B.coef.get(d, 0), cdst[d]
            if b_s != 0:
                Z.append((self.ext[d], a_s, b_s, c_s))
            else:
                M.append((self.ext[d], a_s, 0, c_s))
        M.append((m, a_ax[-2].stride, 0, c_log[0]))
        Nn.append((nn, 0, b_ax[-1].stride, c_log[1]))
        for d in red:
            K.append((self.ext[d], A.coef.get(d, 0), B.coef.get(d, 0), 0))
        K.append((kk, a_ax[-1].stride, b_ax[-2].stride, 0))
        env_a = {self.slot[d]: s for d, s in A.coef.items() if d in ctx.fixed}
        env_b = {self.slot[d]: s for d, s in B.coef.items() if d in ctx.fixed}
        env_c = {self.slot[d]: cdst[d] for d in ctx.fixed if d in cdst}
        ones = None
        if S.id in self.ones_bias:
            # the bias gradient sum(P) of the same points, as a ones column
            rkey = (self.ones_bias[S.id], 0)
            sr = self.storage(rkey)
            rdst = {d: sr.strides[j] for j, d in enumerate(self.bufs[rkey].dims)}
            if any(self.ext[d] != 1 for d in ctx.slab):
                raise LowerError(f"{S.name}: bias-gradient column over a batched contraction")
            g_ = N.rt_gop()
            g_.ptr, g_.dtype, g_.off = sr.ptr, N.DTYPE_CODE[sr.dtype], 0
            for d in ctx.fixed:
                if d in rdst:
                    g_.off_env[self.slot[d]] += rdst[d]
            g_.s2[0] = sr.strides[-1]
            ones = g_
        self._gemm((A.buf, A.off, env_a), (B.buf, B.off, env_b), (st, 0, env_c),
                   Z, M, Nn, K, (S.id, S.name), ones=ones)

    # ---- rng / udf

    def _coord_src(self, ctx):
        src = []
        for d in ctx.node.domain:
            if d in ctx.fixed:
                src.append(-1 - self.slot[d])
            else:
                src.append(ctx.slab.index(d))
        return src

    def _coord_add(self, p, n):
        """Entropy uses GLOBAL env indices when envs are sharded."""
        if self.shard is None:
            return
        for j, d in enumerate(n.domain):
            if d in self.shard.dims:
                p.coord_add[j] = self.shard.offset(self.ext[d])

    @staticmethod
    def words(v):
        if v < 0:
            raise LowerError("negative entropy")
        if v == 0:
            return [0]
        out = []
        while v:
            out.append(v & 0xFFFFFFFF)
            v >>= 32
        return out

    def k_rng(self, ctx: Ctx):
        n = ctx.node
        key = (n.id, 0)
        tag = n.params.get("tag", n.params.get("uid", n.id))
        prefix = self.words(self.seed) + self.words(tag)
        if len(prefix) > 8:
            raise LowerError("entropy prefix too long")
        p = N.rt_rng_params()
        box = list(ctx.slab_ext)
        p.box.nd = len(box)
        for i, x in enumerate(box):
            p.box.ext[i] = x
        p.total = prod(box)
        p.nprefix = len(prefix)
        for i, w in enumerate(prefix):
            p.prefix[i] = w
        cs = self._coord_src(ctx)
        p.ncoord = len(cs)
        for i, c in enumerate(cs):
            p.coord_src[i] = c
        self._coord_add(p, n)
        p.dist = 0 if n.params["dist"] == "normal" else 1
        p.count = prod(self.bufs[key].pshape)
        p.out = self.out_view(ctx, key)
        self.add_rec(N.RT_K_RNG, p, self.grid1(p.total, 128), [128, 1, 1], 0, (n.id, n.name))

    def k_udf(self, ctx: Ctx):
        n = ctx.node
        spec = n.params["spec"]
        if not getattr(spec, "synthetic", False):
            raise LowerError(f"udf {spec.name}: only synthetic (make_udf_fn) bodies run on device")
        tag = n.params.get("tag", n.params.get("uid", n.id))
        prefix = self.words(self.seed) + self.words(tag)
        p = N.rt_udf_params()
        box = list(ctx.slab_ext)
        p.box.nd = len(box)
        for i, x in enumerate(box):
            p.box.ext[i] = x
        p.total = prod(box)
        p.nprefix = len(prefix)
        for i, w in enumerate(prefix):
            p.prefix[i] = w
        cs = self._coord_src(ctx)
        p.ncoord = len(cs)
        for i, c in enumerate(cs):
            p.coord_src[i] = c
        self._coord_add(p, n)
        p.salt = zlib.crc32(spec.name.encode()) % 997 / 997.0
        ins = self.g.in_edges(n.id)
        if len(ins) > 4 or len(n.out_shapes) > 4:
            raise LowerError("udf arity > 4")
        p.nin = len(ins)
        for i, e in enumerate(ins):
            ev = self.edge_val(ctx, e)
            if _ragged(ev) or ev.progs:
                raise LowerError("udf input needs a gather")
            cnt = prod(a.ext for a in ev.axes)
            if [a.stride for a in ev.axes] != cstrides([a.ext for a in ev.axes]):
                raise LowerError("udf input payload not contiguous")
            p.in_count[i] = cnt
            p.in_[i] = self.make_view(ctx, ev, [])
        p.nout = len(n.out_shapes)
        for j in range(p.nout):
            k = (n.id, j)
            p.out_count[j] = prod(self.bufs[k].pshape)
            p.out_kind[j] = N.DTYPE_CODE[n.out_dtypes[j]]
            p.out[j] = self.out_view(ctx, k)
        self.add_rec(N.RT_K_UDF, p, self.grid1(p.total, 128), [128, 1, 1], 0, (n.id, n.name))


def _coords_used(code):
    used = set()
    for i in range(0, len(code), 2):
        if code[i] & 0xFF == OPC["ICOORD"]:
            used.add(code[i + 1])
    return used


def collapse_box(box, views, code):
    """Merge adjacent box dims (d, d+1) that every view walks contiguously
    (stride[d] == stride[d+1] * ext[d+1], same for range-check coefficients)
    and no program reads as a coordinate.  Fewer dims = fewer divides per
    element in the kernels' index decomposition."""
    box = list(box)
    d = len(box) - 2
    while d >= 0:
        used = _coords_used(code)
        e1 = box[d + 1]
        ok = d not in used and (d + 1) not in used
        if ok:
            for v in views:
                if v.stride[d] != v.stride[d + 1] * e1:
                    ok = False
                    break
                for c in range(v.nchk):
                    if v.chk_a[c][d] != v.chk_a[c][d + 1] * e1:
                        ok = False
                        break
                if not ok:
                    break
        if ok:
            for v in views:
                v.stride[d] = v.stride[d + 1]
                for j in range(d + 1, len(box) - 1):
                    v.stride[j] = v.stride[j + 1]
                v.stride[len(box) - 1] = 0
                for c in range(v.nchk):
                    v.chk_a[c][d] = v.chk_a[c][d + 1]
                    for j in range(d + 1, len(box) - 1):
                        v.chk_a[c][j] = v.chk_a[c][j + 1]
                    v.chk_a[c][len(box) - 1] = 0
            for i in range(0, len(code), 2):
                if code[i] & 0xFF == OPC["ICOORD"] and code[i + 1] > d + 1:
                    code[i + 1] -= 1
            box[d] = box[d] * e1
            del box[d + 1]
        d -= 1
        if d > len(box) - 2:
            d = len(box) - 2
    return box


def _ragged(ev):
    return any(a.ext is None for a in ev.axes)


def _merge_reduced(ev, red_axes):
    """Collapse runs of reduced axes that are contiguous in memory into one
    (e.g. the payload of a sumall), keeping at most 4 reduced axes."""
    red = sorted(red_axes)
    axes = list(ev.axes)
    i = 0
    while i + 1 < len(red):
        a, b = red[i], red[i + 1]
        A, B = axes[a], axes[b]
        if b == a + 1 and A.ext is not None and B.ext is not None and \
                A.stride == B.stride * B.ext:
            axes[a] = Axis(A.ext * B.ext, B.stride)
            del axes[b]
            red = [r if r < b else r - 1 for r in red if r != b]
            continue
        i += 1
    ev2 = EdgeVal(buf=ev.buf, off=ev.off, coef=ev.coef, checks=ev.checks, axes=axes,
                  nslices=ev.nslices, progs=ev.progs, psi=ev.psi)
    return ev2, tuple(red)


EW_KINDS = {"add", "sub", "mul", "div", "neg", "exp", "log", "tanh", "sqrt", "pow_const",
            "cmp", "where", "cast", "identity", "detach", "expand", "reshape", "permute",
            "squeeze", "unsqueeze", "eval_symbol", "merge", "scan", "index_select",
            "slice_axis", "set_symbol"}
