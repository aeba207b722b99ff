"""Static demand check: raise where the reference's demand-driven oracle
would evaluate a node outside its domain.

The reference executor evaluates a point only when an output (or a
consumer's read) demands it, and raises `OracleError("<node> evaluated
outside its domain at <point>")` when a demanded read lands outside the
source's domain box (runtime.py:344-355, 396-425).  The B200 executor
computes whole slabs eagerly and masks out-of-domain reads, so
it must decide statically which of those reads the reference would have
performed.  The hazard in practice is SURVEY F5: a `vectorize`-folded node
reads a full-range slice of a per-point node whose first rows read a
shifted predecessor that a guarding merge never demanded.

Demand is propagated from the outputs as unions of boxes (per node, a list
of {dim: (lo, hi)} inclusive ranges):
  * merges pick the first branch whose condition holds (runtime.py:362-371):
    the demanded boxes are split by each condition in order;
  * every other node reads every in-edge whose condition ψ holds
    (runtime.py:375, 400-401);
  * an edge maps a box through φ component by component (affine
    components exactly; slices as the union of their ranges).
Whatever the analysis cannot represent exactly (conditions or index maps
over several dims, non-affine maps) is dropped, i.e. the check
under-approximates demand: it never raises where the reference would not,
and it raises the reference's error class where it proves a demanded
out-of-domain read.
"""

from __future__ import annotations

from . import ir
from .planner import subst_bounds

BUDGET = 200_000


class _Unknown(Exception):
    pass


class _Budget(Exception):
    pass


def _aff1(e, dims):
    """(dim or None, coeff, const) for an expression affine in at most one
    of `dims`; raises _Unknown otherwise."""
    a = ir.as_affine(e)
    if a is None:
        raise _Unknown
    co, c0 = a
    used = [(n, c) for (n, k), c in co.items()]
    if any(n not in dims for n, _ in used) or len(used) > 1:
        raise _Unknown
    if not used:
        return None, 0, c0
    return used[0][0], used[0][1], c0


def _cmp_region(box, op, e):
    """Boxes of `box` where (e op 0) holds, e affine in one dim."""
    d, a, c = _aff1(e, box)
    if d is None or a == 0:
        holds = {"lt": c < 0, "le": c <= 0, "gt": c > 0, "ge": c >= 0, "eq": c == 0,
                 "ne": c != 0}[op]
        return [box] if holds else []
    lo, hi = box[d]
    # a*x + c op 0  ->  x in an interval (or two, for ne)
    if op == "ne":
        return _cmp_region(box, "lt", e) + _cmp_region(box, "gt", e)
    if op == "eq":
        if c % a:
            return []
        x = -c // a
        return [{**box, d: (x, x)}] if lo <= x <= hi else []
    if a < 0:   # flip to a positive coefficient
        a, c = -a, -c
        op = {"lt": "gt", "le": "ge", "gt": "lt", "ge": "le"}[op]
    # a > 0: x op -c/a
    if op == "lt":      # a x + c < 0  <=>  x < -c/a  <=>  x <= ceil(-c/a) - 1
        nhi = -(c // a) - 1 if c % a == 0 else (-c) // a
        nlo = lo
    elif op == "le":    # x <= floor(-c/a)
        nhi, nlo = (-c) // a, lo
    elif op == "gt":    # x > -c/a  <=>  x >= floor(-c/a) + 1
        nlo, nhi = (-c) // a + 1, hi
    else:               # ge: x >= ceil(-c/a)
        nlo, nhi = -((c) // a), hi
    nlo, nhi = max(lo, nlo), min(hi, nhi)
    return [{**box, d: (nlo, nhi)}] if nlo <= nhi else []


_NEG = {"lt": "ge", "le": "gt", "gt": "le", "ge": "lt", "eq": "ne", "ne": "eq"}


def _region(box, c, neg=False):
    """Boxes of `box` where condition c holds (neg: where it fails)."""
    k = c[0]
    if k == "bool":
        return [box] if bool(c[1]) != neg else []
    if k == "not":
        return _region(box, c[1], not neg)
    if k in ("and", "or"):
        if (k == "and") != neg:     # conjunction
            out = []
            for b in _region(box, c[1], neg):
                out += _region(b, c[2], neg)
            return out
        first = _region(box, c[1], neg)
        rest = []
        for b in _region(box, c[1], not neg):
            rest += _region(b, c[2], neg)
        return first + rest
    if k in _NEG:
        return _cmp_region(box, _NEG[k] if neg else k, ("sub", c[1], c[2]))
    raise _Unknown


class Demand:
    def __init__(self, g: ir.Graph, benv: dict):
        self.g = g
        self.benv = benv
        self.ext = {d: benv.get(g.dim_bound[d]) for d in g.dim_order}
        self.seen: dict[int, list] = {}
        self.ops = 0

    def _sub(self, e):
        return subst_bounds(e, self.benv)

    def run(self):
        g = self.g
        if any(v is None for v in self.ext.values()):
            return
        import sys
        old = sys.getrecursionlimit()
        sys.setrecursionlimit(max(old, 100_000))    # as runtime.py:466-472
        try:
            for _, nid, _ in g.outputs:
                n = g.nodes[nid]
                self._demand(nid, {d: (0, self.ext[d] - 1) for d in n.domain})
        except _Budget:
            pass
        finally:
            sys.setrecursionlimit(old)

    def _demand(self, nid, box):
        if any(lo > hi for lo, hi in box.values()):
            return
        boxes = self.seen.setdefault(nid, [])
        for b in boxes:
            if all(b[d][0] <= lo and hi <= b[d][1] for d, (lo, hi) in box.items()):
                return
        # coalesce with a box that differs in one dim and overlaps/touches there
        for i, b in enumerate(boxes):
            diff = [d for d in box if b[d] != box[d]]
            if len(diff) == 1:
                d = diff[0]
                (a0, a1), (b0, b1) = b[d], box[d]
                if b0 <= a1 + 1 and a0 <= b1 + 1:
                    box = {**box, d: (min(a0, b0), max(a1, b1))}
                    boxes.pop(i)
                    break
        boxes.append(box)
        self.ops += 1
        if self.ops > BUDGET:
            raise _Budget
        self._expand(nid, box)      # depth first, in edge order, like the oracle

    def _expand(self, nid, box):
        g = self.g
        n = g.nodes[nid]
        ins = g.in_edges(nid)
        if n.kind == "merge":
            remaining = [box]
            for e, c in zip(ins, n.params["conds"]):
                c = self._sub(c)
                try:
                    picked = [b for r in remaining for b in _region(r, c)]
                    remaining = [b for r in remaining for b in _region(r, c, neg=True)]
                except _Unknown:
                    return
                for b in picked:
                    self._read(n, e, b)
                if not remaining:
                    return
            return
        if n.kind == "set_symbol":
            ins = ins[:1]
        for e in ins:
            if e.psi is None:
                self._read(n, e, box)
                continue
            try:
                boxes = _region(box, self._sub(e.psi))
            except _Unknown:
                continue
            for b in boxes:
                self._read(n, e, b)

    def _read(self, sink, e, box):
        g = self.g
        src = g.nodes[e.src]
        comps = tuple(e.phi)
        if len(comps) != len(src.domain):
            return
        out, exact, used = {}, True, set()
        for d, c in zip(src.domain, comps):
            bound = self.ext[d]
            if bound is None:
                return
            c = self._sub(c)
            try:
                if c[0] == "slice":
                    lo, hi, ex, used_d = self._slice(c, box)
                    if lo is None:      # empty for every demanded point
                        return
                else:
                    dd, a, c0 = _aff1(c, box)
                    if dd is None or a == 0:
                        lo = hi = c0
                    else:
                        x0, x1 = box[dd]
                        lo, hi = sorted((a * x0 + c0, a * x1 + c0))
                    ex = abs(a) <= 1
                    used_d = dd
            except _Unknown:
                return
            if lo < 0 or hi > bound - 1:
                bad = lo if lo < 0 else hi
                pt = tuple(bad if d2 == d else max(0, out.get(d2, (0, 0))[0])
                           for d2 in src.domain)
                from .executor import OracleError
                raise OracleError(f"{src.name} evaluated outside its domain at {pt}")
            if used_d is not None:
                if used_d in used:
                    exact = False
                used.add(used_d)
            exact = exact and ex
            out[d] = (lo, hi)
        if exact:
            self._demand(src.id, out)

    def _slice(self, c, box):
        """Union range of slice c over box: (lo, hi inclusive, exact, dim)
        or (None, ...) when empty at every demanded point."""
        d1, a1, c1 = _aff1(c[1], box)
        d2, a2, c2 = _aff1(c[2], box)
        if d1 is not None and d2 is not None and d1 != d2:
            raise _Unknown
        d = d1 if d1 is not None else d2
        if d is None:
            return (c1, c2 - 1, True, None) if c2 > c1 else (None, None, True, None)
        a1 = a1 if d1 is not None else 0
        a2 = a2 if d2 is not None else 0
        x0, x1 = box[d]
        # points x where the slice is non-empty: (a2 - a1) x + (c2 - c1) > 0
        sub = _cmp_region({d: (x0, x1)}, "gt", ("add", ("mul", ("int", a2 - a1), ("sym", d, "loop")),
                                                    ("int", c2 - c1)))
        if not sub:
            return None, None, True, d
        y0, y1 = sub[0][d]
        los = (a1 * y0 + c1, a1 * y1 + c1)
        his = (a2 * y0 + c2, a2 * y1 + c2)
        return min(los), max(his) - 1, abs(a1) <= 1 and abs(a2) <= 1, d


def check(g: ir.Graph, benv: dict):
    """Raise OracleError where the reference would evaluate out of domain."""
    Demand(g, benv).run()
