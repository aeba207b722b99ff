"""Loop-nest planning: which points of which nodes run in one launch.

The reference evaluates one (node, point) at a time, on demand, recursing
through edges (runtime.py:344-425).  A B200 executor must instead evaluate
whole slabs of points per launch.  The planner derives the loop nest from
the dependence structure itself, the same well-foundedness argument the
reference uses to *validate* cycles (pdg.py:607-668, `_well_founded`):

  * strongly connected components of the graph, in topological order;
  * an acyclic component is one node: evaluated over all its remaining
    dims at once (a "bulk" step);
  * a cyclic component is scheduled by a loop over a dim d common to all
    its members along which every internal dependence reads at distance
    <= 0 (in the loop direction); edges at distance exactly 0 stay, the
    rest are satisfied by the loop, and the body is planned recursively.

Within a loop body every node is evaluated for all values of its free dims
(e.g. all envs b at one step t) — the batching the reference's vectorizer
cannot express across cycles.  Distances come from interval
arithmetic over the concrete box, refined by simple edge conditions.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import ir
from .ir import Graph

INF = float("inf")


class PlanError(Exception):
    pass


# ---------------------------------------------------------------------------
# interval arithmetic over concrete boxes


def subst_bounds(e, benv: dict):
    return ir.substitute(e, {(b, "bound"): ("int", v) for b, v in benv.items()})


def interval(e, box: dict):
    """(lo, hi) inclusive range of integer expression e over box
    {dim: (lo, hi)}; bounds must already be substituted."""
    k = e[0]
    if k == "int":
        return (e[1], e[1])
    if k == "bool":
        v = int(e[1])
        return (v, v)
    if k == "sym":
        if e[2] == "loop" and e[1] in box:
            return box[e[1]]
        return (-INF, INF)
    aff = ir.as_affine(e)
    if aff is not None:
        lo = hi = aff[1]
        for (name, kind), c in aff[0].items():
            if kind != "loop" or name not in box:
                return (-INF, INF)
            a, b = box[name]
            lo += min(c * a, c * b)
            hi += max(c * a, c * b)
        return (lo, hi)
    if k in ("min", "max"):
        ivs = [interval(a, box) for a in e[1:]]
        f = min if k == "min" else max
        return (f(i[0] for i in ivs), f(i[1] for i in ivs))
    if k == "neg":
        a = interval(e[1], box)
        return (-a[1], -a[0])
    if k in ("add", "sub"):
        a, b = interval(e[1], box), interval(e[2], box)
        if k == "add":
            return (a[0] + b[0], a[1] + b[1])
        return (a[0] - b[1], a[1] - b[0])
    if k == "floordiv" and e[2][0] == "int" and e[2][1] > 0:
        a = interval(e[1], box)
        c = e[2][1]
        f = lambda x: x if x in (INF, -INF) else x // c  # noqa: E731
        return (f(a[0]), f(a[1]))
    if k == "mod" and e[2][0] == "int" and e[2][1] != 0:
        return (0, abs(e[2][1]) - 1)
    if k == "mul":
        a, b = interval(e[1], box), interval(e[2], box)
        cands = [x * y for x in a for y in b if not (x in (INF, -INF) and y == 0)
                 and not (y in (INF, -INF) and x == 0)]
        return (min(cands), max(cands)) if cands else (-INF, INF)
    return (-INF, INF)


def refine_box(psi, box: dict):
    """Shrink box by the simple atoms of condition psi (bounds substituted).
    Returns None when psi is unsatisfiable on the box."""
    box = dict(box)
    atoms = []

    def collect(c):
        if c[0] == "and":
            collect(c[1])
            collect(c[2])
        else:
            atoms.append(c)

    collect(psi)
    for a in atoms:
        if a == ("bool", False):
            return None
        if a[0] not in ("eq", "lt", "le", "gt", "ge"):
            continue
        diff = ir.as_affine(("sub", a[1], a[2]))
        if diff is None:
            continue
        co, k = diff
        if len(co) != 1:
            continue
        ((name, kind), c), = co.items()
        if kind != "loop" or name not in box or c not in (1, -1):
            continue
        # c*x + k  op  0
        lo, hi = box[name]
        op = a[0]
        if c == -1:
            op = {"eq": "eq", "lt": "gt", "le": "ge", "gt": "lt", "ge": "le"}[op]
            k = -k
        # x + k op 0  ->  x op -k
        v = -k
        if op == "eq":
            lo, hi = max(lo, v), min(hi, v)
        elif op == "lt":
            hi = min(hi, v - 1)
        elif op == "le":
            hi = min(hi, v)
        elif op == "gt":
            lo = max(lo, v + 1)
        elif op == "ge":
            lo = max(lo, v)
        if lo > hi:
            return None
        box[name] = (lo, hi)
    return box


# ---------------------------------------------------------------------------
# plan structures


@dataclass
class Bulk:
    nid: int
    fixed: tuple          # dims bound by enclosing loops (outer first)


@dataclass
class Loop:
    dim: str
    step: int             # +1 ascending, -1 descending
    body: list = field(default_factory=list)
    fixed: tuple = ()
    lo: int | None = None  # iteration range [lo, hi) (None: the dim's full extent)
    hi: int | None = None


@dataclass
class Shift:
    """Inside a loop over `dim`: evaluate `body` at dim = (loop index) - k
    (a skewed schedule's lag; lowered as env adds around the body)."""
    dim: str
    k: int
    body: list = field(default_factory=list)


@dataclass
class Plan:
    graph: Graph
    benv: dict            # bound name -> int
    ext: dict             # dim name -> int
    steps: list


def sccs(nodes, succ):
    """Tarjan, iterative; components in discovery order."""
    index, low, on, stack, out = {}, {}, set(), [], []
    counter = [0]
    for root in sorted(nodes):
        if root in index:
            continue
        work = [(root, iter(sorted(succ.get(root, ()))))]
        index[root] = low[root] = counter[0]
        counter[0] += 1
        stack.append(root)
        on.add(root)
        while work:
            v, it = work[-1]
            advanced = False
            for w in it:
                if w not in nodes:
                    continue
                if w not in index:
                    index[w] = low[w] = counter[0]
                    counter[0] += 1
                    stack.append(w)
                    on.add(w)
                    work.append((w, iter(sorted(succ.get(w, ())))))
                    advanced = True
                    break
                if w in on:
                    low[v] = min(low[v], index[w])
            if advanced:
                continue
            work.pop()
            if work:
                low[work[-1][0]] = min(low[work[-1][0]], low[v])
            if low[v] == index[v]:
                comp = []
                while True:
                    w = stack.pop()
                    on.discard(w)
                    comp.append(w)
                    if w == v:
                        break
                out.append(sorted(comp))
    return out


class Planner:
    def __init__(self, g: Graph, benv: dict):
        self.g = g
        self.benv = dict(benv)
        self.ext = {d: benv[g.dim_bound[d]] for d in g.dim_order if g.dim_bound[d] in benv}
        self._dist_cache = {}

    # -- distances ----------------------------------------------------------

    def sink_box(self, e):
        n = self.g.nodes[e.sink]
        box = {d: (0, self.ext[d] - 1) for d in n.domain}
        if any(lo > hi for lo, hi in box.values()):
            return None
        if e.psi is not None:
            box = refine_box(subst_bounds(e.psi, self.benv), box)
        return box

    def distance(self, e, d):
        """(min, max) of src_d - snk_d over the edge, or None if vacuous.
        Edges whose source lacks d impose nothing along d: (0, 0)."""
        key = (id(e), d)
        if key in self._dist_cache:
            return self._dist_cache[key]
        src = self.g.nodes[e.src]
        snk = self.g.nodes[e.sink]
        box = self.sink_box(e)
        if box is None:
            res = None
        elif d not in src.domain:
            res = (0, 0)
        else:
            c = subst_bounds(e.phi[src.domain.index(d)], self.benv)
            if d not in snk.domain:
                # sink lacks d: it reads (some) points along d of the source
                res = (-INF, INF)
            elif c[0] == "slice":
                a = interval(("sub", c[1], ("sym", d, "loop")), box)
                b = interval(("sub", ("sub", c[2], ("int", 1)), ("sym", d, "loop")), box)
                res = (min(a[0], b[0]), max(a[1], b[1]))
            else:
                res = interval(("sub", c, ("sym", d, "loop")), box)
        self._dist_cache[key] = res
        return res

    # -- recursive decomposition -----------------------------------------------

    def plan(self, block_dims=()):
        nodes = set(self.g.nodes)
        edges = list(self.g.edges)
        steps = self.level(nodes, edges, ())
        for kb in block_dims:
            steps = group_block_loop(steps, self.g, kb)
        return Plan(self.g, self.benv, self.ext, steps)

    def level(self, nodes: set, edges: list, fixed: tuple):
        succ = {}
        inner = [e for e in edges if e.src in nodes and e.sink in nodes]
        for e in inner:
            succ.setdefault(e.src, set()).add(e.sink)
        comps = sccs(nodes, succ)
        # topological order of the condensation (Kahn, ties by min id)
        cid = {v: i for i, c in enumerate(comps) for v in c}
        indeg = {i: 0 for i in range(len(comps))}
        csucc = {i: set() for i in range(len(comps))}
        for e in inner:
            a, b = cid[e.src], cid[e.sink]
            if a != b and b not in csucc[a]:
                csucc[a].add(b)
                indeg[b] += 1
        ready = sorted((min(comps[i]), i) for i, k in indeg.items() if k == 0)
        order = []
        import heapq
        heapq.heapify(ready)
        while ready:
            _, i = heapq.heappop(ready)
            order.append(i)
            for j in csucc[i]:
                indeg[j] -= 1
                if indeg[j] == 0:
                    heapq.heappush(ready, (min(comps[j]), j))
        steps = []
        for i in order:
            comp = comps[i]
            cedges = [e for e in inner if e.src in comp and e.sink in comp]
            if len(comp) == 1 and not cedges:
                steps.append(Bulk(comp[0], fixed))
                continue
            lp = self.loop_for(set(comp), cedges, fixed)
            steps.extend(lp if isinstance(lp, list) else [lp])
        return steps

    def loop_for(self, comp: set, cedges: list, fixed: tuple):
        live = [e for e in cedges if self.sink_box(e) is not None]
        if len(live) < len(cedges):
            # edges whose condition never holds on the concrete box (e.g. the
            # recurrence o[t] <- o[t-1] at T = 1, anything at B = 0) carry no
            # dependence: plan the component on the edges that remain
            steps = self.level(comp, live, fixed)
            return steps if len(steps) != 1 else steps[0]
        common = [d for d in self.g.dim_order
                  if d not in fixed and all(d in self.g.nodes[v].domain for v in comp)]
        for d in common:
            for step in (1, -1):
                ok = True
                flat = []
                for e in cedges:
                    dist = self.distance(e, d)
                    if dist is None:
                        continue  # vacuous edge
                    lo, hi = dist
                    if step < 0:
                        lo, hi = -hi, -lo
                    if hi > 0:
                        ok = False
                        break
                    if hi == 0:
                        flat.append(e)
                # a loop must carry at least one dependence, or it only
                # serialises independent points (e.g. envs b)
                live = [e for e in cedges if self.distance(e, d) is not None]
                if ok and len(flat) < len(live):
                    body = self.level(comp, flat, fixed + (d,))
                    return Loop(d, step, body, fixed)
        peeled = self.peel_for(comp, cedges, fixed)
        if peeled is not None:
            return peeled
        names = ", ".join(self.g.nodes[v].name for v in sorted(comp))
        raise PlanError(f"unschedulable cycle through [{names}]")

    def peel_for(self, comp: set, cedges: list, fixed: tuple):
        """A cycle whose members do not all share a dim: some members lack d
        and read the d-members only at d == 0 (e.g. a PPO rollout over (b,t)
        reading the parameters theta[i, k=0] that the update loop over k
        then advances).  Peel the first iteration: loop d over [0, 1) with
        every member (the d-less ones evaluated there, once), then over
        [1, n) with the d-members alone.  Point-level, this is the schedule
        theta(v) = 0 along d for the d-less members (polysched's `const`
        placement of a statement without the dim, polysched.py:594-608)."""
        g = self.g
        cands = [d for d in g.dim_order if d not in fixed and self.ext.get(d, 0) > 1
                 and any(d in g.nodes[v].domain for v in comp)]
        for d in cands:
            has = {v for v in comp if d in g.nodes[v].domain}
            lacks = comp - has
            if not lacks:
                continue
            ok = True
            flat0, rest = [], []
            for e in cedges:
                dist = self.distance(e, d)
                if dist is None:
                    continue
                s_has, k_has = e.src in has, e.sink in has
                if s_has and k_has:
                    if dist[1] > 0:
                        ok = False
                        break
                    if dist[1] == 0:
                        rest.append(e)
                        flat0.append(e)
                elif s_has and not k_has:
                    # a d-less member reads d-members: only at d == 0
                    c = subst_bounds(e.phi[g.nodes[e.src].domain.index(d)], self.benv)
                    if interval(c, self.sink_box(e) or {}) != (0, 0):
                        ok = False
                        break
                    flat0.append(e)
                else:
                    # produced once at d == 0, read at any d >= 0
                    flat0.append(e)
            if not ok:
                continue
            first = self.level(comp, flat0, fixed + (d,))
            out = [Loop(d, 1, first, fixed, 0, 1)]
            if self.ext[d] > 1:
                out.append(Loop(d, 1, self.level(has, rest, fixed + (d,)), fixed, 1,
                                self.ext[d]))
            return out
        return None


def _step_nodes(st):
    if isinstance(st, Bulk):
        return {st.nid}
    out = set()
    for b in st.body:
        out |= _step_nodes(b)
    return out


def group_block_loop(steps, g: Graph, kb: str):
    """Put the top-level bulk steps over block dim kb (blocking.block_dim)
    into one loop over kb, so each block's chain runs start to finish and
    its intermediates fold to one block of storage.  Steps the block nodes
    depend on go before the loop, steps depending on them after; unchanged
    if some step sits on a path between two block steps."""
    blk = [st for st in steps if isinstance(st, Bulk) and kb in g.nodes[st.nid].domain]
    if not blk:
        return steps
    bset = {st.nid for st in blk}
    succ = {}
    for e in g.edges:
        succ.setdefault(e.src, set()).add(e.sink)

    def reach(starts):
        seen, work = set(), list(starts)
        while work:
            v = work.pop()
            for w in succ.get(v, ()):
                if w not in seen:
                    seen.add(w)
                    work.append(w)
        return seen

    desc = reach(bset)
    before, after = [], []
    for st in steps:
        if isinstance(st, Bulk) and st.nid in bset:
            continue
        nodes = _step_nodes(st)
        if nodes & desc:
            if reach(nodes) & bset:
                return steps      # a step between two block steps: keep flat
            after.append(st)
        else:
            before.append(st)
    body = [Bulk(st.nid, tuple(st.fixed) + (kb,)) for st in blk]
    return before + [Loop(kb, 1, body, ())] + after


def describe(steps, g: Graph, indent=0) -> str:
    out = []
    for s in steps:
        if isinstance(s, Shift):
            out.append("  " * indent + f"at {s.dim} - {s.k}:")
            out.append(describe(s.body, g, indent + 1))
            continue
        if isinstance(s, Bulk):
            n = g.nodes[s.nid]
            free = [d for d in n.domain if d not in s.fixed]
            out.append("  " * indent + f"bulk {n.name}:{n.kind} over ({','.join(free)})")
        else:
            rng = f" [{s.lo}, {s.hi})" if s.lo is not None else ""
            out.append("  " * indent + f"for {s.dim} {'asc' if s.step > 0 else 'desc'}{rng}:")
            out.append(describe(s.body, g, indent + 1))
    return "\n".join(out)


# ---------------------------------------------------------------------------
# skewed pipelines (a polysched band schedule with constant skews)


def _max_ahead(planner: "Planner", e, d: str):
    """Largest src_d - snk_d an edge reads (None: vacuous).  Interval
    arithmetic loses the correlation in windows like r[t : min(t+2, T)]
    (it gives 7 at T = 8), so the loop dim is enumerated point by point
    when its extent is small."""
    dist = planner.distance(e, d)
    if dist is None or dist[1] <= 0:
        return None if dist is None else dist[1]
    src, snk = planner.g.nodes[e.src], planner.g.nodes[e.sink]
    box = planner.sink_box(e)
    if box is None or d not in snk.domain or d not in src.domain or \
            box[d][1] - box[d][0] > (1 << 16):
        return dist[1]
    c = subst_bounds(e.phi[src.domain.index(d)], planner.benv)
    hi_e = ("sub", c[2], ("int", 1)) if c[0] == "slice" else c
    best = None
    for t in range(int(box[d][0]), int(box[d][1]) + 1):
        b2 = dict(box)
        b2[d] = (t, t)
        v = interval(("sub", hi_e, ("sym", d, "loop")), b2)[1]
        best = v if best is None else max(best, v)
    return best


def skew_steps(planner: "Planner", steps, d: str, lags: dict):
    """Realise a band schedule over d with constant skews (reference
    polysched.py:546-612; e.g. nstep2: s, r at t and the window target g, d
    at t + 1): the top-level recurrence loop over d and
    the bulk steps after it whose nodes the schedule places in the same band
    at d + c (c = lags[nid] >= 0) become ONE loop over the band index tau in
    [0, T + K): the recurrence body at d = tau (tau < T), then every lagged
    node at d = tau - c (0 <= tau - c < T) in plan order.  The steady range
    tau in [K, T) is one loop; the first and last K iterations are peeled
    (the SPEC's "window skew guard peeled for first n iterations",
    SPEC.md:494, 503).  Valid when every dependence of a lagged node on the
    band's nodes reads at most c - c_src ahead along d; else the steps are
    returned unchanged (the executor's own dependence order)."""
    g, ext = planner.g, planner.ext
    T = ext.get(d, 0)
    idx = [i for i, st in enumerate(steps) if isinstance(st, Loop) and st.dim == d and
           not st.fixed and st.lo is None and st.step == 1]
    if not idx or T <= 0:
        return steps
    i = idx[0]
    L = steps[i]
    band = dict.fromkeys(_step_nodes(L), 0)
    if any(lags.get(v, 0) != 0 for v in band if d in g.nodes[v].domain):
        return steps
    cands, late, rest = [], set(), []
    for st in steps[i + 1:]:
        nodes = _step_nodes(st)
        ins = [e for v in nodes for e in g.in_edges(v)]
        if isinstance(st, Bulk) and d in g.nodes[st.nid].domain and st.nid in lags and \
                lags[st.nid] >= 0 and not any(e.src in late for e in ins):
            c = lags[st.nid]
            ok = True
            for e in ins:
                if e.src in band:
                    ahead = _max_ahead(planner, e, d)
                    if ahead is not None and ahead > c - band[e.src]:
                        ok = False
                        break
            if ok:
                band[st.nid] = c
                cands.append(st)
                continue
        late |= nodes
        rest.append(st)
    if not cands or not any(band[st.nid] > 0 for st in cands):
        return steps
    K = max(band[st.nid] for st in cands)

    def items(tau):
        out = list(L.body) if tau is None or tau < T else []
        for st in cands:
            c = band[st.nid]
            if tau is not None and not (0 <= tau - c < T):
                continue
            b = Bulk(st.nid, (d,))
            if c == 0:
                out.append(b)
            elif out and isinstance(out[-1], Shift) and out[-1].k == c:
                out[-1].body.append(b)
            else:
                out.append(Shift(d, c, [b]))
        return out

    loops = []
    for tau in range(0, min(K, T)):
        loops.append(Loop(d, 1, items(tau), (), tau, tau + 1))
    if K < T:
        loops.append(Loop(d, 1, items(None), (), K, T))
    for tau in range(max(K, T), T + K):
        loops.append(Loop(d, 1, items(tau), (), tau, tau + 1))
    planner.lags = dict(band)
    return steps[:i] + loops + rest
