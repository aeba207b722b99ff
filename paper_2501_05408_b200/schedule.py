"""polysched's ScheduleFn -> the band skews the executor can realise.

The reference scheduler (pkg/src/recten/polysched.py:92-143, `schedule`
:546-612) assigns every node a tuple of affine rows, one per level
(`('band', d)`, `('seq',)`, `('const',)`, `('mem',)`).  A program whose
leading level is a band over d with rows `d + c` (c a constant) for the
nodes that have d -- e.g. nstep2: s, r at `t` and the window target g, d at
`t + 1` -- is a software pipeline with skew c.
`band_lags` reads that out; the planner realises it (planner.skew_steps).

Accepts a live ScheduleFn or its JSON form (tests/golden/theta/*.json:
{"levels": [["band", "t"], ["const"]], "rows": {nid: [[[[sym, coef], ...],
const], ...]}}, written by tests/golden/make_theta.py).
"""

from __future__ import annotations


def _levels(theta):
    if isinstance(theta, dict):
        return [tuple(lv) for lv in theta["levels"]]
    out = []
    for lv in theta.levels:
        out.append(tuple(getattr(x, "name", x) for x in lv))
    return out


def _rows(theta):
    """nid -> [(terms {sym name: coef}, const)] per level."""
    if isinstance(theta, dict):
        return {int(k): [({t[0]: int(t[1]) for t in r[0]}, int(r[1])) for r in rows]
                for k, rows in theta["rows"].items()}
    return {int(k): [({getattr(s, "name", s): int(c) for s, c in r.terms}, int(r.const))
                     for r in rows] for k, rows in theta.rows.items()}


def band_lags(theta, g):
    """(dim, {nid: lag}) when theta's first level is a band over a dim d of
    g and every node having d is scheduled there at d + c, c >= 0 an
    integer; None otherwise (the executor keeps its own order)."""
    if theta is None:
        return None
    levels = _levels(theta)
    if not levels or levels[0][0] != "band":
        return None
    d = levels[0][1]
    if d not in g.dim_order:
        return None
    lags = {}
    for nid, rows in _rows(theta).items():
        if nid not in g.nodes or d not in g.nodes[nid].domain:
            continue
        terms, c = rows[0]
        if terms != {d: 1} or c < 0:
            return None
        lags[nid] = c
    if not any(lags.values()):
        return None
    return d, tuple(sorted(lags.items()))


def theta_json(theta):
    """The JSON form of a polysched ScheduleFn (fixtures)."""
    return {"levels": [list(lv) for lv in _levels(theta)],
            "rows": {str(k): [[sorted([s, c] for s, c in t.items()), c0] for t, c0 in rows]
                     for k, rows in _rows(theta).items()}}
