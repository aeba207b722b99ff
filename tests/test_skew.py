"""Skewed band schedules:
polysched's nstep schedule (window targets g, d at t + n - 1 in the band of
the recurrence s, r at t; fixtures tests/golden/theta/, made by
make_theta.py from the reference scheduler) realised as one pipelined loop:
prologue and epilogue iterations peeled, the lagged nodes evaluated at
t - (n - 1) inside the steady loop.  CPU: the plan.  GPU: the outputs equal
the reference's (golden fixtures) and the trace interleaves learning with
acting after step n - 1."""

import json
import os

import numpy as np
import pytest

from golden_cases import load_case

HERE = os.path.dirname(os.path.abspath(__file__))


def theta(name):
    with open(os.path.join(HERE, "golden", "theta", f"{name}.json")) as fh:
        return json.load(fh)


def _plan(case, th):
    from paper_2501_05408_b200 import executor as X, planner
    from paper_2501_05408_b200.schedule import band_lags
    c = load_case(case)
    g = X.as_graph(c.graph())
    benv, _ = X._bind_bounds(g, c.bounds)
    h = X.copy_graph(g)
    X.prepare(h, benv)
    skew = band_lags(th, g)
    an = X.analyze(h, benv, X.payload_shapes(h, benv), skew=skew)
    return h, skew, an, planner.describe(an["plan"].steps, h)


@pytest.mark.parametrize("prog,n", [("nstep2", 2), ("nstep4", 4)])
def test_band_lags_from_polysched(prog, n):
    from paper_2501_05408_b200 import executor as X
    from paper_2501_05408_b200.schedule import band_lags
    g = X.as_graph(load_case(f"corpus_{prog}_plain_s0").graph())
    d, lags = band_lags(theta(prog), g)
    names = {g.nodes[k].name: v for k, v in lags}
    assert d == "t" and names["g"] == n - 1 and names["d"] == n - 1
    assert names["s"] == 0 and names["r"] == 0


@pytest.mark.parametrize("prog,n", [("nstep2", 2), ("nstep4", 4)])
def test_skewed_plan_is_one_pipelined_band(prog, n):
    h, skew, an, text = _plan(f"corpus_{prog}_plain_s0", theta(prog))
    T = 8
    K = n - 1
    lines = text.splitlines()
    loops = [ln for ln in lines if ln.startswith("for t")]
    # K peeled prologue steps, one steady loop over [K, T), K peeled epilogue steps
    assert loops[K] == f"for t asc [{K}, {T}):", text
    assert len(loops) == 2 * K + 1, text
    assert f"  at t - {K}:" in lines, text
    # g and d never run outside the band loops (no bulk over all t after it)
    top_bulk = [ln for ln in lines if ln.startswith("bulk") and ("g:" in ln or "d:" in ln)]
    assert not top_bulk, text
    # the window operand r must keep every step (read one iteration later)
    r = [k for k, b in an["bufs"].items() if h.nodes[k[0]].name == "r"]
    assert r and not an["bufs"][r[0]].folded


def test_non_band_schedule_keeps_the_executor_plan():
    h, skew, an, text = _plan("corpus_nstep2_plain_s0",
                              {"levels": [["seq"], ["const"]], "rows": {}})
    assert skew is None and "at t -" not in text


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["corpus_nstep2_plain_s0", "corpus_nstep2_plain_s3",
                                  "corpus_nstep4_plain_s0", "corpus_nstep4_plain_s3"])
def test_skewed_pipeline_matches_reference(case):
    from paper_2501_05408_b200 import execute, executor as X, get_executable, trace
    c = load_case(case)
    prog = c.meta["program"]
    th = theta(prog)
    X._CACHE.clear()
    got = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed, theta=th)
    for k, want in c.outputs.items():
        np.testing.assert_allclose(got[k], want, rtol=1e-12, atol=1e-14, err_msg=k)
    exe, _ = get_executable(c.graph(), c.bounds, c.inputs, c.seed, theta=th)
    assert exe.skew is not None
    lines = [ln for ln in trace.trace(exe) if ln.startswith("EXEC")]
    n = 2 if prog == "nstep2" else 4
    # learning (g) for step 0 runs after acting (s) reached step n - 1 and
    # before acting finished: interleaved, not all acting first
    first_g = next(i for i, ln in enumerate(lines) if ln.split()[1] == "g")
    s_steps = [i for i, ln in enumerate(lines) if ln.split()[1] == "s"]
    assert s_steps[n - 2] < first_g < s_steps[-1], lines
    X._CACHE.clear()
