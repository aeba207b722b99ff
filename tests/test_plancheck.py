"""The executor's own plan against polysched's (the reference scheduler,
pkg/src/recten/polysched.py), on the CPU: theta = schedule(extract(g)),
donations = donation_analysis, the MemOpSet of augment_memory_ops; the
executor's dry-lowered plan must never free a tensor before polysched's
last-consumer anchor (plancheck.py).  Needs the reference importable (build
container); the GPU-side `execute(..., theta=, memops=)` path is the same
check on a live executable."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tools")]

try:
    import programs as P
    P.recten()
    HAVE_REF = True
except Exception:      # no reference package here
    HAVE_REF = False


def _polysched(g):
    dsl, fe, pdg, tr, rt, ps = P.recten()
    domains, deps, prox = ps.extract(g)
    theta = ps.schedule(domains, deps, prox)
    don = ps.donation_analysis(g, theta)
    _g2, mem = ps.augment_memory_ops(g, theta, donations=don)
    mem.donations = don
    return theta, mem


HAVE_CORPUS = HAVE_REF and os.path.isdir(P.REF_PROGRAMS)


def _program(name):
    """The corpus programs need the reference's .rtl files (build container
    only); the MLP program is built through the front end (baseline/_ref on
    the GPU box)."""
    dsl, fe, pdg, tr, rt, ps = P.recten()
    if name == "mlp":
        g = pdg.build(P.ctx_reinforce_mlp(B=3, T=4, I=1, d_o=4, H=8, d_a=2, dtype="f32", lr=0.05))
        pdg.eliminate_dead(g)
        return g
    g = pdg.build(dsl.load_text(P.corpus_text(name)))
    for d, b in g.dim_bound.items():
        g.bindings[b] = {"I": 2, "B": 2, "T": 4}[b.name] if name == "reinforce" else 8
    return g


@pytest.mark.skipif(not HAVE_REF, reason="reference package not importable")
@pytest.mark.parametrize("name", ["reinforce", "mlp", "nstep2"])
def test_executor_plan_never_frees_before_polysched(name):
    if name != "mlp" and not HAVE_CORPUS:
        pytest.skip("reference .rtl corpus not present")
    from arena_estimate import plan
    from paper_2501_05408_b200 import executor as X, ir, plancheck
    g = _program(name)
    theta, mem = _polysched(g)
    graph = ir.from_pdg(g)
    benv, _ = X._bind_bounds(graph, None)
    h, bufs, low, life, an = plan(graph, benv)

    class A:
        fuse_src, gemm_epi, contract = an["fuse_src"], an["gemm_epi"], an["contract"]
    labels = [lab for (*_, lab) in low.recs]
    prog = [(ins[0], ins[1]) for ins in low.prog]
    rep = plancheck.check(h, bufs, labels, prog, life, plancheck.fused_map(A), theta, mem)
    d = rep["deallocate"]
    assert d["checked"] > 0 and not d["unsafe"], rep
    assert rep["theta_levels"][0].startswith(("band", "seq"))
    assert rep["donation"]["pairs"] == len(mem.donations)


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference package not importable")
def test_execute_takes_polysched_plan():
    """execute(g, theta=, memops=) on a live reference Pdg: the outputs are
    the reference's and the plan report is kept on the executable."""
    import numpy as np
    from paper_2501_05408_b200 import execute, get_executable
    dsl, fe, pdg, tr, rt, ps = P.recten()
    g = _program("mlp")
    theta, mem = _polysched(g)
    inputs = P.mlp_inputs(d_o=4, H=8, d_a=2, dtype="f32")
    want = rt.reference_execute(g, inputs=inputs, seed=0)
    got = execute(g, inputs=inputs, seed=0, theta=theta, memops=mem)
    exe, _ = get_executable(g, None, inputs, 0)
    rep = exe.plan_report
    assert rep and rep["deallocate"]["checked"] > 0 and not rep["deallocate"]["unsafe"]
    for k in want:
        np.testing.assert_allclose(got[k], want[k], rtol=1e-5, atol=1e-6, err_msg=k)
