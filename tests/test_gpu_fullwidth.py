"""Parity of the BENCHMARKED kernels against the real reference.

The fixtures `tests/golden/cases/fw_*` were produced by the reference's own
`reference_execute` (tests/golden/make_golden.py FULLWIDTH) on the full-width
benchmark programs: obs 16, two 256-wide tanh layers, 4 actions (+ the
value head for PPO), I=2 training iterations (REINFORCE) or 2 epochs x 2
minibatches (PPO), f32 and f64.  At B=1024 the lowering picks the same
kernel families the C2/C3 benchmark runs; the tests force the JIT
specialisation on (loop and elementwise thresholds to 0) and assert that
every family of the benchmark's launch list (profiles/*_launches.csv) was
chosen before comparing with the reference at the north_star tolerance
(fp32 rtol 1e-5; reference runtime.py:249 np.matmul, :460-475 layout).
"""

import numpy as np
import pytest

from golden_cases import load_case

pytestmark = pytest.mark.gpu

TOL = {np.float32: dict(rtol=1e-5, atol=1e-6), np.float64: dict(rtol=1e-12, atol=1e-13)}


def _families(exe):
    from paper_2501_05408_b200 import roofline
    fams = {roofline.FAMILY.get(k, str(k)) for k in exe.kernels}
    if any(getattr(exe.recs[ri], "jit_fn", None) for ri in exe.loop_info):
        fams.add("loop_jit")
    from paper_2501_05408_b200 import native as N
    if any(getattr(r, "jit_fn", None) and k == N.RT_K_EW for k, r in zip(exe.kernels, exe.recs)):
        fams.add("ew_jit")
    return fams


def _thin_variants(exe):
    from paper_2501_05408_b200 import native as N
    return {(p.variant, p.epilogue) for k, p in zip(exe.kernels, exe._params)
            if k == N.RT_K_THIN}


def _run(name, monkeypatch):
    from paper_2501_05408_b200 import execute, executor as X, get_executable, jit
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 0)
    monkeypatch.setattr(jit, "JIT_MIN_ELEMS", 0)
    X._CACHE.clear()
    c = load_case(name)
    exe, _ = get_executable(c.graph(), c.bounds, c.inputs, c.seed)
    outs, rb = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed,
                       return_bounds=True)
    assert rb == c.resolved_bounds
    assert sorted(outs) == sorted(c.outputs)
    for k, want in c.outputs.items():
        got = outs[k]
        assert got.shape == want.shape and got.dtype == want.dtype, k
        np.testing.assert_allclose(got, want, err_msg=k, **TOL[want.dtype.type])
    X._CACHE.clear()
    return exe


def test_c2_program_benchmark_kernels_match_reference(monkeypatch):
    """REINFORCE MLP, I=2, B=1024, T=8, f32: JIT acting loop, tcgen05 TMA
    GEMMs (bias+tanh forward epilogue not used here: the learner has no
    forward GEMM; dX and the split-K dW contraction are), the thin row /
    small-K / gate-epilogue kernels, split-K, the reverse return scan."""
    exe = _run("fw_mlp_f32_I2B1024T8", monkeypatch)
    fams = _families(exe)
    for f in ("loop_jit", "gemm_tma", "thin", "splitk", "scan", "reduce", "ew_jit", "rng"):
        assert f in fams, (f, fams)
    v = _thin_variants(exe)
    assert (2, 2) in v, v      # small-K product with the tanh-VJP gate epilogue


def test_c3_program_benchmark_kernels_match_reference(monkeypatch):
    """PPO+GAE, B=1024, T=8, 2 epochs x 2 minibatches, f32: the learner
    re-runs the trunk forward over the gathered minibatch rows, so the
    tcgen05 GEMM with the fused bias+tanh epilogue runs here too."""
    from paper_2501_05408_b200 import native as N
    exe = _run("fw_ppo_f32_I1B1024T8E2M2", monkeypatch)
    fams = _families(exe)
    for f in ("loop_jit", "gemm_tma", "thin", "scan", "reduce", "ew_jit", "rng"):
        assert f in fams, (f, fams)
    epis = {p.epilogue for k, p in zip(exe.kernels, exe._params) if k == N.RT_K_GEMM_TMA}
    assert any(e != 0 for e in epis), epis     # bias / bias+tanh epilogue on tcgen05


@pytest.mark.parametrize("name", ["fw_mlp_f32_I2B8T32", "fw_mlp_f64_I2B8T16",
                                  "fw_ppo_f64_I1B16T8E2M2"])
def test_fullwidth_small_batch_matches_reference(name, monkeypatch):
    """Full width at a handful of envs: the JIT loop with one CTA per few
    rows and the SIMT GEMM paths, f32 and f64 (f64: 1e-12)."""
    exe = _run(name, monkeypatch)
    assert "loop_jit" in _families(exe)
