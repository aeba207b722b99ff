"""Pin the oracle port to the real reference (CPU only).

Every committed golden case was produced by the reference's own
`reference_execute` (tests/golden/make_golden.py).  The port in
oracle/pdg_oracle.py must reproduce it bit for bit — same numpy kernels in
the same order, same per-point RNG streams — or fail the same way.
"""

import os

import numpy as np
import pytest

from golden_cases import case_ids, load_case
from oracle.pdg_oracle import OracleError, oracle_execute


# The B=1024 full-width fixtures take the per-point port 40-90 s each; they
# are reference outputs already and are checked against the CUDA path
# directly (tests/test_gpu_fullwidth.py).  RTB200_PIN_ALL=1 includes them.
SLOW = {"fw_mlp_f32_I2B1024T8", "fw_ppo_f32_I1B1024T8E2M2"}


@pytest.mark.parametrize("name", [c for c in case_ids()
                                  if os.environ.get("RTB200_PIN_ALL") or c not in SLOW])
def test_oracle_port_matches_reference(name):
    c = load_case(name)
    g = c.graph()
    if c.error:
        with pytest.raises(Exception) as exc:
            oracle_execute(g, bounds=c.bounds, inputs=c.inputs, seed=c.seed)
        assert c.error.split(":")[0] == type(exc.value).__name__
        return
    outs, rb = oracle_execute(g, bounds=c.bounds, inputs=c.inputs, seed=c.seed,
                              return_bounds=True)
    assert rb == c.resolved_bounds
    assert sorted(outs) == sorted(c.outputs)
    for k, want in c.outputs.items():
        assert outs[k].dtype == want.dtype, k
        assert outs[k].shape == want.shape, k
        assert np.array_equal(outs[k], want), k


def test_rng_golden_survey():
    """eps[1,0,3] at seed 3, tag 1 of reinforce.rtl."""
    v = np.random.default_rng((3, 1, 1, 0, 3)).standard_normal(())
    assert float(v) == -0.9978302762444449


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_adapter_roundtrip_against_live_reference():
    """from_pdg(live Pdg) -> JSON -> Graph executes identically to the live
    reference on the C1 config (reinforce.rtl, I=2,B=2,T=4, seed 3)."""
    import sys
    sys.path.insert(0, REF)
    from recten import dsl, pdg, runtime
    from paper_2501_05408_b200 import ir
    path = "/root/reference/pkg/programs/reinforce.rtl"
    g = pdg.build(dsl.load_path(path))
    want = runtime.reference_execute(g, bounds={"I": 2, "B": 2, "T": 4},
                                     inputs={"winit": 0.1}, seed=3)
    mine = ir.Graph.from_json(ir.from_pdg(g).to_json())
    got = oracle_execute(mine, bounds={"I": 2, "B": 2, "T": 4},
                         inputs={"winit": 0.1}, seed=3)
    for k in want:
        assert np.array_equal(want[k], got[k])
    # SURVEY §8(c) golden vector
    assert want["w"].tolist() == [0.1, 0.09312935242263691]
    assert float(want["G"].sum()) == pytest.approx(0.5635977569309989, rel=0, abs=1e-15)
