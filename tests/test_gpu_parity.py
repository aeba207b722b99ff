"""Parity of the CUDA executor against the reference (golden fixtures) and
the oracle port, on a B200.  Tolerances (north_star): integer /
bool / index results exact; fp64 programs rtol 1e-12; fp32 programs rtol
1e-5."""

import numpy as np
import pytest

from golden_cases import all_cases, case_ids, load_case

pytestmark = pytest.mark.gpu

TOL = {"f64": dict(rtol=1e-12, atol=1e-13), "f32": dict(rtol=1e-5, atol=1e-6)}


def assert_close(got, want, name):
    assert got.shape == want.shape, (name, got.shape, want.shape)
    assert got.dtype == want.dtype, (name, got.dtype, want.dtype)
    if want.dtype in (np.bool_, np.int64):
        assert np.array_equal(got, want), name
    else:
        tol = TOL["f32" if want.dtype == np.float32 else "f64"]
        np.testing.assert_allclose(got, want, err_msg=name, **tol)


OK_CASES = [c for c in case_ids() if not load_case(c).error]


@pytest.mark.parametrize("name", OK_CASES)
def test_executor_matches_reference(name):
    from paper_2501_05408_b200 import execute
    c = load_case(name)
    outs, rb = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed,
                       return_bounds=True)
    assert rb == c.resolved_bounds
    assert sorted(outs) == sorted(c.outputs)
    for k, want in c.outputs.items():
        if c.alt_outputs:
            from test_gpu_fullwidth import check_output
            check_output(k, outs[k], want, c.alt_outputs.get(k))
        else:
            assert_close(outs[k], want, k)


ERR_CASES = [c for c in case_ids() if load_case(c).error]


@pytest.mark.parametrize("name", ERR_CASES)
def test_executor_fails_like_reference(name):
    """Graphs the reference itself cannot evaluate raise the same exception
    class with the same message: the F5 eager-fold hazard (OracleError,
    runtime.py:352-355, via demand.py) and a zero divisor in a device index
    expression (EvaluationError, symexpr.py:491-506, via the status word)."""
    from paper_2501_05408_b200 import execute
    c = load_case(name)
    with pytest.raises(Exception) as exc:
        execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed)
    kind, msg = c.error.split(": ", 1)
    assert type(exc.value).__name__ == kind
    if kind == "OracleError":
        assert str(exc.value) == msg
    else:
        assert str(exc.value).startswith(msg)


def test_rng_bit_exact_vs_numpy():
    """Device SeedSequence -> PCG64 -> ziggurat equals numpy default_rng bit
    for bit on EVERY draw: 100 000 points x 100 draws = 10 M normals (about
    2.6 k of them from the ziggurat tail, |x| > r = 3.6541528853610088,
    rng.cuh's log1p/exp path) and 10 M uniforms."""
    import ctypes as C
    import torch
    from paper_2501_05408_b200 import native as N
    rows, count = 100_000, 100
    rng = np.random.default_rng(0)
    coords = rng.integers(0, 1 << 20, size=(rows, 3)).astype(np.int64)
    coords[:5] = 0
    prefix = [3, 1]
    for dist in (0, 1):
        out = torch.empty(rows * count, dtype=torch.float64, device="cuda")
        pre = (N.u32 * 8)(*prefix)
        rc = N.lib().rt_rng_fill(out.data_ptr(), pre, len(prefix),
                                 coords.ctypes.data_as(C.POINTER(N.i64)), 3, rows, count, dist, 0)
        N.check(rc, "rng_fill")
        got = out.cpu().numpy().reshape(rows, count)
        want = np.empty_like(got)
        for r in range(rows):
            g = np.random.default_rng(tuple(prefix) + tuple(int(x) for x in coords[r]))
            want[r] = g.standard_normal(count) if dist == 0 else g.uniform(0.0, 1.0, count)
        bad = np.argwhere(got.view(np.int64) != want.view(np.int64))
        assert bad.size == 0, (dist, bad[:5])
        if dist == 0:
            assert int((np.abs(want) > 3.6541528853610088).sum()) > 1000


def test_index_select_error_maps_to_runtime_error():
    """Out-of-range rows raise RuntimeError_ like runtime.py:186-188."""
    from paper_2501_05408_b200 import ir, execute, RuntimeError_
    g = ir.Graph(["t"], {"t": "T"}, {"T": 4})
    g.nodes[0] = ir.Node(0, "x", "input", (), ((4,),), ("f64",))
    g.nodes[1] = ir.Node(1, "y", "index_select", ("t",), ((),), ("f64",),
                         {"dim": ir.SymRef("t"), "expr": ("add", ("sym", "t", "loop"), ("int", 1)),
                          "rows": False, "bound": ir.SymRef("T", "bound")}, 1)
    g.edges.append(ir.Edge(1, 0, (), None, 0, 0))
    g.outputs = [("y", 1, 0)]
    with pytest.raises(RuntimeError_, match="row 4 outside"):
        execute(g, inputs={"x": np.arange(4.0)})


JIT_CASES = ["mlp_f32_I2B3T5", "mlp_f64_I2B3T5", "corpus_reinforce_plain_s3", "kat_if_order_plain",
             "corpus_checkpoint_vecfuse_s3", "corpus_epoch_minibatch_vec_s3", "tr_widesum_inc7",
             "corpus_stream_window_plain_s3", "kat_flag_plain", "corpus_gated_value_vec_s3"]


@pytest.mark.parametrize("name", JIT_CASES)
def test_jit_specialised_kernels_match_reference(name, monkeypatch):
    """Every elementwise launch JIT-compiled (NVRTC, straight-line CUDA)
    gives the same results as the reference."""
    from paper_2501_05408_b200 import execute, jit
    monkeypatch.setattr(jit, "JIT_MIN_ELEMS", 0)
    c = load_case(name)
    outs = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed)
    for k, want in c.outputs.items():
        assert_close(outs[k], want, k)


def test_jit_loop_kernel_matches_interpreter(monkeypatch):
    """The JIT-specialised persistent loop (straight-line body) reproduces
    the interpreting loop kernel on the benchmark program at small scale."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import execute, jit
    from paper_2501_05408_b200.workloads import mlp_inputs
    bounds = {"I": 1, "B": 64, "T": 48}
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 1 << 40)
    ref = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=1)
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 0)
    got = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=1)
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-5, atol=1e-6, err_msg=k)


@pytest.mark.parametrize("name", ["mlp_f32_I1B4T6", "mlp_f64_I1B4T6"])
@pytest.mark.parametrize("bs", [2, 3])
def test_time_blocked_backward_matches_reference(name, bs):
    """Long-horizon mode (blocking.block_dim): the backward chain runs per
    block of bs steps with block-sized intermediates; sums over t become
    per-block partials + totals (incrementalize over the time dim)."""
    from paper_2501_05408_b200 import execute
    c = load_case(name)
    got = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed, block=("t", bs))
    for k, want in c.outputs.items():
        assert_close(got[k], want, k)


@pytest.mark.parametrize("name", ["mlp_f32_I1B4T6", "mlp_f64_I1B4T6"])
@pytest.mark.parametrize("bs", [2, 3])
def test_swapped_time_blocks_match_reference(name, bs):
    """GPU<->host swapping (swap.py): the acting loop's activations keep two
    time blocks in HBM, each block is offloaded to pinned host memory after
    the recurrence writes it and fetched back for the backward block."""
    from paper_2501_05408_b200 import execute, get_executable
    c = load_case(name)
    got = execute(c.graph(), bounds=c.bounds, inputs=c.inputs, seed=c.seed, block=("t", bs),
                  swap=1)
    exe, _ = get_executable(c.graph(), c.bounds, c.inputs, c.seed, block=("t", bs), swap=1)
    assert exe.swap_plan is not None and len(exe.swap_plan.keys) >= 2
    for k, want in c.outputs.items():
        assert_close(got[k], want, k)


def test_pair_cluster_loop_matches_interpreter(monkeypatch):
    """CTA-pair persistent loop (2-CTA clusters, resident K-halves of W2,
    DSMEM exchange of operand rows and partial sums) reproduces the
    interpreting loop kernel."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import execute, jit
    from paper_2501_05408_b200.workloads import mlp_inputs
    bounds = {"I": 1, "B": 96, "T": 40}
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 1 << 40)
    ref = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=2)
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 0)
    monkeypatch.setattr(jit, "PAIR_ENABLED", True)
    monkeypatch.setattr(jit, "DUAL_ENABLED", False)
    from paper_2501_05408_b200 import get_executable
    g = load_graph("reinforce_mlp_c2")
    exe, _ = get_executable(g, bounds, mlp_inputs(), 2)
    assert any(info.get("pair") for info in exe.loop_info.values())
    got = execute(g, bounds=bounds, inputs=mlp_inputs(), seed=2)
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-5, atol=1e-6, err_msg=k)


def test_mma_loop_kernel_matches_interpreter(monkeypatch):
    """8-row CTAs (E=1024): the in-loop layers run on the 3xTF32 warp MMA
    core (loop_lib.cuh mma_core) and match the interpreting loop kernel."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import execute, get_executable, jit
    from paper_2501_05408_b200.workloads import mlp_inputs
    bounds = {"I": 1, "B": 1024, "T": 12}
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 1 << 40)
    ref = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=4)
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 0)
    monkeypatch.setattr(jit, "MMA_ENABLED", True)
    g = load_graph("reinforce_mlp_c2")
    exe, _ = get_executable(g, bounds, mlp_inputs(), 4)
    lp = [exe._params[ri] for ri in exe.loop_info][0]
    assert lp.rows_per_cta == 7
    got = execute(g, bounds=bounds, inputs=mlp_inputs(), seed=4)
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-5, atol=1e-6, err_msg=k)


def test_trace_and_stats_report():
    """SPEC trace/stats (trace.py): one EXEC per launch, DEALLOC at the memory
    plan's lifetime ends, OFFLOAD/FETCH per swapped block; the stats report
    the arena peak, transfers and the eager per-tensor estimate."""
    from paper_2501_05408_b200 import get_executable
    c = load_case("mlp_f32_I1B4T6")
    exe, _ = get_executable(c.graph(), c.bounds, c.inputs, c.seed, block=("t", 2), swap=1)
    exe.run(c.inputs)
    lines = exe.trace()
    assert sum(x.startswith("EXEC ") for x in lines) == exe.launch_count
    assert any(x.startswith("DEALLOC ") for x in lines)
    keys = len(exe.swap_plan.keys)
    assert sum(x.startswith("OFFLOAD ") for x in lines) == 3 * keys
    assert sum(x.startswith("FETCH ") for x in lines) == 3 * keys
    rep = exe.stats()
    assert rep["peak_device_bytes"] >= rep["arena_bytes"] > 0
    assert rep["offloads"] == rep["fetches"] == 3 * keys and rep["bytes_moved"] > 0
    assert rep["static_estimate"]["G"] == 1 * 4 * 6 * 4


@pytest.mark.parametrize("fused", [True, False])
def test_default_loop_at_8_rows_matches_interpreter(monkeypatch, fused):
    """JIT acting loop at 7-row CTAs (E=1024) against the interpreting loop
    kernel: the fused 512-thread MLP step (jit_mlp.py, loop_mlp.cuh; the
    default) and the op-by-op JIT loop (2-columns-per-thread core,
    shared-memory forwarding h1 -> h2 -> mu, jit._forward_pairs)."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import execute, get_executable, jit, jit_mlp
    from paper_2501_05408_b200.workloads import mlp_inputs
    bounds = {"I": 1, "B": 1024, "T": 12}
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 1 << 40)
    ref = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=5)
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 0)
    monkeypatch.setattr(jit_mlp, "ENABLED", fused)
    exe, _ = get_executable(load_graph("reinforce_mlp_c2"), bounds, mlp_inputs(), 5)
    assert any("mlp" in info for info in exe.loop_info.values()) == fused
    got = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=5)
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-5, atol=1e-6, err_msg=k)


def test_tanh_vjp_gate_epilogue_matches_unfused(monkeypatch):
    """The thin GEMM's gate epilogue (d(h2) = d(mu) W3^T times 1 - h2*h2 in
    one launch, executor.find_gate_epilogues) reproduces the unfused
    product + elementwise pair at a size where it is chosen (8192 rows)."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import execute, executor as X, get_executable
    from paper_2501_05408_b200 import native as N
    from paper_2501_05408_b200.workloads import mlp_inputs
    bounds = {"I": 1, "B": 128, "T": 64}
    monkeypatch.setattr(X, "GATE_ENABLED", False)
    X._CACHE.clear()
    ref = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=5)
    monkeypatch.setattr(X, "GATE_ENABLED", True)
    X._CACHE.clear()
    g = load_graph("reinforce_mlp_c2")
    exe, _ = get_executable(g, bounds, mlp_inputs(), 5)
    assert any(k == N.RT_K_THIN and p.variant == 2 and p.epilogue == 2
               for k, p in zip(exe.kernels, exe._params))
    got = execute(g, bounds=bounds, inputs=mlp_inputs(), seed=5)
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-5, atol=1e-6, err_msg=k)


@pytest.mark.parametrize("bs", [8, 10])
def test_time_blocked_jit_loop_matches_interpreter(monkeypatch, bs):
    """Time-blocked acting loop (one persistent launch per block, range from
    the launch) through the JIT path — staged normals / operands take the
    block's own start and stop — reproduces the interpreting loop kernel."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import execute, jit
    from paper_2501_05408_b200.workloads import mlp_inputs
    bounds = {"I": 1, "B": 64, "T": 40}
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 1 << 40)
    ref = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=3,
                  block=("t", bs))
    monkeypatch.setattr(jit, "JIT_LOOP_MIN", 0)
    got = execute(load_graph("reinforce_mlp_c2"), bounds=bounds, inputs=mlp_inputs(), seed=3,
                  block=("t", bs))
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-5, atol=1e-6, err_msg=k)


@pytest.mark.parametrize("B,T,bs", [(128, 400, 100), (32, 256, 64)])
def test_rematerialised_backward_matches_swapped_layers(B, T, bs, monkeypatch):
    """Long-horizon mode: the backward recomputing the loop's tanh layers
    per time block (remat.py) gives the gradients of the run that swaps the
    loop's own layers to the host and back, to the fp32 tolerance (the
    recomputation rounds like the learner GEMMs, the loop like its FMA
    chain: ~1e-7 relative per activation)."""
    from golden_cases import load_graph
    from paper_2501_05408_b200 import execute, executor as X
    from paper_2501_05408_b200.workloads import mlp_inputs
    g = load_graph("reinforce_mlp_c2")
    bounds = {"I": 1, "B": B, "T": T}
    inp = mlp_inputs()
    X._CACHE.clear()
    monkeypatch.setattr(X, "REMAT", False)
    ref = execute(g, bounds=bounds, inputs=inp, seed=4, block=("t", bs), swap=1)
    X._CACHE.clear()
    monkeypatch.setattr(X, "REMAT", True)
    got = execute(g, bounds=bounds, inputs=inp, seed=4, block=("t", bs), swap=1)
    exe, _ = X.get_executable(g, bounds, inp, 4, block=("t", bs), swap=1)
    assert exe.swap_plan is not None and \
        sorted(exe.trace_names[k] for k in exe.swap_plan.keys) == ["a", "mu"]
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=2e-5, atol=1e-5, err_msg=k)
    X._CACHE.clear()
