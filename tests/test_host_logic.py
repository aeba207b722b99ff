"""CPU-only checks of the host side: the C ABI loads and exports what the
header declares, struct layouts match, and every golden graph plans and
lowers (with fake device pointers) without a GPU."""

import ctypes as C
import os
import re
import subprocess

import pytest

from golden_cases import all_cases, load_graph
from paper_2501_05408_b200 import executor as X
from paper_2501_05408_b200 import lower as L
from paper_2501_05408_b200 import native as N
from paper_2501_05408_b200 import planner as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rtb200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rt_\w+)\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(N.LIB_PATH)
    syms = declared_symbols()
    assert syms, "no declarations parsed"
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.EXPORTS), sorted(set(syms) ^ set(N.EXPORTS))
    assert N.lib().rt_version() == 1


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    names = ["rt_box", "rt_view", "rt_hdr", "rt_ew_params", "rt_reduce_params",
             "rt_scan_params", "rt_gemm_params", "rt_splitk_params", "rt_rng_params",
             "rt_udf_params", "rt_launch_rec", "rt_instr", "rt_gop", "rt_thin_params", "rt_coll"]
    src.write_text('#include <stdio.h>\n#include "rtb200.h"\nint main(){' +
                   "".join(f'printf("%zu\\n", sizeof({n}));' for n in names) + "}")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)])
    sizes = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    for n, s in zip(names, sizes):
        assert C.sizeof(getattr(N, n)) == s, n


def dry_lower(g, benv, seed=0, fuse=True):
    h = X.copy_graph(g)
    X.prepare(h, benv)
    pshape = X.payload_shapes(h, benv)
    an = X.analyze(h, benv, pshape, fuse)
    bufs, ptr = an["bufs"], 1 << 20
    for k, b in bufs.items():
        b.ptr = ptr
        ptr += (b.nbytes + 511) // 256 * 256
    low = L.Lowering(an["plan"], bufs, 0, seed, lambda nb: 1 << 40, an["contract"],
                     an["fuse_src"], an["gemm_epi"], absorbed=an["absorbed"]).lower()
    return an["plan"], low, an["contract"], an["alias"]


CASES = [c for c in all_cases() if not c.error]


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_golden_graph_plans_and_lowers(case):
    g = case.graph()
    benv = {g.dim_bound[d]: (case.resolved_bounds or {}).get(g.dim_bound[d],
                                                               g.bindings.get(g.dim_bound[d]))
            for d in g.dim_order}
    for fuse in (True, False):
        plan, low, _, _ = dry_lower(g, benv, fuse=fuse)
        assert low.recs or not g.outputs


def test_c2_plan_batches_envs_and_fuses_dw():
    """The acting recurrence loops over t only (all envs per launch) and the
    three weight gradients are single contraction GEMMs."""
    g = load_graph("reinforce_mlp_c2")
    plan, low, contract, alias = dry_lower(g, {"I": 1, "B": 1024, "T": 1000})
    txt = P.describe(plan.steps, plan.graph)
    assert "for t asc" in txt and "for b" not in txt
    assert "bulk o:merge over (b)" in txt or "bulk o:merge over (i,b)" in txt
    assert len(contract) == 3
    kinds = [k for (k, *_r) in low.recs]
    assert kinds.count(N.RT_K_SCAN) == 1           # G = dsum(r[t:T]) as one reverse scan


def test_interval_and_refine():
    box = {"t": (0, 9)}
    assert P.interval(("sub", ("sym", "t", "loop"), ("int", 1)), box) == (-1, 8)
    assert P.refine_box(("ge", ("sym", "t", "loop"), ("int", 1)), box) == {"t": (1, 9)}
    assert P.refine_box(("lt", ("sym", "t", "loop"), ("int", 0)), box) is None


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_every_touched_buffer_is_materialised(case):
    """No launch may address a buffer that the analysis decided never to
    allocate (fused, absorbed or contracted nodes), directly or via aliases."""
    from paper_2501_05408_b200 import memplan
    g = case.graph()
    benv = {g.dim_bound[d]: (case.resolved_bounds or {}).get(g.dim_bound[d],
                                                               g.bindings.get(g.dim_bound[d]))
            for d in g.dim_order}
    h = X.copy_graph(g)
    X.prepare(h, benv)
    pshape = X.payload_shapes(h, benv)
    an = X.analyze(h, benv, pshape, True)
    bufs = an["bufs"]
    roots = [k for k, b in bufs.items() if b.alias is None and k[0] not in an["virtual"]]
    fake = {k: (i + 1) << 44 for i, k in enumerate(roots)}
    for i, k in enumerate(bufs):
        bufs[k].ptr = (0x7000 + i) << 32          # never-allocated sentinel
    for k, p in fake.items():
        bufs[k].ptr = p
    for k, b in bufs.items():
        r = b
        while r.alias is not None:
            r = bufs[r.alias]
        b.ptr = r.ptr
    low = L.Lowering(an["plan"], bufs, 0, 0, lambda nb: 1 << 60, an["contract"], an["fuse_src"],
                     an["gemm_epi"], absorbed=an["absorbed"]).lower()
    valid = set(fake.values()) | {1 << 60}
    for ri, (kind, p, *_r) in enumerate(low.recs):
        ptrs = memplan.touched_ptrs(p)
        for op in low.loop_subs.get(ri, {}).get("ops", ()):
            ptrs |= memplan.touched_ptrs(op[1])
        assert ptrs <= valid, (ri, [hex(x) for x in ptrs - valid])


def test_thin_gemm_selection():
    """Narrow GEMMs over many points lower to RT_K_THIN, square ones don't."""
    from test_gpu_kernels import mm_graph
    cases = [((20000, 256, 4, True), 1), ((20000, 16, 256, True), 1),
             ((9000, 4, 256, False), 2), ((20000, 256, 256, True), None),
             ((9000, 256, 256, False), None)]
    for (B, K, Nn, contract), variant in cases:
        g = mm_graph(B, K, Nn, contract=contract)
        _, low, _, _ = dry_lower(g, {"B": B})
        thin = [r[1] for r in low.recs if r[0] == N.RT_K_THIN]
        if variant is None:
            assert not thin
        else:
            assert thin and thin[0].variant == variant
            if variant == 1:
                assert any(r[0] == N.RT_K_SPLITK for r in low.recs)


PPO_BOUNDS = {"I": 1, "E": 4, "M": 4, "U": 1024, "B": 4096, "T": 512}


def _ppo_analysis():
    g = load_graph("ppo_c3")
    h = X.copy_graph(g)
    X.prepare(h, PPO_BOUNDS)
    an = X.analyze(h, PPO_BOUNDS, X.payload_shapes(h, PPO_BOUNDS))
    byname = {h.nodes[k[0]].name: b for k, b in an["bufs"].items() if k[1] == 0}
    return h, an, byname


def test_ppo_plan_peels_rollout_into_first_update():
    """The rollout (over b,t) reads theta[i,0,0] that the update loops
    advance: planned as e in [0,1) / j in [0,1) peels holding the rollout,
    then the remaining minibatches and epochs (planner.peel_for)."""
    h, an, _ = _ppo_analysis()
    txt = P.describe(an["plan"].steps, h)
    assert "for e asc [0, 1):" in txt and "for e asc [1, 4):" in txt
    assert "for j asc [0, 1):" in txt and "for j asc [1, 4):" in txt
    assert "bulk o:merge over (b)" in txt or "bulk o:merge over (i,b)" in txt  # all envs


def test_ppo_storage_folding():
    """Minibatch activations keep one (u,t) slab (folded along e and j);
    a permute of the rollout over (i,j,u,t) that later epochs re-read is
    NOT folded along j (it is produced once, in the e = 0 peel)."""
    h, an, bufs = _ppo_analysis()
    assert bufs["h1_n"].folded == frozenset({"e", "j"})
    assert bufs["h2_n"].folded == frozenset({"e", "j"})
    lacking_e = [b for name, b in bufs.items()
                 if "j" in b.dims and "e" not in b.dims and "u" in b.dims]
    assert lacking_e and all(not b.folded for b in lacking_e)
    assert all(not b.folded for name, b in bufs.items() if name in ("A", "R", "o", "a"))


def test_ppo_env_shard_co_shards_minibatch_envs():
    """b = u*M + j: sharding envs b shards every minibatch's u with them;
    the reductions over u (losses, 8 parameter gradients) get all-reduces."""
    from paper_2501_05408_b200.shard import check_shardable
    g = load_graph("ppo_c3")
    b = dict(PPO_BOUNDS, U=512, B=2048)
    h = X.copy_graph(g)
    X.prepare(h, b)
    red = check_shardable(h, "b", ("u",), b)
    assert len(red) == 9
    with pytest.raises(Exception):
        check_shardable(h, "b", (), b)        # without u: b read across envs


def test_ppo_heads_use_row_stream_gemm():
    """mu_n (N=4) and V_n (N=1) over a minibatch's (u,t) rows are narrow-N
    row streams (thin variant 3), not 128x256 tensor-core tiles -- and ONE
    launch per minibatch writes both (find_sibling_rows: the trunk's h2_n
    is read once)."""
    g = load_graph("ppo_c3")
    plan, low, _, _ = dry_lower(g, PPO_BOUNDS)
    fam = {}
    for (k, p, *_r, lab) in low.recs:
        if lab[1] in ("mu_n", "V_n", "V"):
            fam.setdefault(lab[1], set()).add((k, getattr(p, "variant", None),
                                               getattr(p, "r", None), getattr(p, "r2", None)))
    assert fam["mu_n"] == {(N.RT_K_THIN, 3, 5, 1)} and "V_n" not in fam


def test_time_blocking_shrinks_long_horizon_plan():
    """C4 (E=256, T=100k): blocking t by 10k puts the backward chain in a
    loop over blocks with block-sized storage: the static peak drops from
    ~159 GB (over one B200's HBM with the env noise) to ~68 GB."""
    from paper_2501_05408_b200 import blocking
    g = load_graph("reinforce_mlp_c2")
    benv = {"I": 1, "B": 256, "T": 100000}
    h = X.copy_graph(g)
    X.prepare(h, benv)
    b2 = blocking.block_dim(h, benv, "t", 10000)
    an = X.analyze(h, b2, X.payload_shapes(h, b2))
    txt = P.describe(an["plan"].steps, h)
    assert "for t_blk asc:" in txt
    folded = [k for k, b in an["bufs"].items() if "t_blk" in b.folded]
    assert len(folded) >= 15
    # every block-chain buffer of real size keeps one block of storage
    roots = [k for k, b in an["bufs"].items() if b.alias is None and k[0] not in an["virtual"]]
    big = [k for k in roots if "t_blk" in an["bufs"][k].dims and
           "t_blk" not in an["bufs"][k].folded and an["bufs"][k].nbytes > 16 << 20]
    assert not big, big
    assert an["bufs"][[k for k in an["bufs"] if h.nodes[k[0]].name == "v126"][0]].nbytes \
        == 256 * 10000 * 256 * 4


def test_swap_plan_manages_acting_activations():
    """C4 blocked: h1, h2 (26 GB each at E=256, T=100k) are swap-managed
    (written by the acting loop, read per time block); o is not (the
    recurrence reads o[t-1] across block boundaries)."""
    from paper_2501_05408_b200 import blocking, swap as SW
    g = load_graph("reinforce_mlp_c2")
    benv = {"I": 1, "B": 256, "T": 100000}
    h = X.copy_graph(g)
    X.prepare(h, benv)
    b2 = blocking.block_dim(h, benv, "t", 10000)
    an = X.analyze(h, b2, X.payload_shapes(h, b2))
    sp = SW.plan_swap(h, an["plan"], an["bufs"], an["virtual"], b2)
    names = {h.nodes[k[0]].name for k in sp.keys}
    assert {"h1", "h2"} <= names and "o" not in names
    assert sp.DI == 10 and sp.bs == 10000


def test_gae_delta_fused_into_the_scan():
    """GAE: delta = r + gamma*V[t+1] - V is formed inside the scan kernel (no
    delta buffer) for the kernel program and for the PPO program."""
    for name, benv in (("k_gae_bt", {"B": 4096, "T": 512}), ("ppo_c3", PPO_BOUNDS)):
        g = load_graph(name)
        plan, low, _, _ = dry_lower(g, benv)
        scans = [p for (k, p, *_r) in low.recs if k == N.RT_K_SCAN]
        assert any(p.gae for p in scans), name
        assert not any(lab[1] == "delta" for (*_r, lab) in low.recs), name


def test_c2_tanh_vjp_gate_fuses_into_the_narrow_head_product():
    """d(h2) = d(mu) @ W3^T followed by the tanh VJP `gy * (1 - h2*h2)`
    (reference frontend.py:961-963) lowers to ONE thin variant-2 launch with
    the gate epilogue (no elementwise launch, no d(h2) buffer); small
    problems keep the unfused path (the thin kernel would not be chosen)."""
    g = load_graph("reinforce_mlp_c2")
    _plan, low, _c, _a = dry_lower(g, {"I": 1, "B": 1024, "T": 1000})
    gates = [p for (k, p, *_r) in low.recs if k == N.RT_K_THIN and p.variant == 2 and p.epilogue == 2]
    assert len(gates) == 1 and gates[0].k == 4 and gates[0].r == 256
    assert any(isinstance(t, tuple) and t[0] == "gate" for (_x, _b, t) in low.gemm_epi.values())
    _plan, low2, _c, _a = dry_lower(g, {"I": 1, "B": 4, "T": 8})
    assert not any(isinstance(t, tuple) for (_x, _b, t) in low2.gemm_epi.values())


def test_c2_acting_loop_kernel_source_builds_for_sm100a():
    """The JIT-specialised acting loop of C2 carries every on-chip mechanism
    (W2 in registers + shared memory with the row-split epilogue, normals and
    eps staged by cp.async, env inputs and the carried observation read from
    shared memory) and NVRTC compiles it for sm_100a (no GPU needed)."""
    import ctypes as C
    from paper_2501_05408_b200 import jit
    g = load_graph("reinforce_mlp_c2")
    _p, low, _c, _a = dry_lower(g, {"I": 1, "B": 1024, "T": 1000})
    subs = list(low.loop_subs.items())
    assert len(subs) == 1
    ri, info = subs[0]
    lp = low.recs[ri][1]
    assert info["hybrid"] and info["hybrid"]["kr"] == 128 and info["hybrid"]["ncol"] == 2
    src = jit.loop_source(lp, info["ops"], "loop_jit", info)
    for needle in ("hyb_core<8, 256, 256, 2, 64, true>",   # W2 on chip, row-split epilogue
                   "hyb_core<8, 16, 256, 2, 0, true>",     # W1 resident through the same core
                   "cp_async8", "cp_async4",               # normals / eps one step ahead
                   "warp_pairwise_sum_s",                  # env inputs from shared memory
                   "T0_ ?",                                # carried observation / staged eps
                   "tanh_fast"):
        assert needle in src, needle
    lib = N.lib()
    opts = jit._opts()
    blob = b"\0".join(opts) + b"\0"
    size = C.c_uint64(0)
    rc = lib.rt_jit_cubin(src.encode(), blob, len(opts), None, C.byref(size))
    assert rc == 0 and size.value > 0
    # resource usage: the 128 weight registers per thread must not spill
    import shutil
    import subprocess
    import tempfile
    if shutil.which("cuobjdump"):
        buf = C.create_string_buffer(size.value)
        assert lib.rt_jit_cubin(src.encode(), blob, len(opts), buf, C.byref(size)) == 0
        with tempfile.NamedTemporaryFile(suffix=".cubin") as fh:
            fh.write(buf.raw[:size.value])
            fh.flush()
            res = subprocess.run(["cuobjdump", "--dump-resource-usage", fh.name],
                                 capture_output=True, text=True).stdout
        line = [x for x in res.splitlines() if "REG:" in x][0]
        fields = dict(f.split(":") for f in line.split() if ":" in f and f.split(":")[1].isdigit())
        assert int(fields["REG"]) <= 255 and int(fields.get("LOCAL", "0")) == 0, line


def test_c2_fused_mlp_step_source_builds_for_sm100a():
    """The fused MLP acting step of C2 (jit_mlp.py: four-column h2 core,
    warp-per-row head/action/env) matches the C2 loop and NVRTC compiles it
    for sm_100a without spills (no GPU needed)."""
    import ctypes as C
    from paper_2501_05408_b200 import jit, jit_mlp
    g = load_graph("reinforce_mlp_c2")
    _p, low, _c, _a = dry_lower(g, {"I": 1, "B": 1024, "T": 1000})
    (ri, info), = list(low.loop_subs.items())
    lp = low.recs[ri][1]
    m = jit_mlp.match(lp, info["ops"], info)
    assert m is not None and m["R"] == 7
    src = jit_mlp.source(lp, info["ops"], info, m)
    for needle in ("mlp_h2q<8, 7, 32, 256>", "mlp_head<4, 256>",
                   "warp_pairwise_sum_s", "cp_async8", "tanh_fast"):
        assert needle in src, needle
    lib = N.lib()
    opts = jit._opts()
    blob = b"\0".join(opts) + b"\0"
    size = C.c_uint64(0)
    assert lib.rt_jit_cubin(src.encode(), blob, len(opts), None, C.byref(size)) == 0
    buf = C.create_string_buffer(size.value)
    assert lib.rt_jit_cubin(src.encode(), blob, len(opts), buf, C.byref(size)) == 0
    import shutil
    import subprocess
    import tempfile
    if shutil.which("cuobjdump"):
        with tempfile.NamedTemporaryFile(suffix=".cubin") as fh:
            fh.write(buf.raw[:size.value])
            fh.flush()
            res = subprocess.run(["cuobjdump", "--dump-resource-usage", fh.name],
                                 capture_output=True, text=True).stdout
        line = [x for x in res.splitlines() if "REG:" in x][0]
        fields = dict(f.split(":") for f in line.split() if ":" in f and f.split(":")[1].isdigit())
        assert int(fields["REG"]) <= 255 and int(fields.get("LOCAL", "0")) == 0, line


def test_remat_replaces_swapping_of_the_tanh_layers():
    """C4 (E=256, T=100k, blocked by 10k, swap): the backward gets its own
    copies of the loop's two tanh layers (remat.remat_chains), recomputed per
    time block from the kept observation; only the narrow mu / a stay
    swap-managed and the static footprint drops from ~73 GB to ~16 GB."""
    from paper_2501_05408_b200 import blocking, remat, swap as SW
    g = load_graph("reinforce_mlp_c2")
    benv = {"I": 1, "B": 256, "T": 100000}
    h = X.copy_graph(g)
    X.prepare(h, benv)
    cl = remat.remat_chains(h, "t")
    assert sorted(h.nodes[k].name for k in cl) == ["h1", "h2"]
    for k in cl:        # the loop's layers are read only inside the loop now
        assert all(h.nodes[e.sink].name in ("v66", "v69") for e in h.out_edges(k))
    b2 = blocking.block_dim(h, benv, "t", 10000)
    an = X.analyze(h, b2, X.payload_shapes(h, b2))
    sp = SW.plan_swap(h, an["plan"], an["bufs"], an["virtual"], b2)
    assert sorted(h.nodes[k[0]].name for k in sp.keys) == ["a", "mu"]
    roots = [k for k, b in an["bufs"].items() if b.alias is None and k[0] not in an["virtual"]]
    assert sum(an["bufs"][k].nbytes for k in roots) < 20e9
