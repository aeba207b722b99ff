"""Env sharding: host logic on CPU with a world-size-2 gloo
group, and the real sharded CUDA path with two ranks sharing one GPU (gloo
all-reduce over CUDA tensors) checked against the unsharded run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from golden_cases import load_case, load_graph
from paper_2501_05408_b200 import executor as X
from paper_2501_05408_b200 import lower as L
from paper_2501_05408_b200 import native as N
from paper_2501_05408_b200.shard import ShardError, ShardSpec, TorchComm, check_shardable


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_c2_program_is_env_shardable():
    g = load_graph("reinforce_mlp_c2")
    red = check_shardable(g, "b")
    names = sorted(g.nodes[n].name for n in red)
    # objective sum over envs + the six parameter-gradient reductions
    assert len(red) == 7, names


def test_cross_env_reads_are_refused():
    c = load_case("corpus_stream_window_plain_s3")     # x[b, t:min(t+3,T)] is fine along b
    check_shardable(c.graph(), "b")
    with pytest.raises(ShardError):
        check_shardable(c.graph(), "t")                 # windows along t cross shards


def _dry(g, benv, shard):
    h = X.copy_graph(g)
    X.prepare(h, benv)
    red = check_shardable(h, shard.dim)
    an = X.analyze(h, benv, X.payload_shapes(h, benv), True)
    ptr = 1 << 20
    for k, b in an["bufs"].items():
        b.ptr = ptr
        ptr += b.nbytes + 256
    return L.Lowering(an["plan"], an["bufs"], 0, 0, lambda nb: 1 << 40, an["contract"],
                      an["fuse_src"], an["gemm_epi"], absorbed=an["absorbed"], shard=shard,
                      shard_reduce=red).lower()


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    g = load_graph("reinforce_mlp_c2")
    low = _dry(g, {"I": 1, "B": 8, "T": 16}, ShardSpec("b", rank, world))
    offs = set()
    for (k, p, *_r) in low.recs:
        if k in (N.RT_K_RNG, N.RT_K_UDF):
            offs |= {p.coord_add[j] for j in range(p.ncoord)}
    for info in low.loop_subs.values():
        for op in info["ops"]:
            if op[0] == N.RT_K_UDF:
                offs |= {op[1].coord_add[j] for j in range(op[1].ncoord)}
    t = torch.full((5,), float(rank + 1))
    TorchComm().allreduce_(t)
    q.put((rank, len(low.hooks), sorted(offs), t.tolist()))
    dist.destroy_process_group()


def test_sharded_lowering_and_allreduce_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, nhooks, offs, t in res:
        assert nhooks == 7
        assert offs == sorted({0, rank * 8})            # global env index offset
        assert t == [3.0] * 5                           # 1 + 2 summed over ranks


def _gpu_worker(rank, world, port, q, B, T):
    import torch.distributed as dist
    from paper_2501_05408_b200 import execute
    from paper_2501_05408_b200.workloads import mlp_inputs
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    g = load_graph("reinforce_mlp_c2")
    outs = execute(g, bounds={"I": 1, "B": B // world, "T": T}, inputs=mlp_inputs(), seed=0,
                   shard=ShardSpec("b", rank, world))
    q.put((rank, {k: v for k, v in outs.items()}))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_run_matches_unsharded_on_one_gpu():
    from paper_2501_05408_b200 import execute
    from paper_2501_05408_b200.workloads import mlp_inputs
    B, T = 64, 32
    g = load_graph("reinforce_mlp_c2")
    full = execute(g, bounds={"I": 1, "B": B, "T": T}, inputs=mlp_inputs(), seed=0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q, B, T)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    half = B // 2
    for r in range(2):
        np.testing.assert_allclose(res[r]["G"], full["G"][:, r * half:(r + 1) * half],
                                   rtol=1e-5, atol=1e-6)
        for k in ("W1_next", "b1_next", "W2_next", "b2_next", "W3_next", "b3_next", "objective"):
            np.testing.assert_allclose(res[r][k], full[k], rtol=1e-4, atol=1e-6, err_msg=k)


def _ppo_gpu_worker(rank, world, port, q, case):
    import torch.distributed as dist
    from paper_2501_05408_b200 import execute
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    c = load_case(case)
    g = c.graph()
    outs = execute(g, bounds={"B": 8 // world, "U": 2 // world},
                   inputs=c.inputs, seed=c.seed,
                   shard=ShardSpec("b", rank, world, ("u",)))
    q.put((rank, {k: v for k, v in outs.items()}))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_ppo_matches_reference_on_one_gpu():
    """PPO with every minibatch gradient all-reduced across 2 env shards
    (envs b and minibatch envs u co-sharded) reproduces the reference's
    unsharded outputs: replicated parameters, summed losses, local A."""
    case = "ppo_f32_I1B8T6E2M4"
    c = load_case(case)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ppo_gpu_worker, args=(r, 2, port, q, case)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        np.testing.assert_allclose(res[r]["A"], c.outputs["A"][:, r * 4:(r + 1) * 4],
                                   rtol=1e-5, atol=1e-6)
        for k, want in c.outputs.items():
            if k != "A":
                np.testing.assert_allclose(res[r][k], want, rtol=1e-5, atol=1e-6, err_msg=k)


def test_sharded_ppo_lowering_offsets_and_hooks():
    """Rank 1 of 2: env entropy uses global env indices (offset B_local),
    and every minibatch loss/gradient reduction over u is all-reduced."""
    g = load_graph("ppo_c3")
    b = {"I": 1, "E": 2, "M": 2, "U": 4, "B": 8, "T": 6}
    low = _dry_shard(g, b, ShardSpec("b", 1, 2, ("u",)))
    offs = set()
    for (k, p, *_r) in low.recs:
        if k in (N.RT_K_RNG, N.RT_K_UDF):
            offs |= {p.coord_add[j] for j in range(p.ncoord)}
    for info in low.loop_subs.values():
        for op in info["ops"]:
            if op[0] == N.RT_K_UDF:
                offs |= {op[1].coord_add[j] for j in range(op[1].ncoord)}
    assert offs == {0, 8}
    names = {h["node"] for h in low.hooks}
    assert len(names) == 9


def _dry_shard(g, benv, shard):
    h = X.copy_graph(g)
    X.prepare(h, benv)
    red = check_shardable(h, shard.dim, shard.also, benv)
    an = X.analyze(h, benv, X.payload_shapes(h, benv), True)
    ptr = 1 << 20
    for k, bb in an["bufs"].items():
        bb.ptr = ptr
        ptr += bb.nbytes + 256
    return L.Lowering(an["plan"], an["bufs"], 0, 0, lambda nb: 1 << 40, an["contract"],
                      an["fuse_src"], an["gemm_epi"], absorbed=an["absorbed"], shard=shard,
                      shard_reduce=red).lower()


def _nccl_worker(port, q, B, T):
    import torch.distributed as dist
    from paper_2501_05408_b200 import execute
    from paper_2501_05408_b200.shard import ShardSpec
    from paper_2501_05408_b200.workloads import mlp_inputs
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    g = load_graph("reinforce_mlp_c2")
    side = torch.cuda.Stream()
    outs = execute(g, bounds={"I": 1, "B": B, "T": T}, inputs=mlp_inputs(), seed=0,
                   shard=ShardSpec("b", 0, 1), stream=side)
    side.synchronize()
    q.put({k: v for k, v in outs.items()})
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_run_over_nccl_on_a_side_stream():
    """The sharded program's gradient all-reduce hooks over a real NCCL
    communicator (one rank: the multi-GPU plumbing — hook segments, prefix
    CUDA graph, the collective ordered on the program's own non-default
    stream) reproduce the unsharded run."""
    from paper_2501_05408_b200 import execute
    from paper_2501_05408_b200.workloads import mlp_inputs
    B, T = 64, 32
    full = execute(load_graph("reinforce_mlp_c2"), bounds={"I": 1, "B": B, "T": T},
                   inputs=mlp_inputs(), seed=0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(free_port(), q, B, T))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    for k, want in full.items():
        np.testing.assert_allclose(res[k], want, rtol=1e-5, atol=1e-6, err_msg=k)


def test_gradient_allreduces_bucket_into_one_collective():
    """The sharded C2 program's seven sum all-reduces (six gradients and the
    objective) all precede their first consumer, so only the last hook
    flushes: one collective per optimizer step; PPO flushes
    once per minibatch update."""
    g = load_graph("reinforce_mlp_c2")
    low = _dry(g, {"I": 1, "B": 8, "T": 16}, ShardSpec("b", 0, 2))
    flags = [h["flush"] for h in low.hooks]
    assert len(flags) == 7 and flags.count(True) == 1 and flags[-1]
    lowp = _dry_shard(load_graph("ppo_c3"), {"I": 1, "E": 2, "M": 2, "U": 4, "B": 8, "T": 6},
                      ShardSpec("b", 1, 2, ("u",)))
    assert any(h["flush"] for h in lowp.hooks)
    assert sum(h["flush"] for h in lowp.hooks) < len(lowp.hooks)


def test_allreduce_bucket_sums_each_tensor():
    from paper_2501_05408_b200.executor import _allreduce_bucket

    class Twice:
        def allreduce_(self, t):
            t.mul_(2)
            return t
    a, b, c = torch.ones(3), torch.arange(4.0), torch.ones(2, dtype=torch.float64)
    _allreduce_bucket(Twice(), [a, b, c], torch)
    assert a.tolist() == [2.0] * 3 and b.tolist() == [0.0, 2.0, 4.0, 6.0] and c.tolist() == [2.0, 2.0]


def _native_worker(port, q, B, T, workload):
    import torch.distributed as dist
    from paper_2501_05408_b200 import execute, get_executable, native as N
    from paper_2501_05408_b200.shard import NcclComm, ShardSpec
    from paper_2501_05408_b200.workloads import mlp_inputs, ppo_inputs
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    comm = NcclComm()
    if workload == "c2":
        g, bounds, inp = load_graph("reinforce_mlp_c2"), {"I": 1, "B": B, "T": T}, mlp_inputs()
        spec = ShardSpec("b", 0, 1)
    else:
        g = load_graph("ppo_c3")
        bounds = {"I": 1, "E": 2, "M": 2, "U": B // 2, "B": B, "T": T}
        inp, spec = ppo_inputs(), ShardSpec("b", 0, 1, ("u",))
    exe, _ = get_executable(g, bounds, inp, 0, shard=spec, comm=comm)
    exe.GRAPH_MIN_LAUNCHES = 0          # capture however short the program is
    ncoll = sum(1 for i in range(exe.nprog) if exe.prog[i].op == N.RT_OP_COLL)
    outs = execute(g, bounds=bounds, inputs=inp, seed=0, shard=spec, comm=comm)
    outs = execute(g, bounds=bounds, inputs=inp, seed=0, shard=spec, comm=comm)   # graph replay
    q.put(({k: v for k, v in outs.items()}, ncoll, len(exe.hooks), exe.graph_exec is not None))
    comm.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c2", "c3"])
def test_sharded_run_with_in_graph_nccl_collectives(workload):
    """NcclComm: the gradient all-reduces of the sharded program become
    in-program NCCL collectives (RT_OP_COLL, csrc/coll.cu) -- no host hook
    is left and the whole step replays as one CUDA graph with them inside.
    One rank (one GPU in this environment: NCCL refuses two ranks on one
    device); the collective path, bucketing and capture are exercised and
    the result equals the unsharded run."""
    from paper_2501_05408_b200 import execute
    from paper_2501_05408_b200.workloads import mlp_inputs, ppo_inputs
    if workload == "c2":
        B, T = 64, 32
        full = execute(load_graph("reinforce_mlp_c2"), bounds={"I": 1, "B": B, "T": T},
                       inputs=mlp_inputs(), seed=0)
    else:
        B, T = 16, 8
        full = execute(load_graph("ppo_c3"), bounds={"I": 1, "E": 2, "M": 2, "U": B // 2, "B": B,
                                                     "T": T}, inputs=ppo_inputs(), seed=0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_native_worker, args=(free_port(), q, B, T, workload))
    p.start()
    res, ncoll, nhooks, graphed = q.get(timeout=300)
    p.join(timeout=60)
    assert ncoll > 0 and nhooks == 0 and graphed
    for k, want in full.items():
        np.testing.assert_allclose(res[k], want, rtol=1e-5, atol=1e-6, err_msg=k)
