"""Benchmark: training iterations of recurrent-tensor RL programs through
the B200 executor (BASELINE.json metric: env-steps/s per train iter, peak
HBM).  Workloads:

  c2 (default): REINFORCE, E=1024 envs x T=1000 steps per GPU, 2-hidden-
      layer 256-wide tanh MLP policy (BASELINE.json configs[1]).
  c3: PPO with GAE(lambda), 4 epochs x 4 minibatches, E=4096 x T=512,
      shared policy/value MLP (configs[2]).
  c5: c3's program with E=32768 envs in total, split E/N per GPU, NCCL
      all-reduce of every minibatch gradient (configs[4]; strong scaling).

One step = one call of the program at I=1: roll out, returns/advantages
(suffix scans), backward through the MLP, parameter updates (outputs
`*_next`, fed back as the next step's inputs).  env-steps per step = E*T.

  value : device-resident (weights already in HBM, outputs left in HBM)
  e2e   : public API `execute()` with host numpy weights in and updated
          weights + outputs out (H2D/D2H inside the timed region)

`--impl reference` times the reference's own CPU executor on the same
program: recten.runtime.reference_execute from the installed reference
package (baseline/_ref; the oracle port oracle/pdg_oracle.py when it is
absent) on a bounded sample (the real horizon, fewer envs) on every host
core.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


class Workload:
    def __init__(self, name, graph, T, env_total=None, env_per_gpu=None, minibatches=None,
                 ppo=False, desc="", block=None, swap=False):
        self.name, self.graph, self.T, self.block, self.swap = name, graph, T, block, swap
        self.env_total, self.env_per_gpu = env_total, env_per_gpu
        self.minibatches, self.ppo, self.desc = minibatches, ppo, desc

    def local_envs(self, world):
        if self.env_per_gpu:
            return self.env_per_gpu
        assert self.env_total % world == 0
        return self.env_total // world

    def bounds(self, B):
        if self.ppo:
            return {"I": 1, "E": 4, "M": self.minibatches, "U": B // self.minibatches,
                    "B": B, "T": self.T}
        return {"I": 1, "B": B, "T": self.T}

    def inputs(self):
        from paper_2501_05408_b200.workloads import mlp_inputs, ppo_inputs
        return ppo_inputs() if self.ppo else mlp_inputs()

    def params(self):
        from paper_2501_05408_b200.workloads import PARAMS, PPO_PARAMS
        return PPO_PARAMS if self.ppo else PARAMS

    def shard(self, rank, world):
        from paper_2501_05408_b200.shard import ShardSpec
        return ShardSpec("b", rank, world, ("u",) if self.ppo else ())

    @property
    def scaling(self):
        return "strong" if self.env_total else "weak"


WORKLOADS = {
    "c2": Workload("reinforce_mlp_c2", "reinforce_mlp_c2", 1000, env_per_gpu=1024,
                   desc="REINFORCE, E=1024/GPU x T=1000, MLP 16-256-256-4"),
    "c3": Workload("ppo_gae_c3", "ppo_c3", 512, env_per_gpu=4096, minibatches=4, ppo=True,
                   desc="PPO+GAE(0.95), E=4096 x T=512, 4 epochs x 4 minibatches, "
                        "shared MLP 16-256-256-(4|1)"),
    "c4": Workload("reinforce_mlp_c4", "reinforce_mlp_c2", 100000, env_per_gpu=256,
                   block=("t", 10000), swap=True,
                   desc="long-horizon REINFORCE, E=256/GPU x T=100k, MLP 16-256-256-4, "
                        "backward time-blocked by 10k steps (blocking.block_dim), acting "
                        "activations swapped to pinned host per block (swap.py)"),
    "c4_noswap": Workload("reinforce_mlp_c4_noswap", "reinforce_mlp_c2", 100000,
                          env_per_gpu=256, block=("t", 10000),
                          desc="C4 time-blocked, activations resident in HBM (no swap)"),
    "c5": Workload("ppo_gae_c5", "ppo_c3", 512, env_total=32768, minibatches=4, ppo=True,
                   desc="PPO+GAE(0.95), E=32768 total split over GPUs x T=512, "
                        "4 epochs x 4 minibatches"),
}
WL = WORKLOADS["c2"]


def load_graph():
    from paper_2501_05408_b200 import ir
    with open(os.path.join(ROOT, "tests", "golden", "graphs", f"{WL.graph}.json")) as fh:
        return ir.Graph.from_json(fh.read())


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz (boost clock seen under load)
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12

# kernel family -> the kernel name in the committed ncu --set full capture
_NCU_NAME = {"loop": "loop_mlp", "gemm_tma": "k_gemm_tmap", "ew": "ew_jit", "scan": "k_scan"}


def ncu_traffic(family):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the family's
    kernel, from the committed `ncu --set full` capture under profiles/ (the
    newest round's), or None."""
    import csv
    import glob
    name = _NCU_NAME.get(family)
    if not name:
        return None
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{name}_raw.csv")))
    if not files:
        return None
    try:
        rows = list(csv.reader(open(files[-1])))
        h, units, row = rows[0], rows[1], rows[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += float(row[i].replace(",", "")) * scale[units[i]]
        return tot
    except Exception:
        return None


class Clocks:
    def __init__(self):
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,"
                         "clocks_event_reasons.hw_slowdown,"
                         "clocks_event_reasons.hw_thermal_slowdown,"
                         "clocks_event_reasons.sw_thermal_slowdown,"
                         "clocks_event_reasons.sw_power_cap",
                         "--format=csv,noheader,nounits", "-i", "0"],
                        capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples)}


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _ref_importable():
    """The reference package itself (`pip install --target baseline/_ref
    /root/reference`, git-ignored, shipped to the GPU box), else None."""
    try:
        import programs as P   # tests/golden/programs.py builds through recten's front end
        P.recten()
        return P
    except Exception:
        return None


def _ref_sample():
    """A bounded sample of WL's program for the CPU: the REAL horizon (C2:
    T=1000, so the reference's O(T^2) r[t:T] gather is paid as in the real
    workload) over fewer envs (envs are independent: the per-point
    interpreter's cost is linear in them).  PPO: 4 envs x T=128, 4 epochs x
    4 minibatches.  Returns (kind, graph, inputs, bounds, env-steps per call)."""
    P = _ref_importable()
    if WL.ppo:
        B, T = 4, min(WL.T, 128)
        bounds = {"I": 1, "E": 4, "M": 4, "U": 1, "B": B, "T": T}
    else:
        B, T = 1, min(WL.T, 1000)
        bounds = {"I": 1, "B": B, "T": T}
    inputs = WL.inputs()
    if P is not None:
        dsl, fe, pdg, tr, rt, ps = P.recten()
        ctx = (P.ctx_ppo_mlp(B=B, T=T, I=1, epochs=4, minibatches=4) if WL.ppo
               else P.ctx_reinforce_mlp(B=B, T=T, I=1))
        g = pdg.build(ctx)
        pdg.eliminate_dead(g)
        return "reference", g, inputs, None, B * T
    return "port", load_graph(), inputs, bounds, B * T


def _ref_worker(args):
    """One host process: run the reference executor (recten.runtime.
    reference_execute on the untransformed graph; else the oracle port) on
    distinct seeds for `seconds`."""
    wl, seconds, seed0 = args
    global WL
    WL = WORKLOADS[wl]
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    kind, g, inputs, bounds, per = _ref_sample()
    if kind == "reference":
        import recten.runtime as rt
        run = rt.reference_execute
    else:
        from oracle.pdg_oracle import oracle_execute as run
    t0 = time.perf_counter()
    n = 0
    while True:
        run(g, bounds=bounds, inputs=inputs, seed=seed0 + n)
        n += 1
        if time.perf_counter() - t0 > seconds:
            break
    return kind, n * per, time.perf_counter() - t0


def cpu_baseline(seconds=12.0, processes=1):
    """The reference's own CPU executor on a bounded sample of WL's program
    (_ref_sample), single-threaded Python + numpy per process; processes > 1
    runs independent samples in parallel host processes (the reference arm:
    every host core the process may use)."""
    name = [k for k, v in WORKLOADS.items() if v is WL][0]
    if processes <= 1:
        kind, steps, dt = _ref_worker((name, seconds, 0))
        value = steps / dt
    else:
        import multiprocessing as mp
        with mp.get_context("spawn").Pool(processes) as pool:
            res = pool.map(_ref_worker, [(name, seconds, 100000 * i) for i in range(processes)])
        kind = res[0][0]
        steps = sum(r[1] for r in res)
        dt = max(r[2] for r in res)
        value = sum(r[1] / r[2] for r in res)
    B, T = (4, min(WL.T, 128)) if WL.ppo else (1, min(WL.T, 1000))
    what = ("recten.runtime.reference_execute (the reference package, baseline/_ref)"
            if kind == "reference" else "oracle/pdg_oracle.py (reference_execute restated)")
    return {"value": value, "unit": "env-steps/s", "cores": processes, "kind": kind,
            "sample": f"{int(steps // (B * T))} calls of {what} on the untransformed {WL.name} "
                      f"program at E={B} x T={T} (full width, H=256), {processes} process(es) x "
                      f"{dt:.1f}s, single-threaded Python+numpy each; host cores available "
                      f"{_host_cores()}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps_total = args.warmup + args.steps
    procs = max(1, min(_host_cores(), 64))
    base = cpu_baseline(seconds=max(12.0, 2.0 * steps_total), processes=procs)
    line = {"impl": "reference", "metric": "env-steps/s per train iter",
            "value": base["value"], "unit": "env-steps/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": WL.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{WL.name} (bounded CPU sample)",
                       "sample": base["sample"], "hidden": [256, 256], "obs": 16, "act": 4},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    global WL
    WL = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    from paper_2501_05408_b200 import execute, get_executable
    from paper_2501_05408_b200.workloads import next_inputs

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; BENCH_DIST_BACKEND=gloo lets several ranks share
    # one GPU (a functional check of the sharded path, not a measurement)
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(os.environ.get("BENCH_DIST_BACKEND", "nccl"))
    g = load_graph()
    B = WL.local_envs(world)
    T_STEPS = WL.T
    bounds = WL.bounds(B)
    host = WL.inputs()
    params = WL.params()
    dev_in = {k: torch.from_numpy(v).cuda() for k, v in host.items()}
    shard, comm = None, None
    if world > 1:
        shard = WL.shard(rank, world)     # envs [rank*B, (rank+1)*B) of B*world
        if dist.get_backend() == "nccl":
            # the library's own NCCL communicator: gradient all-reduces run
            # inside the program (RT_OP_COLL), one CUDA graph per step
            from paper_2501_05408_b200.shard import NcclComm
            comm = NcclComm()
    exe, _ = get_executable(g, bounds, dev_in, seed=0, shard=shard, comm=comm, block=WL.block,
                            swap=WL.swap)

    def step_dev(inp, graph=None):
        if graph is None:
            exe.run(inp)
        else:
            exe.launch_graph(graph, inp)
        outs = exe.outputs(device_outputs=True)
        return next_inputs(outs, params)

    # warmup (device path, CUDA graph)
    inp = dev_in
    for w in range(args.warmup):
        inp = step_dev(inp)
    torch.cuda.synchronize()

    # per-kernel breakdown: one profiled step (event pair around every launch)
    prof = exe.profile(inp)
    from paper_2501_05408_b200 import roofline as RF
    fam_ms, rows = {}, []
    for r in prof:
        fam = RF.FAMILY.get(r["kernel"], "?")
        fam_ms[fam] = fam_ms.get(fam, 0.0) + r["ms"]
        rows.append(r)
    rows.sort(key=lambda r: -r["ms"])
    dom = rows[0]
    if exe.hooks:      # sharded: all-reduce hooks between program segments, no single graph
        graph_ev, kev = None, []
    else:
        graph_ev, kev = exe.capture_with_events(dom["rec"])

    if dist:
        dist.barrier()
    clocks = Clocks()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dom_ms = []
    ev0.record()
    for s in range(args.steps):
        inp = step_dev(inp, graph_ev)
        if kev:
            ev1.record()
            ev1.synchronize()
            dom_ms.append(sum(kev[2 * i].elapsed_time(kev[2 * i + 1])
                              for i in range(len(kev) // 2)))
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    clk = clocks.stop()
    exe.check_status()
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * B * T_STEPS / (ms / 1e3)

    # roofline of the dominant kernel (live, inside the timed region)
    hbm, tfl, src = peaks()
    bytes_, flops = RF.cost(dom["kernel"], dom["params"], exe.loop_info.get(dom["rec"]))
    n_inst = max(1, len(kev) // 2)
    if dom_ms:
        kms = sum(dom_ms) / len(dom_ms) / n_inst   # per launch, live in the timed graph
    else:
        kms = dom["ms"] / max(1, dom["count"])     # per launch, from the profiled step
    if flops and RF.FAMILY[dom["kernel"]] in ("gemm", "gemm_tc", "loop"):
        ach = flops / (kms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": tfl, "unit": "TFLOP/s",
                "frac": ach / tfl, "traffic": None}
    else:
        ach = bytes_ / (kms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": None}
    roof["traffic"] = ncu_traffic(RF.FAMILY[dom["kernel"]])
    if roof["unit"] == "TFLOP/s":
        # the acting loop runs FP32 FMAs on the SIMT pipe: its own ceiling
        roof["fp32_simt_peak"] = FP32_SIMT_TFLOPS
        roof["fp32_simt_frac"] = ach / FP32_SIMT_TFLOPS
    roof.update({"kernel": RF.FAMILY[dom["kernel"]], "node": dom["label"][1],
                 "ms_per_launch": kms, "launches_per_step": dom["count"],
                 "share_of_step": dom["ms"] / max(1e-9, sum(r["ms"] for r in prof)),
                 "peak_source": src})
    # whole-step roofline: sum over launches of max(bytes / HBM,
    # flops / compute ceiling) against the measured step time
    floor = sum(RF.floor_ms(r["kernel"], r["params"], exe.loop_info.get(r["rec"]), hbm, tfl,
                            FP32_SIMT_TFLOPS) * max(1, r["count"]) for r in prof)
    whole = {"floor_ms_per_step": round(floor, 4), "measured_ms_per_step": round(ms, 4),
             "frac": floor / ms if ms > 0 else None,
             "ceilings": {"hbm_gbs": hbm, "tensor_3xtf32_tflops": tfl / 6.0,
                          "fp32_simt_tflops": FP32_SIMT_TFLOPS}}
    top = []
    for r in rows[:8]:
        b_, f_ = RF.cost(r["kernel"], r["params"], exe.loop_info.get(r["rec"]))
        per = r["ms"] / max(1, r["count"])
        top.append({"kernel": RF.FAMILY.get(r["kernel"]), "node": r["label"][1],
                    "ms_step": round(r["ms"], 3), "launches": r["count"],
                    "gbs": round(b_ / (per / 1e3) / 1e9, 1) if per > 0 else None,
                    "tflops": round(f_ / (per / 1e3) / 1e12, 2) if f_ and per > 0 else None})

    # e2e through the public API with host buffers
    hin = host
    for w in range(max(1, args.warmup)):
        outs = execute(g, bounds=bounds, inputs=hin, seed=0, shard=shard, comm=comm,
                       block=WL.block, swap=WL.swap)
        hin = next_inputs(outs, params)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for s in range(args.steps):
        outs = execute(g, bounds=bounds, inputs=hin, seed=0, shard=shard, comm=comm,
                       block=WL.block, swap=WL.swap)
        hin = next_inputs(outs, params)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    h2d = sum(v.nbytes for v in host.values())
    d2h = sum(np.asarray(v).nbytes for v in outs.values())
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = world * B * T_STEPS / (e2e_ms / 1e3)

    line = {"metric": "env-steps/s per train iter", "value": value, "unit": "env-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": WL.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": WL.name, "desc": WL.desc, "E_per_gpu": B,
                       "E_total": B * world, "T": T_STEPS, "bounds": bounds,
                       "time_block": WL.block,
                       "hidden": [256, 256], "obs": 16, "act": 4, "iters_per_step": 1,
                       "l2": "activations (GBs) exceed L2 every step",
                       "parallelism": f"env-shard x{world}"},
            "e2e": {"value": e2e, "unit": "env-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
            "gpu_launches": exe.launch_count * args.steps,
            "in_graph_collectives_per_step": 0 if exe.colls is None else len(exe.colls),
            "host_hooks_per_step": len(exe.hooks),
            "peak_hbm_bytes": exe.peak_bytes,
            "peak_hbm_allocated_bytes": int(torch.cuda.max_memory_allocated()),
            "swap": None if exe.swap_rt is None else {
                "managed": [exe.g.nodes[k[0]].name for k in exe.swap_plan.keys],
                "pinned_host_bytes": exe.swap_rt.host_bytes,
                "offload_bytes_per_step": exe.swap_rt.host_bytes,
                "fetch_bytes_per_step": exe.swap_rt.host_bytes,
                "time_block": exe.swap_plan.bs},
            "naive_hbm_bytes": exe.naive_bytes,
            "roofline": roof,
            "roofline_step": whole,
            "breakdown": {"family_ms_per_step": {k: round(v, 3) for k, v in fam_ms.items()},
                          "top": top},
            "clocks": clk}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
