"""Generate the golden parity fixtures from the REAL reference.

Runs only in the build container (imports /root/reference/pkg/src).  For
each case it builds the reference dependence graph (optionally transformed
by the reference's own passes), serialises it with
`paper_2501_05408_b200.ir.from_pdg(...).to_json()`, runs the reference
oracle `recten.runtime.reference_execute`, and writes

    tests/golden/cases/<case>.json   graph + bounds + seed + meta
    tests/golden/cases/<case>.npz    inputs (in_*) and reference outputs (out_*)

Cases the reference itself cannot evaluate (eager-fold hazard on
transformed graphs) are recorded with their error text, not skipped
silently.  Also writes the benchmark graphs under tests/golden/graphs/.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import programs as P  # noqa: E402
from paper_2501_05408_b200 import ir  # noqa: E402

CASES = os.path.join(HERE, "cases")
GRAPHS = os.path.join(HERE, "graphs")


def variants():
    dsl, fe, pdg, tr, rt, ps = P.recten()

    def plain(g):
        return g

    def vec(g):
        tr.vectorize_all(g)
        return g

    def vec_fuse(g):
        tr.vectorize_all(g)
        tr.fuse(g)
        return g

    def lift(g):
        tr.lift_incremental_patterns(g)
        return g

    return {"plain": plain, "vec": vec, "vecfuse": vec_fuse, "lift": lift}


def bind(g, bounds):
    for d, b in g.dim_bound.items():
        if bounds and b.name in bounds:
            g.bindings[b] = bounds[b.name]


class alt_accumulation:
    """Context: the reference's reduction kernels (matmul, sum, discounted
    sums, windows, cumsums) accumulate in float64 and round once.  An
    equally valid fp32 evaluation of the same program; its distance to the
    reference's own result is the fp32 rounding noise each output carries
    (the band a different-but-correct fp32 implementation lands in)."""

    KINDS = ("matmul", "sum", "discounted_sum", "window_reduce", "cumsum", "discounted_cumsum")

    def __enter__(self):
        dsl, fe, pdg, tr, rt, ps = P.recten()
        self.rt, self.saved = rt, dict(rt.KERNELS)

        def up(fn):
            def k(node, vals, env, rng):
                v = [x.astype(np.float64) if isinstance(x, np.ndarray) and x.dtype == np.float32
                     else x for x in vals]
                return fn(node, v, env, rng)
            return k
        for kind in self.KINDS:
            rt.KERNELS[kind] = up(self.saved[kind])
        return self

    def __exit__(self, *exc):
        self.rt.KERNELS.clear()
        self.rt.KERNELS.update(self.saved)


def write_case(name, g, bounds, inputs, seed, meta, alt=False):
    dsl, fe, pdg, tr, rt, ps = P.recten()
    doc = {"name": name, "bounds": bounds, "seed": seed, "meta": meta}
    arrays = {}
    for k, v in (inputs or {}).items():
        arrays[f"in_{k}"] = np.asarray(v)
    doc["inputs"] = sorted((inputs or {}).keys())
    t0 = time.time()
    try:
        outs, rb = rt.reference_execute(g, bounds=bounds, inputs=inputs, seed=seed,
                                        return_bounds=True)
        doc["error"] = None
        doc["resolved_bounds"] = rb
        for k, v in outs.items():
            arrays[f"out_{k}"] = v
        doc["outputs"] = sorted(outs.keys())
    except Exception as exc:  # the reference's own failure is the fixture
        doc["error"] = f"{type(exc).__name__}: {exc}"
        doc["outputs"] = []
    doc["ref_seconds"] = round(time.time() - t0, 4)
    if alt and doc["error"] is None:
        with alt_accumulation():
            outs2 = rt.reference_execute(g, bounds=bounds, inputs=inputs, seed=seed)
        for k, v in outs2.items():
            arrays[f"alt_{k}"] = v
        doc["alt_outputs"] = sorted(outs2.keys())
    doc["graph"] = json.loads(ir.from_pdg(g).to_json())
    with open(os.path.join(CASES, f"{name}.json"), "w") as fh:
        json.dump(doc, fh)
    np.savez_compressed(os.path.join(CASES, f"{name}.npz"), **arrays)
    print(f"{name:40s} {'ERR ' + doc['error'][:60] if doc['error'] else 'ok'} "
          f"{doc['ref_seconds']}s")


def ppo_inputs(d_o, H, d_a, dtype, seed=1234):
    """PPO trunk + heads ~ N(0, 1/fan_in) from default_rng(seed), biases zero."""
    sys.path.insert(0, ROOT)
    from paper_2501_05408_b200.workloads import ppo_inputs as mk
    return mk(d_o=d_o, H=H, d_a=d_a, dtype=dtype, seed=seed)


def ppo_cases():
    dsl, fe, pdg, tr, rt, ps = P.recten()
    # (I, B, T, epochs, minibatches)
    for dt, (I, B, T, ep, mb) in (("f64", (2, 4, 5, 2, 2)), ("f32", (2, 4, 5, 2, 2)),
                                  ("f32", (1, 8, 6, 2, 4)), ("f64", (1, 6, 7, 3, 2))):
        ctx = P.ctx_ppo_mlp(B=B, T=T, I=I, epochs=ep, minibatches=mb, d_o=4, H=8, d_a=2,
                            dtype=dt, lr=0.002)
        g = pdg.build(ctx)
        pdg.eliminate_dead(g)
        inputs = ppo_inputs(4, 8, 2, dt)
        write_case(f"ppo_{dt}_I{I}B{B}T{T}E{ep}M{mb}", g, None, inputs, 0,
                   {"program": "ppo_mlp", "dtype": dt})
    # benchmark graphs: C3 (E=4096 x T=512) and the per-GPU shard of C5
    for name, B in (("ppo_c3", 4096),):
        ctx = P.ctx_ppo_mlp(B=B)
        g = pdg.build(ctx)
        pdg.eliminate_dead(g)
        with open(os.path.join(GRAPHS, f"{name}.json"), "w") as fh:
            fh.write(ir.from_pdg(g).to_json())
        print(f"wrote graphs/{name}.json")


def kernel_graphs():
    """Single-kernel programs for bench_kernels.py (HBM-roofline checks of
    the scan and gather kernels at full HBM scale) + small oracle cases."""
    dsl, fe, pdg, tr, rt, ps = P.recten()
    import numpy as np
    for name in P.KERNEL_NAMES:
        g = pdg.build(P.ctx_kernel(name))
        with open(os.path.join(GRAPHS, f"{name}.json"), "w") as fh:
            fh.write(ir.from_pdg(g).to_json())
        rng = np.random.default_rng(7)
        inputs = {}
        for n in g.sorted_nodes():
            if n.kind == "input":
                dom = tuple(g.bindings[g.dim_bound[d]] for d in n.domain)
                inputs[n.name] = rng.standard_normal(dom + tuple(n.out_shapes[0])).astype(
                    np.float32)
        write_case(name, g, None, inputs, 0, {"program": name})


def edge_cases():
    """Degenerate extents the executor must get right: a single env or step,
    no envs at all (empty slabs, sums of nothing), a one-epoch PPO with one
    env per minibatch, a one-step PPO horizon."""
    dsl, fe, pdg, tr, rt, ps = P.recten()
    for (I, B, T) in ((1, 1, 1), (2, 1, 3), (1, 3, 1), (1, 0, 3)):
        ctx = P.ctx_reinforce_mlp(B=max(B, 1), T=T, I=I, d_o=4, H=8, d_a=2, dtype="f32", lr=0.05)
        g = pdg.build(ctx)
        pdg.eliminate_dead(g)
        write_case(f"edge_mlp_I{I}B{B}T{T}", g, {"I": I, "B": B, "T": T},
                   P.mlp_inputs(d_o=4, H=8, d_a=2, dtype="f32"), 0,
                   {"program": "reinforce_mlp", "edge": True})
    for (B, T, ep, mb) in ((2, 4, 1, 2), (4, 1, 2, 2)):
        ctx = P.ctx_ppo_mlp(B=B, T=T, I=1, epochs=ep, minibatches=mb, d_o=4, H=8, d_a=2,
                            dtype="f32", lr=0.002)
        g = pdg.build(ctx)
        pdg.eliminate_dead(g)
        write_case(f"edge_ppo_B{B}T{T}E{ep}M{mb}", g, None, ppo_inputs(4, 8, 2, "f32"), 0,
                   {"program": "ppo_mlp", "edge": True})


# Full-width benchmark programs (obs 16, H=256 x 2, act 4 [+ value head]) at
# sizes where the executor picks the kernels the benchmark runs: the JIT
# acting loop (forced on by the test), tcgen05 TMA GEMMs with the bias+tanh
# epilogue, the thin row/small-K/gate kernels and split-K.  (name, kind,
# dtype, I, B, T, epochs, minibatches)
FULLWIDTH = (
    ("fw_mlp_f32_I2B1024T8", "mlp", "f32", 2, 1024, 8, 0, 0),
    ("fw_mlp_f32_I2B8T32", "mlp", "f32", 2, 8, 32, 0, 0),
    ("fw_mlp_f64_I2B8T16", "mlp", "f64", 2, 8, 16, 0, 0),
    ("fw_ppo_f32_I1B1024T8E2M2", "ppo", "f32", 1, 1024, 8, 2, 2),
    ("fw_ppo_f64_I1B16T8E2M2", "ppo", "f64", 1, 16, 8, 2, 2),
)


def fullwidth_case(spec):
    dsl, fe, pdg, tr, rt, ps = P.recten()
    name, kind, dt, I, B, T, ep, mb = spec
    if kind == "mlp":
        ctx = P.ctx_reinforce_mlp(B=B, T=T, I=I, dtype=dt)
        inputs = P.mlp_inputs(dtype=dt)
    else:
        ctx = P.ctx_ppo_mlp(B=B, T=T, I=I, epochs=ep, minibatches=mb, dtype=dt)
        inputs = ppo_inputs(16, 256, 4, dt)
    g = pdg.build(ctx)
    pdg.eliminate_dead(g)
    write_case(name, g, None, inputs, 0,
               {"program": "reinforce_mlp" if kind == "mlp" else "ppo_mlp", "dtype": dt,
                "fullwidth": True}, alt=dt == "f32")


def teacher_forced_case(src="fw_mlp_f32_I2B1024T8", name="fw_mlp_f32_I1B1024T8_tf"):
    """Iteration 2 of `src` in isolation: one iteration (I=1) started from the
    REFERENCE's own updated weights W*_next[0].  A chained run's second
    rollout amplifies 1e-6-level weight differences (fp32 rounding of the
    gradient sums) by up to ~100x; this pins every iteration at the strict
    tolerance instead."""
    dsl, fe, pdg, tr, rt, ps = P.recten()
    sys.path.insert(0, os.path.dirname(HERE))
    from golden_cases import load_case
    c = load_case(src)
    inputs = {f"{k}_0": c.outputs[f"{k}_next"][0] for k in ("W1", "b1", "W2", "b2", "W3", "b3")}
    ctx = P.ctx_reinforce_mlp(B=1024, T=8, I=1, dtype="f32")
    g = pdg.build(ctx)
    pdg.eliminate_dead(g)
    write_case(name, g, None, inputs, 0,
               {"program": "reinforce_mlp", "dtype": "f32", "fullwidth": True,
                "teacher_forced_from": src}, alt=True)


def fullwidth_cases():
    from multiprocessing import Pool
    with Pool(len(FULLWIDTH)) as pool:
        pool.map(fullwidth_case, FULLWIDTH)
    teacher_forced_case()


def opset_cases():
    """The remaining KERNELS kinds (div, log, sqrt, where, cast, reshape,
    squeeze, identity, eval_symbol, cumsum), the unit-gamma cumsum lift
    (reference test_transforms.py:223-237), Euclidean index KATs with
    negative operands and a zero divisor (symexpr.py:491-506)."""
    dsl, fe, pdg, tr, rt, ps = P.recten()
    V = variants()
    for dt in ("f64", "f32"):
        for vname in ("plain", "vec"):
            g = pdg.build(P.ctx_opset(dtype=dt))
            V[vname](g)
            write_case(f"ops_{dt}_{vname}", g, None, None, 3, {"program": "opset", "variant": vname})
    for vname in ("plain", "vec"):
        g = pdg.build(P.ctx_unit_cumsum())
        V[vname](g)
        write_case(f"tr_unit_cumsum_{vname}", g, None, None, 1,
                   {"program": "unit_cumsum", "variant": vname})
    x = np.arange(9.0) * 1.5 - 2.0
    g = pdg.build(P.ctx_euclid())
    write_case("kat_euclid", g, None, {"x": x}, 0, {"program": "euclid"})
    g = pdg.build(P.ctx_divzero())
    write_case("kat_divzero", g, None, {"x": np.arange(5.0)}, 0, {"program": "divzero"})


def main():
    dsl, fe, pdg, tr, rt, ps = P.recten()
    os.makedirs(CASES, exist_ok=True)
    os.makedirs(GRAPHS, exist_ok=True)
    if "--only" in sys.argv:
        what = sys.argv[sys.argv.index("--only") + 1]
        return {"ppo": ppo_cases, "kernels": kernel_graphs, "edge": edge_cases,
                "fullwidth": fullwidth_cases, "opset": opset_cases}[what]()
    ppo_cases()
    opset_cases()
    V = variants()

    # corpus x variants x seeds (reference pkg/tests/test_dsl.py:240-248)
    for name, (bounds, inp) in sorted(P.CORPUS_BINDS.items()):
        inputs = {k: P.make_input(v) for k, v in (inp or {}).items()}
        for vname, fn in V.items():
            for seed in (3, 0):
                g = pdg.build(dsl.load_text(P.corpus_text(name)))
                bind(g, bounds)  # transforms read static bindings
                fn(g)
                write_case(f"corpus_{name}_{vname}_s{seed}", g, bounds, inputs, seed,
                           {"program": name, "variant": vname})
    # wider reinforce (more points through the per-point executor)
    for (I, B, T) in ((2, 8, 16), (3, 4, 32)):
        g = pdg.build(dsl.load_text(P.corpus_text("reinforce")))
        write_case(f"reinforce_I{I}B{B}T{T}", g, {"I": I, "B": B, "T": T},
                   {"winit": 0.1}, 3, {"program": "reinforce"})

    # KAT programs (reference pkg/tests/test_dsl.py:106-188) and appendices
    for name, (text, bounds, inp) in P.KAT_TEXTS.items():
        inputs = {k: P.make_input(v) for k, v in (inp or {}).items()}
        for vname in ("plain", "vec"):
            g = pdg.build(dsl.load_text(text))
            V[vname](g)
            write_case(f"{name}_{vname}", g, bounds, inputs, 0,
                       {"program": name, "variant": vname})

    # transform-test programs (reference pkg/tests/test_transforms.py)
    for name, mk in (("gated", P.ctx_gated), ("reverse_scan", P.ctx_reverse_scan)):
        for vname in ("plain", "lift", "vec"):
            g = pdg.build(mk())
            V[vname](g)
            write_case(f"tr_{name}_{vname}", g, None, None, 5,
                       {"program": name, "variant": vname})
    for bs in (10, 7):
        g = pdg.build(P.ctx_widesum())
        (tgt,) = [n for n in g.sorted_nodes()
                  if n.kind == "sum" and n.params["dims"] == (0,)
                  and g.nodes[g.in_edges(n.id)[0].src].kind == "mul"]
        tr.incrementalize(g, tgt, bs=bs)
        write_case(f"tr_widesum_inc{bs}", g, None, None, 7,
                   {"program": "widesum", "variant": f"incrementalize bs={bs}"})
    g = pdg.build(P.ctx_widesum())
    write_case("tr_widesum_plain", g, None, None, 7, {"program": "widesum"})

    # the benchmark program at parity scale, f32 and f64
    for dt in ("f32", "f64"):
        for I, B, T in ((1, 4, 6), (2, 3, 5)):
            ctx = P.ctx_reinforce_mlp(B=B, T=T, I=I, d_o=4, H=8, d_a=2, dtype=dt,
                                      lr=0.05)
            g = pdg.build(ctx)
            pdg.eliminate_dead(g)
            inputs = P.mlp_inputs(d_o=4, H=8, d_a=2, dtype=dt, seed=1234)
            write_case(f"mlp_{dt}_I{I}B{B}T{T}", g, None, inputs, 0,
                       {"program": "reinforce_mlp", "dtype": dt})

    # benchmark graphs (too large for the oracle; structure only)
    ctx = P.ctx_reinforce_mlp()
    g = pdg.build(ctx)
    pdg.eliminate_dead(g)
    with open(os.path.join(GRAPHS, "reinforce_mlp_c2.json"), "w") as fh:
        fh.write(ir.from_pdg(g).to_json())
    print("wrote graphs/reinforce_mlp_c2.json")


if __name__ == "__main__":
    main()
