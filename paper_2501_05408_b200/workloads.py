"""Synthetic inputs for the benchmark workloads (no reference imports).

C2 (BASELINE.json configs[1]): REINFORCE, E=1024 envs x T=1000 steps, a
2-hidden-layer 256-wide tanh MLP policy, obs 16, action 4.
Weights ~ N(0, 1/fan_in) from default_rng(1234), biases zero.
"""
import numpy as np


def mlp_inputs(d_o=16, H=256, d_a=4, dtype="f32", seed=1234):
    rng = np.random.default_rng(seed)
    dt = np.float32 if dtype == "f32" else np.float64
    out = {}
    for k, (fi, fo) in {"W1": (d_o, H), "W2": (H, H), "W3": (H, d_a)}.items():
        out[f"{k}_0"] = (rng.standard_normal((fi, fo)) / np.sqrt(fi)).astype(dt)
    for k, n in {"b1": H, "b2": H, "b3": d_a}.items():
        out[f"{k}_0"] = np.zeros((1, n), dt)
    return out


PARAMS = ("W1", "b1", "W2", "b2", "W3", "b3")
PPO_PARAMS = ("W1", "b1", "W2", "b2", "W3", "b3", "Wv", "bv")


def ppo_inputs(d_o=16, H=256, d_a=4, dtype="f32", seed=1234):
    """C3/C5: shared tanh trunk (W1, W2), policy head W3 (d_a), value head
    Wv (1); weights ~ N(0, 1/fan_in) from default_rng(seed), biases zero."""
    rng = np.random.default_rng(seed)
    dt = np.float32 if dtype == "f32" else np.float64
    out = {}
    for k, (fi, fo) in {"W1": (d_o, H), "W2": (H, H), "W3": (H, d_a), "Wv": (H, 1)}.items():
        out[f"{k}_0"] = (rng.standard_normal((fi, fo)) / np.sqrt(fi)).astype(dt)
    for k, n in {"b1": H, "b2": H, "b3": d_a, "bv": 1}.items():
        out[f"{k}_0"] = np.zeros((1, n), dt)
    return out


def next_inputs(outs, params=PARAMS):
    """Feed a training step's updated weights into the next step."""
    return {f"{k}_0": outs[f"{k}_next"][-1] for k in params}
