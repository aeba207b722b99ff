"""Loader for the committed golden fixtures (tests/golden/cases)."""

import glob
import json
import os

import numpy as np

from paper_2501_05408_b200 import ir

CASES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cases")
GRAPHS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "graphs")


class Case:
    def __init__(self, path):
        with open(path) as fh:
            doc = json.load(fh)
        self.name = doc["name"]
        self.bounds = doc["bounds"]
        self.seed = doc["seed"]
        self.error = doc["error"]
        self.meta = doc["meta"]
        self.resolved_bounds = doc.get("resolved_bounds")
        self.graph_doc = doc["graph"]
        arrs = np.load(path[:-5] + ".npz")
        self.inputs = {k: arrs[f"in_{k}"] for k in doc["inputs"]}
        self.outputs = {k: arrs[f"out_{k}"] for k in doc["outputs"]}
        # fp32 cases: the same program with float64-accumulated reductions
        # (make_golden.alt_accumulation): the reference's own rounding noise
        self.alt_outputs = {k: arrs[f"alt_{k}"] for k in doc.get("alt_outputs", [])}

    def graph(self):
        return ir.Graph.from_json(json.dumps(self.graph_doc))

    def __repr__(self):
        return self.name


def all_cases():
    return [Case(p) for p in sorted(glob.glob(os.path.join(CASES, "*.json")))]


def case_ids():
    return [os.path.basename(p)[:-5] for p in sorted(glob.glob(os.path.join(CASES, "*.json")))]


def load_case(name):
    return Case(os.path.join(CASES, f"{name}.json"))


def load_graph(name):
    with open(os.path.join(GRAPHS, f"{name}.json")) as fh:
        return ir.Graph.from_json(fh.read())
