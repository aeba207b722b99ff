"""Executor-side mirror of the reference's polyhedral dependence graph.

The B200 backend consumes the graph the reference front end produces
(`recten.pdg.Pdg`, reference `pkg/src/recten/pdg.py:88-158`) after any of
the reference transforms.  It never imports the reference: `from_pdg`
reads a live `Pdg` by duck typing, and `Graph.to_json`/`from_json` carry the
same information as a self-contained document, so a graph built in one
process (with the reference front end) can be executed in another (on a
GPU box without it).

Index expressions mirror `recten.symexpr.SymExpr` (reference
`pkg/src/recten/symexpr.py:102-265`) as nested tuples:

    ("int", v) ("bool", v) ("sym", name, kind)
    (op, a, b)            op in add sub mul floordiv mod eq le lt ge gt and or
    ("neg", a) ("not", a) ("min", *args) ("max", *args)
    ("slice", lo, hi)     half-open
    ("tuple", *components)

Tuples compare and hash structurally, which is what the reference gets from
hash-consing.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

LOOP = "loop"
BOUND = "bound"

DTYPES = {"f64": np.float64, "f32": np.float32, "i64": np.int64, "bool": np.bool_}
ITEMSIZE = {"f64": 8, "f32": 4, "i64": 8, "bool": 1}


class IRError(Exception):
    pass


# ---------------------------------------------------------------------------
# expressions


def cint(v: int):
    return ("int", int(v))


def csym(name: str, kind: str = LOOP):
    return ("sym", name, kind)


TRUE = ("bool", True)
FALSE = ("bool", False)


def components(e) -> tuple:
    """Reference `symexpr.components` (`pkg/src/recten/symexpr.py:263-265`)."""
    return tuple(e[1:]) if e[0] == "tuple" else (e,)


def free_syms(e) -> set:
    if e[0] == "sym":
        return {(e[1], e[2])}
    if e[0] in ("int", "bool"):
        return set()
    out = set()
    for a in e[1:]:
        out |= free_syms(a)
    return out


def expr_text(e) -> str:
    k = e[0]
    if k in ("int", "bool"):
        return str(e[1])
    if k == "sym":
        return e[1]
    if k == "slice":
        return f"{expr_text(e[1])}:{expr_text(e[2])}"
    if k == "tuple":
        return "[" + ", ".join(expr_text(a) for a in e[1:]) + "]"
    if k in ("neg", "not"):
        return f"{'-' if k == 'neg' else 'not '}({expr_text(e[1])})"
    if k in ("min", "max"):
        return f"{k}(" + ", ".join(expr_text(a) for a in e[1:]) + ")"
    ops = {"add": "+", "sub": "-", "mul": "*", "floordiv": "//", "mod": "%",
           "eq": "==", "le": "<=", "lt": "<", "ge": ">=", "gt": ">",
           "and": " and ", "or": " or "}
    return f"({expr_text(e[1])}{ops[k]}{expr_text(e[2])})"


def substitute(e, mapping: dict):
    """Replace ("sym", name, kind) leaves found in mapping[(name, kind)]."""
    k = e[0]
    if k == "sym":
        return mapping.get((e[1], e[2]), e)
    if k in ("int", "bool"):
        return e
    return (k,) + tuple(substitute(a, mapping) for a in e[1:])


def as_affine(e):
    """(coeffs {(name, kind): int}, const) when e is integer-affine, else None."""
    k = e[0]
    if k == "int":
        return {}, e[1]
    if k == "sym":
        return {(e[1], e[2]): 1}, 0
    if k == "neg":
        a = as_affine(e[1])
        if a is None:
            return None
        return {s: -c for s, c in a[0].items()}, -a[1]
    if k in ("add", "sub"):
        a, b = as_affine(e[1]), as_affine(e[2])
        if a is None or b is None:
            return None
        sg = 1 if k == "add" else -1
        co = dict(a[0])
        for s, c in b[0].items():
            co[s] = co.get(s, 0) + sg * c
        return {s: c for s, c in co.items() if c}, a[1] + sg * b[1]
    if k == "mul":
        a, b = as_affine(e[1]), as_affine(e[2])
        if a is None or b is None:
            return None
        if not a[0]:
            a, b = b, a
        if b[0]:
            return None  # product of two symbolic terms
        return {s: c * b[1] for s, c in a[0].items() if c * b[1]}, a[1] * b[1]
    return None


# ---------------------------------------------------------------------------
# graph


@dataclass(frozen=True)
class SymRef:
    """A Symbol held in node params (scan/index_select/... `dim`, `bound`)."""
    name: str
    kind: str = LOOP


@dataclass(frozen=True)
class UdfRef:
    """UDF spec without its Python body.  `synthetic` marks bodies made by
    the reference's `dsl.make_udf_fn` (`pkg/src/recten/dsl.py:288-307`),
    whose semantics the device environment kernel reproduces."""
    name: str
    out_shapes: tuple
    out_dtypes: tuple
    synthetic: bool = True


@dataclass(frozen=True)
class InnerOp:
    name: str
    kind: str
    params: dict
    inputs: tuple


@dataclass(frozen=True)
class InnerGraph:
    ops: tuple
    out: int


@dataclass
class Node:
    id: int
    name: str
    kind: str
    domain: tuple          # dim names, canonical order
    out_shapes: tuple      # tuple of tuples of int | expr
    out_dtypes: tuple
    params: dict = field(default_factory=dict)
    nin: int = 0

    @property
    def shape(self):
        return self.out_shapes[0]

    @property
    def dtype(self):
        return self.out_dtypes[0]

    def __repr__(self):
        return f"<n{self.id} {self.name}:{self.kind} ({','.join(self.domain)})>"


@dataclass
class Edge:
    sink: int
    iid: int
    phi: tuple             # components, one per source-domain dim
    psi: object            # expr | None
    oid: int
    src: int


class Graph:
    def __init__(self, dim_order, dim_bound, bindings):
        self.dim_order = tuple(dim_order)
        self.dim_bound = dict(dim_bound)     # dim name -> bound name
        self.bindings = dict(bindings)       # bound name -> int | "dyn"
        self.nodes: dict[int, Node] = {}
        self.edges: list[Edge] = []
        self.outputs: list[tuple[str, int, int]] = []
        self._in: dict | None = None

    # -- queries (reference `Pdg.in_edges`/`out_edges`, pdg.py:110-114) -------

    def _index(self):
        if self._in is None:
            self._in, self._out = {}, {}
            for e in self.edges:
                self._in.setdefault(e.sink, []).append(e)
                self._out.setdefault(e.src, []).append(e)
            for v in self._in.values():
                v.sort(key=lambda e: e.iid)

    def invalidate(self):
        self._in = None

    def in_edges(self, nid) -> list[Edge]:
        self._index()
        return self._in.get(nid, [])

    def out_edges(self, nid) -> list[Edge]:
        self._index()
        return self._out.get(nid, [])

    def sorted_nodes(self) -> list[Node]:
        return [self.nodes[k] for k in sorted(self.nodes)]

    def bound_of(self, dim: str) -> str:
        return self.dim_bound[dim]

    # -- JSON ---------------------------------------------------------------

    def to_json(self) -> str:
        doc = {
            "format": "rtb200-pdg/1",
            "dim_order": list(self.dim_order),
            "dim_bound": self.dim_bound,
            "bindings": self.bindings,
            "nodes": [
                {"id": n.id, "name": n.name, "kind": n.kind, "domain": list(n.domain),
                 "out_shapes": [[_enc(s) for s in shp] for shp in n.out_shapes],
                 "out_dtypes": list(n.out_dtypes),
                 "params": {k: _enc(v) for k, v in n.params.items()},
                 "nin": n.nin}
                for n in self.sorted_nodes()],
            "edges": [
                {"sink": e.sink, "iid": e.iid, "phi": [_enc_expr(c) for c in e.phi],
                 "psi": None if e.psi is None else _enc_expr(e.psi),
                 "oid": e.oid, "src": e.src} for e in self.edges],
            "outputs": [list(o) for o in self.outputs],
        }
        return json.dumps(doc)

    @staticmethod
    def from_json(text: str) -> "Graph":
        doc = json.loads(text)
        if doc.get("format") != "rtb200-pdg/1":
            raise IRError("not an rtb200 graph document")
        g = Graph(doc["dim_order"], doc["dim_bound"], doc["bindings"])
        for nd in doc["nodes"]:
            n = Node(nd["id"], nd["name"], nd["kind"], tuple(nd["domain"]),
                     tuple(tuple(_dec(s) for s in shp) for shp in nd["out_shapes"]),
                     tuple(nd["out_dtypes"]),
                     {k: _dec(v) for k, v in nd["params"].items()}, nd["nin"])
            g.nodes[n.id] = n
        for ed in doc["edges"]:
            g.edges.append(Edge(ed["sink"], ed["iid"],
                                tuple(_dec_expr(c) for c in ed["phi"]),
                                None if ed["psi"] is None else _dec_expr(ed["psi"]),
                                ed["oid"], ed["src"]))
        g.outputs = [tuple(o) for o in doc["outputs"]]
        return g


def _enc_expr(e):
    if e[0] in ("int", "bool"):
        return [e[0], e[1]]
    if e[0] == "sym":
        return ["sym", e[1], e[2]]
    return [e[0]] + [_enc_expr(a) for a in e[1:]]


def _dec_expr(v):
    if v[0] in ("int", "bool"):
        return (v[0], v[1])
    if v[0] == "sym":
        return ("sym", v[1], v[2])
    return (v[0],) + tuple(_dec_expr(a) for a in v[1:])


def _is_expr(v) -> bool:
    return isinstance(v, tuple) and v and isinstance(v[0], str) and v[0] in _EXPR_KINDS


_EXPR_KINDS = {"int", "bool", "sym", "add", "sub", "mul", "floordiv", "mod", "neg",
               "eq", "le", "lt", "ge", "gt", "and", "or", "not", "min", "max",
               "slice", "tuple"}


def _enc(v):
    if v is None or isinstance(v, (bool, str)):
        return v
    if isinstance(v, (int, np.integer)):
        return int(v)
    if isinstance(v, (float, np.floating)):
        return {"$f": float(v).hex()}
    if isinstance(v, SymRef):
        return {"$sym": [v.name, v.kind]}
    if isinstance(v, UdfRef):
        return {"$udf": {"name": v.name,
                         "out_shapes": [list(s) for s in v.out_shapes],
                         "out_dtypes": list(v.out_dtypes),
                         "synthetic": v.synthetic}}
    if isinstance(v, InnerGraph):
        return {"$graph": {"out": v.out, "ops": [
            {"name": o.name, "kind": o.kind,
             "params": {k: _enc(x) for k, x in o.params.items()},
             "inputs": [list(i) for i in o.inputs]} for o in v.ops]}}
    if isinstance(v, np.ndarray):
        arr = np.array(v, order="C", copy=True)
        return {"$arr": {"dtype": arr.dtype.str, "shape": list(arr.shape),
                         "hex": arr.tobytes().hex()}}
    if _is_expr(v):
        return {"$expr": _enc_expr(v)}
    if isinstance(v, (tuple, list)):
        return {"$tuple": [_enc(x) for x in v]}
    raise IRError(f"cannot encode param value {v!r}")


def _dec(v):
    if not isinstance(v, dict):
        return v
    (tag, body), = v.items()
    if tag == "$f":
        return float.fromhex(body)
    if tag == "$sym":
        return SymRef(body[0], body[1])
    if tag == "$udf":
        return UdfRef(body["name"], tuple(tuple(s) for s in body["out_shapes"]),
                      tuple(body["out_dtypes"]), body["synthetic"])
    if tag == "$graph":
        return InnerGraph(tuple(InnerOp(o["name"], o["kind"],
                                        {k: _dec(x) for k, x in o["params"].items()},
                                        tuple(tuple(i) for i in o["inputs"]))
                                for o in body["ops"]), body["out"])
    if tag == "$arr":
        arr = np.frombuffer(bytes.fromhex(body["hex"]), dtype=np.dtype(body["dtype"]))
        return arr.reshape(tuple(body["shape"])).copy()
    if tag == "$expr":
        return _dec_expr(body)
    if tag == "$tuple":
        return tuple(_dec(x) for x in body)
    raise IRError(f"unknown tag {tag}")


# ---------------------------------------------------------------------------
# adapter from a live reference Pdg (duck-typed; the reference is not imported)


def _conv_expr(e):
    k = e.kind
    if k in ("int", "bool"):
        return (k, e.value)
    if k == "sym":
        return ("sym", e.value.name, e.value.kind)
    return (k,) + tuple(_conv_expr(a) for a in e.args)


def _is_symexpr(v) -> bool:
    return hasattr(v, "kind") and hasattr(v, "args") and hasattr(v, "value") \
        and type(v).__name__ == "SymExpr"


def _is_symbol(v) -> bool:
    return type(v).__name__ == "Symbol" and hasattr(v, "name") and hasattr(v, "kind")


def _conv_param(v):
    if _is_symexpr(v):
        return _conv_expr(v)
    if _is_symbol(v):
        return SymRef(v.name, v.kind)
    if type(v).__name__ == "UdfSpec":
        fn = getattr(v, "fn", None)
        qn = getattr(fn, "__qualname__", "")
        return UdfRef(v.name, tuple(tuple(s) for s in v.out_shapes),
                      tuple(v.out_dtypes), synthetic=qn.startswith("make_udf_fn"))
    if type(v).__name__ == "InnerGraph":
        return InnerGraph(tuple(InnerOp(o.name, o.kind,
                                        {k: _conv_param(x) for k, x in o.params.items()},
                                        tuple(tuple(i) for i in o.inputs))
                                for o in v.ops), v.out)
    if isinstance(v, np.ndarray):
        return v.copy()
    if isinstance(v, np.generic):
        return v.item()
    if isinstance(v, (tuple, list)):
        return tuple(_conv_param(x) for x in v)
    return v


def from_pdg(p) -> Graph:
    """Mirror a reference `Pdg` (`pkg/src/recten/pdg.py:88-101`)."""
    g = Graph([d.name for d in p.dim_order],
              {d.name: b.name for d, b in p.dim_bound.items()},
              {b.name: v for b, v in p.bindings.items()})
    for nid in sorted(p.nodes):
        n = p.nodes[nid]
        shapes = tuple(tuple(s if isinstance(s, (int, np.integer)) else _conv_expr(s)
                             for s in shp) for shp in n.out_shapes)
        shapes = tuple(tuple(int(s) if isinstance(s, np.integer) else s for s in shp)
                       for shp in shapes)
        g.nodes[nid] = Node(n.id, n.name, n.kind, tuple(d.name for d in n.domain),
                            shapes, tuple(n.out_dtypes),
                            {k: _conv_param(v) for k, v in n.params.items()}, n.nin)
    for e in p.edges:
        comps = e.phi.args if e.phi.kind == "tuple" else (e.phi,)
        g.edges.append(Edge(e.sink, e.iid, tuple(_conv_expr(c) for c in comps),
                            None if e.psi is None else _conv_expr(e.psi), e.oid, e.src))
    g.outputs = [(nm, nid, oid) for nm, nid, oid in p.outputs]
    return g


def as_graph(g) -> Graph:
    if isinstance(g, Graph):
        return g
    if isinstance(g, str):
        return Graph.from_json(g)
    if hasattr(g, "nodes") and hasattr(g, "edges") and hasattr(g, "dim_bound"):
        return from_pdg(g)
    raise IRError(f"cannot interpret {type(g).__name__} as a dependence graph")
