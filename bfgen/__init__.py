"""bfgen -- seeded synthetic bipartite graphs (input generators only).

Shared by the oracle side (tests) and the product side (bench.py, GPU tests).
This module holds none of the butterfly-counting arithmetic; it only draws
edge lists.  The recipe is in DESIGN.md ("Input recipe") and bfgen.c's header;
it follows SURVEY.md 8(d).  Edges are returned as a C-contiguous
``uint32[m, 2]`` numpy array of (u, v) pairs with side-local ids.

The paper measures on KONECT graphs (Table table-graphs
P:2034-2051), which are not available; CONFIGS stand in for them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libbfgen.so")
# bumped whenever bfgen.c or a CONFIGS entry changes the graphs it draws (keys the
# cached full-size oracle hashes in tests/golden/fullsize_oracle.json)
GEN_VERSION = 1
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "bfgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.bfgen_uniform.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                      ctypes.c_uint64, u32p]
        lib.bfgen_uniform.restype = ctypes.c_int
        lib.bfgen_chung_lu.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_uint32,
                                       ctypes.c_uint32, ctypes.c_uint64, u32p, u32p, u32p]
        lib.bfgen_chung_lu.restype = ctypes.c_int
        lib.bfgen_geo_zipf.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_uint64, u32p]
        lib.bfgen_geo_zipf.restype = ctypes.c_int64
        lib.bfgen_splitmix64.argtypes = [ctypes.c_uint64]
        lib.bfgen_splitmix64.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


@dataclass
class Graph:
    n_u: int
    n_v: int
    edges: np.ndarray  # uint32 [m, 2]
    name: str = ""
    planted_u: np.ndarray | None = None
    planted_v: np.ndarray | None = None

    @property
    def m(self) -> int:
        return int(self.edges.shape[0])


def uniform(n_u: int, n_v: int, m: int, seed: int) -> Graph:
    """m distinct (u, v) pairs drawn uniformly (config 1 recipe)."""
    out = np.zeros((m, 2), dtype=np.uint32)
    rc = _load().bfgen_uniform(n_u, n_v, m, seed, _ptr(out))
    if rc != 0:
        raise ValueError(f"bfgen_uniform failed rc={rc}")
    return Graph(n_u, n_v, out, f"uniform({n_u},{n_v},{m},seed={seed})")


def chung_lu(n_u: int, n_v: int, m: int, gamma_u: float, gamma_v: float, seed: int,
             planted: tuple[int, int] = (0, 0)) -> Graph:
    """Chung-Lu power-law bipartite graph with m distinct edges, optional planted K_{a,b}."""
    out = np.zeros((m, 2), dtype=np.uint32)
    pa, pb = planted
    pu = np.zeros(max(pa, 1), dtype=np.uint32)
    pv = np.zeros(max(pb, 1), dtype=np.uint32)
    rc = _load().bfgen_chung_lu(n_u, n_v, m, gamma_u, gamma_v, pa, pb, seed, _ptr(out),
                                _ptr(pu), _ptr(pv))
    if rc != 0:
        raise ValueError(f"bfgen_chung_lu failed rc={rc}")
    g = Graph(n_u, n_v, out, f"chung_lu({n_u},{n_v},{m},{gamma_u},{gamma_v},seed={seed},planted={planted})")
    if pa:
        g.planted_u, g.planted_v = pu[:pa].copy(), pv[:pb].copy()
    return g


def geo_zipf(n_u: int, n_v: int, p: float, s: float, seed: int) -> Graph:
    """Users with Geometric(p) degrees x items with Zipf(s) popularity (config 4 recipe)."""
    lib = _load()
    m = lib.bfgen_geo_zipf(n_u, n_v, p, s, seed, None)
    if m < 0:
        raise ValueError("bfgen_geo_zipf failed")
    out = np.zeros((m, 2), dtype=np.uint32)
    m2 = lib.bfgen_geo_zipf(n_u, n_v, p, s, seed, _ptr(out))
    assert m2 == m
    return Graph(n_u, n_v, out, f"geo_zipf({n_u},{n_v},p={p},s={s},seed={seed})")


def splitmix64(x: int) -> int:
    return int(_load().bfgen_splitmix64(x))


# ---- BASELINE.json configs ----
CONFIGS = {
    1: dict(kind="uniform", n_u=2000, n_v=1500, m=20000, seed=1,
            ranking=("side", "degree"), modes=("total", "vertex")),
    2: dict(kind="chung_lu", n_u=1_000_000, n_v=200_000, m=10_000_000, gamma_u=2.1, gamma_v=2.1,
            seed=2, ranking=("degree",), modes=("vertex",)),
    3: dict(kind="chung_lu", n_u=3_000_000, n_v=3_000_000, m=100_000_000, gamma_u=2.0, gamma_v=2.5,
            seed=3, planted=(200, 300), ranking=("approx_degree",), modes=("total", "edge")),
    4: dict(kind="geo_zipf", n_u=20_000_000, n_v=30_000, p=1.0 / 7.0, s=1.2, seed=4,
            ranking=("degree",), modes=("vertex",)),
    5: dict(kind="chung_lu", n_u=8_000_000, n_v=3_000_000, m=300_000_000, gamma_u=1.9, gamma_v=1.9,
            seed=5, ranking=("degree",), modes=("total", "vertex", "edge")),
}


def config_graph(k: int, scale: float = 1.0) -> Graph:
    """Generate config k.  ``scale`` < 1 shrinks vertex and edge counts
    proportionally (same shape) for parity tests the oracle finishes."""
    c = CONFIGS[k]
    sc = lambda x: max(1, int(round(x * scale)))
    if c["kind"] == "uniform":
        g = uniform(sc(c["n_u"]), sc(c["n_v"]), sc(c["m"]), c["seed"])
    elif c["kind"] == "chung_lu":
        planted = c.get("planted", (0, 0))
        g = chung_lu(sc(c["n_u"]), sc(c["n_v"]), sc(c["m"]), c["gamma_u"], c["gamma_v"], c["seed"],
                     planted=planted)
    else:
        g = geo_zipf(sc(c["n_u"]), c["n_v"] if scale == 1.0 else sc(c["n_v"]), c["p"], c["s"], c["seed"])
    g.name = f"c{k}" + ("" if scale == 1.0 else f"@{scale:g}") + ":" + g.name
    return g


# ---- small structured fixtures (tests) ----
def complete(a: int, b: int) -> Graph:
    u, v = np.meshgrid(np.arange(a, dtype=np.uint32), np.arange(b, dtype=np.uint32), indexing="ij")
    return Graph(a, b, np.stack([u.ravel(), v.ravel()], 1).copy(), f"K({a},{b})")


def from_pairs(n_u: int, n_v: int, pairs) -> Graph:
    e = np.asarray(list(pairs), dtype=np.uint32).reshape(-1, 2)
    return Graph(n_u, n_v, np.ascontiguousarray(e), "pairs")


def disjoint_union(g1: Graph, g2: Graph) -> Graph:
    e2 = g2.edges.astype(np.uint64).copy()
    e2[:, 0] += g1.n_u
    e2[:, 1] += g1.n_v
    e = np.concatenate([g1.edges, e2.astype(np.uint32)], 0)
    return Graph(g1.n_u + g2.n_u, g1.n_v + g2.n_v, np.ascontiguousarray(e), f"{g1.name}+{g2.name}")


def permute_edges(g: Graph, seed: int) -> Graph:
    """Same graph, edges in a different (seeded) order."""
    keys = np.array([splitmix64((seed << 32) ^ i) for i in range(g.m)], dtype=np.uint64) \
        if g.m < 5000 else (np.arange(g.m, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
                             ^ np.uint64(seed))
    order = np.argsort(keys, kind="stable")
    return Graph(g.n_u, g.n_v, np.ascontiguousarray(g.edges[order]), g.name + f"/perm{seed}")
