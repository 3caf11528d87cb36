"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration.

Configs 2-4: the library's per-vertex (Eq. (1)), per-edge
(Eq. (2)) and total counts are compared with the exact oracle
outputs over EVERY element: each output array's SHA-256 must equal the cached
hash of the sharded CPU oracle's array (tests/golden/fullsize_oracle.json,
written by tools/oracle_cache.py, which calls only oracle/; the plain
definition), and for configs 2 and 4 the oracle also runs
live on the box's host cores and the arrays are compared element by element
(config 3's oracle takes about 2,000 CPU-seconds; BF_FULL_LIVE=1 adds it).  The
generator is pinned by the cached SHA-256 of the edge list.

Config 5 (300M edges, about 7.7e13 oracle steps -- days of single-core CPU)
is checked on a stratified sample of exact oracle values
(tests/golden/c5_sample.json, tools/oracle_cache.py --c5-sample: vertices and
edges from every degree stratum on both sides, including the highest-degree
vertices the oracle can afford) plus properties that hold at any size:
sum_U b = sum_V b = 2T, sum_E b = 4T and, for EVERY vertex z, the sum of b(e)
over z's edges = 2 b(z) (each butterfly through z uses two of z's edges).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import bfgen
import oracle

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
# configs whose oracle also runs live in the test (c3's needs about 2,000
# CPU-seconds; its arrays are checked by the cached hashes unless BF_FULL_LIVE=1)
LIVE = {2, 4} | ({3} if os.environ.get("BF_FULL_LIVE") == "1" else set())


def _cache():
    return json.load(open(os.path.join(GOLDEN, "fullsize_oracle.json")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u8", copy=False).tobytes()).hexdigest()


def _edges_sha(e):
    return hashlib.sha256(np.ascontiguousarray(e).astype("<u4", copy=False).tobytes()).hexdigest()


def _counts(g, rank):
    from paper_1907_08607_b200 import bf
    with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank) as bg:  # bench's defaults (orient auto)
        bu, bv, t = bg.vertex()
        be, t2 = bg.edge()
        t3 = bg.total()
    assert t == t2 == t3
    return bu, bv, be, t


def _segment_sum(idx, vals, n):
    """Exact u64 sum of vals per index (mod 2^64): bincount over 16-bit pieces,
    each partial sum < 2^53 so float64 holds it exactly."""
    out = np.zeros(n, np.uint64)
    v = vals.astype(np.uint64)
    for q in range(4):
        piece = ((v >> np.uint64(16 * q)) & np.uint64(0xFFFF)).astype(np.float64)
        part = np.bincount(idx, weights=piece, minlength=n)
        out += part.astype(np.uint64) << np.uint64(16 * q)
    return out


def _first_diff(a, b):
    d = np.flatnonzero(a != b)
    return f"{len(d)} differ, first {int(d[0])}: got {int(a[d[0]])} want {int(b[d[0]])}" if len(d) else ""


@pytest.mark.parametrize("k", [2, 3, 4])
def test_fullsize_exact(k):
    """north_star: per-vertex and per-edge counts bit-exact with the CPU oracle."""
    c = _cache()[str(k)]
    g = bfgen.config_graph(k)
    assert (g.n_u, g.n_v, g.m) == (c["n_u"], c["n_v"], c["m"])
    assert _edges_sha(g.edges) == c["edges_sha256"], "generator drifted from the cached oracle run"
    rank = bfgen.CONFIGS[k]["ranking"][0]
    bu, bv, be, T = _counts(g, rank)
    assert T == c["total"]
    live = k in LIVE
    if live:  # element by element against the oracle run here, on the host cores
        with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
            ref = og.count_sharded()
        assert ref["total"] == c["total"]
    for name, got in (("b_u", bu), ("b_v", bv), ("b_e", be)):
        if live:
            assert np.array_equal(got, ref[name]), f"c{k} {name}: " + _first_diff(got, ref[name])
            assert _sha(ref[name]) == c[name + "_sha256"], f"live oracle disagrees with the cached hash ({name})"
        # the whole array's SHA-256 against the cached oracle output: equal hashes = equal arrays
        assert _sha(got) == c[name + "_sha256"], f"c{k} {name} differs from the cached oracle output"


def test_fullsize_c5_sample():
    """Config 5: stratified sample of exact oracle values + invariants at full size."""
    path = os.path.join(GOLDEN, "c5_sample.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c5_sample.json not generated yet (tools/oracle_cache.py --c5-sample)")
    smp = json.load(open(path))
    g = bfgen.config_graph(5)
    assert _edges_sha(g.edges) == smp["edges_sha256"]
    bu, bv, be, T = _counts(g, bfgen.CONFIGS[5]["ranking"][0])
    U = g.edges[:, 0].astype(np.int64)
    V = g.edges[:, 1].astype(np.int64)
    su = int(bu.sum(dtype=np.uint64))
    sv = int(bv.sum(dtype=np.uint64))
    se = int(be.sum(dtype=np.uint64))
    assert T < 2**62  # the wrap-around checks below are exact
    assert su == sv == 2 * T and se == 4 * T
    assert np.array_equal(_segment_sum(U, be, g.n_u), 2 * bu)
    assert np.array_equal(_segment_sum(V, be, g.n_v), 2 * bv)
    for side, x, val in smp["vertices"]:
        assert int((bu, bv)[side][x]) == val, (side, x)
    for e, val in smp["edges"]:
        assert int(be[e]) == val, e
