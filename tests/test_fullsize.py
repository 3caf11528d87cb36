"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration.

The CPU oracle cannot count a 10^8-edge graph whole, so at full size the GPU
outputs are checked (a) on sampled outputs the oracle computes one by one --
Eq. (1) per vertex and Eq. (2) per edge -- for
random vertices, random edges and the highest-degree vertices the oracle can
afford, and (b) by properties that hold at any size: sum_U b = sum_V b = 2T,
sum_E b = 4T, and sum over the edges of z of b(e) = 2 b(z) for EVERY vertex z
(each butterfly through z uses exactly two of z's edges), plus the planted
K_{200,300} lower bounds of config 3.  Config 5 (300M edges; its
generator alone takes minutes on the host) runs when BF_FULL_C5=1.
"""
import os
from math import comb

import numpy as np
import pytest

import bfgen
import oracle

pytestmark = pytest.mark.gpu

CONFIGS = [2, 3, 4] + ([5] if os.environ.get("BF_FULL_C5") == "1" else [])
ORACLE_STEP_BUDGET = 2e8  # sum of deg over a sampled vertex's neighbours


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


@pytest.mark.parametrize("k", CONFIGS)
def test_fullsize_sampled(k):
    g = bfgen.config_graph(k)
    rank = bfgen.CONFIGS[k]["ranking"][0]
    bu, bv, be, T = _counts(g, rank)
    U = g.edges[:, 0].astype(np.int64)
    V = g.edges[:, 1].astype(np.int64)
    # invariants at full size (exact integer sums; u64 arrays summed as Python ints via object-free splits)
    su = int(bu.astype(np.uint64).sum(dtype=np.uint64))
    sv = int(bv.astype(np.uint64).sum(dtype=np.uint64))
    se = int(be.astype(np.uint64).sum(dtype=np.uint64))
    assert su == sv == (2 * T) % 2**64
    assert se == (4 * T) % 2**64
    assert T < 2**63  # the wrap-around checks above are exact
    # sum over the edges at z of b(e) = 2 b(z), every vertex
    assert np.array_equal(_segment_sum(U, be, g.n_u), 2 * bu)
    assert np.array_equal(_segment_sum(V, be, g.n_v), 2 * bv)

    # sampled outputs, one by one from the oracle
    rng = np.random.default_rng(100 + k)
    deg_u = np.bincount(U, minlength=g.n_u)
    deg_v = np.bincount(V, minlength=g.n_v)
    cost_u = np.bincount(U, weights=deg_v[V].astype(np.float64), minlength=g.n_u)  # sum_{v in N(u)} deg v
    cost_v = np.bincount(V, weights=deg_u[U].astype(np.float64), minlength=g.n_v)
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        for side, b, cost, deg in ((0, bu, cost_u, deg_u), (1, bv, cost_v, deg_v)):
            n_side = len(b)
            xs = list(rng.integers(0, n_side, 48))
            by_deg = np.argsort(-deg)  # the highest-degree vertices the oracle can afford
            hubs = [int(x) for x in by_deg[cost[by_deg] <= ORACLE_STEP_BUDGET][:8]]
            xs += hubs
            assert hubs, "no affordable hub sampled"
            for x in xs:
                assert og.vertex(side, int(x)) == int(b[x]), (k, side, int(x))
        for e in rng.integers(0, g.m, 48):
            if cost_u[U[e]] <= ORACLE_STEP_BUDGET:
                assert og.edge(int(e)) == int(be[e]), (k, int(e))
    if k == 3:  # planted K_{200,300}: lower bounds
        assert T >= comb(200, 2) * comb(300, 2)
        assert (bu >= 0).all()
        top_u = np.sort(bu)[-200:]
        assert int(top_u.min()) >= 199 * comb(300, 2)
        top_v = np.sort(bv)[-300:]
        assert int(top_v.min()) >= 299 * comb(200, 2)
