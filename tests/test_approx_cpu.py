"""Approximate counting by sparsification (PAPER.md 4.4; SURVEY
8(f) row 3), oracle side: the counter-based hash against the published
splitmix64 test vector, exactness at p = 1, and unbiasedness of both
estimators over seeds (each butterfly survives edge sparsification with
probability p^4 and colorful sparsification with probability p^3)."""
import math

import numpy as np

import bfgen
import oracle


def test_h64_is_splitmix64():
    # splitmix64 seeded with 0: first outputs 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4
    assert oracle.h64(0, 0) == 0xE220A8397B1DCDAF
    assert oracle.h64(0, 1) == 0x6E789E6AA1B965F4


def test_p1_keeps_everything():
    g = bfgen.chung_lu(300, 200, 2500, 2.1, 2.1, seed=11)
    for method in ("edge", "color"):
        kept = oracle.sparsify(g.n_u, g.edges, method, 1.0, seed=5)
        assert np.array_equal(kept, g.edges)


def test_edge_keep_rate():
    g = bfgen.uniform(500, 400, 20000, seed=3)
    kept = oracle.sparsify(g.n_u, g.edges, "edge", 0.3, seed=9)
    # Binomial(20000, 0.3): sd ~ 65
    assert abs(len(kept) - 6000) < 6 * 65


def _estimates(g, method, p, seeds):
    out = []
    for sd in seeds:
        kept = oracle.sparsify(g.n_u, g.edges, method, p, seed=sd)
        t = oracle.count(g.n_u, g.n_v, kept, vertex=False, edge=False)["total"] if len(kept) else 0
        out.append(t / p ** 4 if method == "edge" else t * math.ceil(1 / p) ** 3)
    return np.array(out, dtype=np.float64)


def test_unbiased_over_seeds():
    g = bfgen.chung_lu(120, 90, 1400, 2.0, 2.2, seed=21)
    T = oracle.count(g.n_u, g.n_v, g.edges, vertex=False, edge=False)["total"]
    assert T > 1000
    for method, p in (("edge", 0.5), ("color", 0.5)):
        est = _estimates(g, method, p, range(400))
        se = est.std(ddof=1) / math.sqrt(len(est))
        assert abs(est.mean() - T) < 5 * se, (method, est.mean(), T, se)
