"""Pins for the CPU oracle (SURVEY.md 8(c) table "What pins each part of the oracle").

Each test checks oracle/ against something other than itself: values the paper
prints (Fig. 1 / Fig. fig-count-ex, tests/golden/fig1.json), closed forms
(K_{a,b}), brute force over 4-tuples (tests/brute.py), exhaustive enumeration of
small graphs, a library integer matmul, the trace identity of closed 4-walks,
invariants, and the literal Alg. 1+2 wedge listing.
"""
import itertools
import json
import os
from math import comb

import numpy as np
import pytest

import bfgen
import oracle
from oracle import wedges_py
from tests import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def fig1():
    d = json.load(open(os.path.join(GOLDEN, "fig1.json")))
    return d, np.array(d["edges"], dtype=np.uint32)


# ---------------------------------------------------------------- P1-P3 ----
def test_fig1_counts():
    """P1-P3: Fig. 1 has exactly 3 butterflies; per-vertex and
    per-edge values from Fig. fig-count-ex Step 4."""
    d, e = fig1()
    with oracle.OracleGraph(d["n_u"], d["n_v"], e) as g:
        for side in (0, 1):
            r = g.count(side=side)
            assert r["total"] == d["total"] == 3
            assert r["b_u"].tolist() == d["b_u"]
            assert r["b_v"].tolist() == d["b_v"]
            assert r["b_e"].tolist() == d["b_e"]
        assert [g.vertex(0, u) for u in range(3)] == d["b_u"]
        assert [g.vertex(1, v) for v in range(3)] == d["b_v"]
        assert [g.edge(i) for i in range(7)] == d["b_e"]
    # the three listed butterflies are exactly brute force's
    T, bu, bv, be = brute.butterflies(d["n_u"], d["n_v"], e)
    assert T == 3 and bu.tolist() == d["b_u"] and bv.tolist() == d["b_v"] and be.tolist() == d["b_e"]


def test_fig2_wedge_listing():
    """P4: under Fig. fig-count-ex's order (v3,u1,u2,v1,v2,u3) Alg. 2 retrieves
    exactly the 6 wedges of Step 2, grouped as in Step 3."""
    d, e = fig1()
    name = {0: "u1", 1: "u2", 2: "u3", 3: "v1", 4: "v2", 5: "v3"}
    gid = {v: k for k, v in name.items()}
    rank = [0] * 6
    for r, nm in enumerate(d["fig2_order"]):
        rank[gid[nm]] = r
    w = wedges_py.get_wedges(3, 3, e, rank)
    got = sorted(((name[a], name[b]), name[y]) for (a, b), y in w)
    want = sorted(((a, b), y) for (a, b), y in d["fig2_wedges"])
    assert got == want
    freq = {f"{name[a]},{name[b]}": c for (a, b), c in wedges_py.get_freq(w).items()}
    assert freq == d["fig2_groups"]
    # the oracle's W definition agrees with the literal listing
    with oracle.OracleGraph(3, 3, e) as g:
        W, per = g.wedges(np.array(rank, np.uint32))
        assert W == 6
        assert per.tolist() == [sum(1 for (a, _), _y in w if a == z) for z in range(6)]


def test_fig1_rankings_and_wedge_counts():
    """Readings Z1-Z4 on Fig. 1: W = 5 (degree, gid ties), 5 (side, U first), 6 (V first)."""
    d, e = fig1()
    with oracle.OracleGraph(3, 3, e) as g:
        rdeg = g.rank("degree")
        assert rdeg.tolist() == [0, 1, 5, 3, 4, 2]  # u1,u2,v3,v1,v2,u3
        assert g.wedges(rdeg)[0] == d["wedges_degree_gid_ties"]
        rside = g.rank("side")
        assert rside.tolist() == [0, 1, 2, 3, 4, 5]  # U first
        assert g.wedges(rside)[0] == d["wedges_side_u_first"]
        vfirst = np.array([3, 4, 5, 0, 1, 2], np.uint32)
        assert g.wedges(vfirst)[0] == d["wedges_side_v_first"]
        # approx degree: floor(log2 3)=1 for u1,u2,v3 and floor(log2 2)=1 for v1,v2; 0 for u3
        assert g.rank("approx_degree").tolist() == [0, 1, 5, 2, 3, 4]


# ---------------------------------------------------------------- P5 -------
@pytest.mark.parametrize("a,b", [(1, 1), (1, 5), (2, 2), (2, 3), (3, 4), (5, 7), (12, 9), (30, 2)])
def test_complete_bipartite_closed_form(a, b):
    """P5: K_{a,b}: T=C(a,2)C(b,2) (north_star); b(u)=(a-1)C(b,2);
    b(v)=(b-1)C(a,2); b(u,v)=(a-1)(b-1)."""
    g = bfgen.complete(a, b)
    r = oracle.count(g.n_u, g.n_v, g.edges)
    assert r["total"] == comb(a, 2) * comb(b, 2)
    assert np.all(r["b_u"] == (a - 1) * comb(b, 2))
    assert np.all(r["b_v"] == (b - 1) * comb(a, 2))
    assert np.all(r["b_e"] == (a - 1) * (b - 1))


# ---------------------------------------------------------------- P6, P7 ---
def test_zero_cases():
    """P6: stars, matchings, forests, empty graphs have no butterflies."""
    cases = [
        bfgen.complete(1, 40),  # star K_{1,40}
        bfgen.complete(40, 1),
        bfgen.from_pairs(10, 10, [(i, i) for i in range(10)]),  # matching
        bfgen.from_pairs(5, 6, [(0, 0), (0, 1), (1, 1), (1, 2), (2, 2), (2, 3), (3, 3), (3, 4), (4, 5)]),  # path
        bfgen.from_pairs(4, 4, []),
        bfgen.from_pairs(0, 3, []),
        bfgen.from_pairs(3, 0, []),
    ]
    for g in cases:
        r = oracle.count(g.n_u, g.n_v, g.edges)
        assert r["total"] == 0
        assert not r["b_u"].any() and not r["b_v"].any() and not r["b_e"].any()


def test_disjoint_union_additive():
    """P7: counts of a disjoint union are the per-component counts."""
    g1 = bfgen.uniform(30, 25, 200, seed=11)
    g2 = bfgen.complete(4, 6)
    g = bfgen.disjoint_union(g1, g2)
    r1, r2, r = (oracle.count(x.n_u, x.n_v, x.edges) for x in (g1, g2, g))
    assert r["total"] == r1["total"] + r2["total"]
    assert r["b_u"].tolist() == r1["b_u"].tolist() + r2["b_u"].tolist()
    assert r["b_v"].tolist() == r1["b_v"].tolist() + r2["b_v"].tolist()
    assert r["b_e"].tolist() == r1["b_e"].tolist() + r2["b_e"].tolist()


# ---------------------------------------------------------------- P8 -------
@pytest.mark.parametrize("seed", range(40))
def test_brute_force_random(seed):
    """P8: oracle == brute-force 4-tuple enumeration on random tiny graphs
    (SPEC.md:545's idea: sizes up to 30+30, densities 0.05..0.5)."""
    rng = np.random.default_rng(seed)
    n_u, n_v = int(rng.integers(1, 31)), int(rng.integers(1, 31))
    p = [0.05, 0.2, 0.5][seed % 3]
    A = rng.random((n_u, n_v)) < p
    e = np.argwhere(A).astype(np.uint32)
    e = e[rng.permutation(len(e))]
    T, bu, bv, be = brute.butterflies(n_u, n_v, e)
    with oracle.OracleGraph(n_u, n_v, e) as g:
        r = g.count_full()
        assert r["total"] == T
        assert r["b_u"].tolist() == bu.tolist()
        assert r["b_v"].tolist() == bv.tolist()
        assert r["b_e"].tolist() == be.tolist()
        for x in range(0, n_u, 7):
            assert g.vertex(0, x) == bu[x]
        for i in range(0, len(e), 5):
            assert g.edge(i) == be[i]


# ---------------------------------------------------------------- P9 -------
@pytest.mark.parametrize("n_u,n_v", [(2, 2), (3, 3), (2, 4), (4, 3), (4, 4)])
def test_exhaustive_small(n_u, n_v):
    """P9: every labelled bipartite graph with |U|,|V| <= 4 (2^16 graphs at 4x4)
    against vectorised brute force over 4-tuples."""
    k = n_u * n_v
    G = 1 << k
    bits = (np.arange(G)[:, None] >> np.arange(k)[None, :]) & 1
    A = bits.reshape(G, n_u, n_v).astype(bool)
    pu = list(itertools.combinations(range(n_u), 2))
    pv = list(itertools.combinations(range(n_v), 2))
    T = np.zeros(G, np.int64)
    BU = np.zeros((G, n_u), np.int64)
    BV = np.zeros((G, n_v), np.int64)
    BE = np.zeros((G, n_u, n_v), np.int64)
    for (a, b) in pu:
        for (c, d) in pv:
            m = A[:, a, c] & A[:, a, d] & A[:, b, c] & A[:, b, d]
            T += m
            for x in (a, b):
                BU[:, x] += m
            for y in (c, d):
                BV[:, y] += m
            for x in (a, b):
                for y in (c, d):
                    BE[:, x, y] += m
    cells = [(u, v) for u in range(n_u) for v in range(n_v)]
    for gi in range(G):
        e = np.array([cells[i] for i in range(k) if bits[gi, i]], dtype=np.uint32).reshape(-1, 2)
        r = oracle.count(n_u, n_v, e)
        assert r["total"] == T[gi]
        assert r["b_u"].tolist() == BU[gi].tolist()
        assert r["b_v"].tolist() == BV[gi].tolist()
        assert r["b_e"].tolist() == [int(BE[gi, u, v]) for u, v in e]


# ---------------------------------------------------------------- P10 ------
def test_integer_matmul_identity():
    """P10: with C = A A^T (int64 numpy matmul), T = Σ_{i<j} C(C_ij,2), b_U = off-diagonal
    row sums of C(C,2), b_V likewise from A^T A, b_E[u,v] = (D0 A)[u,v] with
    D0 = C - 1 and zero diagonal.  Run on config 1 (2000x1500, 20K edges)."""
    g = bfgen.config_graph(1)
    A = np.zeros((g.n_u, g.n_v), np.int64)
    A[g.edges[:, 0], g.edges[:, 1]] = 1
    C = A @ A.T
    C2 = C * (C - 1) // 2
    np.fill_diagonal(C2, 0)
    D = A.T @ A
    D2 = D * (D - 1) // 2
    np.fill_diagonal(D2, 0)
    D0 = C - 1
    np.fill_diagonal(D0, 0)
    BE = D0 @ A
    r = oracle.count(g.n_u, g.n_v, g.edges)
    assert r["total"] == int(np.triu(C2, 1).sum())
    assert r["b_u"].tolist() == C2.sum(1).tolist()
    assert r["b_v"].tolist() == D2.sum(1).tolist()
    assert r["b_e"].tolist() == BE[g.edges[:, 0], g.edges[:, 1]].tolist()


# ---------------------------------------------------------------- P11 ------
@pytest.mark.parametrize("seed", range(6))
def test_trace_identity(seed):
    """P11: tr(B^4) = 8T + 2m + 4 Σ_z C(deg z, 2) for the full n x n adjacency B
    (closed 4-walks: back-and-forth, two spokes at z, two spokes at a neighbour,
    and the 8 traversals of each 4-cycle)."""
    rng = np.random.default_rng(100 + seed)
    n_u, n_v = int(rng.integers(5, 40)), int(rng.integers(5, 40))
    e = np.argwhere(rng.random((n_u, n_v)) < 0.25).astype(np.uint32)
    n = n_u + n_v
    B = np.zeros((n, n), np.int64)
    B[e[:, 0], n_u + e[:, 1]] = 1
    B[n_u + e[:, 1], e[:, 0]] = 1
    B2 = B @ B
    tr4 = int(np.trace(B2 @ B2))
    deg = B.sum(1)
    r = oracle.count(n_u, n_v, e)
    assert tr4 == 8 * r["total"] + 2 * len(e) + 4 * int((deg * (deg - 1) // 2).sum())


# ---------------------------------------------------------------- P12 ------
@pytest.mark.parametrize("seed", range(5))
def test_invariants(seed):
    """P12: Σ_U b = Σ_V b = 2T; Σ_E b = 4T; Σ_{e∋z} b(e) = 2 b(z) for every z."""
    g = bfgen.chung_lu(400, 300, 4000, 2.1, 2.3, seed=seed)
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        r = og.count_full()
    T = r["total"]
    assert int(r["b_u"].sum()) == 2 * T == int(r["b_v"].sum())
    assert int(r["b_e"].sum()) == 4 * T
    su = np.zeros(g.n_u, np.uint64)
    sv = np.zeros(g.n_v, np.uint64)
    np.add.at(su, g.edges[:, 0], r["b_e"])
    np.add.at(sv, g.edges[:, 1], r["b_e"])
    assert (su == 2 * r["b_u"]).all() and (sv == 2 * r["b_v"]).all()


# ---------------------------------------------------------------- P14 ------
def test_planted_biclique_isolated():
    """P14 (exact variant): a K_{20,30} as its own component adds exactly the
    closed form to the total and to its vertices (P5 + P7)."""
    base = bfgen.chung_lu(300, 300, 2500, 2.0, 2.5, seed=3)
    g = bfgen.disjoint_union(base, bfgen.complete(20, 30))
    rb = oracle.count(base.n_u, base.n_v, base.edges)
    r = oracle.count(g.n_u, g.n_v, g.edges)
    assert r["total"] == rb["total"] + comb(20, 2) * comb(30, 2)
    assert np.all(r["b_u"][base.n_u:] == 19 * comb(30, 2))
    assert np.all(r["b_v"][base.n_v:] == 29 * comb(20, 2))


# ---------------------------------------------------------------- P15 ------
@pytest.mark.parametrize("seed", range(8))
def test_wedge_count_closed_form(seed):
    """P15: the oracle's W (Alg. 2 loop bounds) equals the closed form
    W = Σ_y (k_y d_y - k_y(k_y+1)/2), k_y = #neighbours ranked below y
    (SURVEY App. B item 4), under every ranking and a random one; and equals the
    literal Alg. 1+2 listing (oracle/wedges_py.py) per start vertex on tiny graphs."""
    rng = np.random.default_rng(seed)
    g = bfgen.chung_lu(60, 40, 400, 2.1, 2.2, seed=seed)
    n = g.n_u + g.n_v
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        ranks = [og.rank(k) for k in ("side", "approx_degree", "degree")]
        ranks.append(rng.permutation(n).astype(np.uint32))
        for rank in ranks:
            assert sorted(rank.tolist()) == list(range(n))
            W, per = og.wedges(rank)
            ru = rank[g.edges[:, 0]].astype(np.int64)
            rv = rank[g.n_u + g.edges[:, 1]].astype(np.int64)
            closed = 0
            for z_is_u in (True, False):
                cnt = np.zeros(n, np.int64)
                below = np.zeros(n, np.int64)
                zs = g.edges[:, 0].astype(np.int64) if z_is_u else g.n_u + g.edges[:, 1].astype(np.int64)
                rz, ro = (ru, rv) if z_is_u else (rv, ru)
                np.add.at(cnt, zs, 1)
                np.add.at(below, zs, (ro < rz).astype(np.int64))
                closed += int((below * cnt - below * (below + 1) // 2).sum())
            assert W == closed
            w = wedges_py.get_wedges(g.n_u, g.n_v, g.edges, rank.tolist())
            assert len(w) == W
            lit = np.zeros(n, np.int64)
            for (a, _b), _y in w:
                lit[a] += 1
            assert per.tolist() == lit.tolist()


def test_side_ranking_direction():
    """Reading Z1 on K_{1,5}: U endpoints give Σ_V C(1,2)=0 wedges, V endpoints
    C(5,2)=10, so U goes first."""
    g = bfgen.complete(1, 5)
    with oracle.OracleGraph(1, 5, g.edges) as og:
        r = og.rank("side")
        assert r.tolist() == [0, 1, 2, 3, 4, 5]
        assert og.wedges(r)[0] == 0
    g = bfgen.complete(5, 1)
    with oracle.OracleGraph(5, 1, g.edges) as og:
        r = og.rank("side")
        assert r.tolist() == [1, 2, 3, 4, 5, 0]  # V first


def test_rejects_bad_input():
    with pytest.raises(oracle.OracleError, match="ERANGE"):
        oracle.OracleGraph(2, 2, np.array([[0, 2]], np.uint32))
    with pytest.raises(oracle.OracleError, match="EDUP"):
        oracle.OracleGraph(2, 2, np.array([[0, 1], [1, 1], [0, 1]], np.uint32))


def test_edge_order_invariance():
    """Per-edge output follows the input order (reading Z7)."""
    g = bfgen.uniform(50, 40, 500, seed=7)
    gp = bfgen.permute_edges(g, 3)
    r, rp = oracle.count(g.n_u, g.n_v, g.edges), oracle.count(gp.n_u, gp.n_v, gp.edges)
    key = lambda e: (e[:, 0].astype(np.int64) << 32) | e[:, 1]
    d = dict(zip(key(g.edges).tolist(), r["b_e"].tolist()))
    assert [d[k] for k in key(gp.edges).tolist()] == rp["b_e"].tolist()


@pytest.mark.parametrize("procs", [1, 3, 7])
def test_sharded_equals_unsharded(procs):
    """the sharded oracle (forked workers over x ranges,
    disjoint b(x)/b(e), centre partials summed) equals the single-process run
    bit for bit, on either enumeration side, with ragged shard counts."""
    g = bfgen.chung_lu(900, 700, 9000, 2.0, 2.3, seed=11)
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        for side in (0, 1):
            a = og.count(side=side)
            b = og.count_sharded(procs=procs, side=side)
            assert a["total"] == b["total"]
            for k in ("b_u", "b_v", "b_e"):
                assert np.array_equal(a[k], b[k]), (side, k)
        e = bfgen.from_pairs(5, 3, [])
        with oracle.OracleGraph(5, 3, e.edges) as og0:
            r = og0.count_sharded(procs=procs)
            assert r["total"] == 0 and not r["b_u"].any() and not r["b_v"].any() and len(r["b_e"]) == 0


# ------------------------------------- approximate complement degeneracy ----
def test_approx_codegen_hand_worked():
    """Approximate complement degeneracy: rounds remove every
    remaining vertex of the largest floor(log2 current degree).
    Fig. 1: degrees u1 3, u2 3, u3 1, v1 2, v2 2, v3 3 -> buckets 1,1,0,1,1,1;
    round 1 removes {u1,u2,v1,v2,v3} (gid order), leaving u3 at degree 0
    (bucket -1): round 2.  Order u1,u2,v1,v2,v3,u3; W = 5 (x1=u1: v1->u2,
    v2->u2, v3->u2, v3->u3; x1=u2: v3->u3).
    A graph where the degree updates matter (U: h,x,y; V: p,q,a,b,c; edges
    h-p,h-a,h-b,h-c,x-p,x-q,y-q): round 1 {h} (bucket 2); then p drops to
    degree 1 but q keeps 2, so round 2 is {x,q} (bucket 1), not {x,p,q};
    round 3 the rest at degree 0 in gid order: h,x,q,y,p,a,b,c."""
    d, e = fig1()
    with oracle.OracleGraph(3, 3, e) as og:
        r = og.rank("approx_codegen")
        assert r.tolist() == [0, 1, 5, 2, 3, 4]
        assert og.wedges(r)[0] == 5
    e2 = np.array([[0, 0], [0, 2], [0, 3], [0, 4], [1, 0], [1, 1], [2, 1]], np.uint32)
    with oracle.OracleGraph(3, 5, e2) as og:
        assert og.rank("approx_codegen").tolist() == [0, 1, 3, 4, 2, 5, 6, 7]


@pytest.mark.parametrize("a,b", [(3, 9), (9, 3), (4, 5), (1, 6)])
def test_approx_codegen_complete_bipartite(a, b):
    """K_{a,b}: U vertices have degree b, V vertices degree a.  Different
    log-buckets: the higher side goes in round 1 and the other side drops to
    degree 0 (round 2) -- the side order with that side first.  Same bucket:
    one round, gid order."""
    g = bfgen.complete(a, b)
    with oracle.OracleGraph(a, b, g.edges) as og:
        r = og.rank("approx_codegen").tolist()
    la, lb = (a).bit_length() - 1, (b).bit_length() - 1
    if lb > la:
        assert r == list(range(a + b))
    elif la > lb:
        assert r == list(range(b, a + b)) + list(range(b))
    else:
        assert r == list(range(a + b))


@pytest.mark.parametrize("seed", range(6))
def test_approx_codegen_work_bound(seed):
    """The paper's work bound for this order: when x is peeled,
    every remaining neighbour y has deg^r(y) <= 2 deg^r(x), hence for every edge
    with rank(x) < rank(y): deg_x(y) = #{z in N(y): rank(z) > rank(x)} <= 2 deg(x).
    The order is a permutation."""
    g = bfgen.chung_lu(300 + 40 * seed, 200 + 30 * seed, 3000 + 500 * seed, 2.0, 2.3, seed=seed)
    n = g.n_u + g.n_v
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        r = og.rank("approx_codegen").astype(np.int64)
    assert sorted(r.tolist()) == list(range(n))
    gu = g.edges[:, 0].astype(np.int64)
    gv = g.n_u + g.edges[:, 1].astype(np.int64)
    deg = np.bincount(np.concatenate([gu, gv]), minlength=n)
    nbrs = [[] for _ in range(n)]
    for u, v in zip(gu.tolist(), gv.tolist()):
        nbrs[u].append(v)
        nbrs[v].append(u)
    for x, y in list(zip(gu.tolist(), gv.tolist())) + list(zip(gv.tolist(), gu.tolist())):
        if r[x] < r[y]:
            degxy = sum(1 for z in nbrs[y] if r[z] > r[x])
            assert degxy <= 2 * deg[x], (x, y)


def test_fullsize_cache_reproduces():
    """tests/golden/fullsize_oracle.json (tools/oracle_cache.py) is what the
    oracle computes: config 1 in full from a fresh sharded run, and the cached
    generator keys (edge-list SHA-256) of configs 1-2 from fresh generation."""
    import hashlib
    cache = json.load(open(os.path.join(GOLDEN, "fullsize_oracle.json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).astype("<u8").tobytes()).hexdigest()
    for k in (1, 2):
        g = bfgen.config_graph(k)
        c = cache[str(k)]
        assert c["gen_version"] == bfgen.GEN_VERSION
        assert hashlib.sha256(np.ascontiguousarray(g.edges).astype("<u4").tobytes()).hexdigest() == c["edges_sha256"]
        if k == 1:
            with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
                r = og.count_sharded(procs=3)
            assert r["total"] == c["total"]
            for name in ("b_u", "b_v", "b_e"):
                assert sha(r[name]) == c[name + "_sha256"]
