"""GPU parity: libbf (through the C ABI) vs the CPU oracle, element by element.

Integer results must be bit-exact (north_star).  Sizes: tiny
fixtures, random small graphs, config 1 in full, shrunken copies of configs
2-5 (same generators) that span many tiles, both tiers and a ragged tail, and
every code path forced on (warp-only, CTA-only, small shared window -> global
overflow rows, multi-rank shares via the virtual world).
"""
import json
import os
from math import comb

import numpy as np
import pytest

import bfgen
import oracle

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RANKS = ("side", "approx_degree", "degree", "approx_codegen")
ORIENTS = ("high", "low")


@pytest.fixture(scope="module")
def bf():
    from paper_1907_08607_b200 import bf as _bf
    return _bf


def run_all(bf, g, rank, orient, **opts):
    with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank, orient=orient, **opts) as bg:
        t = bg.total()
        bu, bv, t2 = bg.vertex()
        be, t3 = bg.edge()
        w = bg.wedges()
    return dict(total=t, b_u=bu, b_v=bv, b_e=be, t2=t2, t3=t3, W=w)


def assert_same(got, ref, ctx=""):
    assert got["total"] == ref["total"] == got["t2"] == got["t3"], ctx
    assert np.array_equal(got["b_u"], ref["b_u"]), ctx + " b_u"
    assert np.array_equal(got["b_v"], ref["b_v"]), ctx + " b_v"
    assert np.array_equal(got["b_e"], ref["b_e"]), ctx + " b_e"


def test_fig1(bf):
    d = json.load(open(os.path.join(GOLDEN, "fig1.json")))
    e = np.array(d["edges"], np.uint32)
    g = bfgen.from_pairs(3, 3, e)
    ref = dict(total=d["total"], b_u=np.array(d["b_u"], np.uint64), b_v=np.array(d["b_v"], np.uint64),
               b_e=np.array(d["b_e"], np.uint64))
    Ws = {}
    for rank in RANKS:
        for orient in ORIENTS:
            got = run_all(bf, g, rank, orient)
            assert_same(got, ref, f"{rank}/{orient}")
            Ws[(rank, orient)] = got["W"]
    assert Ws[("degree", "low")] == d["wedges_degree_gid_ties"] == Ws[("degree", "high")]
    assert Ws[("side", "low")] == d["wedges_side_u_first"]


@pytest.mark.parametrize("a,b", [(1, 1), (2, 2), (3, 5), (17, 9), (40, 33)])
def test_complete_bipartite(bf, a, b):
    g = bfgen.complete(a, b)
    for rank in RANKS:
        for orient in ORIENTS:
            got = run_all(bf, g, rank, orient)
            assert got["total"] == comb(a, 2) * comb(b, 2)
            assert (got["b_u"] == (a - 1) * comb(b, 2)).all()
            assert (got["b_v"] == (b - 1) * comb(a, 2)).all()
            assert (got["b_e"] == (a - 1) * (b - 1)).all()


@pytest.mark.parametrize("seed", range(24))
def test_random_small(bf, seed):
    rng = np.random.default_rng(1000 + seed)
    n_u, n_v = int(rng.integers(1, 80)), int(rng.integers(1, 80))
    p = [0.02, 0.1, 0.3, 0.6][seed % 4]
    e = np.argwhere(rng.random((n_u, n_v)) < p).astype(np.uint32)
    e = e[rng.permutation(len(e))]
    g = bfgen.from_pairs(n_u, n_v, e)
    ref = oracle.count(n_u, n_v, e)
    with oracle.OracleGraph(n_u, n_v, e) as og:
        for rank in RANKS:
            W_ref = og.wedges(og.rank(rank))[0]
            for orient in ORIENTS:
                got = run_all(bf, g, rank, orient)
                assert_same(got, ref, f"seed {seed} {rank}/{orient}")
                assert got["W"] == W_ref


@pytest.mark.parametrize("flags", ["warp", "cta", "dense", "small_window", "dense+small_window", "light8",
                                   "small_chunk", "dense+small_chunk", "dense+small_window+small_chunk",
                                   "cta+small_window", "small_chunk+small_window", "dense+no_split+small_chunk",
                                   "unpacked_sort", "no_dense_row", "dense+no_dense_row",
                                   "small_chunk+no_dense_row", "dense+small_chunk+no_dense_row", "key_buffer",
                                   "dense+key_buffer", "dense+small_chunk+key_buffer", "hub_pos",
                                   "hub_pos+unpacked_sort"])
@pytest.mark.parametrize("orient", ORIENTS)
def test_forced_paths(bf, flags, orient):
    """T3: every start through one tier; tiny windows force the overflow paths
    (warp/medium hash, heavy global rows); tiny chunks force the multi-chunk walk."""
    g = bfgen.chung_lu(1500, 900, 12000, 2.0, 2.3, seed=5)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    f = 0
    if "warp" in flags:
        f |= bf.BF_FLAG_FORCE_WARP
    if "cta" in flags:
        f |= bf.BF_FLAG_FORCE_CTA
    if "dense" in flags:
        f |= bf.BF_FLAG_FORCE_DENSE
    if "small_window" in flags:
        f |= bf.BF_FLAG_SMALL_WINDOW
    if "small_chunk" in flags:
        f |= bf.BF_FLAG_SMALL_CHUNK  # also drops the split threshold: giant-start pieces
    if "no_split" in flags:
        f |= bf.BF_FLAG_NO_SPLIT
    if "key_buffer" in flags:
        f |= bf.BF_FLAG_KEY_BUFFER  # slot-mode walks keep their keys for pass 2
    if "no_dense_row" in flags:
        f |= bf.BF_FLAG_NO_DENSE_ROW  # heavy tier: 4096-key window + global overflow rows
    if "unpacked_sort" in flags:
        f |= bf.BF_FLAG_UNPACKED_SORT  # the c5-size slot sort (key and value arrays)
    if "hub_pos" in flags:
        f |= bf.BF_FLAG_HUB_POS  # U-side twin positions of the hub items ranked in slot order
    opts = dict(test_flags=f)
    if flags == "light8":
        opts["test_light_max_wedges"] = 8
    for rank in ("degree", "side"):
        got = run_all(bf, g, rank, orient, **opts)
        assert_same(got, ref, f"{flags} {rank}/{orient}")


def test_config1_full(bf):
    """Config 1 in full (BASELINE.json configs[0]) under side and degree ranking."""
    g = bfgen.config_graph(1)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    for rank in ("side", "degree", "approx_degree"):
        for orient in ORIENTS:
            assert_same(run_all(bf, g, rank, orient), ref, f"c1 {rank}/{orient}")


@pytest.mark.parametrize("k,scale", [(2, 0.02), (3, 0.01), (4, 0.01), (5, 0.004)])
def test_configs_scaled(bf, k, scale):
    """Shrunken configs 2-5 (same generators, same shape): heavy and light tiers,
    planted biclique (c3), extreme item skew (c4), hub saturation (c5)."""
    g = bfgen.config_graph(k, scale)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    rank = bfgen.CONFIGS[k]["ranking"][0]
    for orient in ORIENTS:
        assert_same(run_all(bf, g, rank, orient), ref, f"c{k}@{scale} {rank}/{orient}")


@pytest.mark.parametrize("V", [2, 5])
def test_virtual_world_split_starts(bf, V):
    """Split starts are dealt whole to ranks (snake order); with tiny chunks the
    split threshold drops to 256 wedges, so many split starts exist and every
    virtual rank gets some."""
    g = bfgen.config_graph(4, 0.01)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    for orient in ORIENTS:
        got = run_all(bf, g, "degree", orient, virtual_world=V, test_flags=bf.BF_FLAG_SMALL_CHUNK)
        assert_same(got, ref, f"V={V} {orient}")


@pytest.mark.parametrize("V", [2, 3, 8])
def test_virtual_world(bf, V):
    """T4 on one GPU: each virtual rank counts its share (snake-dealt heavy starts,
    equal-wedge light slices) and the shares are summed on device."""
    g = bfgen.config_graph(2, 0.01)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    for orient in ORIENTS:
        assert_same(run_all(bf, g, "degree", orient, virtual_world=V), ref, f"V={V} {orient}")


def test_edge_cases(bf):
    cases = [bfgen.from_pairs(0, 0, []), bfgen.from_pairs(5, 0, []), bfgen.from_pairs(0, 7, []),
             bfgen.from_pairs(4, 4, []), bfgen.complete(1, 50), bfgen.complete(50, 1),
             bfgen.from_pairs(10, 10, [(i, i) for i in range(10)]),
             bfgen.from_pairs(100, 100, [(3, 4), (3, 7), (9, 4), (9, 7)])]
    for g in cases:
        ref = oracle.count(g.n_u, g.n_v, g.edges)
        for rank in RANKS:
            for orient in ORIENTS:
                assert_same(run_all(bf, g, rank, orient), ref, f"{g.name} {rank}/{orient}")


def test_errors(bf):
    with pytest.raises(bf.BFError) as ei:
        bf.ButterflyGraph(2, 2, np.array([[0, 2]], np.uint32))
    assert ei.value.status == bf.BF_ERANGE
    with pytest.raises(bf.BFError) as ei:
        bf.ButterflyGraph(3, 3, np.array([[0, 1], [2, 2], [0, 1]], np.uint32))
    assert ei.value.status == bf.BF_EDUP
    g = bf.ButterflyGraph(2, 2, np.array([[0, 1]], np.uint32), rank=None)
    with pytest.raises(bf.BFError) as ei:
        g.total()
    assert ei.value.status == bf.BF_ENORANK
    with pytest.raises(bf.BFError) as ei:
        bf.bf_rank(g.h, 7)
    assert ei.value.status == bf.BF_EINVAL
    g.rank("side")
    assert g.total() == 0
    g.close()


def test_csr_export(bf):
    """Alg. 1 invariants on the exported ranked CSR: rid is a permutation grouping
    U before V; lists strictly decreasing; hi/pos per definition; W equals the
    oracle's W for each ranking."""
    g = bfgen.chung_lu(700, 500, 5000, 2.1, 2.1, seed=9)
    n = g.n_u + g.n_v
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        for rank in RANKS:
            rref = og.rank(rank)
            W_ref, w_ref = og.wedges(rref)
            with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank, orient="low") as bg:
                c = bg.export_csr()
                assert bg.wedges() == W_ref
            rid = c["rid_of_gid"].astype(np.int64)
            assert sorted(rid.tolist()) == list(range(n))
            assert (rid[:g.n_u] < g.n_u).all() and (rid[g.n_u:] >= g.n_u).all()
            # rid order within a side == oracle rank order within the side
            for lo, hi in ((0, g.n_u), (g.n_u, n)):
                assert (np.argsort(rid[lo:hi]) == np.argsort(rref[lo:hi])).all()
            gid_of = np.empty(n, np.int64)
            gid_of[rid] = np.arange(n)
            off, nbr, pos, hi_ = c["off"].astype(np.int64), c["nbr"].astype(np.int64), c["pos"], c["hi"]
            for x in range(0, n, 37):
                lst = nbr[off[x]:off[x + 1]]
                assert (np.diff(lst) < 0).all()
                rx = rref[gid_of[x]]
                assert hi_[x] == int((rref[gid_of[lst]] > rx).sum())
                for i, y in enumerate(lst):
                    assert nbr[off[y] + pos[off[x] + i]] == x
            # per-start wedges (LOW orientation = Alg. 2 per x1)
            assert (c["wstart"][rid] == w_ref).all()


@pytest.mark.parametrize("g", [("C", 700, 500, 5000, 2.1, 2.1, 9), ("cfg", 4, 0.002), ("cfg", 3, 0.002), ("K", 40, 33)])
def test_hub_pos_same_csr(bf, g):
    """BF_FLAG_HUB_POS (the U-side twin positions of the hub items ranked in slot
    order instead of scattered by the V half's decode) builds the same ranked CSR,
    array for array, in both slot-sort record forms and under every ranking."""
    g = bfgen.complete(*g[1:]) if g[0] == "K" else (bfgen.config_graph(*g[1:]) if g[0] == "cfg" else bfgen.chung_lu(*g[1:4], *g[4:6], seed=g[6]))
    for rank in RANKS:
        for extra in (0, bf.BF_FLAG_UNPACKED_SORT):
            with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank, test_flags=extra) as bg:
                a = bg.export_csr()
            with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank, test_flags=extra | bf.BF_FLAG_HUB_POS) as bg:
                b = bg.export_csr()
            for k in ("rid_of_gid", "off", "nbr", "pos", "hi", "wstart"):
                assert np.array_equal(a[k], b[k]), (rank, extra, k)


@pytest.mark.parametrize("orient", ORIENTS)
def test_repeated_graphs_same_process(bf, orient):
    """Library state that outlives a graph (the per-device pool of heavy-tier
    overflow rows) must be clean for the next graph, whatever the mode order."""
    g = bfgen.config_graph(3, 0.01)
    ref = oracle.count(g.n_u, g.n_v, g.edges, edge=False)
    rank = bfgen.CONFIGS[3]["ranking"][0]
    for rep in range(3):
        for flags in (0, bf.BF_FLAG_FORCE_DENSE):
            with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank, orient=orient, test_flags=flags) as bg:
                assert bg.total() == ref["total"], (rep, flags)
                bu, bv_, t = bg.vertex()
                assert t == ref["total"] and np.array_equal(bu, ref["b_u"]) and np.array_equal(bv_, ref["b_v"])
                assert bg.total() == ref["total"], (rep, flags)
        bf.bf_release_device_cache(0)  # rows and pool go back to the driver; the next graph reallocates


@pytest.mark.parametrize("k,scale", [(1, 1.0), (2, 0.02), (3, 0.01), (4, 0.01), (5, 0.004)])
def test_rank_auto_f_metric(bf, k, scale):
    """BF_RANK_AUTO: the wedge counts of the four candidate orders
    computed before ranking equal the oracle's W for each order; the choice
    follows f = (w_s - w_r)/w_s < 0.1 -> side, else the cheapest other order;
    the counts stay exact."""
    g = bfgen.config_graph(k, scale)
    kinds = ("side", "approx_degree", "degree", "approx_codegen")
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        W = {kind: og.wedges(og.rank(kind))[0] for kind in kinds}
    ref = oracle.count(g.n_u, g.n_v, g.edges, edge=False)
    with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank="auto") as bg:
        kind, w = bg.rank_info()
        assert w == [W[x] for x in kinds]
        wr = min(W["degree"], W["approx_degree"], W["approx_codegen"])
        side = wr >= W["side"] or 10 * (W["side"] - wr) < W["side"]
        expect = "side" if side else next(x for x in ("degree", "approx_degree", "approx_codegen") if W[x] == wr)
        assert kind == expect
        assert bg.wedges() == W[kind]
        bu, bv, t = bg.vertex()
        assert t == ref["total"] and np.array_equal(bu, ref["b_u"]) and np.array_equal(bv, ref["b_v"])


@pytest.mark.parametrize("k,scale", [(1, 1.0), (2, 0.02), (3, 0.01), (4, 0.01), (5, 0.004)])
def test_rank_approx_codegen(bf, k, scale):
    """Approximate complement degeneracy on the GPU (bucketed peel, <= 33
    rounds): the rank order inside each side equals the oracle's order, W equals
    the oracle's W under it, and every output is exact."""
    g = bfgen.config_graph(k, scale)
    n = g.n_u + g.n_v
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        rref = og.rank("approx_codegen")
        W_ref = og.wedges(rref)[0]
    for orient in ORIENTS:
        with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank="approx_codegen", orient=orient) as bg:
            assert bg.wedges() == W_ref
            rid = bg.export_csr()["rid_of_gid"].astype(np.int64)
        for lo, hi in ((0, g.n_u), (g.n_u, n)):
            assert (np.argsort(rid[lo:hi]) == np.argsort(rref[lo:hi])).all()
        assert_same(run_all(bf, g, "approx_codegen", orient), ref, f"c{k} approx_codegen/{orient}")


@pytest.mark.parametrize("method", ["edge", "color"])
@pytest.mark.parametrize("p", [1.0, 0.5, 0.2])
def test_sparsify_matches_oracle(bf, method, p):
    """Approximate counting: the device filter keeps exactly the
    oracle's edges (same counter-based hash, implemented on both sides), the
    sparsified graph's count is exact, and p = 1 reproduces T."""
    g = bfgen.config_graph(2, 0.01)
    for seed in (1, 77):
        kept = bf.bf_sparsify(g.n_u, g.n_v, g.edges, method, p, seed)
        ref_kept = oracle.sparsify(g.n_u, g.edges, method, p, seed)
        assert np.array_equal(kept, ref_kept), (method, p, seed)
        ref = oracle.count(g.n_u, g.n_v, ref_kept, vertex=False, edge=False)["total"] if len(ref_kept) else 0
        est, t_s, m_s = bf.bf_approx_total(g.n_u, g.n_v, g.edges, method, p, seed)
        assert t_s == ref and m_s == len(ref_kept)
        scale = p ** -4 if method == "edge" else float(np.ceil(1.0 / p)) ** 3
        assert est == pytest.approx(ref * scale, rel=1e-12)
    if p == 1.0:
        T = oracle.count(g.n_u, g.n_v, g.edges, vertex=False, edge=False)["total"]
        assert bf.approx_total(g.n_u, g.n_v, g.edges, 1.0, method=method) == T


def test_duplicate_in_large_graph(bf):
    """Reading Z8: a single repeated pair anywhere in the list is rejected (by
    bf_rank: the ranked slot sort makes the two copies adjacent)."""
    g = bfgen.chung_lu(3000, 2000, 30000, 2.1, 2.2, seed=7)
    for pick in (0, 12345, g.m - 1):
        e = np.concatenate([g.edges, g.edges[pick:pick + 1]])
        e = e[np.random.default_rng(pick).permutation(len(e))]
        for f in (0, bf.BF_FLAG_UNPACKED_SORT):
            with pytest.raises(bf.BFError) as ei:
                bf.ButterflyGraph(g.n_u, g.n_v, e, test_flags=f)
            assert ei.value.status == bf.BF_EDUP


@pytest.mark.parametrize("seed", range(16))
def test_random_graphs_random_paths(bf, seed):
    """Randomised T3: random power-law graphs, random ranking, orientation and
    path-forcing flags (tiers, tiny windows/chunks, no split, virtual ranks);
    every mode bit-exact with the oracle."""
    rng = np.random.default_rng(7000 + seed)
    n_u, n_v = int(rng.integers(50, 2500)), int(rng.integers(50, 2500))
    m = int(min(n_u * n_v // 3, rng.integers(200, 25000)))
    g = bfgen.chung_lu(n_u, n_v, m, float(rng.uniform(1.8, 2.6)), float(rng.uniform(1.8, 2.6)), seed=seed + 1)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    names = ["FORCE_WARP", "FORCE_CTA", "FORCE_DENSE", "SMALL_WINDOW", "SMALL_CHUNK", "NO_SPLIT", "UNPACKED_SORT",
             "NO_DENSE_ROW", "KEY_BUFFER", "HUB_POS"]
    f = 0
    for nm in names:
        if rng.random() < 0.3:
            f |= getattr(bf, "BF_FLAG_" + nm)
    rank = ["side", "approx_degree", "degree", "auto", "approx_codegen"][int(rng.integers(0, 5))]
    orient = ORIENTS[int(rng.integers(0, 2))]
    opts = dict(test_flags=f)
    if rng.random() < 0.3:
        opts["virtual_world"] = int(rng.integers(2, 6))
    got = run_all(bf, g, rank, orient, **opts)
    assert_same(got, ref, f"seed {seed} flags {f:#x} {rank}/{orient} {opts}")


@pytest.mark.parametrize("k,scale,rank,flags", [
    (3, 0.02, "approx_degree", 0),
    (4, 0.01, "degree", 0x20),         # SMALL_CHUNK: split starts, multi-chunk heavy starts
    (2, 0.02, "degree", 0x4 | 0x200),  # SMALL_WINDOW + KEY_BUFFER: hash / global-row / slot paths
])
def test_race_stress_grid_jitter(bf, k, scale, rank, flags):
    """Race stress (a racecheck stand-in: compute-sanitizer is not on the pool):
    every wedge-kernel launch takes a pseudo-random grid (BF_FLAG_GRID_JITTER),
    so each repetition maps starts to CTAs and interleaves the shared-memory
    CAS hash, owner lists, window resets and global rows differently; every
    repetition and mode must stay bit-exact with the oracle."""
    g = bfgen.config_graph(k, scale)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    f = flags | bf.BF_FLAG_GRID_JITTER
    for orient in ORIENTS:
        with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank, orient=orient, test_flags=f) as bg:
            for rep in range(4):
                ctx = f"c{k} {orient} rep {rep}"
                assert bg.total() == ref["total"], ctx
                bu, bv_, t = bg.vertex()
                assert t == ref["total"] and np.array_equal(bu, ref["b_u"]) and np.array_equal(bv_, ref["b_v"]), ctx
                be, t = bg.edge()
                assert t == ref["total"] and np.array_equal(be, ref["b_e"]), ctx


def test_nccl_bootstrap_single_rank(bf):
    """The multi-GPU bootstrap on one GPU: NCCL loads at run time, a 1-rank
    communicator is created from the 128-byte id and destroyed."""
    uid = bf.bf_nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128
    comm = bf.bf_nccl_comm_create(uid, 0, 1, 0)
    assert comm
    bf.bf_nccl_comm_destroy(comm)


@pytest.mark.parametrize("V", [1, 3])
def test_nccl_allreduce_combine(bf, V):
    """a9 through the real ncclAllReduce: with a communicator attached (here a
    1-rank one, the only kind one GPU can host) every count call combines its
    [counts | total] buffer with ncclAllReduce(u64, sum) on the graph's stream;
    with virtual ranks the on-device share sum feeds that same allreduce.  All
    three modes stay bit-exact with the oracle."""
    g = bfgen.config_graph(2, 0.01)
    ref = oracle.count(g.n_u, g.n_v, g.edges)
    comm = bf.bf_nccl_comm_create(bf.bf_nccl_unique_id(), 0, 1, 0)
    try:
        for orient in ORIENTS:
            got = run_all(bf, g, "degree", orient, nccl_comm=comm, virtual_world=V)
            assert_same(got, ref, f"nccl V={V} {orient}")
    finally:
        bf.bf_nccl_comm_destroy(comm)


@pytest.mark.parametrize("k,scale", [(2, 0.02), (4, 0.01)])
def test_rank_shares_partition(bf, k, scale):
    """bf_rank_shares: the per-rank wedge loads of the kernels' deal partition W
    exactly, for G = 1..8, and a virtual world of G ranks counts exactly."""
    g = bfgen.config_graph(k, scale)
    with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank="degree") as bg:
        W = bg.wedges()
        for G in (1, 2, 3, 4, 8):
            sh = bf.bf_rank_shares(bg.h, G)
            assert len(sh) == G and sum(sh) == W, (G, sh, W)
