"""Full-size oracle outputs for BASELINE.json's configs, cached as SHA-256s.

Calls only oracle/ (the sharded plain-definition oracle)
and bfgen/ (the seeded input generator).  Writes tests/golden/fullsize_oracle.json:
per config the generator key (config, GEN_VERSION, seed, sizes, SHA-256 of the
edge list) and the SHA-256 of each exact output array -- b_u, b_v (Eq. (1),
PAPER.md:703-705) and b_e (Eq. (2)) as little-endian uint64 in
input-id / input-edge order -- plus the total.  The GPU tests and bench.py
compare the library's outputs against these hashes; no value here comes from
the CUDA path.

  python tools/oracle_cache.py [k ...]      # default: 1 2 3 4
  python tools/oracle_cache.py --c5-sample  # config 5: stratified sample (c5_sample.json)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bfgen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize_oracle.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u8", copy=False).tobytes()).hexdigest()


def edges_sha(e: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(e).astype("<u4", copy=False).tobytes()).hexdigest()


def entry(k: int, procs: int | None = None) -> dict:
    t0 = time.time()
    g = bfgen.config_graph(k)
    tg = time.time() - t0
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        t1 = time.time()
        r = og.count_sharded(procs=procs)
        tc = time.time() - t1
    c = bfgen.CONFIGS[k]
    return {
        "config": k, "gen_version": bfgen.GEN_VERSION, "seed": c["seed"], "n_u": g.n_u, "n_v": g.n_v, "m": g.m,
        "edges_sha256": edges_sha(g.edges), "total": int(r["total"]),
        "b_u_sha256": sha(r["b_u"]), "b_v_sha256": sha(r["b_v"]), "b_e_sha256": sha(r["b_e"]),
        "oracle": {"enumeration_side": "UV"[r["side"]], "shards": r["shards"], "wall_s": round(tc, 1),
                   "gen_s": round(tg, 1), "host_cores": len(os.sched_getaffinity(0))},
    }


_OG = None


def _vertex_task(t):
    side, x = t
    return side, x, _OG.vertex(side, x)


def _edge_task(e):
    return e, _OG.edge(e)


def c5_sample(budget: float = 4e9, per_stratum: int = 4, hubs: int = 12, n_edges: int = 64, procs=None):
    """Config 5 is beyond a full oracle run (about 7.7e13 steps); store exact
    oracle values for a stratified sample instead: per side, `per_stratum`
    random vertices from each of ten degree strata (quantiles over vertices with
    degree >= 1) plus a few isolated ones, and the `hubs` highest-degree
    vertices whose oracle cost sum_{y in N(x)} deg(y) fits `budget`; random
    edges plus the edges of affordable hubs.  Written to tests/golden/c5_sample.json."""
    import multiprocessing as mp
    global _OG
    g = bfgen.config_graph(5)
    rng = np.random.default_rng(2024)
    U = g.edges[:, 0].astype(np.int64)
    V = g.edges[:, 1].astype(np.int64)
    deg = [np.bincount(U, minlength=g.n_u), np.bincount(V, minlength=g.n_v)]
    cost = [np.bincount(U, weights=deg[1][V].astype(np.float64), minlength=g.n_u),
            np.bincount(V, weights=deg[0][U].astype(np.float64), minlength=g.n_v)]
    tasks = []
    for side in (0, 1):
        d, cs = deg[side], cost[side]
        nz = np.flatnonzero(d > 0)
        qs = np.quantile(d[nz], np.linspace(0, 1, 11))
        for lo, hi in zip(qs[:-1], qs[1:]):
            cand = nz[(d[nz] >= lo) & (d[nz] <= hi) & (cs[nz] <= budget)]
            if len(cand):
                tasks += [(side, int(x)) for x in rng.choice(cand, min(per_stratum, len(cand)), replace=False)]
        zero = np.flatnonzero(d == 0)
        tasks += [(side, int(x)) for x in zero[:2]]
        by_deg = np.argsort(-d, kind="stable")
        tasks += [(side, int(x)) for x in by_deg[cs[by_deg] <= budget][:hubs]]
    tasks = sorted(set(tasks))
    ecost = cost[0][U]
    edges = [int(e) for e in rng.integers(0, g.m, n_edges) if ecost[e] <= budget]
    hub_u = [x for s, x in tasks if s == 0][-hubs:]
    for u in hub_u[:4]:
        es = np.flatnonzero(U == u)
        edges += [int(e) for e in rng.choice(es, min(4, len(es)), replace=False)]
    edges = sorted(set(edges))
    t0 = time.time()
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        _OG = og
        P = procs or len(os.sched_getaffinity(0))
        with mp.get_context("fork").Pool(P) as pool:
            vals = pool.map(_vertex_task, tasks, chunksize=1)
            evals = pool.map(_edge_task, edges, chunksize=1)
        _OG = None
    out = {"_doc": "exact oracle values (oracle/, Eq. (1)/(2)) for a stratified sample of config 5 "
                   "(tools/oracle_cache.py --c5-sample); [side, id, b] and [edge index, b]",
           "config": 5, "gen_version": bfgen.GEN_VERSION, "edges_sha256": edges_sha(g.edges),
           "budget_steps_per_value": budget, "wall_s": round(time.time() - t0, 1),
           "vertices": [[s, x, int(v)] for s, x, v in vals], "edges": [[e, int(v)] for e, v in evals]}
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c5_sample.json"), "w"), indent=0)
    print(f"c5 sample: {len(vals)} vertices, {len(evals)} edges, {out['wall_s']} s", flush=True)


def main(ks):
    d = json.load(open(OUT)) if os.path.exists(OUT) else {}
    d["_doc"] = ("SHA-256 of the exact oracle outputs at BASELINE.json's full sizes (tools/oracle_cache.py: "
                 "sharded oracle/, plain definition Eq. (1)/(2)); arrays little-endian uint64 in input order")
    for k in ks:
        e = entry(k)
        d[str(k)] = e
        print(json.dumps(e), flush=True)
        json.dump(d, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if "--c5-sample" in sys.argv:
        c5_sample()
    else:
        main([int(x) for x in sys.argv[1:]] or [1, 2, 3, 4])
