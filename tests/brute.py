"""Brute-force butterfly enumeration for tiny graphs (pin P8).

Independent of oracle/: it enumerates every 4-tuple {u<u'} x {v<v'} and keeps
those whose four edges (u,v), (u,v'), (u',v), (u',v') are all present -- the
definition of a butterfly (§2).  Incidences give per-vertex
and per-edge counts.  Vectorised over tuples with numpy; intended for graphs
with at most a few dozen vertices per side.
"""
from __future__ import annotations

import itertools

import numpy as np


def adjacency(n_u, n_v, edges):
    A = np.zeros((n_u, n_v), dtype=bool)
    if len(edges):
        A[edges[:, 0], edges[:, 1]] = True
    return A


def butterflies(n_u, n_v, edges):
    """Returns (total, b_u, b_v, b_e) by enumerating all 4-tuples."""
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    A = adjacency(n_u, n_v, edges)
    eid = -np.ones((n_u, n_v), dtype=np.int64)
    eid[edges[:, 0], edges[:, 1]] = np.arange(len(edges))
    pu = np.array(list(itertools.combinations(range(n_u), 2)), dtype=np.int64).reshape(-1, 2)
    pv = np.array(list(itertools.combinations(range(n_v), 2)), dtype=np.int64).reshape(-1, 2)
    b_u = np.zeros(n_u, np.int64)
    b_v = np.zeros(n_v, np.int64)
    b_e = np.zeros(len(edges), np.int64)
    if len(pu) == 0 or len(pv) == 0:
        return 0, b_u, b_v, b_e
    u1, u2 = pu[:, 0][:, None], pu[:, 1][:, None]
    v1, v2 = pv[:, 0][None, :], pv[:, 1][None, :]
    mask = A[u1, v1] & A[u1, v2] & A[u2, v1] & A[u2, v2]
    iu, iv = np.nonzero(mask)
    a, b = pu[iu, 0], pu[iu, 1]
    c, d = pv[iv, 0], pv[iv, 1]
    for x in (a, b):
        np.add.at(b_u, x, 1)
    for y in (c, d):
        np.add.at(b_v, y, 1)
    for (x, y) in ((a, c), (a, d), (b, c), (b, d)):
        np.add.at(b_e, eid[x, y], 1)
    return int(mask.sum()), b_u, b_v, b_e


def all_graphs(n_u, n_v):
    """Every bipartite graph on n_u x n_v labelled vertices, as edge arrays."""
    cells = [(u, v) for u in range(n_u) for v in range(n_v)]
    for bits in range(1 << len(cells)):
        yield np.array([cells[i] for i in range(len(cells)) if bits >> i & 1], dtype=np.uint32).reshape(-1, 2)
