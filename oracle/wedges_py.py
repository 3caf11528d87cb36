"""Literal Alg. 1 + Alg. 2 for tiny graphs (pure Python).  TEST INFRASTRUCTURE ONLY.

PREPROCESS (Alg. 1): rename every vertex to its rank and sort
each neighbour list by decreasing rank, storing deg_x(x) and deg_y(x).
GET-WEDGES (Alg. 2): for x1, for i < deg_{x1}(x1), y = N(x1)[i],
for j < deg_{x1}(y), x2 = N(y)[j], emit ((x1, x2), y) (reading Z6: exclusive bounds).
get-freq: group by endpoint pair.

Used only to pin the wedge listing of Fig. fig-count-ex and the
wedge-count definition on tiny cases.  Names are global ids gid = u | n_u + v.
"""
from __future__ import annotations

from collections import Counter


def preprocess(n_u, n_v, edges, rank):
    """Alg. 1: returns (N, deg_self) in rank space, N[r] sorted by decreasing rank."""
    n = n_u + n_v
    N = [[] for _ in range(n)]
    for u, v in edges:
        a, b = rank[int(u)], rank[n_u + int(v)]
        N[a].append(b)
        N[b].append(a)
    for r in range(n):
        N[r].sort(reverse=True)
    # deg_x(x) = #neighbours with rank > rank(x)
    deg_self = [sum(1 for z in N[r] if z > r) for r in range(n)]
    return N, deg_self


def get_wedges(n_u, n_v, edges, rank):
    """Alg. 2 in rank space; returns [((x1, x2), y)] with ids mapped back to gid."""
    n = n_u + n_v
    inv = [0] * n
    for g, r in enumerate(rank):
        inv[r] = g
    N, deg_self = preprocess(n_u, n_v, edges, rank)
    out = []
    for x1 in range(n):
        for i in range(deg_self[x1]):
            y = N[x1][i]
            deg_x1_y = sum(1 for z in N[y] if z > x1)  # deg_{x1}(y)
            for j in range(deg_x1_y):
                x2 = N[y][j]
                out.append(((inv[x1], inv[x2]), inv[y]))
    return out


def get_freq(wedges):
    return Counter(e for e, _ in wedges)
