"""oracle -- plain CPU oracle for exact butterfly counting.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.  The
product (``paper_1907_08607_b200``) never imports it, and it never imports the
product.  The arithmetic lives in ``oracle.c`` (see its header for the paper
passages each function follows); this file is ctypes marshalling plus the
assembly of the per-side arrays.

Pins (tests/test_oracle_pins.py): Fig. 1 golden values, K_{a,b} closed forms,
brute force over 4-tuples, every bipartite graph up to 4x4, the integer-matmul
identity, the trace identity tr(B^4), invariants, Fig. 2's wedge listing, and
the wedge-count closed form.  No oracle function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

ORC_ERRORS = {1: "ERANGE", 2: "EDUP", 3: "ENOMEM", 4: "EOVERFLOW", 5: "EINVAL"}
RANK_KINDS = {"side": 0, "approx_degree": 1, "degree": 2, "explicit": 3, "approx_codegen": 4}


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _SO, src])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, u32p, u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)
        lib.orc_build.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u32p, ctypes.c_uint64,
                                  ctypes.POINTER(vp)]
        lib.orc_free.argtypes = [vp]
        lib.orc_count.argtypes = [vp, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, u64p, u64p,
                                  u64p, u64p]
        lib.orc_cheap_side.argtypes = [vp]
        lib.orc_vertex.argtypes = [vp, ctypes.c_int, ctypes.c_uint32, u64p]
        lib.orc_edge.argtypes = [vp, u32p, ctypes.c_uint64, u64p]
        lib.orc_rank.argtypes = [vp, ctypes.c_int, u32p]
        lib.orc_wedges.argtypes = [vp, u32p, u64p, u64p]
        lib.orc_h64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.orc_h64.restype = ctypes.c_uint64
        lib.orc_sparsify.argtypes = [ctypes.c_uint32, u32p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                     ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, vp]
        _lib = lib
    return _lib


def _p32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)) if a is not None else None


def _p64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if a is not None else None


def _check(rc):
    if rc != 0:
        raise OracleError(ORC_ERRORS.get(rc, str(rc)))


class OracleGraph:
    """Per-side sorted adjacency of a simple bipartite graph."""

    def __init__(self, n_u: int, n_v: int, edges: np.ndarray):
        self.lib = _load()
        self.n_u, self.n_v = int(n_u), int(n_v)
        self.edges = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
        self.m = self.edges.shape[0]
        h = ctypes.c_void_p()
        _check(self.lib.orc_build(self.n_u, self.n_v, _p32(self.edges), self.m, ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.orc_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def n(self):
        return (self.n_u, self.n_v)

    def cheap_side(self) -> int:
        return int(self.lib.orc_cheap_side(self.h))

    def count_range(self, X: int, x_lo: int, x_hi: int, vertex=True, edge=True):
        """One shard: x in [x_lo, x_hi) of side X.  Returns (bx, by, be, sum_bx)."""
        nX, nY = self.n[X], self.n[1 - X]
        bx = np.zeros(nX, np.uint64) if vertex else None
        by = np.zeros(nY, np.uint64) if vertex else None
        be = np.zeros(self.m, np.uint64) if edge else None
        s = ctypes.c_uint64(0)
        _check(self.lib.orc_count(self.h, X, x_lo, x_hi, _p64(bx), _p64(by), _p64(be), ctypes.byref(s)))
        return bx, by, be, int(s.value)

    def count(self, side: int | None = None, vertex=True, edge=True):
        """Exact counts.  Returns dict(total, b_u, b_v, b_e) (arrays None if not asked).
        side: enumeration side X (None = cheap side)."""
        X = self.cheap_side() if side is None else side
        bx, by, be, s = self.count_range(X, 0, self.n[X], vertex, edge)
        if s % 2:
            raise OracleError("sum of b(x) over a side is odd")
        b_u, b_v = (bx, by) if X == 0 else (by, bx)
        return dict(total=s // 2, b_u=b_u, b_v=b_v, b_e=be, side=X)

    def count_full(self):
        """'Full mode': enumerate both sides literally and
        require that they agree."""
        a = self.count(side=0)
        b = self.count(side=1)
        for k in ("b_u", "b_v", "b_e"):
            if not np.array_equal(a[k], b[k]):
                raise OracleError(f"side-0 and side-1 enumerations disagree on {k}")
        if a["total"] != b["total"]:
            raise OracleError("side-0 and side-1 totals disagree")
        return a

    def count_sharded(self, procs: int | None = None, side: int | None = None, vertex=True, edge=True):
        """The same exact counts as ``count``, computed by ``procs`` forked
        single-threaded workers over disjoint x-ranges of the enumeration side X
        (SURVEY 8(c) step 7).  b(x) and b(e) (edges grouped by their X endpoint)
        are disjoint per shard and written in place into shared memory; the
        centre-rule partials b(y) overlap and are summed here, exactly (u64 with
        a carry check; the C code checks each shard's values).  Shards are cut
        at equal cost sum_{y in N(x)} deg(y), so they finish together."""
        import mmap
        import multiprocessing as mp

        X = self.cheap_side() if side is None else side
        Y = 1 - X
        nX, nY = self.n[X], self.n[Y]
        P = max(1, int(procs or len(os.sched_getaffinity(0))))
        deg_y = np.bincount(self.edges[:, Y], minlength=nY).astype(np.float64)
        cost = np.bincount(self.edges[:, X], weights=deg_y[self.edges[:, Y]], minlength=nX) + 1.0
        csum = np.cumsum(cost)
        cuts = np.searchsorted(csum, np.linspace(0, csum[-1], P + 1)[1:-1]) if nX else np.zeros(0, np.int64)
        bounds = list(zip([0] + [int(c) for c in cuts], [int(c) for c in cuts] + [nX]))
        P = len(bounds)

        def shared(nelem):
            buf = mmap.mmap(-1, max(nelem, 1) * 8)
            return buf, np.frombuffer(buf, np.uint64, count=max(nelem, 1))

        keep = []
        bx = by = be = None
        if vertex:
            b1, bx = shared(nX)
            b2, by = shared(P * nY)
            by = by[:P * nY].reshape(P, nY) if nY else np.zeros((P, 0), np.uint64)
            keep += [b1, b2]
        if edge:
            b3, be = shared(self.m)
            keep.append(b3)
        b4, sums = shared(P)
        b5, rcs = shared(P)
        keep += [b4, b5]

        def work(i):
            lo, hi = bounds[i]
            s = ctypes.c_uint64(0)
            rc = self.lib.orc_count(self.h, X, lo, hi, _p64(bx) if vertex else None,
                                    _p64(by[i]) if vertex and nY else None, _p64(be) if edge else None,
                                    ctypes.byref(s))
            sums[i] = s.value
            rcs[i] = rc

        import warnings
        ctx = mp.get_context("fork")
        ps = [ctx.Process(target=work, args=(i,)) for i in range(P)]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", DeprecationWarning)  # the workers only call the C oracle
            for p in ps:
                p.start()
        for p in ps:
            p.join()
        if any(p.exitcode != 0 for p in ps):
            raise OracleError("oracle shard died")
        for rc in rcs[:P]:
            _check(int(rc))
        total2 = sum(int(s) for s in sums[:P])
        if total2 >= 1 << 64:
            raise OracleError("EOVERFLOW")
        if total2 % 2:
            raise OracleError("sum of b(x) over a side is odd")
        out_y = None
        if vertex:
            out_y = np.zeros(nY, np.uint64)
            for i in range(P):
                nxt = out_y + by[i]
                if (nxt < out_y).any():
                    raise OracleError("EOVERFLOW")
                out_y = nxt
            bx = np.array(bx[:nX])
        if edge:
            be = np.array(be[:self.m])
        del keep
        b_u, b_v = (bx, out_y) if X == 0 else (out_y, bx)
        return dict(total=total2 // 2, b_u=b_u, b_v=b_v, b_e=be, side=X, shards=P)

    def vertex(self, side: int, x: int) -> int:
        out = ctypes.c_uint64(0)
        _check(self.lib.orc_vertex(self.h, side, x, ctypes.byref(out)))
        return int(out.value)

    def edge(self, e: int) -> int:
        out = ctypes.c_uint64(0)
        _check(self.lib.orc_edge(self.h, _p32(self.edges), e, ctypes.byref(out)))
        return int(out.value)

    def rank(self, kind: str, explicit: np.ndarray | None = None) -> np.ndarray:
        """rank[gid] with gid = u or n_u + v (readings Z1-Z4)."""
        n = self.n_u + self.n_v
        r = np.zeros(max(n, 1), np.uint32) if explicit is None else np.ascontiguousarray(explicit, np.uint32).copy()
        _check(self.lib.orc_rank(self.h, RANK_KINDS[kind], _p32(r)))
        return r[:n]

    def wedges(self, rank: np.ndarray):
        """(W, w[gid]) under a ranking: Alg. 2's loop bounds."""
        n = self.n_u + self.n_v
        r = np.ascontiguousarray(rank, np.uint32)
        w = np.zeros(max(n, 1), np.uint64)
        t = ctypes.c_uint64(0)
        _check(self.lib.orc_wedges(self.h, _p32(r), _p64(w), ctypes.byref(t)))
        return int(t.value), w[:n]


def count(n_u, n_v, edges, **kw):
    with OracleGraph(n_u, n_v, edges) as g:
        return g.count(**kw)


def h64(seed: int, x: int) -> int:
    """The sparsifiers' counter-based hash (splitmix64 step of seed + (x+1)*golden)."""
    _load()
    return int(_lib.orc_h64(ctypes.c_uint64(seed & (2**64 - 1)), ctypes.c_uint64(x)))


def sparsify(n_u: int, edges: np.ndarray, method: str, p: float, seed: int) -> np.ndarray:
    """Edge / colorful sparsification (PAPER.md 4.4): the kept edges
    in input order.  Edge: keep e iff h(seed, e) < p*2^64; colour: c = ceil(1/p)
    colours by h(seed ^ salt, gid), keep iff the endpoints share a colour."""
    lib = _load()
    e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
    keep = np.zeros(max(len(e), 1), np.uint8)
    keep_all = int(p >= 1.0)
    thr = 2**64 - 1 if keep_all else int(math.ldexp(p, 64))
    colors = int(math.ceil(1.0 / p))
    _check(lib.orc_sparsify(n_u, _p32(e), len(e), {"edge": 0, "color": 1}[method], ctypes.c_uint64(thr), keep_all,
                            colors, ctypes.c_uint64(seed & (2**64 - 1)), keep.ctypes.data_as(ctypes.c_void_p)))
    return e[keep[:len(e)].astype(bool)]
