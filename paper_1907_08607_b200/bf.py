"""Thin ctypes binding of libbf (include/bf.h).  Argument marshalling only:
every step of the counting path runs in libbf's CUDA kernels.  There is no CPU
fallback -- importing this module fails loudly if libbf.so is missing.

Names mirror the C ABI (bf_graph_create, bf_rank, bf_count_total,
bf_count_vertex, bf_count_edge, bf_wedge_count, ...).  Host buffers are numpy
arrays; device buffers are torch CUDA tensors (PyTorch is used only for device
memory, streams and process groups).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BF_LIB selects another in-tree build (libbf_debug.so: device bounds checks)
LIB_PATH = os.path.join(_HERE, os.environ.get("BF_LIB", "libbf.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

BF_OK, BF_EINVAL, BF_ERANGE, BF_EDUP, BF_ENOMEM, BF_ECUDA, BF_ENCCL, BF_ENORANK, BF_EOVERFLOW = range(9)
BF_RANK_SIDE, BF_RANK_APPROX_DEGREE, BF_RANK_DEGREE, BF_RANK_AUTO, BF_RANK_APPROX_CODEGEN = 0, 1, 2, 3, 4
RANK_KINDS = {"side": BF_RANK_SIDE, "approx_degree": BF_RANK_APPROX_DEGREE, "degree": BF_RANK_DEGREE,
              "auto": BF_RANK_AUTO, "approx_codegen": BF_RANK_APPROX_CODEGEN}
RANK_NAMES = {v: k for k, v in RANK_KINDS.items()}
BF_ORIENT_AUTO, BF_ORIENT_LOW, BF_ORIENT_HIGH = 0, 1, 2
ORIENTS = {"auto": BF_ORIENT_AUTO, "low": BF_ORIENT_LOW, "high": BF_ORIENT_HIGH}
BF_FLAG_FORCE_WARP, BF_FLAG_FORCE_CTA, BF_FLAG_SMALL_WINDOW, BF_FLAG_FORCE_DENSE = 0x1, 0x2, 0x4, 0x10
BF_FLAG_SMALL_CHUNK, BF_FLAG_NO_SPLIT, BF_FLAG_UNPACKED_SORT, BF_FLAG_NO_DENSE_ROW = 0x20, 0x40, 0x80, 0x100
BF_FLAG_KEY_BUFFER, BF_FLAG_GRID_JITTER, BF_FLAG_HUB_POS = 0x200, 0x400, 0x800


class bf_options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("nccl_comm", ctypes.c_void_p),
                ("world_rank", ctypes.c_int), ("world_size", ctypes.c_int), ("edges_on_device", ctypes.c_int),
                ("outputs_on_device", ctypes.c_int), ("orient", ctypes.c_int),
                ("test_light_max_wedges", ctypes.c_uint32), ("test_flags", ctypes.c_uint32),
                ("virtual_world", ctypes.c_int)]


_vp, _u32p, _u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)
_sig = {
    "bf_options_default": (None, [ctypes.POINTER(bf_options)]),
    "bf_graph_create": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, _vp, ctypes.c_uint64,
                                       ctypes.POINTER(bf_options), ctypes.POINTER(_vp)]),
    "bf_rank": (ctypes.c_int, [_vp, ctypes.c_int]),
    "bf_count_total": (ctypes.c_int, [_vp, _vp]),
    "bf_count_vertex": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "bf_count_edge": (ctypes.c_int, [_vp, _vp, _vp]),
    "bf_wedge_count": (ctypes.c_int, [_vp, _u64p]),
    "bf_last_stats": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float), _u64p]),
    "bf_rank_info": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), _u64p]),
    "bf_sparsify": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, _vp, ctypes.c_uint64, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_uint64, _vp, _u64p, ctypes.POINTER(bf_options)]),
    "bf_launch_count": (ctypes.c_uint64, [_vp]),
    "bf_deal_index": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                        ctypes.c_uint64]),
    "bf_export_csr": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bf_rank_shares": (ctypes.c_int, [_vp, ctypes.c_int, _u64p]),
    "bf_approx_total": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, _vp, ctypes.c_uint64, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_uint64, ctypes.POINTER(bf_options),
                                       ctypes.POINTER(ctypes.c_double), _u64p, _u64p]),
    "bf_nccl_unique_id": (ctypes.c_int, [_vp]),
    "bf_nccl_comm_create": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]),
    "bf_nccl_comm_destroy": (ctypes.c_int, [_vp]),
    "bf_graph_destroy": (None, [_vp]),
    "bf_release_device_cache": (ctypes.c_int, [ctypes.c_int]),
    "bf_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "bf_last_error": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    if os.environ.get("BF_LIB") and not hasattr(_lib, _name):
        continue  # an older build under A/B comparison (tools/ab.sh) may lack newer entry points
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args

EXPORTED = tuple(_sig)


class BFError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.bf_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_lib.bf_status_str(status).decode()} ({msg})")


def _check(st, where):
    if st != BF_OK:
        raise BFError(st, where)


def _ptr(x):
    """Address of a numpy array or torch tensor (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()  # torch tensor


def _on_device(x) -> bool:
    return x is not None and not isinstance(x, np.ndarray) and getattr(x, "is_cuda", False)


def bf_options_default() -> bf_options:
    o = bf_options()
    _lib.bf_options_default(ctypes.byref(o))
    return o


def bf_graph_create(n_u: int, n_v: int, edges, opt: bf_options | None = None):
    """edges: uint32 [m, 2] numpy array (host) or torch int32/uint32 CUDA tensor (device)."""
    o = opt if opt is not None else bf_options_default()
    if _on_device(edges):
        o.edges_on_device = 1
        m = int(edges.shape[0]) if edges.dim() == 2 else int(edges.numel() // 2)
    else:
        edges = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
        m = edges.shape[0]
    h = ctypes.c_void_p()
    _check(_lib.bf_graph_create(n_u, n_v, _ptr(edges), m, ctypes.byref(o), ctypes.byref(h)), "bf_graph_create")
    return h


def bf_rank(g, kind) -> None:
    k = RANK_KINDS[kind] if isinstance(kind, str) else int(kind)
    _check(_lib.bf_rank(g, k), "bf_rank")


def bf_count_total(g, out=None) -> int:
    """Global count.  out: optional 1-element uint64 buffer (host numpy or device tensor
    when the graph was created with outputs_on_device)."""
    buf = out if out is not None else np.zeros(1, np.uint64)
    _check(_lib.bf_count_total(g, _ptr(buf)), "bf_count_total")
    return int(buf[0]) if isinstance(buf, np.ndarray) else None


def bf_count_vertex(g, out_u, out_v, total=None) -> None:
    _check(_lib.bf_count_vertex(g, _ptr(out_u), _ptr(out_v), _ptr(total)), "bf_count_vertex")


def bf_count_edge(g, out_e, total=None) -> None:
    _check(_lib.bf_count_edge(g, _ptr(out_e), _ptr(total)), "bf_count_edge")


def bf_wedge_count(g) -> int:
    w = ctypes.c_uint64(0)
    _check(_lib.bf_wedge_count(g, ctypes.byref(w)), "bf_wedge_count")
    return int(w.value)


def bf_rank_info(g):
    """(ranking in effect, [w_side, w_approx_degree, w_degree, w_approx_codegen]) -- the w's only
    after BF_RANK_AUTO."""
    k = ctypes.c_int(0)
    w = (ctypes.c_uint64 * 4)()
    _check(_lib.bf_rank_info(g, ctypes.byref(k), w), "bf_rank_info")
    return RANK_NAMES[k.value], [int(x) for x in w]


BF_SPARSIFY_EDGE, BF_SPARSIFY_COLOR = 0, 1
SPARSIFY_METHODS = {"edge": BF_SPARSIFY_EDGE, "color": BF_SPARSIFY_COLOR}


def bf_sparsify(n_u: int, n_v: int, edges, method, p: float, seed: int, opt: bf_options | None = None):
    """Device edge filter of approximate counting.  Host numpy in,
    host numpy out (the kept edges in input order)."""
    o = opt if opt is not None else bf_options_default()
    e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
    out = np.zeros((max(e.shape[0], 1), 2), np.uint32)
    k = ctypes.c_uint64(0)
    mth = SPARSIFY_METHODS[method] if isinstance(method, str) else int(method)
    _check(_lib.bf_sparsify(n_u, n_v, _ptr(e), e.shape[0], mth, float(p), int(seed) & (2**64 - 1), _ptr(out),
                            ctypes.byref(k), ctypes.byref(o)), "bf_sparsify")
    return out[:int(k.value)]


def bf_approx_total(n_u: int, n_v: int, edges, method, p: float, seed: int = 0, opt: bf_options | None = None):
    """Approximate total count by sparsification, all in libbf.
    Returns (estimate, exact count of the sparsified graph, its edge count)."""
    o = opt if opt is not None else bf_options_default()
    if _on_device(edges):
        o.edges_on_device = 1
        m = int(edges.numel() // 2)
    else:
        edges = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
        m = edges.shape[0]
    est, t, km = ctypes.c_double(0), ctypes.c_uint64(0), ctypes.c_uint64(0)
    mth = SPARSIFY_METHODS[method] if isinstance(method, str) else int(method)
    _check(_lib.bf_approx_total(n_u, n_v, _ptr(edges), m, mth, float(p), int(seed) & (2**64 - 1), ctypes.byref(o),
                                ctypes.byref(est), ctypes.byref(t), ctypes.byref(km)), "bf_approx_total")
    return float(est.value), int(t.value), int(km.value)


def approx_total(n_u: int, n_v: int, edges, p: float, method="edge", seed: int = 0) -> float:
    """Unbiased estimate of the total butterfly count (bf_approx_total)."""
    return bf_approx_total(n_u, n_v, edges, method, p, seed)[0]


def bf_last_stats(g):
    """(kernel_ms, call_ms, pairs) of the last bf_count_* on g."""
    a, b, p = ctypes.c_float(0), ctypes.c_float(0), ctypes.c_uint64(0)
    _check(_lib.bf_last_stats(g, ctypes.byref(a), ctypes.byref(b), ctypes.byref(p)), "bf_last_stats")
    return float(a.value), float(b.value), int(p.value)


def bf_launch_count(g) -> int:
    return int(_lib.bf_launch_count(g))


def bf_deal_index(q: int, rank: int, world: int, t0: int, t1: int) -> int:
    return int(_lib.bf_deal_index(q, rank, world, t0, t1))


def bf_rank_shares(g, world: int) -> list[int]:
    """Wedges each of `world` ranks would process under the current plan."""
    w = (ctypes.c_uint64 * max(world, 1))()
    _check(_lib.bf_rank_shares(g, world, w), "bf_rank_shares")
    return [int(x) for x in w[:world]]


def bf_export_csr(g, n: int, m: int):
    rid = np.zeros(max(n, 1), np.uint32)
    off = np.zeros(n + 1, np.uint32)
    nbr = np.zeros(max(2 * m, 1), np.uint32)
    pos = np.zeros(max(2 * m, 1), np.uint32)
    hi = np.zeros(max(n, 1), np.uint32)
    ws = np.zeros(max(n, 1), np.uint64)
    _check(_lib.bf_export_csr(g, _ptr(rid), _ptr(off), _ptr(nbr), _ptr(pos), _ptr(hi), _ptr(ws)), "bf_export_csr")
    return dict(rid_of_gid=rid[:n], off=off, nbr=nbr[:2 * m], pos=pos[:2 * m], hi=hi[:n], wstart=ws[:n])


def bf_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.bf_nccl_unique_id(buf), "bf_nccl_unique_id")
    return bytes(buf)


def bf_nccl_comm_create(uid: bytes, rank: int, world: int, device: int):
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    c = ctypes.c_void_p()
    _check(_lib.bf_nccl_comm_create(buf, rank, world, device, ctypes.byref(c)), "bf_nccl_comm_create")
    return c


def bf_nccl_comm_destroy(comm) -> None:
    _check(_lib.bf_nccl_comm_destroy(comm), "bf_nccl_comm_destroy")


def bf_graph_destroy(g) -> None:
    _lib.bf_graph_destroy(g)


def bf_release_device_cache(device: int = 0) -> None:
    _check(_lib.bf_release_device_cache(device), "bf_release_device_cache")


class ButterflyGraph:
    """Convenience owner of a bf_graph handle (host numpy in, host numpy out)."""

    def __init__(self, n_u: int, n_v: int, edges, rank: str | None = "degree", **opts):
        o = bf_options_default()
        for k, v in opts.items():
            if k == "orient" and isinstance(v, str):
                v = ORIENTS[v]
            setattr(o, k, v)
        self.n_u, self.n_v = int(n_u), int(n_v)
        self.m = int(edges.shape[0])
        self.opt = o
        self.h = bf_graph_create(n_u, n_v, edges, o)
        if rank is not None:
            bf_rank(self.h, rank)

    def rank(self, kind: str):
        bf_rank(self.h, kind)

    def total(self) -> int:
        return bf_count_total(self.h)

    def vertex(self):
        bu = np.zeros(max(self.n_u, 1), np.uint64)
        bv = np.zeros(max(self.n_v, 1), np.uint64)
        t = np.zeros(1, np.uint64)
        bf_count_vertex(self.h, bu, bv, t)
        return bu[:self.n_u], bv[:self.n_v], int(t[0])

    def edge(self):
        be = np.zeros(max(self.m, 1), np.uint64)
        t = np.zeros(1, np.uint64)
        bf_count_edge(self.h, be, t)
        return be[:self.m], int(t[0])

    def wedges(self) -> int:
        return bf_wedge_count(self.h)

    def rank_info(self):
        return bf_rank_info(self.h)

    def export_csr(self):
        return bf_export_csr(self.h, self.n_u + self.n_v, self.m)

    def close(self):
        if self.h:
            bf_graph_destroy(self.h)
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
