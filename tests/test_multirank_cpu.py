"""N > 1 host path on CPU: world-size 2 and 3 process groups over gloo (127.0.0.1).

Covers what the multi-GPU path does outside the kernels -- the same helpers
bench.py's N > 1 branch calls (paper_1907_08607_b200/dist.py): the NCCL
bootstrap (rank 0's 128-byte id broadcast over the process group, every rank
joining with it), the max-over-ranks timing reduction,
and the per-rank share of the wedge-sorted start lists (libbf's own deal
function, bf_deal_index, which the kernels call): every start is processed by
exactly one rank and the ranks' wedge loads are balanced.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1907_08607_b200 import bf
        from paper_1907_08607_b200 import dist as bfd
        payload = bytes((np.arange(128) * 7 + 3) % 256) if rank == 0 else None
        got = bfd.broadcast_bytes(payload)
        # bench.py's bootstrap (dist.nccl_comm_for_group) with libbf's NCCL calls
        # stubbed (no GPU here): rank 0 makes the id, every rank joins with it
        made = []
        bf.bf_nccl_unique_id = lambda: (made.append(1), bytes(range(128)))[1]
        bf.bf_nccl_comm_create = lambda uid, r, w, d: ("comm", uid, r, w, d)
        comm = bfd.nccl_comm_for_group(0)
        assert comm == ("comm", bytes(range(128)), rank, world, 0)
        assert len(made) == (1 if rank == 0 else 0)
        mx = bfd.max_over_ranks([rank * 1.5, 10.0 - rank])
        # a wedge-sorted list (descending) with a heavy head, cut into three tier segments
        rng = np.random.default_rng(0)
        w = np.sort(rng.zipf(1.6, 5000).astype(np.int64))[::-1]
        segs = [(0, 40), (40, 900), (900, 5000)]
        mine = [bfd.rank_share(rank, world, t0, t1) for t0, t1 in segs]
        box = [None] * world
        dist.all_gather_object(box, (got, mx, mine))
        if rank == 0:
            q.put((box, w.tolist(), segs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_multirank(world):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, q), nprocs=world, join=True, start_method="spawn")
    box, w, segs = q.get()
    w = np.array(w)
    want = bytes((np.arange(128) * 7 + 3) % 256)
    for r, (got, mx, mine) in enumerate(box):
        assert got == want
        assert mx == [(world - 1) * 1.5, 10.0]
    for si, (t0, t1) in enumerate(segs):
        parts = [box[r][2][si] for r in range(world)]
        allidx = sorted(i for p in parts for i in p)
        assert allidx == list(range(t0, t1)), "every start processed by exactly one rank"
        loads = [int(w[p].sum()) for p in parts]
        # snake dealing over a descending list: loads differ by at most the largest item
        assert max(loads) - min(loads) <= int(w[t0:t1].max())
