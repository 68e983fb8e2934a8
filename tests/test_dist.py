"""N>1 host logic on CPU with gloo, world_size 2 (no GPU): sharding covers the
batch exactly once, the timing reduction is a MAX, and the checking gather
reassembles rows in rank order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_15949_b200.dist import gather_rows, max_over_ranks, shard_range


def test_shard_range_partitions():
    for gb in (1, 7, 256, 1024):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(gb, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == gb
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(10, rank, world)
        rows = torch.arange(lo, hi, dtype=torch.float32).unsqueeze(1).repeat(1, 3)
        allrows = gather_rows(rows)
        m = max_over_ranks(1.5 + rank)
        q.put((rank, allrows[:, 0].tolist(), m))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, rows, m in res:
        assert rows == [float(i) for i in range(10)]
        assert m == 2.5
