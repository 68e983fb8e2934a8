"""bench.py's N>1 rank logic on CPU (gloo, world 2) with the forward mocked:
the global batch is sharded exactly once, every rank sees the same global
images, the NCCL-style logits gather reassembles rank order and matches a
single-process recomputation, per-rank scalars (P, ratio) come back in order."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def test_image_range_is_world_size_independent():
    whole = bench.image_range(0, 70, 8, 8)
    parts = np.concatenate([bench.image_range(0, 23, 8, 8), bench.image_range(23, 64, 8, 8),
                            bench.image_range(64, 70, 8, 8)])
    assert np.array_equal(whole, parts)
    assert not np.array_equal(bench.calib_images(4, 8, 8), whole[:4])  # held-out set


def test_plan_shard_weak_and_strong():
    a = SimpleNamespace(global_batch=None, batch=256)
    assert bench.plan_shard(a, 4, 3) == (1024, 768, 1024, "weak")
    a = SimpleNamespace(global_batch=1024, batch=256)
    spans = [bench.plan_shard(a, 8, r) for r in range(8)]
    assert all(s[0] == 1024 and s[3] == "strong" and s[2] - s[1] == 128 for s in spans)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


W = torch.arange(3 * 5, dtype=torch.float32).reshape(3, 5) / 7.0


def _mock_forward(a, b):
    x = torch.from_numpy(bench.image_range(a, b, 8, 8)).float()
    return x.mean(dim=(1, 2)) @ W


def _worker(rank, world, port, q, g):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        args = SimpleNamespace(global_batch=g, batch=4)
        gb, lo, hi, scaling = bench.plan_shard(args, world, rank)
        local = _mock_forward(lo, hi)
        chk = bench.check_shards(local, gb, world, rank, _mock_forward)
        per = bench.gather_scalars([100 + rank, 0.5, hi - lo])
        q.put((rank, chk, per, (lo, hi)))
    finally:
        dist.destroy_process_group()


def _run(world, g):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, g)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    return res


def test_gloo_world2_shards_gather_and_check():
    res = _run(2, 11)  # ragged: 6 + 5 images
    (r0, chk, per, span0), (r1, chk1, per1, span1) = res
    assert chk1 is None
    assert chk["rows"] == chk["rows_expected"] == 11 and chk["bitwise_equal"] and chk["max_abs_diff"] == 0.0
    assert span0 == (0, 6) and span1 == (6, 11)
    assert per == per1 == [[100.0, 0.5, 6.0], [101.0, 0.5, 5.0]]


def test_gloo_world2_weak_default():
    res = _run(2, None)  # batch 4 per rank -> global 8
    assert res[0][1]["rows"] == 8 and res[0][1]["bitwise_equal"]
