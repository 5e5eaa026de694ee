"""N>1 host-side path on CPU: two gloo ranks (world_size 2) run the same unit
assignment and reductions bench.py uses under torchrun."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2605_18071_b200.dist import rank_requests, unit_partition


def test_rank_requests_disjoint_cover():
    world, per = 4, 16
    seen = [r for rank in range(world) for r in rank_requests(rank, world, per)]
    assert sorted(seen) == list(range(world * per))


@pytest.mark.parametrize("B,Hkv,world", [(4, 4, 8), (64, 8, 4), (16, 8, 2), (4, 4, 1), (1, 8, 8)])
def test_unit_partition_covers_every_unit_once(B, Hkv, world):
    parts = unit_partition(B, Hkv, world)
    assert len(parts) == world
    units = [(req, h) for rank in parts for (req, h0, h1) in rank for h in range(h0, h1)]
    assert sorted(units) == [(r, h) for r in range(B) for h in range(Hkv)]
    per = B * Hkv // world
    assert all(sum(h1 - h0 for _, h0, h1 in rank) == per for rank in parts)


def test_unit_partition_c4_heads_sharded():
    # BASELINE c4: 4 requests x 4 KV heads over 8 GPUs -> 2 heads of one request per rank (R21)
    parts = unit_partition(4, 4, 8)
    assert parts[0] == [(0, 0, 2)] and parts[1] == [(0, 2, 4)] and parts[7] == [(3, 2, 4)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2605_18071_b200 import dist as kdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        reqs = kdist.rank_requests(rank, world, 3)
        step_ms = 1.0 + rank                     # rank 1 is the slow one
        q.put((rank, reqs, kdist.max_over_ranks(step_ms), kdist.sum_over_ranks(len(reqs))))
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_reduce_like_bench():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0][1] == [0, 1, 2] and res[1][1] == [3, 4, 5]
    for _, _, mx, sm in res:
        assert mx == 2.0 and sm == 6.0            # max-over-ranks time, whole-job token count
