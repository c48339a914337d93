"""N>1 host logic on CPU: world_size-2 gloo ranks shard the pair list with no
overlap and agree on the max-over-ranks timing (bench.py's reduction)."""

import os
import socket

import pytest
import torch.multiprocessing as tmp

from paper_1504_01441_b200.dist import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_pairs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist

    from paper_1504_01441_b200 import dist as hd
    hd.init("gloo")
    mine = list(hd.shard(n_pairs, world, rank))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    t = hd.max_over_ranks(10.0 + rank)
    hd.barrier()
    q.put((rank, gathered, t))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_pairs", [16, 17, 3])
def test_gloo_two_ranks_shard_and_max(n_pairs):
    world = 2
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_pairs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, gathered, t in res:
        flat = [i for part in gathered for i in part]
        assert sorted(flat) == list(range(n_pairs))
        assert len(flat) == len(set(flat))
        assert t == 11.0


def test_shard_sizes():
    for n in range(0, 40):
        for world in (1, 2, 4, 8):
            parts = [shard(n, world, r) for r in range(world)]
            assert sum(len(p) for p in parts) == n
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_band_rows_partition():
    """banded.py's row bands: contiguous, whole 32-row blocks, balanced."""
    from paper_1504_01441_b200.banded import band_rows
    for h in (100, 480, 481, 1944, 3000):
        for world in (1, 2, 3, 5, 8):
            bands = [band_rows(h, world, r, 32) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == h
            for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
                assert a1 == b0 and (a0 % 32 == 0 or a0 == h)
            sizes = [b - a for a, b in bands]
            # full bands, then at most one partial band, then empty ones
            full = max(sizes)
            assert sizes == sorted(sizes, reverse=True)
            assert full % 32 == 0 or world == 1 or full == h
            assert sum(0 < sz < full for sz in sizes) <= 1
