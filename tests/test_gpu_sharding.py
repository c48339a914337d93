"""Sharded runs on the GPU (weeding.py:114-145's "units are
independent"): two gloo ranks in separate processes share cuda:0, each runs
its dist.shard of the pair list through its own BatchRunner (different stream
counts), and the per-pair output digests gathered over the ranks equal those
of one process running every pair -- the result of a pair does not depend on
the rank, stream or order it ran on."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

W, H, N = 320, 240, 5
SEEDS = (2, 7, 9, 11, 4)


FIELDS = ("composite", "flow", "warped", "valid", "ssim", "matches", "raw_matches", "homography", "info")


def _digest(bufs):
    info = bufs.info.cpu().numpy()
    # match buffers are sized for the worst case: only the first m / n rows are outputs
    rows = {"matches": int(info[16]), "raw_matches": int(info[17]),
            "homography": 3 if info[1] else 0}  # no H when the pair did not register
    return tuple(hashlib.sha256(getattr(bufs, f)[:rows[f]].cpu().numpy().tobytes() if f in rows
                                else getattr(bufs, f).cpu().numpy().tobytes()).hexdigest()[:16]
                 for f in FIELDS)


def _run(pairs, streams):
    from paper_1504_01441_b200.pipeline import PairBuffers
    from paper_1504_01441_b200.runner import BatchRunner
    from harness import synth
    r = BatchRunner(W, H, streams=streams)
    dev = []
    for k in pairs:
        st = synth.synth_stack(synth.working_spec(W, H), SEEDS[k])
        dev.append((torch.from_numpy(st.ref).cuda(), torch.from_numpy(st.src).cuda()))
    outs = [PairBuffers(W, H, 0) for _ in pairs]
    r.run_device(dev, outs)
    torch.cuda.synchronize()
    d = {k: _digest(o) for k, o in zip(pairs, outs)}
    r.close()
    return d


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_1504_01441_b200 import dist as hd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    mine = list(hd.shard(N, world, rank))
    d = _run(list(reversed(mine)), streams=1 + rank)  # reversed order, rank-specific streams
    got = [None] * world
    dist.all_gather_object(got, d)
    if rank == 0:
        merged = {}
        for g in got:
            merged.update(g)
        q.put(merged)
    dist.destroy_process_group()


def test_pair_outputs_independent_of_rank_and_stream(cuda):
    alone = _run(list(range(N)), streams=3)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    bad = {k: [f for f, a, b in zip(FIELDS, alone[k], merged[k]) if a != b] for k in alone if alone[k] != merged[k]}
    assert not bad, bad
