"""One pair split across ranks by row bands (SURVEY.md §8(f)4,
paper_1504_01441_b200/banded.py): every rank must return exactly what the
single-GPU pair returns when it takes the same kernels (the chunk
agg/link/apply column sweep and the dense splat), whatever the number of
ranks, and the reference's result within the usual bars. Ranks are gloo
processes sharing cuda:0 (collectives staged through the host) -- the
NCCL path differs only in the transport."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from golden_util import digest, load, scene_inputs

pytestmark = pytest.mark.gpu

FIELDS = ("composite", "flow", "warped", "valid", "ssim", "matches", "raw_matches", "homography")


def _outputs_digest(res):
    return {f: digest(np.asarray(getattr(res, f))) for f in FIELDS}


def _scene(name="vga_s0"):
    return scene_inputs(load(name))


def _single_pair_same_kernels(ref, src):
    from paper_1504_01441_b200 import _native, pipeline
    lib = _native.lib()
    try:
        _native.check(lib.hdr_set_option(b"dt_cluster_columns", 0))
        _native.check(lib.hdr_set_option(b"dt_sparse_first", 0))
        return pipeline.register_and_fuse(ref, src)
    finally:
        lib.hdr_set_option(b"dt_cluster_columns", 1)
        lib.hdr_set_option(b"dt_sparse_first", 1)


@pytest.mark.parametrize("name", ["vga_s0", "r960_s3"])
def test_banded_one_rank_equals_pair(cuda, name):
    from oracle import hdr_oracle as O
    from paper_1504_01441_b200.banded import register_and_fuse_banded
    ref, src = _scene(name)
    want = _single_pair_same_kernels(ref, src)
    got = register_and_fuse_banded(ref, src)
    assert _outputs_digest(got) == _outputs_digest(want)
    assert got.level_counts == want.level_counts
    o = O.register_and_fuse(ref, src)
    assert np.abs(got.flow - o.flow).max() < 1e-4
    assert np.abs(got.composite - o.composite).max() < 1e-3


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    from paper_1504_01441_b200.banded import register_and_fuse_banded
    ref, src = _scene(name)
    res = register_and_fuse_banded(ref, src)
    got = [None] * world
    dist.all_gather_object(got, _outputs_digest(res))
    if rank == 0:
        q.put(got)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "r960_s3"), (3, "r960_s3"), (5, "qvga_s2")])
def test_banded_ranks_equal_one_rank(cuda, world, name):
    """qvga_s2 (240 rows) over 5 ranks: 64-row bands, the last one empty."""
    from paper_1504_01441_b200.banded import register_and_fuse_banded
    ref, src = _scene(name)
    want = _outputs_digest(register_and_fuse_banded(ref, src))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r, d in enumerate(got):
        assert d == want, (r, [f for f in FIELDS if d[f] != want[f]])


def _nccl_worker(port, name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1",
                      LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda:0"))
    from paper_1504_01441_b200.banded import register_and_fuse_banded
    ref, src = _scene(name)
    q.put(_outputs_digest(register_and_fuse_banded(ref, src)))
    dist.destroy_process_group()


def test_banded_nccl_collectives(cuda):
    """The NCCL path (in-place all-gathers, all-reduce of the histogram) on a
    one-rank group -- the only NCCL group one GPU allows -- gives the same
    bits as no group at all."""
    from paper_1504_01441_b200.banded import register_and_fuse_banded
    name = "vga_rot_s1"
    want = _outputs_digest(register_and_fuse_banded(*_scene(name)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(port, name, q))
    p.start()
    got = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert got == want
