"""bench.py's multi-rank plumbing on CPU (gloo, world size 2): `--gpus 2`
outside torchrun re-launches itself under torch.distributed.run, every rank
runs the same pair assignment / barrier / max-over-ranks / digest gathering
code as the GPU path, and rank 0 alone prints one line with n_gpus == 2."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*extra):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--selftest-cpu", *extra]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    return lines[0]


@pytest.mark.parametrize("mode", [("--pairs", "3"), ("--total-pairs", "13")])
def test_bench_self_launches_two_gloo_ranks(mode):
    line = run_bench("--gpus", "2", *mode)
    assert line["n_gpus"] == 2
    owned = line["pairs_per_rank"]
    flat = [g for part in owned for g in part]
    if mode[0] == "--total-pairs":
        assert line["scaling"] == "strong"
        assert sorted(flat) == list(range(13))          # dist.shard covers every pair once
        assert [len(p) for p in owned] == [7, 6]
    else:
        assert line["scaling"] == "weak"
        assert sorted(flat) == list(range(6))           # --pairs per rank, disjoint
    assert line["ms"] == 11.0                           # max over ranks (10 + rank)
    assert line["checks"]["replicas_identical"]


def test_bench_single_rank_selftest():
    line = run_bench("--gpus", "1", "--pairs", "2")
    assert line["n_gpus"] == 1 and line["pairs_per_rank"] == [[0, 1]]
