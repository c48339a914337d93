#!/usr/bin/env python
"""Benchmark: 5MP two-exposure pairs/sec registered+merged (BASELINE.json).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU). Pairs are independent,
so each rank owns its own resident batch: per-GPU work is fixed ("weak"
scaling) and no collective touches the data path (timings are max-reduced
over ranks with one tiny all-reduce after the timed region).

A step = one batch of `--pairs` 5MP pairs per GPU (synthetic scenes of
SURVEY.md §8(d) C2, rendered on the host, resident in HBM, each pair its own
buffers so the batch (~1.9 GB of inputs) is far larger than the 126 MB L2).
`e2e` is the same metric through the public batch API (runner.BatchRunner
.run_host) with pinned host inputs: H2D of both frames and D2H of the
composite + verdict words happen inside the timed region.

--impl reference times the CPU oracle port of the reference (oracle/, the
reference itself is pure Python and cannot travel to this box) on all host
cores: one pair per process per step.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W5, H5 = 2592, 1944
METRIC = "5MP 2-exposure pairs/sec registered+merged (1/2/4/8 B200) vs host-CPU ref"
WORKLOAD = "5MP (2592x1944) two-exposure pair, registered + merged (BASELINE configs[1])"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pairs", type=int, default=16, help="resident pairs per GPU per step")
    ap.add_argument("--streams", type=int, default=8, help="compute streams of the device-resident runs")
    ap.add_argument("--e2e-streams", type=int, default=8, help="compute streams of the host-buffer runs")
    ap.add_argument("--scenes", type=int, default=4, help="distinct synthetic scenes")
    ap.add_argument("--e2e-pairs", type=int, default=32, help="pairs per end-to-end step (32 amortises the H2D ramp-up and D2H drain at step boundaries: 406 vs 395 pairs/s f32, 799 vs 764 png8)")
    ap.add_argument("--width", type=int, default=W5)
    ap.add_argument("--height", type=int, default=H5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="hdr_set_option before the run (tuning hooks, e.g. dt_cols_grid_div=2)")
    return ap.parse_args()


# ------------------------------------------------------------------ scenes
def _render(args):
    from harness import synth
    w, h, seed = args
    st = synth.synth_stack(synth.working_spec(w, h), seed)
    return st.ref, st.src


def render_scenes(n, w, h, base_seed):
    jobs = [(w, h, base_seed + i) for i in range(n)]
    with mp.get_context("fork").Pool(min(n, os.cpu_count() or 1)) as pool:
        return pool.map(_render, jobs)


# ------------------------------------------------------------------ CPU reference
_CPU_PAIRS = None


def _cpu_pair(i):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import hdr_oracle as O
    ref, src = _CPU_PAIRS[i % len(_CPU_PAIRS)]
    t = time.perf_counter()
    out = O.register_and_fuse(ref, src)
    return time.perf_counter() - t, len(out.matches)


def cpu_pool(pairs, procs):
    global _CPU_PAIRS
    _CPU_PAIRS = pairs
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    return mp.get_context("fork").Pool(procs)


def cpu_step(pool, procs):
    t = time.perf_counter()
    res = pool.map(_cpu_pair, range(procs), chunksize=1)
    return time.perf_counter() - t, res


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.path = index, None, f"/tmp/hdr_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ roofline bookkeeping
def stage_bytes(w, h, passes=3):
    """HBM bytes each stage must move per pair."""
    P = w * h
    return {
        # both RGB frames in; lum_ref f32, q_src u8, eq_src f32, pyramids out
        "raster": P * (24 + 4 + 1 + 4) + 2 * 4 * P // 3,
        # splat memsets (3 f64 planes), then per pass a row sweep and a column
        # sweep pair, each reading the guide (4 B) and the 3 f64 planes (24 B)
        # and writing the planes (24 B); the last column pass writes the f32
        # flow (8 B) instead of the planes
        "dt_filter": P * 24 + passes * 2 * P * 52 - P * 16,
        # warp_image: flow 8 + src 12 in; warped 12, valid 1, q 1 out
        "finalize_warp": P * (8 + 12 + 12 + 1 + 1),
        "ssim": P * (4 + 1 + 4),
        # SURVEY.md §8(d) merge: ref 12, warped 12, SSIM 4, valid 1, composite 12
        "fuse": P * 41,
    }


def kernel_bytes(w, h, passes=3):
    """Algorithmic HBM bytes per pair of each probed kernel family (all its
    launches in one pair) and the launch count."""
    P = w * h
    return {
        # read guide 4 + 3 f64 planes 24, write the planes 24
        "dt_rows": (passes * P * 52, passes),
        # same per column sweep pair; the last one writes the f32 flow (8)
        "dt_cols": ((passes - 1) * P * 52 + P * 36, passes),
        # flow 8 + src 12 in; warped 12, valid 1, q 1 out
        "warp": (P * 34, 1),
        # lum_ref 4 + q(warped) 1 in, ssim 4 out
        "ssim": (P * 9, 1),
        # ref 12, warped 12, ssim 4, valid 1 in; weights 8 + level-1 Gaussian (8 ch / 4) 8 out
        "fuse_weights0": (P * 45, 1),
        # ref 12, warped 12, weights 8, level-1 G (8 ch / 4) 8 + C (3 ch / 4) 3 in; composite 12 out
        "fuse_collapse0": (P * 55, 1),
    }


def peaks():
    """HBM peak for the roofline: the driver-measured STREAM-style copy
    bandwidth (MEASURED_PEAKS.json `hbm_gbs`), else the profiling guide's
    6.65 TB/s fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            v = float(json.load(f)["hbm_gbs"])
        if v > 0:
            return v, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, ValueError, KeyError, TypeError):
        pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch, by kernel
    family, from the committed ncu --set full captures (profiles/)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        return json.load(open(path))
    return {}


# ------------------------------------------------------------------ arms
def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def emit(obj):
    print(json.dumps(obj), flush=True)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    procs = min(os.cpu_count() or 1, 16)
    scenes = render_scenes(min(args.scenes, procs), args.width, args.height, 0)
    pool = cpu_pool(scenes, procs)
    # one step = one 5MP pair per host core (~13 s of wall on this box); the
    # step counts are capped so the whole run stays within a few minutes
    warm, steps = min(args.warmup, 1), max(1, min(args.steps, 8))
    for _ in range(warm):
        cpu_step(pool, procs)
    t0 = time.perf_counter()
    for _ in range(steps):
        cpu_step(pool, procs)
    dt = time.perf_counter() - t0
    pool.close()
    value = procs * steps / dt
    sample = (f"{procs} synthetic {args.width}x{args.height} pairs per step, one per process "
              f"(oracle port of hdrflow.register_and_fuse, OMP/OpenBLAS threads = 1); "
              f"steps capped at 8 and warm-up at 1 to bound the run")
    emit({"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
          "steps": steps, "warmup": warm, "steps_requested": args.steps,
          "warmup_requested": args.warmup, "ms_per_step": 1e3 * dt / steps,
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
          "dtype": "f32/f64", "data": "synthetic",
          "config": {"workload": WORKLOAD, "width": args.width, "height": args.height,
                     "pairs_per_step": procs, "parallelism": "process per core"},
          "impl": "reference",
          "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": procs, "kind": "port",
                           "sample": sample},
          "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 0}})


def run_ours(args):
    rank, world, local = dist_env()
    cpu_base = None
    scenes = render_scenes(args.scenes, args.width, args.height, 1000 * rank)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = min(os.cpu_count() or 1, 16)
        pool = cpu_pool(scenes, procs)
        dt, res = cpu_step(pool, procs)
        pool.close()
        cpu_base = {"value": procs / dt, "unit": "pairs/s", "cores": procs, "kind": "port",
                    "sample": f"{procs} {args.width}x{args.height} pairs, one per process, "
                              f"{dt:.1f} s wall (oracle port of the reference)"}

    import torch
    import torch.distributed as dist

    from paper_1504_01441_b200.pipeline import PairBuffers, PipelineParams
    from paper_1504_01441_b200.runner import BatchRunner

    from paper_1504_01441_b200 import dist as hd
    from paper_1504_01441_b200 import _native as _nat
    for opt in args.option:
        name, val = opt.split("=")
        _nat.check(_nat.lib().hdr_set_option(name.encode(), int(val)))
    torch.cuda.set_device(local)
    if world > 1:
        hd.init("nccl", local)
    dev = f"cuda:{local}"
    w, h, B = args.width, args.height, args.pairs
    pairs = []
    for k in range(B):
        ref, src = scenes[k % len(scenes)]
        pairs.append((torch.from_numpy(ref).to(dev), torch.from_numpy(src).to(dev)))
    outs = [PairBuffers(w, h, local) for _ in range(B)]
    runner = BatchRunner(w, h, streams=args.streams, params=PipelineParams(), device=local,
                         graph=not args.no_graph)
    from paper_1504_01441_b200 import _native
    nst = _native.NUM_STAGES
    probes = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nst)] for _ in range(B)]
    for evs in probes:
        for e in evs:
            e.record()
    torch.cuda.synchronize()

    def step():
        cur = torch.cuda.current_stream()
        for s in runner.streams:
            s.wait_stream(cur)
        for k in range(B):
            runner.set_probes(k, probes[k])
            runner.enqueue(k, pairs[k][0], pairs[k][1], outs[k])
        for s in runner.streams:
            cur.wait_stream(s)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    infos = [o.info.cpu().numpy() for o in outs]
    ok = all(int(i[0]) == 0 for i in infos)
    by_scene = {}
    for k, i in enumerate(infos):
        by_scene.setdefault(k % len(scenes), set()).add(tuple(i[:18].tolist()))
    consistent = all(len(v) == 1 for v in by_scene.values())

    clocks = Clocks(local)
    hd.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step()
    t1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = hd.max_over_ranks(t0.elapsed_time(t1), device=dev)
    hd.barrier()
    # per-stage durations of the last timed step (probes inside the graphs);
    # with 4 streams in flight these include time-sharing with other pairs
    stage_ms_conc = {}
    for s_i, name in enumerate(_native.STAGES):
        v = [probes[k][2 * s_i].elapsed_time(probes[k][2 * s_i + 1]) for k in range(B)]
        stage_ms_conc[name] = statistics.mean(v)
    kernels_per_pair = runner.graph_kernels()
    # isolated stage and kernel times: the same pipeline, one pair at a time
    # on one stream, events recorded on that stream between the stages and
    # around every launch of the probed kernel families
    NI = 3
    iso = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nst)] for _ in range(NI)]
    kfam = _native.KPROBES
    kev = [[[torch.cuda.Event(enable_timing=True) for _ in range(16)] for _ in kfam] for _ in range(NI)]
    for evs in iso + [e for run in kev for e in run]:
        for e in evs:
            e.record()
    torch.cuda.synchronize()
    s0 = runner.streams[0]
    for j in range(NI):
        runner.set_probes(0, iso[j])
        for f in range(len(kfam)):
            runner.set_kernel_probes(0, f, kev[j][f])
        s0.wait_stream(torch.cuda.current_stream())
        runner.enqueue(0, pairs[j % B][0], pairs[j % B][1], outs[0])
        torch.cuda.current_stream().wait_stream(s0)
        torch.cuda.synchronize()
    runner.set_probes(0, None)
    for f in range(len(kfam)):
        runner.set_kernel_probes(0, f, None)
    stage_ms = {}
    for s_i, name in enumerate(_native.STAGES):
        stage_ms[name] = statistics.median(
            iso[j][2 * s_i].elapsed_time(iso[j][2 * s_i + 1]) for j in range(NI))
    # single-pair latency, device-resident inputs: first stage start to last stage end
    pair_latency_ms = statistics.median(iso[j][0].elapsed_time(iso[j][2 * nst - 1]) for j in range(NI))
    kb = kernel_bytes(w, h)
    kernel_ms = {}
    for f, name in enumerate(kfam):
        n = kb[name][1]
        kernel_ms[name] = statistics.median(
            sum(kev[j][f][2 * i].elapsed_time(kev[j][f][2 * i + 1]) for i in range(n))
            for j in range(NI))

    # ---- end to end through the public batch API (host buffers); the host
    # link is the bottleneck (--e2e-streams may differ from --streams)
    E = args.e2e_pairs
    if args.e2e_streams != args.streams:
        runner.close()
        runner = BatchRunner(w, h, streams=args.e2e_streams, params=PipelineParams(), device=local,
                             graph=not args.no_graph)
    # one pinned copy per distinct scene (every pair still moves its own
    # 121 MB H2D each step); outputs are distinct per pair
    pinned = [(torch.from_numpy(ref).pin_memory(), torch.from_numpy(src).pin_memory()) for ref, src in scenes]
    hpairs = [pinned[k % len(pinned)] for k in range(E)]
    hout = [(torch.empty((h, w, 3), dtype=torch.float32).pin_memory(),
             torch.empty((_native.INFO_WORDS,), dtype=torch.int32).pin_memory()) for _ in range(E)]
    runner.set_probes(0, None)
    for k in range(len(runner.streams)):
        runner.set_probes(k, None)
    for _ in range(max(args.warmup, 1)):
        runner.run_host(hpairs, hout)
    torch.cuda.synchronize()
    hd.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h2d = d2h = 0
    for _ in range(args.steps):
        a, b = runner.run_host(hpairs, hout)
        h2d, d2h = a, b
    e1.record()
    torch.cuda.synchronize()
    e2e_ok = all(int(x[1][0]) == 0 for x in hout)
    ems = hd.max_over_ranks(e0.elapsed_time(e1), device=dev)

    # ---- end to end on the file path: the same scenes as
    # 8-bit PNG samples (what run_hdr reads), raw bytes over PCIe, the 8-bit
    # composite (save_png's samples) back
    q8 = lambda a: np.clip(np.floor(a.astype(np.float64) * 255.0 + 0.5), 0, 255).astype(np.uint8)
    rpairs = []
    for k in range(E):
        ref, src = scenes[k % len(scenes)]
        rpairs.append((torch.from_numpy(q8(ref)).pin_memory(), torch.from_numpy(q8(src)).pin_memory()))
    rout = [(torch.empty((h, w, 3), dtype=torch.uint8).pin_memory(),
             torch.empty((_native.INFO_WORDS,), dtype=torch.int32).pin_memory()) for _ in range(E)]
    for _ in range(max(args.warmup, 1)):
        runner.run_host_raw(rpairs, rout, 8)
    torch.cuda.synchronize()
    hd.barrier()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record()
    rh2d = rd2h = 0
    for _ in range(args.steps):
        rh2d, rd2h = runner.run_host_raw(rpairs, rout, 8)
    r1.record()
    torch.cuda.synchronize()
    raw_ok = all(int(x[1][0]) == 0 for x in rout)
    rms = hd.max_over_ranks(r0.elapsed_time(r1), device=dev)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    value = world * B * args.steps / (ms / 1e3)
    e2e_value = world * E * args.steps / (ems / 1e3)
    png8_value = world * E * args.steps / (rms / 1e3)
    peak, peak_src = peaks()
    traffic_all = ncu_traffic()

    def kroof(name):
        nbytes, n = kb[name]
        t = kernel_ms[name] / 1e3
        a = nbytes / t / 1e9
        tr = traffic_all.get(name)
        return {"kernel": name, "launches_per_pair": n, "bytes_per_launch": nbytes / n,
                "us_per_launch": 1e3 * kernel_ms[name] / n, "achieved": a, "frac": a / peak,
                "traffic": tr}
    dom = max(kernel_ms, key=lambda k: kernel_ms[k])
    d = kroof(dom)
    sb = stage_bytes(w, h)

    def sroof(stage):
        a = sb[stage] / (stage_ms[stage] / 1e3) / 1e9
        return {"stage": stage, "achieved": a, "frac": a / peak, "bytes": sb[stage],
                "ms": stage_ms[stage]}
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "width": w, "height": h, "pairs_per_step_per_gpu": B,
                   "global_pairs_per_step": B * world, "streams": args.streams,
                   "e2e_streams": args.e2e_streams,
                   "distinct_scenes": len(scenes), "graph": not args.no_graph,
                   "options": args.option,
                   "l2": "inputs larger than L2 (each pair 121 MB, %d resident pairs)" % B,
                   "parallelism": f"pair-sharded x{world}, no collective"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": d["achieved"], "peak": peak,
                     "unit": "GB/s", "frac": d["frac"], "traffic": d["traffic"],
                     "bytes_per_launch": d["bytes_per_launch"],
                     "us_per_launch": d["us_per_launch"], "launches_per_pair": d["launches_per_pair"],
                     "peak_source": peak_src,
                     "note": "dominant kernel by device time per pair; achieved = algorithmic "
                             "bytes per launch (DESIGN.md §4) / mean launch duration, CUDA events "
                             "on the launching stream around each launch (kernel probes), pairs "
                             "run one at a time after the timed region; traffic = ncu dram bytes "
                             "per launch (profiles/)"},
        "kernel_rooflines": {k: kroof(k) for k in kernel_ms},
        "stage_rooflines": {k: sroof(k) for k in ("dt_filter", "finalize_warp", "fuse")},
        "pair_latency_ms": pair_latency_ms,
        "stage_ms": stage_ms, "stage_ms_concurrent": stage_ms_conc, "kernel_ms": kernel_ms,
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "pairs_per_step": E},
        "e2e_png8": {"value": png8_value, "unit": "pairs/s", "h2d_bytes_per_step": rh2d,
                     "d2h_bytes_per_step": rd2h, "pairs_per_step": E,
                     "note": "file path (run_hdr): the same scenes as 8-bit PNG samples, "
                             "raw uint8 H2D, device decode, pair graph, 8-bit composite D2H"},
        "gpu_launches": kernels_per_pair * B * args.steps,
        "kernels_per_pair": kernels_per_pair,
        "clocks": clk,
        "checks": {"all_registered": ok, "replicas_identical": consistent, "e2e_ok": e2e_ok,
                   "e2e_png8_ok": raw_ok},
    }
    if cpu_base is not None:
        line["cpu_baseline"] = cpu_base
    emit(line)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
