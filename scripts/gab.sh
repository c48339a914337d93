# kernel A/B after a change: kbench warp sweep, targeted GPU tests, bench per option value
# (usage: OPT=name VALS="a b" TESTS="-k expr" bash scripts/gab.sh)
mkdir -p gpurun_out
timeout 300 python scripts/kbench.py warp > gpurun_out/gab_kbench.log 2>&1; tail -4 gpurun_out/gab_kbench.log
timeout 300 python scripts/fuse_bench.py > gpurun_out/gab_fuse.log 2>&1; tail -2 gpurun_out/gab_fuse.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x ${TESTS:-} 2>&1 | tail -20 > gpurun_out/gab_tests.log
tail -3 gpurun_out/gab_tests.log
OPT=${OPT:-pdl} VALS=${VALS:-1} 
for v in $VALS; do
  timeout 600 python bench.py --steps 20 --no-extra-workloads --no-cpu-baseline --option $OPT=$v > gpurun_out/gab_bench_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
line = [l for l in open(f"gpurun_out/gab_bench_{sys.argv[1]}.log") if l.startswith("{")][-1]
d = json.loads(line)
print(sys.argv[1], "value", round(d["value"], 1), "lat", round(d["pair_latency_ms"], 3), "e2e", round(d["e2e"]["value"], 1),
      {k: round(v, 3) for k, v in d["stage_ms"].items()}, {k: round(v * 1e3, 1) for k, v in d["kernel_ms"].items()})
PY
done
