# tests + A/B bench of one option (usage: OPT=name bash scripts/g2.sh)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x 2>&1 | tail -30 > gpurun_out/g2_tests.log
tail -3 gpurun_out/g2_tests.log
for v in ${VALS:-1 0}; do
  timeout 600 python bench.py --steps 20 --no-extra-workloads --no-cpu-baseline --option ${OPT:-pdl}=$v > gpurun_out/g2_bench_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
line = [l for l in open(f"gpurun_out/g2_bench_{sys.argv[1]}.log") if l.startswith("{")][-1]
d = json.loads(line)
print(sys.argv[1], "value", round(d["value"], 1), "lat", round(d["pair_latency_ms"], 3), "e2e", round(d["e2e"]["value"], 1),
      {k: round(v, 3) for k, v in d["stage_ms"].items()}, {k: round(v * 1e3, 1) for k, v in d["kernel_ms"].items()})
PY
done
