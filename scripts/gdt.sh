# column-sweep A/B: kbench dt at 5MP and 12MP, DT + headline parity tests, bench per dt_cols_tile value
mkdir -p gpurun_out
timeout 300 python scripts/kbench.py dt > gpurun_out/gdt_kbench.log 2>&1; cat gpurun_out/gdt_kbench.log | tail -6
timeout 300 python scripts/kbench.py dt 4000 3000 > gpurun_out/gdt_kbench12.log 2>&1; tail -6 gpurun_out/gdt_kbench12.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -q -p no:cacheprovider -rf -x 2>&1 | tail -15 > gpurun_out/gdt_tests.log
tail -4 gpurun_out/gdt_tests.log
OPT=dt_cols_tile VALS="0 4 2" bash -c 'for v in $VALS; do timeout 600 python bench.py --steps 20 --no-extra-workloads --no-cpu-baseline --option $OPT=$v > gpurun_out/gdt_bench_$v.log 2>&1; python - "$v" <<PY
import json, sys
line = [l for l in open(f"gpurun_out/gdt_bench_{sys.argv[1]}.log") if l.startswith("{")][-1]
d = json.loads(line)
print(sys.argv[1], "value", round(d["value"], 1), "lat", round(d["pair_latency_ms"], 3), {k: round(v, 3) for k, v in d["stage_ms"].items()}, {k: round(v * 1e3, 1) for k, v in d["kernel_ms"].items()}, d.get("parity"))
PY
done'
