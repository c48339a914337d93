mkdir -p gpurun_out
HDR_NVCC_FLAGS="-DHDR_FINISH_TIMING" python -m paper_1504_01441_b200.build --force >/dev/null 2>&1
python scripts/one_pair.py 2592 1944 2 2>&1 | tail -4
python -m paper_1504_01441_b200.build --force >/dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --no-extra-workloads --no-cpu-baseline > gpurun_out/gfit_bench.log 2>&1
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/gfit_bench.log") if l.startswith("{")][-1])
print("value", round(d["value"], 1), "lat", round(d["pair_latency_ms"], 3), {k: round(v, 3) for k, v in d["stage_ms"].items()})
PY
