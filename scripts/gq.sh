# quick A/B: bench summary line (usage: bash scripts/gq.sh [extra bench args])
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --no-extra-workloads --no-cpu-baseline "$@" > gpurun_out/gq_bench.log 2>&1
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/gq_bench.log") if l.startswith("{")][-1])
print("value", round(d["value"], 1), "lat", round(d["pair_latency_ms"], 3), "e2e", round(d["e2e"]["value"], 1),
      {k: round(v, 3) for k, v in d["stage_ms"].items()}, {k: round(v * 1e3, 1) for k, v in d["kernel_ms"].items()})
PY
