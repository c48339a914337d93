# throughput vs concurrent streams (device value only)
for s in 2 4 6 8; do
  timeout 300 python bench.py --steps 3 --warmup 3 --pairs 16 --streams $s --no-cpu-baseline > gpurun_out/sweep_s$s.log 2>&1
  python3 -c "import json,sys; d=json.loads(open('gpurun_out/sweep_s$s.log').read().strip().splitlines()[-1]); print('streams', $s, round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
