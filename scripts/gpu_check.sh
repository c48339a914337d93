# quick GPU check: tests, smoke, short bench, launch list
set -x
timeout 900 python -m pytest tests -m "gpu" -q -p no:cacheprovider -rf 2>&1 | tail -80 > gpurun_out/t_tests.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/t_smoke.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --pairs 8 --no-cpu-baseline > gpurun_out/t_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t_launches.csv python bench.py --steps 1 --warmup 1 --pairs 1 --streams 1 --e2e-pairs 1 --no-cpu-baseline --no-graph > gpurun_out/t_ncu_bench.log 2>&1
tail -5 gpurun_out/t_tests.log; tail -3 gpurun_out/t_smoke.log; tail -3 gpurun_out/t_bench.log
