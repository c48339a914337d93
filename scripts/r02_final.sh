# round-2 closing evidence on one B200: GPU tests, smoke, bench +
# reference arm, launch list of full pairs, ncu --set full of the heavy kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -30 > gpurun_out/fin_tests.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/fin_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/fin_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv \
  python bench.py --steps 1 --warmup 1 --pairs 1 --streams 1 --e2e-streams 1 --e2e-pairs 1 --no-cpu-baseline --no-graph --no-extra-workloads > gpurun_out/fin_launches.log 2>&1
bash scripts/ncu_top.sh dt_rows dt_cols ssd finish weed ssim weights0 collapse0 warp > gpurun_out/fin_ncu.log 2>&1
tail -3 gpurun_out/fin_tests.log; tail -2 gpurun_out/fin_smoke.log; cat gpurun_out/fin_san.log
python scripts/bench_summary.py gpurun_out/fin_bench.log; tail -c 600 gpurun_out/fin_ref.log
ls gpurun_out
