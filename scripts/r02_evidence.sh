# round-2 evidence: sanitizers, launch list of full pairs, ncu --set full of the heavy kernels
mkdir -p gpurun_out
bash scripts/sanitize.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 1 --warmup 1 --pairs 1 --streams 1 --e2e-streams 1 --e2e-pairs 1 --no-cpu-baseline --no-graph --no-extra-workloads > gpurun_out/r02_launches.log 2>&1
bash scripts/ncu_top.sh dt_rows dt_cols ssd finish weed ssim weights0 collapse0 warp
ls -la gpurun_out | tail -30
