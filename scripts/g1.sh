mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x 2>&1 | tail -60 > gpurun_out/g1_tests.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/g1_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g1_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/g1_ref.log 2>&1
tail -5 gpurun_out/g1_tests.log; tail -3 gpurun_out/g1_smoke.log; tail -c 3000 gpurun_out/g1_bench.log; tail -c 1500 gpurun_out/g1_ref.log
