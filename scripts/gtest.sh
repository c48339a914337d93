# GPU test pass: all -m gpu tests (or the ones named in $1), log under gpurun_out/
mkdir -p gpurun_out
timeout ${T:-1500} python -m pytest ${1:-tests} -m gpu -q -p no:cacheprovider -rf -x 2>&1 | tail -40 > gpurun_out/gtest.log
tail -15 gpurun_out/gtest.log
