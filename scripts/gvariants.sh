# build-time variants on the box: rebuild with each HDR_NVCC_FLAGS set, run
# $CMD (default: the warp kbench + the merge bench), then restore the default
# build (usage: VARIANTS="-DA=1|-DB=2 -DC=3" [CMD="..."] bash scripts/gvariants.sh)
mkdir -p gpurun_out
IFS='|' read -ra VS <<< "${VARIANTS:-}"
CMD=${CMD:-"python scripts/kbench.py warp 2>&1 | grep 'unroll=1:'; python scripts/fuse_bench.py 2>&1 | tail -1"}
for v in "" "${VS[@]}"; do
  echo "=== variant: ${v:-default}" >> gpurun_out/gvar.log
  HDR_NVCC_FLAGS="$v" python -c "from paper_1504_01441_b200 import build as b; b.build(force=True)" >> gpurun_out/gvar.log 2>&1
  timeout 600 bash -c "$CMD" >> gpurun_out/gvar.log 2>&1
done
python -c "from paper_1504_01441_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
cat gpurun_out/gvar.log
