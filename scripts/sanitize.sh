# compute-sanitizer memcheck / racecheck / initcheck over one VGA pair (GPU box)
for tool in memcheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/one_pair.py 640 480 1 \
    > gpurun_out/san_$tool.txt 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.txt)"
done
