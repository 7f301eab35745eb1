mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize.py > gpurun_out/r2_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_sanitizer_$tool.txt
  tail -4 gpurun_out/r2_sanitizer_$tool.txt
done
