mkdir -p gpurun_out/job57
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/job57/sanitizer_$tool.log 2>&1
  tail -3 gpurun_out/job57/sanitizer_$tool.log
done
