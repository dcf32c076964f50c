mkdir -p gpurun_out/job9
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/job9/sanitizer_$tool.log 2>&1
  tail -3 gpurun_out/job9/sanitizer_$tool.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:f1_kernel -s 1 -c 1 -o gpurun_out/job9/dominant python tools/prof_one.py simt 8 8 4 8 16 50176 2304 256 1 2 > gpurun_out/job9/ncu_dom.log 2>&1; tail -2 gpurun_out/job9/ncu_dom.log
