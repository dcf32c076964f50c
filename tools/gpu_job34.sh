mkdir -p gpurun_out/job34
for S in 0 1 2 3 4 5 6 7 8; do
  KPGEMM_FORCE_SLICES=$S timeout 600 python tools/wave_probe2.py >> gpurun_out/job34/probe2.jsonl 2>> gpurun_out/job34/err.log
done
wc -l gpurun_out/job34/probe2.jsonl
