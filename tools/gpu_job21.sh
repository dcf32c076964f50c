mkdir -p gpurun_out/job21
for S in 0 1 2 3 4 5 6 7 8; do
  KPGEMM_FORCE_SLICES=$S timeout 300 python tools/wave_probe.py simt >> gpurun_out/job21/simt.jsonl 2>&1
  KPGEMM_FORCE_SLICES=$S timeout 300 python tools/wave_probe.py bf16 >> gpurun_out/job21/bf16.jsonl 2>&1
done
wc -l gpurun_out/job21/*.jsonl
