mkdir -p gpurun_out/job22
for S in 0 2 3 4; do
  KPGEMM_FORCE_SLICES=$S timeout 300 python tools/wave_probe.py simt_many >> gpurun_out/job22/simt_many.jsonl 2>&1
done
wc -l gpurun_out/job22/*.jsonl
