mkdir -p gpurun_out/job27
for L in default exp/libkpgemm_w12.so default exp/libkpgemm_w12.so; do
  if [ "$L" = default ]; then timeout 600 python tools/exp_f1.py >> gpurun_out/job27/exp.jsonl 2>&1;
  else KPGEMM_LIB=$L timeout 600 python tools/exp_f1.py >> gpurun_out/job27/exp.jsonl 2>&1; fi
done
