mkdir -p gpurun_out/job10
for L in default exp/libkpgemm_v2.so exp/libkpgemm_bk16.so exp/libkpgemm_bk16w8.so exp/libkpgemm_zz.so; do
  if [ "$L" = default ]; then timeout 600 python tools/exp_f1.py >> gpurun_out/job10/exp.jsonl 2>&1;
  else KPGEMM_LIB=$L timeout 600 python tools/exp_f1.py >> gpurun_out/job10/exp.jsonl 2>&1; fi
done
KPGEMM_LIB=exp/libkpgemm_v2.so timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -2
