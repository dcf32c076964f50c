mkdir -p gpurun_out/job5
for L in default exp/libkpgemm_ilp8.so exp/libkpgemm_ilp16.so exp/libkpgemm_w8.so; do
  if [ "$L" = default ]; then timeout 600 python tools/exp_f1.py >> gpurun_out/job5/exp.jsonl 2>&1;
  else KPGEMM_LIB=$L timeout 600 python tools/exp_f1.py >> gpurun_out/job5/exp.jsonl 2>&1; fi
done
timeout 600 python -m pytest tests/test_tc_gpu.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --workload vgg16-infer --batch 16 > gpurun_out/job5/bench_vgg16.json 2> gpurun_out/job5/bench_vgg16.err; tail -c 1500 gpurun_out/job5/bench_vgg16.json
timeout 900 python bench.py --workload vgg16-infer --batch 1 --steps 50 > gpurun_out/job5/bench_vgg16_b1.json 2>&1; tail -c 600 gpurun_out/job5/bench_vgg16_b1.json
