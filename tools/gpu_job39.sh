mkdir -p gpurun_out/job39
make -s -C oracle
timeout 900 python -m pytest tests/test_vgg16_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/job39/pytest.log 2>&1; tail -3 gpurun_out/job39/pytest.log
for B in 1 16 64; do
  timeout 900 python bench.py --workload vgg16-infer --batch $B --steps 20 > gpurun_out/job39/vgg16_b$B.json 2>&1; tail -c 150 gpurun_out/job39/vgg16_b$B.json; echo
done
timeout 600 python tools/exp_f1.py > gpurun_out/job39/exp.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/job39/launches_b16.csv python bench.py --workload vgg16-infer --batch 16 --steps 1 --warmup 1 > /dev/null 2>&1
