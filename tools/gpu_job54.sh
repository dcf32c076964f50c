mkdir -p gpurun_out/job54
make -s -C oracle
timeout 900 python -m pytest tests/test_vgg16_gpu.py -q -x -s > gpurun_out/job54/pytest.log 2>&1; tail -3 gpurun_out/job54/pytest.log; grep "relative error" gpurun_out/job54/pytest.log
for B in 1 16 64; do
  timeout 900 python bench.py --workload vgg16-infer --family bf16 --table data/sweeps/vgg16_bf16.csv --batch $B --steps 20 > gpurun_out/job54/vgg16_bf16_b$B.json 2>&1
done
