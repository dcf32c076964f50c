mkdir -p gpurun_out/job49
for B in 1 16 64; do
  timeout 900 python bench.py --workload vgg16-infer --batch $B --steps 20 > gpurun_out/job49/vgg16_b$B.json 2>&1
  timeout 900 python bench.py --workload vgg16-infer --family tf32 --table data/sweeps/vgg16_tf32.csv --batch $B --steps 20 > gpurun_out/job49/vgg16_tf32_b$B.json 2>&1
done
