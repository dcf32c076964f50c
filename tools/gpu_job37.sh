mkdir -p gpurun_out/job37
for B in 4 64; do
  timeout 900 python bench.py --workload vgg16-infer --batch $B --steps 10 > gpurun_out/job37/vgg16_b$B.json 2>&1; tail -c 250 gpurun_out/job37/vgg16_b$B.json; echo
done
