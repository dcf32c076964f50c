# TF32/BF16 tables after the tail split, ResNet-50 simt+tf32, full GPU suite, TF32 VGG16 inference
mkdir -p gpurun_out/job47/sweeps
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job47/pytest_gpu.log 2>&1; tail -2 gpurun_out/job47/pytest_gpu.log
S=gpurun_out/job47/sweeps
for spec in "vgg16 tf32" "vgg16 bf16" "resnet50 bf16" "square tf32" "square bf16" "square16k tf32" "square16k bf16" "resnet50 simt+tf32"; do
  set -- $spec
  timeout 2400 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
cp $S/vgg16_tf32.csv data/sweeps/vgg16_tf32.csv
for B in 1 16 64; do
  timeout 900 python bench.py --workload vgg16-infer --family tf32 --table data/sweeps/vgg16_tf32.csv --batch $B --steps 20 > gpurun_out/job47/vgg16_tf32_b$B.json 2>&1
done
