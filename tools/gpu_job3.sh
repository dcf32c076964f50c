# full GPU test suite, bench (both arms), then the remaining sweeps
mkdir -p gpurun_out/job3/sweeps
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job3/pytest_gpu.log 2>&1; tail -5 gpurun_out/job3/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/job3/bench.json 2> gpurun_out/job3/bench.err; tail -c 2500 gpurun_out/job3/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/job3/bench_ref.json 2>&1; cat gpurun_out/job3/bench_ref.json
S=gpurun_out/job3/sweeps
for spec in "vgg16 tf32" "vgg16 bf16" "square tf32" "square bf16" "square16k tf32" "square16k bf16" "resnet50 simt+tf32" "square simt" "resnet50 bf16" "square paper" "resnet50 paper"; do
  set -- $spec
  timeout 1800 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
