# full GPU suite; re-measure the TF32/BF16 tables (and the ResNet-50 simt+tf32 table) after the TMA-store epilogue
mkdir -p gpurun_out/job26
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job26/pytest_gpu.log 2>&1; tail -3 gpurun_out/job26/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/job26/smoke.log 2>&1; tail -2 gpurun_out/job26/smoke.log
S=gpurun_out/job26/sweeps
mkdir -p $S
for spec in "vgg16 tf32" "vgg16 bf16" "resnet50 bf16" "square tf32" "square bf16" "square16k tf32" "square16k bf16" "resnet50 simt+tf32"; do
  set -- $spec
  timeout 2400 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
