# full GPU suite, SIMT slicing probe, then re-measure every SIMT/TF32/BF16 table
mkdir -p gpurun_out/job19
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job19/pytest_gpu.log 2>&1; tail -3 gpurun_out/job19/pytest_gpu.log
timeout 600 python tools/kslice_probe.py 1,8 > gpurun_out/job19/probe.jsonl 2>&1
S=gpurun_out/job19/sweeps
mkdir -p $S
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 5000 > $S/clocks.csv &
SMI=$!
for spec in "vgg16 tf32" "vgg16 bf16" "resnet50 bf16" "square tf32" "square bf16" "square16k tf32" "square16k bf16" "vgg16 simt" "resnet50 simt+tf32" "square simt"; do
  set -- $spec
  timeout 2400 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
kill $SMI
timeout 900 python bench.py --table $S/vgg16_simt.csv > gpurun_out/job19/bench.json 2> gpurun_out/job19/bench.err; tail -c 600 gpurun_out/job19/bench.json
