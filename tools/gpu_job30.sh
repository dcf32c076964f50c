# GPU suite + SIMT re-sweeps after the 1-3-wave slicing rule, then both bench arms
mkdir -p gpurun_out/job30
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job30/pytest_gpu.log 2>&1; tail -3 gpurun_out/job30/pytest_gpu.log
S=gpurun_out/job30/sweeps
mkdir -p $S
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 5000 > $S/clocks.csv &
SMI=$!
for spec in "vgg16 simt" "resnet50 simt+tf32" "square simt"; do
  set -- $spec
  timeout 2400 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
kill $SMI
timeout 900 python bench.py --table $S/vgg16_simt.csv > gpurun_out/job30/bench.json 2> gpurun_out/job30/bench.err; tail -c 800 gpurun_out/job30/bench.json
