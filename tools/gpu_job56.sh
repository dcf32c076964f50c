# final round-1 validation: GPU suite, smoke, default bench + reference arm, gemm-layers on TF32/BF16
J=gpurun_out/job56
mkdir -p $J
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > $J/pytest_gpu.log 2>&1; tail -2 $J/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $J/smoke.log 2>&1; tail -1 $J/smoke.log
timeout 900 python bench.py > $J/bench.json 2> $J/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $J/bench_ref.json 2> $J/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --family tf32 --table data/sweeps/vgg16_tf32.csv --no-cpu > $J/bench_tf32.json 2> $J/bench_tf32.err; echo "tf32 rc=$?"
timeout 900 python bench.py --family bf16 --table data/sweeps/vgg16_bf16.csv --no-cpu > $J/bench_bf16.json 2> $J/bench_bf16.err; echo "bf16 rc=$?"; tail -3 $J/bench_bf16.err
