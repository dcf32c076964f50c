# re-entry check: smoke, full GPU suite, default bench, reference arm
mkdir -p gpurun_out/job11
make -s -C oracle
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/job11/smoke.log 2>&1; tail -3 gpurun_out/job11/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job11/pytest_gpu.log 2>&1; tail -3 gpurun_out/job11/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/job11/bench.json 2> gpurun_out/job11/bench.err; tail -c 1500 gpurun_out/job11/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/job11/bench_ref.json 2>&1; tail -c 800 gpurun_out/job11/bench_ref.json
