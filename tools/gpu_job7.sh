mkdir -p gpurun_out/job7
make -s -C oracle
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/job7/smoke.log 2>&1; tail -3 gpurun_out/job7/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job7/pytest_gpu.log 2>&1; tail -3 gpurun_out/job7/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/job7/bench.json 2> gpurun_out/job7/bench.err; tail -c 1200 gpurun_out/job7/bench.json
