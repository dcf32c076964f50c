mkdir -p gpurun_out/job36
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job36/pytest_gpu.log 2>&1; tail -3 gpurun_out/job36/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/job36/smoke.log 2>&1; tail -1 gpurun_out/job36/smoke.log
