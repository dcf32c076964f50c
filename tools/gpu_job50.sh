mkdir -p gpurun_out/job50
make -s -C oracle
timeout 900 python -m pytest tests/test_dispatch_gpu.py tests/test_cli_gpu.py -q -x > gpurun_out/job50/pytest.log 2>&1; tail -3 gpurun_out/job50/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/job50/smoke.log 2>&1; tail -1 gpurun_out/job50/smoke.log
timeout 900 python -m paper_2008_13145_b200.sweep --set square --family tf32 --out gpurun_out/job50/square_tf32.csv --work gpurun_out/job50/parts 2>&1 | tail -1
head -3 gpurun_out/job50/parts/shard0.csv
