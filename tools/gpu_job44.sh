mkdir -p gpurun_out/job44
timeout 900 python -m pytest tests/test_tc_gpu.py -q -x > gpurun_out/job44/pytest.log 2>&1; tail -3 gpurun_out/job44/pytest.log
timeout 600 python tools/tc_ab.py 8 > gpurun_out/job44/new.json 2>&1
timeout 600 python tools/tc_ab.py 1 > gpurun_out/job44/cap1.json 2>&1
