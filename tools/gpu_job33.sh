mkdir -p gpurun_out/job33
timeout 900 python -m pytest tests/test_tc_gpu.py -q -x > gpurun_out/job33/pytest.log 2>&1; tail -2 gpurun_out/job33/pytest.log
timeout 600 python tools/tc_ab.py 8 > gpurun_out/job33/new.json 2>&1
