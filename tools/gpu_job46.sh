mkdir -p gpurun_out/job46
timeout 900 python -m pytest tests/test_tc_gpu.py -q -x > gpurun_out/job46/pytest.log 2>&1; tail -3 gpurun_out/job46/pytest.log
