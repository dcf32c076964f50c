mkdir -p gpurun_out/job15
make -s -C oracle
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_tc_gpu.py tests/test_dispatch_gpu.py tests/test_vgg16_gpu.py -q -x > gpurun_out/job15/pytest.log 2>&1; tail -15 gpurun_out/job15/pytest.log
timeout 900 python tools/kslice_probe.py 8 > gpurun_out/job15/probe.jsonl 2> gpurun_out/job15/probe.err; cat gpurun_out/job15/probe.jsonl; tail -3 gpurun_out/job15/probe.err
