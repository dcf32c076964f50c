mkdir -p gpurun_out/job29
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_dispatch_gpu.py tests/test_vgg16_gpu.py -q -x > gpurun_out/job29/pytest.log 2>&1; tail -4 gpurun_out/job29/pytest.log
timeout 600 python tools/exp_f1.py > gpurun_out/job29/exp.jsonl 2>&1
timeout 600 python tools/tail_probe.py > gpurun_out/job29/tail.jsonl 2>&1; cat gpurun_out/job29/tail.jsonl
