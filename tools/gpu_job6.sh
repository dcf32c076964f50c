mkdir -p gpurun_out/job6
timeout 600 python tools/exp_f1.py > gpurun_out/job6/exp.jsonl 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -2
