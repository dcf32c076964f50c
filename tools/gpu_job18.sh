mkdir -p gpurun_out/job18
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/job18/pytest.log 2>&1; tail -5 gpurun_out/job18/pytest.log
timeout 600 python tools/tc_ab.py 8 > gpurun_out/job18/new_cap8.json 2>&1
timeout 600 python tools/tc_ab.py 1 > gpurun_out/job18/new_cap1.json 2>&1
KPGEMM_LIB=exp/libkpgemm_oldtc.so timeout 600 python tools/tc_ab.py 1 > gpurun_out/job18/old.json 2>&1
tail -c 200 gpurun_out/job18/*.json
