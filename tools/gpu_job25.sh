mkdir -p gpurun_out/job25
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_cli_gpu.py -q -x > gpurun_out/job25/pytest.log 2>&1; tail -5 gpurun_out/job25/pytest.log
timeout 600 python tools/tc_ab.py 8 > gpurun_out/job25/new.json 2>&1
KPGEMM_LIB=exp/libkpgemm_oldtc.so timeout 600 python tools/tc_ab.py 1 > gpurun_out/job25/old.json 2>&1
timeout 600 python tools/square_compare.py > gpurun_out/job25/square_cublas.json 2> gpurun_out/job25/square_cublas.err; tail -3 gpurun_out/job25/square_cublas.json
