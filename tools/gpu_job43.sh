mkdir -p gpurun_out/job43
make -s -C oracle
timeout 900 python -m pytest tests/test_vgg16_gpu.py -q -x -k tf32 -s > gpurun_out/job43/pytest.log 2>&1; tail -3 gpurun_out/job43/pytest.log
