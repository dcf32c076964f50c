mkdir -p gpurun_out/job13
make -s -C oracle
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/job13/smoke.log 2>&1; tail -3 gpurun_out/job13/smoke.log
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_dispatch_gpu.py tests/test_vgg16_gpu.py -q -x > gpurun_out/job13/pytest.log 2>&1; tail -15 gpurun_out/job13/pytest.log
timeout 600 python tools/kslice_probe.py > gpurun_out/job13/kslice.jsonl 2> gpurun_out/job13/kslice.err; cat gpurun_out/job13/kslice.jsonl | head -100; tail -3 gpurun_out/job13/kslice.err
