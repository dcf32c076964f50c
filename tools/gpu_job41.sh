# round-end rehearsal on a fresh box: what the driver runs
mkdir -p gpurun_out/job41
make -s -C oracle
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/job41/pytest_gpu.log 2>&1; tail -2 gpurun_out/job41/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/job41/smoke.log 2>&1; tail -1 gpurun_out/job41/smoke.log
timeout 900 python bench.py > gpurun_out/job41/bench.json 2> gpurun_out/job41/bench.err; echo "bench rc=$?"; head -c 400 gpurun_out/job41/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/job41/bench_ref.json 2> gpurun_out/job41/bench_ref.err; echo "ref rc=$?"; head -c 300 gpurun_out/job41/bench_ref.json
