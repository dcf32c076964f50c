# flakiness check: the GPU suite three times on one box
mkdir -p gpurun_out/job60
make -s -C oracle
for i in 1 2 3; do timeout 1200 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/job60/pytest_$i.log 2>&1; tail -1 gpurun_out/job60/pytest_$i.log; done
