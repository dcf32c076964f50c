# multi-rank code path on one GPU (2 ranks share cuda:0: timings meaningless, plumbing real),
# full GPU suite, default bench (N=1) with the numpy-BLAS CPU line
mkdir -p gpurun_out/job32
make -s -C oracle
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555"
timeout 600 $TR bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/job32/bench_n2.json 2> gpurun_out/job32/bench_n2.err; echo "n2 rc=$?"; tail -c 400 gpurun_out/job32/bench_n2.json
timeout 600 $TR bench.py --gpus 2 --workload vgg16-infer --batch 4 --steps 5 --warmup 3 > gpurun_out/job32/vgg_n2.json 2> gpurun_out/job32/vgg_n2.err; echo "vgg n2 rc=$?"; tail -c 300 gpurun_out/job32/vgg_n2.json
timeout 600 $TR bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/job32/ref_n2.json 2> gpurun_out/job32/ref_n2.err; echo "ref n2 rc=$?"; tail -c 300 gpurun_out/job32/ref_n2.json
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job32/pytest_gpu.log 2>&1; tail -3 gpurun_out/job32/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/job32/bench.json 2> gpurun_out/job32/bench.err; tail -c 700 gpurun_out/job32/bench.json
