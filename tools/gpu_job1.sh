set -x
mkdir -p gpurun_out/sweeps
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 1000 > gpurun_out/sweeps/clocks.csv &
SMI=$!
timeout 1500 python -m paper_2008_13145_b200.sweep --set vgg16 --family simt --out gpurun_out/sweeps/vgg16_simt.csv --work gpurun_out/sweeps/vgg16_simt.parts 2> gpurun_out/sweeps/vgg16_simt.log
timeout 1500 python -m paper_2008_13145_b200.sweep --set vgg16 --family paper --out gpurun_out/sweeps/vgg16_paper.csv --work gpurun_out/sweeps/vgg16_paper.parts 2> gpurun_out/sweeps/vgg16_paper.log
kill $SMI
