# full GPU suite, then the VGG16 SIMT sweep with k-slicing, then bench on the new table
mkdir -p gpurun_out/job14/sweeps
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/job14/pytest_gpu.log 2>&1; tail -3 gpurun_out/job14/pytest_gpu.log
S=gpurun_out/job14/sweeps
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 2000 > $S/clocks.csv &
SMI=$!
timeout 2400 python -m paper_2008_13145_b200.sweep --set vgg16 --family simt --out $S/vgg16_simt.csv --work $S/vgg16_simt.parts 2> $S/vgg16_simt.log
tail -n 2 $S/vgg16_simt.log
kill $SMI
timeout 900 python bench.py --table $S/vgg16_simt.csv > gpurun_out/job14/bench.json 2> gpurun_out/job14/bench.err; tail -c 2500 gpurun_out/job14/bench.json
