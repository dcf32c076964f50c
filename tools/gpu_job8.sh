mkdir -p gpurun_out/job8
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/job8/traffic.csv python tools/bench_layers_once.py > gpurun_out/job8/layers.log 2>&1
python tools/traffic_from_ncu.py gpurun_out/job8/layers.log gpurun_out/job8/traffic.csv gpurun_out/job8/dominant_kernel_traffic.json | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/job8/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/job8/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"f1_kernel<8, 8, 4, 8, 16>" -s 1 -c 1 -o gpurun_out/job8/dominant python tools/prof_one.py simt 8 8 4 8 16 50176 2304 256 1 2 > gpurun_out/job8/ncu_dom.log 2>&1
