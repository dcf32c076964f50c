# tests, bench, ncu launch list + dominant-kernel capture, perf probe
mkdir -p gpurun_out/job2
make -s -C oracle
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/job2/pytest_gpu.log 2>&1; tail -5 gpurun_out/job2/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/job2/bench.json 2> gpurun_out/job2/bench.err; tail -c 3000 gpurun_out/job2/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/job2/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/job2/bench_under_ncu.log 2>&1
python - <<'PY' > gpurun_out/job2/dominant.txt
import json
line = json.loads(open("gpurun_out/job2/bench.json").read().strip().splitlines()[-1])
k = line["roofline"]["kernel"]
fam = k.split("(")[0]
cfg = k[k.index("(")+1:k.index(")")].replace(",", " ")
prob = k[k.index("[")+1:k.index("]")].replace(",", " ")
print(fam, cfg, prob)
PY
cat gpurun_out/job2/dominant.txt
read FAM R A C WR WC M K N BATCH < gpurun_out/job2/dominant.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"f1_kernel|f0_kernel|tc_gemm" -s 1 -c 1 -o gpurun_out/job2/dominant python tools/prof_one.py $FAM $R $A $C $WR $WC $M $K $N $BATCH 2 > gpurun_out/job2/ncu_dominant.log 2>&1
timeout 900 python tools/probe_gpu.py perf > gpurun_out/job2/probe.log 2>&1; tail -60 gpurun_out/job2/probe.log
