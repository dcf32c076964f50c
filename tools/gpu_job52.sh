# profiles + benches on the SURVEY-protocol tables
set -x
J=gpurun_out/job52
mkdir -p $J
make -s -C oracle
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $J/traffic.csv python tools/bench_layers_once.py > $J/layers.log 2>&1
python tools/traffic_from_ncu.py $J/layers.log $J/traffic.csv $J/dominant_kernel_traffic.json | tail -3
cp $J/dominant_kernel_traffic.json profiles/dominant_kernel_traffic.json
timeout 900 python bench.py > $J/bench.json 2> $J/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $J/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $J/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $J/bench_under_ncu.log 2>&1
python - <<'PY' > $J/dominant.txt
import json
line = json.loads(open("gpurun_out/job52/bench.json").read().strip().splitlines()[-1])
k = line["roofline"]["kernel"]
fam = k.split("(")[0]
cfg = k[k.index("(")+1:k.index(")")].replace(",", " ")
prob = k[k.index("[")+1:k.index("]")].replace(",", " ")
print(fam, cfg, prob)
PY
read FAM R A C WR WC M K N BATCH < $J/dominant.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"f1_kernel|f0_kernel|tc_gemm" -s 1 -c 1 -o $J/dominant python tools/prof_one.py $FAM $R $A $C $WR $WC $M $K $N $BATCH 2 > $J/ncu_dominant.log 2>&1
for B in 1 16 64; do
  timeout 900 python bench.py --workload vgg16-infer --batch $B --steps 20 > $J/vgg16_b$B.json 2>&1
  timeout 900 python bench.py --workload vgg16-infer --family tf32 --table data/sweeps/vgg16_tf32.csv --batch $B --steps 20 > $J/vgg16_tf32_b$B.json 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q > $J/pytest_gpu.log 2>&1; tail -2 $J/pytest_gpu.log
