# fitted SIMT slice planner: parity, planner-vs-forced check, SIMT re-sweeps, bench + profiles
set -x
J=gpurun_out/job35
mkdir -p $J/sweeps
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > $J/pytest_gpu.log 2>&1; tail -3 $J/pytest_gpu.log
KPGEMM_FORCE_SLICES=0 timeout 600 python tools/wave_probe2.py > $J/probe2_planner.jsonl 2>> $J/err.log
S=$J/sweeps
for spec in "vgg16 simt" "resnet50 simt+tf32" "square simt"; do
  set -- $spec
  timeout 2400 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
cp $S/vgg16_simt.csv data/sweeps/vgg16_simt.csv
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $J/traffic.csv python tools/bench_layers_once.py > $J/layers.log 2>&1
python tools/traffic_from_ncu.py $J/layers.log $J/traffic.csv $J/dominant_kernel_traffic.json | tail -3
cp $J/dominant_kernel_traffic.json profiles/dominant_kernel_traffic.json
timeout 900 python bench.py > $J/bench.json 2> $J/bench.err; tail -c 1500 $J/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $J/bench_ref.json 2>&1; tail -c 400 $J/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $J/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $J/bench_under_ncu.log 2>&1
python - <<'PY' > $J/dominant.txt
import json
line = json.loads(open("gpurun_out/job35/bench.json").read().strip().splitlines()[-1])
k = line["roofline"]["kernel"]
fam = k.split("(")[0]
cfg = k[k.index("(")+1:k.index(")")].replace(",", " ")
prob = k[k.index("[")+1:k.index("]")].replace(",", " ")
print(fam, cfg, prob)
PY
cat $J/dominant.txt
read FAM R A C WR WC M K N BATCH < $J/dominant.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"f1_kernel|f0_kernel|tc_gemm" -s 1 -c 1 -o $J/dominant python tools/prof_one.py $FAM $R $A $C $WR $WC $M $K $N $BATCH 2 > $J/ncu_dominant.log 2>&1
timeout 900 python bench.py --workload vgg16-infer --batch 16 > $J/bench_vgg16_b16.json 2>&1
timeout 900 python bench.py --workload vgg16-infer --batch 1 --steps 50 > $J/bench_vgg16_b1.json 2>&1
