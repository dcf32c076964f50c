# run-to-run reproducibility of the headline bench line (3 fresh processes)
J=gpurun_out/job59
mkdir -p $J
for i in 1 2 3; do timeout 900 python bench.py --no-cpu > $J/bench_$i.json 2> $J/bench_$i.err; done
