# PAPER-family tables with the SURVEY protocol (part 1)
S=gpurun_out/job53/sweeps
mkdir -p $S
for spec in "square paper" "vgg16 paper"; do
  set -- $spec
  timeout 3300 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
