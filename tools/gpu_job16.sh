# re-measure every table whose family now k-slices (SIMT, TF32, BF16); PAPER tables unchanged
S=gpurun_out/job16/sweeps
mkdir -p $S
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 5000 > $S/clocks.csv &
SMI=$!
for spec in "vgg16 tf32" "vgg16 bf16" "resnet50 bf16" "square tf32" "square bf16" "square16k tf32" "square16k bf16" "resnet50 simt+tf32" "square simt"; do
  set -- $spec
  timeout 2400 python -m paper_2008_13145_b200.sweep --set $1 --family $2 --out $S/$1_$2.csv --work $S/$1_$2.parts 2> $S/$1_$2.log
  tail -n 1 $S/$1_$2.log
done
kill $SMI
