# usage: bash tools/gpu_sweep_chunk.sh NAME SET FAMILY SECONDS
# Resumable chunk of a measured sweep: partial shard files travel in sweep_parts/NAME
# (pushed with the repo) and come back in gpurun_out/sweep_NAME; the final CSV is written
# when the sweep completes inside the chunk.
N=$1; SET=$2; FAM=$3; SECS=$4
W=gpurun_out/sweep_$N; mkdir -p $W
cp sweep_parts/$N/* $W/ 2>/dev/null
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $W/smi_start.csv 2>&1
timeout -s INT $SECS python -m paper_2008_13145_b200.sweep --set $SET --family $FAM --out $W/table.csv --work $W > $W/log.txt 2>&1
echo "rc=$?" >> $W/log.txt
