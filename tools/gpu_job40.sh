mkdir -p gpurun_out/job40
for i in 1 2; do ./tools/micro/f1_inner >> gpurun_out/job40/f1_inner.json; done
cat gpurun_out/job40/f1_inner.json
