J=gpurun_out/job58
mkdir -p $J
timeout 900 ncu --set full --clock-control none -k regex:"tc_gemm" -s 2 -c 1 -o $J/tc_bf16 python tools/prof_one.py bf16 128 64 256 4 192 8192 8192 8192 1 3 > $J/ncu_tc.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"tc_gemm" -s 2 -c 1 -o $J/tc_tf32 python tools/prof_one.py tf32 128 32 256 4 192 8192 8192 8192 1 3 > $J/ncu_tc32.log 2>&1
tail -2 $J/ncu_tc.log $J/ncu_tc32.log
