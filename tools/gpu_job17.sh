mkdir -p gpurun_out/job17
timeout 600 python tools/tc_ab.py 8 > gpurun_out/job17/new_cap8.json 2>&1
timeout 600 python tools/tc_ab.py 1 > gpurun_out/job17/new_cap1.json 2>&1
KPGEMM_LIB=exp/libkpgemm_oldtc.so timeout 600 python tools/tc_ab.py 1 > gpurun_out/job17/old.json 2>&1
timeout 600 python tools/tc_ab.py 8 > gpurun_out/job17/new_cap8b.json 2>&1
tail -c 300 gpurun_out/job17/*.json
