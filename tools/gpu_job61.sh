mkdir -p gpurun_out/job61
timeout 1500 python tools/occ_probe.py gpurun_out/job61/w16.csv > gpurun_out/job61/w16.log 2>&1; tail -1 gpurun_out/job61/w16.log
KPGEMM_LIB=exp/libkpgemm_w12.so timeout 1500 python tools/occ_probe.py gpurun_out/job61/w12.csv > gpurun_out/job61/w12.log 2>&1; tail -1 gpurun_out/job61/w12.log
