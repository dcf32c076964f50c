# persistent TC kernel validation + perf, LDS pattern micro-benchmark, cuBLAS square lines
mkdir -p gpurun_out/job4
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_vgg16_gpu.py -q -x > gpurun_out/job4/pytest_tc.log 2>&1; tail -3 gpurun_out/job4/pytest_tc.log
timeout 600 python tools/probe_gpu.py perf > gpurun_out/job4/probe.log 2>&1; grep -E "bf16|tf32|cublas" gpurun_out/job4/probe.log
timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum --csv tools/micro/lds_patterns > gpurun_out/job4/lds.csv 2>&1
timeout 600 python tools/square_compare.py > gpurun_out/job4/square_cublas.json 2> gpurun_out/job4/square_cublas.err; tail -3 gpurun_out/job4/square_cublas.json
timeout 600 ncu --set full --clock-control none -k regex:"tc_gemm" -s 2 -c 1 -o gpurun_out/job4/tc_bf16 python tools/prof_one.py bf16 128 64 256 4 192 8192 8192 8192 1 3 > gpurun_out/job4/ncu_tc.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"gemm|sgemm|cutlass" -s 3 -c 1 -o gpurun_out/job4/cublas_fp32 python -c "
import torch; torch.backends.cuda.matmul.allow_tf32=False
a=torch.rand(8192,8192,device='cuda'); b=torch.rand(8192,8192,device='cuda')
[torch.matmul(a,b) for _ in range(5)]; torch.cuda.synchronize()" > gpurun_out/job4/ncu_cublas.log 2>&1
