"""Quick on-GPU probe: FFMA peak, F0/F1 parity, a few timings vs cuBLAS fp32."""
import sys, time, json
import torch
sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm
from paper_2008_13145_b200.dataset import KernelConfig

torch.manual_seed(0)
dev = torch.device("cuda:0")
print("device", torch.cuda.get_device_name(0), flush=True)
print("ffma peak TF/s", [round(gemm.ffma_peak_tflops(), 2) for _ in range(3)], flush=True)
print("ffma2 peak TF/s", [round(gemm.ffma_peak_tflops(True), 2) for _ in range(3)], flush=True)

def check(m, k, n, batch, cfgs):
    A = torch.rand(batch, m, k, device=dev) * 2 - 1
    B = torch.rand(batch, k, n, device=dev) * 2 - 1
    ref = torch.matmul(A.double(), B.double())
    outs = {}
    for fam, cfg in cfgs:
        C = gemm.matmul(A, B, cfg, fam)
        torch.cuda.synchronize()
        err = ((C.double() - ref).abs() / (A.double().abs() @ B.double().abs() + 1e-30)).max().item()
        outs[(fam, cfg)] = C
        print(f"  {m}x{k}x{n}x{batch} {fam} {cfg.as_tuple()} max rel-to-|A||B| err {err:.3e}", flush=True)
    vals = list(outs.values())
    same = all(torch.equal(vals[0], v) for v in vals[1:])
    print("  all variants bit-identical:", same, flush=True)

cfgs = [("paper", KernelConfig(4, 4, 4, 16, 16)), ("paper", KernelConfig(1, 8, 2, 8, 8)),
        ("simt", KernelConfig(8, 4, 8, 16, 16)), ("simt", KernelConfig(1, 1, 1, 1, 64)),
        ("simt", KernelConfig(2, 8, 4, 128, 1)), ("simt", KernelConfig(8, 2, 1, 8, 32))]
PERF_ONLY = 'perf' in sys.argv
for shp in [] if PERF_ONLY else [(256, 256, 256, 1), (37, 27, 61, 3), (1, 1000, 1000, 1), (129, 147, 64, 2), (500, 36, 31, 1)]:
    check(*shp, cfgs)

def tflops(fam, cfg, m, k, n, batch=1):
    dt = gemm.input_dtype(fam)
    A = torch.rand(batch, m, k, device=dev).to(dt); B = torch.rand(batch, k, n, device=dev).to(dt)
    ops = gemm.GemmOperands(A, B, None, dt)
    vid = gemm.variant_id(cfg, fam)
    ms, it = gemm.bench(vid, ops, warmup=2, min_ms=50)
    return 2.0 * m * k * n * batch / (ms * 1e-3) / 1e12

res = {}
for N in ((4096, 8192) if PERF_ONLY else (1024, 4096, 8192)):
    for A_ in (1, 2, 4, 8):
        cfg = KernelConfig(8, A_, 8, 16, 16)
        res[f"simt{cfg.as_tuple()}@{N}"] = tflops("simt", cfg, N, N, N)
    for cfg in (KernelConfig(8, 4, 8, 8, 16), KernelConfig(8, 4, 8, 16, 8), KernelConfig(4, 4, 8, 16, 16), KernelConfig(8, 4, 4, 16, 16)):
        res[f"simt{cfg.as_tuple()}@{N}"] = tflops("simt", cfg, N, N, N)
    res[f"paper(4,4,4,16,16)@{N}"] = tflops("paper", KernelConfig(4, 4, 4, 16, 16), N, N, N)
    for fam in ("bf16", "tf32"):
        for cfg in gemm.family_configs(fam):
            try:
                res[f"{fam}{cfg.as_tuple()}@{N}"] = tflops(fam, cfg, N, N, N)
            except Exception as exc:  # report and continue
                print(f"{fam}{cfg.as_tuple()} failed: {exc}", flush=True)
    for dt, name in ((torch.bfloat16, "cublas_bf16"),):
        a = torch.rand(N, N, device=dev).to(dt); b = torch.rand(N, N, device=dev).to(dt)
        for _ in range(3): torch.matmul(a, b)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = max(3, int(2e14 / (2 * N**3)))
        e0.record()
        for _ in range(reps): torch.matmul(a, b)
        e1.record(); torch.cuda.synchronize()
        res[f"{name}@{N}"] = 2.0 * N**3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.rand(N, N, device=dev); b = torch.rand(N, N, device=dev)
    for _ in range(3): torch.matmul(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = max(3, int(1e14 / (2 * N**3)))
    e0.record()
    for _ in range(reps): torch.matmul(a, b)
    e1.record(); torch.cuda.synchronize()
    res[f"cublas_tf32@{N}"] = 2.0 * N**3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    res[f"paper(8,4,8,16,16)@{N}"] = tflops("paper", KernelConfig(8, 4, 8, 16, 16), N, N, N)
    torch.backends.cuda.matmul.allow_tf32 = False
    a = torch.rand(N, N, device=dev); b = torch.rand(N, N, device=dev)
    for _ in range(3): torch.matmul(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = max(3, int(2e13 / (2 * N**3)))
    e0.record()
    for _ in range(reps): torch.matmul(a, b)
    e1.record(); torch.cuda.synchronize()
    res[f"cublas_fp32@{N}"] = 2.0 * N**3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    for kk, v in res.items():
        if kk.endswith(f"@{N}"): print(f"{kk:40s} {v:8.2f} TF/s", flush=True)
json.dump(res, open("gpurun_out/probe.json", "w"), indent=1)
