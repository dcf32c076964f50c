"""Small launches of every family / code path for compute-sanitizer (memcheck, racecheck,
synccheck): F0 and F1 vector + scalar (unaligned) paths, tcgen05 TMA and LSU paths,
k-sliced cluster launches (F1 and tcgen05: DSMEM slice reduction), the tcgen05
partial-last-wave split, the TMA-store epilogue, epilogue bias/ReLU, kp_bench_sets,
im2col (plain, padded, bf16), the bf16 cast and max-pool; round 2: unaligned-row repack
and in-kernel staging (both modes), 16-CTA k-slice clusters, tcgen05 CTA pairs and the
TMA-im2col implicit-GEMM convolution."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import _lib, gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

dev = torch.device("cuda")
cases = [("paper", KernelConfig(4, 4, 4, 16, 16)), ("paper", KernelConfig(1, 8, 2, 8, 8)),
         ("simt", KernelConfig(8, 4, 8, 16, 16)), ("simt", KernelConfig(4, 8, 8, 16, 8)),
         ("simt", KernelConfig(2, 1, 1, 128, 1)), ("simt", KernelConfig(1, 2, 8, 1, 128))]
cases += [(f, c) for f in ("bf16", "tf32") for c in gemm.family_configs(f)[:2]]
for fam, cfg in cases:
    dt = gemm.input_dtype(fam)
    for (m, k, n) in ((70, 64, 72), (33, 27, 45)):  # aligned / unaligned rows
        A = torch.rand(m, k, device=dev).to(dt)
        B = torch.rand(k, n, device=dev).to(dt)
        gemm.matmul(A, B, cfg, fam)
# k-sliced launches (under-filled grid, long k): F1 float4 and scalar reduce paths, tcgen05
for fam, cfg, (m, k, n) in (("simt", KernelConfig(4, 8, 8, 16, 8), (50, 2048, 70)),
                            ("simt", KernelConfig(2, 1, 2, 64, 1), (33, 1100, 5)),
                            ("bf16", gemm.family_configs("bf16")[1], (100, 3072, 200)),
                            ("tf32", gemm.family_configs("tf32")[2], (64, 2001, 64))):
    dt = gemm.input_dtype(fam)
    from paper_2008_13145_b200.dataset import ProblemSize
    assert gemm.k_slice_plan(cfg, ProblemSize(m, k, n, 1), family=fam)[0] > 1, (fam, cfg)
    gemm.matmul(torch.rand(m, k, device=dev).to(dt), torch.rand(k, n, device=dev).to(dt), cfg, fam)
# tensor-core partial-last-wave split (persistent head + sliced tail launch)
from paper_2008_13145_b200.dataset import ProblemSize  # noqa: E402
cfg = gemm.family_configs("tf32")[3]
assert gemm.k_slice_plan(cfg, ProblemSize(1280, 3456, 4096, 1), family="tf32")[0] > 1
gemm.matmul(torch.rand(1280, 3456, device=dev), torch.rand(3456, 4096, device=dev), cfg, "tf32")
# the sweep's rotating / median harness
ops = [gemm.GemmOperands(torch.rand(40, 64, device=dev), torch.rand(64, 24, device=dev), None, torch.float32)
       for _ in range(2)]
gemm.bench_sets(gemm.variant_id(KernelConfig(4, 4, 4, 16, 16), "simt"), ops, warmup=1, min_ms=0.05, repeats=3)
lib = _lib.load()
# padded / bf16 im2col and the bf16 cast (VGG16 conv1_1 and the BF16 family)
xi = torch.rand(2, 6, 6, 3, device=dev)
pad = torch.empty(72, 28, device=dev)
_lib.check(lib.kp_im2col3x3_nhwc_pad(xi.data_ptr(), 2, 6, 6, 3, pad.data_ptr(), 28, None), "im2col pad")
colsb = torch.empty(72, 32, device=dev, dtype=torch.bfloat16)
_lib.check(lib.kp_im2col3x3_nhwc_bf16(xi.data_ptr(), 2, 6, 6, 3, colsb.data_ptr(), 32, None), "im2col bf16 c3")
x8 = torch.rand(2, 6, 6, 8, device=dev)
cols8 = torch.empty(72, 72, device=dev, dtype=torch.bfloat16)
_lib.check(lib.kp_im2col3x3_nhwc_bf16(x8.data_ptr(), 2, 6, 6, 8, cols8.data_ptr(), 72, None), "im2col bf16 c8")
v = torch.rand(64, device=dev)
vb = torch.empty(64, device=dev, dtype=torch.bfloat16)
_lib.check(lib.kp_cast_bf16(v.data_ptr(), 64, vb.data_ptr(), None), "cast")
A = torch.rand(70, 64, device=dev)
W = torch.rand(64, 72, device=dev)
C = torch.empty(70, 72, device=dev)
bias = torch.rand(72, device=dev)
vid = gemm.variant_id(KernelConfig(8, 4, 8, 16, 16), "simt")
_lib.check(lib.kp_gemm_ex(vid, 70, 64, 72, 1, A.data_ptr(), 64, 0, W.data_ptr(), 72, 0, C.data_ptr(), 72, 0,
                          bias.data_ptr(), 1, None), "gemm_ex")
x = torch.rand(2, 6, 6, 5, device=dev)
cols = torch.empty(2 * 36, 45, device=dev)
_lib.check(lib.kp_im2col3x3_nhwc(x.data_ptr(), 2, 6, 6, 5, cols.data_ptr(), 45, None), "im2col")
y = torch.empty(2, 3, 3, 5, device=dev)
_lib.check(lib.kp_maxpool2x2_nhwc(x.data_ptr(), 2, 6, 6, 5, y.data_ptr(), None), "pool")
# round 2: unaligned rows through the repack pass and through in-kernel staging
for mode in ("always", "never"):
    prev = gemm.set_operand_repack(mode)
    for fam, cfg in (("simt", KernelConfig(8, 4, 4, 8, 8)), ("bf16", gemm.family_configs("bf16")[0]),
                     ("tf32", gemm.family_configs("tf32")[1])):
        dt = gemm.input_dtype(fam)
        gemm.matmul(torch.rand(300, 27, device=dev).to(dt), torch.rand(27, 61, device=dev).to(dt), cfg, fam)
    gemm.set_operand_repack(prev)
# a 16-CTA (non-portable) k-slice cluster: a grid under 0.15 tiles per SM
cfg16 = KernelConfig(8, 4, 2, 1, 64)
p16 = ProblemSize(8, 4096, 1000, 1)
assert gemm.k_slice_plan(cfg16, p16)[0] > 8, gemm.k_slice_plan(cfg16, p16)
gemm.matmul(torch.rand(8, 4096, device=dev), torch.rand(4096, 1000, device=dev), cfg16, "simt")
# tcgen05 CTA pairs (256-row tiles), both families
for fam in ("bf16", "tf32"):
    pair = next(c for c in gemm.family_configs(fam) if c.tile_rows == 256)
    dt = gemm.input_dtype(fam)
    gemm.matmul(torch.rand(600, 256, device=dev).to(dt), torch.rand(256, 520, device=dev).to(dt), pair, fam)
# implicit-GEMM 3x3 convolution (TMA im2col copies)
xc = torch.rand(2, 8, 8, 64, device=dev)
wc = torch.rand(9 * 64, 64, device=dev)
gemm.conv3x3(xc, wc, gemm.variant_id(KernelConfig(8, 8, 8, 16, 8), "simt"))
torch.cuda.synchronize()
print("sanitize run ok")
