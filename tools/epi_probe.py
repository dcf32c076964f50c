"""Probe: tensor-core GEMM time on VGG16 conv shapes with/without the fused epilogue,
fp32 vs bf16 output, explicit vs implicit conv.  python tools/epi_probe.py [batch]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2008_13145_b200 import _lib, gemm  # noqa: E402

lib = _lib.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = "cuda:0"


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for fam in ("bf16", "tf32"):
    dt = gemm.input_dtype(fam)
    cfgs = gemm.family_configs(fam)
    for (H, C, Co, kk) in [(224, 3, 64, 32), (224, 64, 64, None), (112, 64, 128, None), (56, 128, 256, None),
                           (28, 256, 512, None), (14, 512, 512, None)]:
        m, k = B * H * H, kk or 9 * C
        A = torch.randn(m, k, device=dev).to(dt)
        W = (torch.randn(k, Co, device=dev) * 0.05).to(dt)
        bias = torch.randn(Co, device=dev)
        o32 = torch.empty(m, Co, device=dev)
        o16 = torch.empty(m, Co, device=dev, dtype=torch.bfloat16)
        x = torch.randn(B, H, H, C, device=dev).to(dt)
        for ci, cfg in enumerate(cfgs):
            vid = gemm.variant_id(cfg, fam)
            res = {}
            res["plain"] = t(lambda: lib.kp_gemm(vid, m, k, Co, 1, A.data_ptr(), k, 0, W.data_ptr(), Co, 0, o32.data_ptr(), Co, 0, None))
            res["bias_relu"] = t(lambda: lib.kp_gemm_ex(vid, m, k, Co, 1, A.data_ptr(), k, 0, W.data_ptr(), Co, 0, o32.data_ptr(), Co, 0, bias.data_ptr(), 1, None))
            res["bf16out"] = t(lambda: lib.kp_gemm_ex(vid, m, k, Co, 1, A.data_ptr(), k, 0, W.data_ptr(), Co, 0, o16.data_ptr(), Co, 0, bias.data_ptr(), 3, None))
            if kk is None:
                res["implicit"] = t(lambda: lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), B, H, H, C, W.data_ptr(), Co, o32.data_ptr(), bias.data_ptr(), 1, None))
                res["implicit16"] = t(lambda: lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), B, H, H, C, W.data_ptr(), Co, o16.data_ptr(), bias.data_ptr(), 3, None))
            print(fam, (m, k, Co), cfg.as_tuple(), " ".join(f"{a}={b:.1f}" for a, b in res.items()), flush=True)
