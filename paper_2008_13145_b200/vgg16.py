"""VGG16 inference with tree-dispatched GEMMs (BASELINE.json configs[2]; the paper's
system-level check).

Every convolution is 3x3 / stride 1 / pad 1 and runs as im2col (``kp_im2col3x3_nhwc``)
+ one GEMM (m = B*H*W, k = 9*Cin, n = Cout) launched through the C dispatch table with
the bias add and ReLU fused into the GEMM epilogue (``kp_gemm_ex``); 2x2 max pooling
is ``kp_maxpool2x2_nhwc``; fc6/fc7/fc8 are GEMMs with m = B.  Activations are NHWC
fp32, so each GEMM output is directly the next layer's input.  Weights are He-normal
random (no network access for trained weights), seeded, identical on every rank.

Convolutions whose dispatched variant supports it run as implicit GEMMs instead
(``kp_conv3x3_nhwc_ex``: TMA im2col copies gather the patches from the activation, no
im2col buffer).  On the BF16 family, when every conv after conv1_1 is implicit, the
activations are bf16 end to end: each GEMM epilogue rounds its output to bf16
(``KP_EPI_BF16_OUT``) and pooling runs on bf16 (``kp_maxpool2x2_nhwc_bf16``).  Otherwise
activations are fp32 and a BF16 layer rounds its input in the bf16 im2col / cast.  Both
are the same round-to-nearest of the same fp32 values, so the logits are identical.

Data parallelism (configs[2] at 1/2/4/8 GPUs): each rank runs its own images with
replicated weights; there is no collective on the data path.  The whole forward for a
fixed batch can be captured once in a CUDA graph (``Vgg16.capture``) because all
buffers are preallocated.
"""

from __future__ import annotations

import math

import torch

from . import _lib, gemm
from .dataset import ProblemSize

# (Cin, Cout) per conv, "M" = 2x2 max pool (configuration D).
VGG16_PLAN = ((3, 64), (64, 64), "M", (64, 128), (128, 128), "M", (128, 256), (256, 256), (256, 256), "M",
              (256, 512), (512, 512), (512, 512), "M", (512, 512), (512, 512), (512, 512), "M")
VGG16_FC = ((7 * 7 * 512, 4096, True), (4096, 4096, True), (4096, 1000, False))


def init_weights(seed: int = 0, device="cpu"):
    """He-normal conv/fc weights ((9*Cin) x Cout / in x out, row-major) and small
    biases, deterministic for a seed (generated on CPU so every device agrees)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    convs, fcs = [], []
    for item in VGG16_PLAN:
        if item == "M":
            continue
        cin, cout = item
        w = torch.randn(9 * cin, cout, generator=g) * math.sqrt(2.0 / (9 * cin))
        b = torch.randn(cout, generator=g) * 0.01
        convs.append((w.to(device), b.to(device)))
    for fin, fout, _ in VGG16_FC:
        w = torch.randn(fin, fout, generator=g) * math.sqrt(2.0 / fin)
        b = torch.randn(fout, generator=g) * 0.01
        fcs.append((w.to(device), b.to(device)))
    return convs, fcs


class Vgg16:
    """Preallocated VGG16 forward for a fixed batch on one device."""

    def __init__(self, dispatcher, batch: int, device, seed: int = 0, weights=None, implicit: bool = True):
        self.disp = dispatcher
        # implicit: conv layers whose dispatched variant supports it run as implicit
        # GEMMs (kp_conv3x3_nhwc_ex, TMA im2col) instead of im2col + GEMM
        self.implicit = implicit
        self.batch = batch
        self.device = torch.device(device)
        convs, fcs = weights if weights is not None else init_weights(seed)
        # BF16 family: bf16 weights and im2col rows (fp32 accumulation, fp32 activations in
        # between -- the GEMM epilogue writes fp32 and the next im2col rounds to bf16)
        self.bf16 = dispatcher.family == "bf16"
        wdt = torch.bfloat16 if self.bf16 else torch.float32
        self.convs = [(w.to(self.device).contiguous(), b.to(self.device).contiguous()) for w, b in convs]
        # conv1_1 (Cin = 3): rows padded from 27 to 28 floats (16-byte aligned, so the GEMM
        # takes its vector / TMA paths) against a zero 28th weight row: fma(0, 0, acc) ==
        # acc keeps the fp32 chain over the 27 real taps bit for bit (32 for bf16 rows)
        w0, b0 = self.convs[0]
        align = 8 if self.bf16 else 4
        self.k_pad0 = (w0.shape[0] + align - 1) // align * align
        self.convs[0] = (torch.cat([w0, w0.new_zeros(self.k_pad0 - w0.shape[0], w0.shape[1])]).contiguous(), b0)
        self.convs = [(w.to(wdt).contiguous(), b) for w, b in self.convs]
        self.fcs = [(w.to(self.device).to(wdt).contiguous(), b.to(self.device).contiguous()) for w, b in fcs]
        B = batch
        # per conv layer: (B, H, Cin, Cout, m, k as launched, variant, implicit?)
        self.layers = []
        H = 224
        for item in VGG16_PLAN:
            if item == "M":
                H //= 2
                continue
            cin, cout = item
            m, k = B * H * H, 9 * cin
            k_launch = k if k % align == 0 else self.k_pad0
            vid = self.disp.variant(ProblemSize(m, k, cout, 1))
            implicit = self.implicit and gemm.conv3x3_supported(vid, cin, cout)
            self.layers.append((B, H, cin, cout, m, k_launch, vid, implicit))
        # BF16 family with every conv after conv1_1 implicit: activations stay bf16 end to end
        # -- each GEMM epilogue rounds its output (KP_EPI_BF16_OUT), pools run on bf16 -- the
        # same roundings of the same fp32 values as the fp32-activation path below
        self.bf16_acts = self.bf16 and all(lay[-1] for lay in self.layers[1:])
        # ping-pong activation buffers sized for the largest layer output (B*224*224*64)
        act = B * 224 * 224 * 64
        self.act = [torch.empty(8 if self.bf16_acts else act, device=self.device) for _ in range(2)]
        # im2col rows for the explicit layers only (conv1_1 alone when the rest are implicit)
        cols = max([m * k for (_, _, _, _, m, k, _, imp) in self.layers if not imp], default=8)
        self.cols = torch.empty(cols, device=self.device, dtype=wdt)
        # bf16 activations: the ping-pong pair (bf16_acts), else one bf16 copy of an
        # implicit conv's fp32 input (kp_cast_bf16 / a bf16 pool)
        n16 = 2 if self.bf16_acts else 1 if self.bf16 and any(lay[-1] for lay in self.layers) else 0
        self.act16 = [torch.empty(act, device=self.device, dtype=torch.bfloat16) for _ in range(n16)]
        self.fc_in = torch.empty(B, 7 * 7 * 512, device=self.device, dtype=wdt)  # bf16 fc operands
        self.fc_in2 = torch.empty(B, 4096, device=self.device, dtype=wdt)
        self.fc16 = [torch.empty(B, 4096, device=self.device, dtype=wdt) for _ in range(2 if self.bf16_acts else 0)]
        self.input = torch.empty(B, 224, 224, 3, device=self.device)
        self.logits = torch.empty(B, 1000, device=self.device)
        self.fc_buf = [torch.empty(B, 4096, device=self.device) for _ in range(2)]
        self.launches = []  # (problem, variant) per GEMM, filled on first forward
        self.graph = None

    def problems(self) -> list[ProblemSize]:
        out, H, B = [], 224, self.batch
        for item in VGG16_PLAN:
            if item == "M":
                H //= 2
                continue
            cin, cout = item
            align = 8 if getattr(self, "bf16", False) else 4
            out.append(ProblemSize(B * H * H, (9 * cin + align - 1) // align * align, cout, 1))  # as launched
        out += [ProblemSize(B, fin, fout, 1) for fin, fout, _ in VGG16_FC]
        return out

    def _gemm(self, A, W, bias, C, m, k, n, relu, stream, flags=0):
        lib = _lib.load()
        vid = self.disp.variant(ProblemSize(m, k, n, 1))
        _lib.check(lib.kp_gemm_ex(vid, m, k, n, 1, A.data_ptr(), k, 0, W.data_ptr(), n, 0, C.data_ptr(), n, 0,
                                  bias.data_ptr(), flags | (_lib.KP_EPI_RELU if relu else 0), stream),
                   f"kp_gemm_ex({m},{k},{n})")
        return vid

    def _forward_bf16(self, stream_handle):
        """BF16 activations end to end: conv1_1 by bf16 im2col + GEMM, every other conv an
        implicit GEMM, each writing bf16 (KP_EPI_BF16_OUT); bf16 pools; fc6/fc7 bf16 out,
        fc8 fp32 logits."""
        lib = _lib.load()
        B, H, C = self.batch, 224, 3
        src = self.input  # fp32: only conv1_1's im2col reads it
        di = 0
        ci = 0
        out16 = _lib.KP_EPI_RELU | _lib.KP_EPI_BF16_OUT
        for pi, item in enumerate(VGG16_PLAN):
            if item == "M":
                dst = self.fc_in if pi == len(VGG16_PLAN) - 1 else self.act16[di]
                _lib.check(lib.kp_maxpool2x2_nhwc_bf16(src.data_ptr(), B, H, H, C, dst.data_ptr(), stream_handle),
                           "kp_maxpool2x2_nhwc_bf16")
                H //= 2
            else:
                _, _, cin, cout, m, k, vid, implicit = self.layers[ci]
                w, b = self.convs[ci]
                ci += 1
                dst = self.act16[di]
                if implicit:
                    _lib.check(lib.kp_conv3x3_nhwc_ex(vid, src.data_ptr(), B, H, H, cin, w.data_ptr(), cout,
                                                      dst.data_ptr(), b.data_ptr(), out16, stream_handle),
                               f"kp_conv3x3_nhwc_ex({B}x{H}x{H}x{cin} -> {cout}, bf16 out)")
                else:  # conv1_1 (C = 3): bf16 im2col rows of the fp32 input
                    _lib.check(lib.kp_im2col3x3_nhwc_bf16(src.data_ptr(), B, H, H, cin, self.cols.data_ptr(), k,
                                                          stream_handle), "kp_im2col3x3_nhwc_bf16")
                    self._gemm(self.cols, w, b, dst, m, k, cout, True, stream_handle, _lib.KP_EPI_BF16_OUT)
                C = cout
            src = dst
            di ^= 1
        x = self.fc_in
        for j, ((fin, fout, relu), (w, b)) in enumerate(zip(VGG16_FC, self.fcs)):
            last = j == len(self.fcs) - 1
            out = self.logits if last else self.fc16[j % 2]
            self._gemm(x, w, b, out, B, fin, fout, relu, stream_handle, 0 if last else _lib.KP_EPI_BF16_OUT)
            x = out
        return self.logits

    def _forward(self, stream_handle):
        if self.bf16_acts:
            return self._forward_bf16(stream_handle)
        lib = _lib.load()
        B, H, C = self.batch, 224, 3
        src = self.input
        dst_i = 0
        ci = 0
        for item in VGG16_PLAN:
            dst = self.act[dst_i]
            if item == "M":
                _lib.check(lib.kp_maxpool2x2_nhwc(src.data_ptr(), B, H, H, C, dst.data_ptr(), stream_handle),
                           "kp_maxpool2x2_nhwc")
                H //= 2
            else:
                _, _, cin, cout, m, k, vid, implicit = self.layers[ci]
                w, b = self.convs[ci]
                ci += 1
                if implicit:
                    # implicit GEMM: TMA im2col copies gather the patches from the activation
                    x = src
                    if self.bf16:  # a bf16 copy of the fp32 activation
                        _lib.check(lib.kp_cast_bf16(src.data_ptr(), B * H * H * cin, self.act16[0].data_ptr(),
                                                    stream_handle), "kp_cast_bf16")
                        x = self.act16[0]
                    _lib.check(lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), B, H, H, cin, w.data_ptr(), cout,
                                                      dst.data_ptr(), b.data_ptr(), _lib.KP_EPI_RELU, stream_handle),
                               f"kp_conv3x3_nhwc_ex({B}x{H}x{H}x{cin} -> {cout})")
                elif self.bf16:
                    _lib.check(lib.kp_im2col3x3_nhwc_bf16(src.data_ptr(), B, H, H, cin, self.cols.data_ptr(), k,
                                                          stream_handle), "kp_im2col3x3_nhwc_bf16")
                    self._gemm(self.cols, w, b, dst, m, k, cout, True, stream_handle)
                elif k != 9 * cin:  # conv1_1: 16-byte-aligned padded rows
                    _lib.check(lib.kp_im2col3x3_nhwc_pad(src.data_ptr(), B, H, H, cin, self.cols.data_ptr(), k,
                                                         stream_handle), "kp_im2col3x3_nhwc_pad")
                    self._gemm(self.cols, w, b, dst, m, k, cout, True, stream_handle)
                else:
                    _lib.check(lib.kp_im2col3x3_nhwc(src.data_ptr(), B, H, H, cin, self.cols.data_ptr(), k,
                                                     stream_handle), "kp_im2col3x3_nhwc")
                    self._gemm(self.cols, w, b, dst, m, k, cout, True, stream_handle)
                C = cout
            src = dst
            dst_i ^= 1
        x = src  # (B, 7, 7, 512) NHWC flattened per image = fc6 input rows
        for j, ((fin, fout, relu), (w, b)) in enumerate(zip(VGG16_FC, self.fcs)):
            out = self.logits if j == len(self.fcs) - 1 else self.fc_buf[j % 2]
            if self.bf16:
                xin = self.fc_in if j == 0 else self.fc_in2
                _lib.check(lib.kp_cast_bf16(x.data_ptr(), B * fin, xin.data_ptr(), stream_handle), "kp_cast_bf16")
                x = xin
            self._gemm(x, w, b, out, B, fin, fout, relu, stream_handle)
            x = out
        return self.logits

    def forward(self, x: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """x: (B, 224, 224, 3) NHWC fp32 (copied into the input buffer) -> logits (B, 1000)."""
        stream = stream or torch.cuda.current_stream(self.device)
        if x is not None:
            with torch.cuda.stream(stream):
                self.input.copy_(x, non_blocking=True)
        if self.graph is not None:
            with torch.cuda.stream(stream):
                self.graph.replay()
            return self.logits
        return self._forward(stream.cuda_stream)

    def capture(self, stream: torch.cuda.Stream | None = None) -> None:
        """Capture the whole forward in a CUDA graph (launch-bound small batches)."""
        stream = stream or torch.cuda.Stream(self.device)
        with torch.cuda.stream(stream):
            self._forward(stream.cuda_stream)  # warm: resolves variants, sets kernel attributes
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            self._forward(torch.cuda.current_stream().cuda_stream)
        self.graph = g

    @property
    def flops(self) -> int:
        """Convolution + fc flops of one forward (conv1_1 counted at its true k = 27)."""
        probs = self.problems()
        first = probs[0]
        return sum(p.flops for p in probs) - 2 * first.m * first.n * (first.k - 27)
