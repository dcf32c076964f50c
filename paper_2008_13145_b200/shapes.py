"""GEMM shape sets of the paper's workloads (VGG, ResNet, MobileNet
layer sizes) as reference ``ProblemSize`` rows.

Convolutions are lowered im2col-style: per image m = Ho*Wo, k = Cin*kh*kw,
n = Cout.  The image batch is folded into m
(m = B*Ho*Wo, batch = 1) so every CTA tile is full -- one GEMM per layer with the
weights shared -- and fully connected layers have m = B.  Rows are de-duplicated in
first-appearance order (a table may not repeat a problem, dataset.py:102-103).
"""

from __future__ import annotations

from dataclasses import dataclass

from .dataset import ProblemSize

DEFAULT_BATCHES = (1, 2, 4, 8, 16, 32, 64)


@dataclass(frozen=True)
class GemmLayer:
    """One network layer as a GEMM: per-image m (or 1 for fc), k, n, and how many
    layers of the network share the shape."""

    name: str
    m_per_image: int
    k: int
    n: int
    count: int = 1
    fc: bool = False

    def problem(self, batch: int) -> ProblemSize:
        m = batch if self.fc else self.m_per_image * batch
        return ProblemSize(m, self.k, self.n, 1)

    def flops(self, batch: int) -> int:
        return self.problem(batch).flops * self.count


# VGG16 (configuration D): 13 conv 3x3 pad 1 + 3 fc; 16 GEMM layers, 12 unique.
VGG16_LAYERS: tuple[GemmLayer, ...] = (
    GemmLayer("conv1_1", 224 * 224, 3 * 9, 64),
    GemmLayer("conv1_2", 224 * 224, 64 * 9, 64),
    GemmLayer("conv2_1", 112 * 112, 64 * 9, 128),
    GemmLayer("conv2_2", 112 * 112, 128 * 9, 128),
    GemmLayer("conv3_1", 56 * 56, 128 * 9, 256),
    GemmLayer("conv3_2", 56 * 56, 256 * 9, 256, count=2),  # conv3_2, conv3_3
    GemmLayer("conv4_1", 28 * 28, 256 * 9, 512),
    GemmLayer("conv4_2", 28 * 28, 512 * 9, 512, count=2),  # conv4_2, conv4_3
    GemmLayer("conv5_1", 14 * 14, 512 * 9, 512, count=3),  # conv5_1..conv5_3
    GemmLayer("fc6", 1, 512 * 7 * 7, 4096, fc=True),
    GemmLayer("fc7", 1, 4096, 4096, fc=True),
    GemmLayer("fc8", 1, 4096, 1000, fc=True),
)

# ResNet-50 v1.5 (stride on the 3x3), 54 GEMM layers incl. projections, 21 unique.
RESNET50_LAYERS: tuple[GemmLayer, ...] = (
    GemmLayer("conv1", 112 * 112, 3 * 49, 64),
    GemmLayer("l1_reduce_in", 56 * 56, 64, 64),
    GemmLayer("l1_3x3", 56 * 56, 64 * 9, 64, count=3),
    GemmLayer("l1_expand_proj", 56 * 56, 64, 256, count=4),
    GemmLayer("l1_reduce", 56 * 56, 256, 64, count=2),
    GemmLayer("l2_reduce_in", 56 * 56, 256, 128),
    GemmLayer("l2_3x3", 28 * 28, 128 * 9, 128, count=4),
    GemmLayer("l2_expand", 28 * 28, 128, 512, count=4),
    GemmLayer("l2_proj", 28 * 28, 256, 512),
    GemmLayer("l2_reduce", 28 * 28, 512, 128, count=3),
    GemmLayer("l3_reduce_in", 28 * 28, 512, 256),
    GemmLayer("l3_3x3", 14 * 14, 256 * 9, 256, count=6),
    GemmLayer("l3_expand", 14 * 14, 256, 1024, count=6),
    GemmLayer("l3_proj", 14 * 14, 512, 1024),
    GemmLayer("l3_reduce", 14 * 14, 1024, 256, count=5),
    GemmLayer("l4_reduce_in", 14 * 14, 1024, 512),
    GemmLayer("l4_3x3", 7 * 7, 512 * 9, 512, count=3),
    GemmLayer("l4_expand", 7 * 7, 512, 2048, count=3),
    GemmLayer("l4_proj", 7 * 7, 1024, 2048),
    GemmLayer("l4_reduce", 7 * 7, 2048, 512, count=2),
    GemmLayer("fc", 1, 2048, 1000, fc=True),
)

NETWORKS = {"vgg16": VGG16_LAYERS, "resnet50": RESNET50_LAYERS}


def _unique(problems) -> list[ProblemSize]:
    seen: set[ProblemSize] = set()
    out = []
    for p in problems:
        if p not in seen:
            seen.add(p)
            out.append(p)
    return out


# The paper's three sample problems (its Figure "sample"):
# square-ish m=512 k=784 n=512 batch 16, rectangular m=512 k=4608 n=784, and the long
# accumulation m=32 k=12321 n=27 -- swept beside the VGG16 rows.
PAPER_SAMPLES: tuple[ProblemSize, ...] = (
    ProblemSize(512, 784, 512, 16),
    ProblemSize(512, 4608, 784, 1),
    ProblemSize(32, 12321, 27, 1),
)


def network_problems(network: str, batches=DEFAULT_BATCHES) -> list[ProblemSize]:
    """Unique GEMM problems of a network over a batch list, batch-major order."""
    layers = NETWORKS[network]
    return _unique(layer.problem(b) for b in batches for layer in layers)


def network_flops(network: str, batch: int) -> int:
    """Total GEMM flops of one forward pass (every layer, duplicates counted)."""
    return sum(layer.flops(batch) for layer in NETWORKS[network])


def square_skinny_problems(sizes=(64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384)) -> list[ProblemSize]:
    """BASELINE config 5: square M=N=K sweep plus skinny extremes."""
    rows = [ProblemSize(s, s, s, 1) for s in sizes]
    rows += [ProblemSize(16384, 64, 16384, 1), ProblemSize(64, 16384, 16384, 1),
             ProblemSize(16384, 16384, 64, 1)]
    return _unique(rows)
