"""Launch each unique (variant, problem) of bench.py's gemm-layers step once, in a fixed
order, and print that order as JSON -- run under ncu to attribute DRAM traffic per
launch (tools/profile_traffic.sh)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2008_13145_b200.dispatch import Dispatcher  # noqa: E402

args = bench.parse_args(sys.argv[1:])
pm, subset, tree, *_ = bench.train_selector(args.table, args.k, args.method, args.classifier)
disp = Dispatcher(tree, subset, pm.configs, args.family)
dev = torch.device("cuda")
order = []
seen = set()
for name, p in bench.vgg16_layers(args.batch):
    vid = disp.variant(p)
    if (vid, p) in seen:
        continue
    seen.add((vid, p))
    A = torch.rand(p.m, -(-p.k // 4) * 4, device=dev)[:, :p.k]  # rows pitched to 16 bytes, as bench.py
    W = torch.rand(p.k, p.n, device=dev)
    C = torch.empty(p.m, p.n, device=dev)
    torch.cuda.synchronize()
    disp.matmul(A, W, out=C)
    torch.cuda.synchronize()
    cfg, fam = disp.select(p), args.family
    order.append({"layer": name, "variant": list(cfg.as_tuple()), "problem": [p.m, p.k, p.n, p.batch]})
print("ORDER " + json.dumps(order))
