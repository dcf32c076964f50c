"""Per-launch profile of one VGG16 inference forward (eager, no graph) for ncu:
python tools/prof_infer.py FAMILY TABLE BATCH [implicit=1] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_13145_b200.dispatch import Dispatcher  # noqa: E402
from paper_2008_13145_b200.vgg16 import Vgg16  # noqa: E402

fam, table, batch = sys.argv[1], sys.argv[2], int(sys.argv[3])
implicit = len(sys.argv) <= 4 or sys.argv[4] == "1"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
pm, subset, tree, *_ = bench.train_selector(table, 4, "kmeans", "treeA")
disp = Dispatcher(tree, subset, pm.configs, fam)
model = Vgg16(disp, batch, "cuda:0", seed=0, implicit=implicit)
model.input.normal_()
for lay in model.layers:
    print(lay, flush=True)
s = torch.cuda.Stream()
for _ in range(reps):
    model.forward(stream=s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(10):
        model.forward(stream=s)
    e1.record(s)
torch.cuda.synchronize()
print(f"eager forward {e0.elapsed_time(e1) / 10:.3f} ms (b{batch} {fam} implicit={implicit})")
