"""Round-2 prep (dev tool): every SIMT config on the bench's 12 unique VGG16 b16 layer
shapes, with the library named by KPGEMM_LIB; writes a reference-format CSV."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2008_13145_b200.sweep import CudaEventTimer, benchmark_sweep, write_benchmark_csv  # noqa: E402

probs = list(dict.fromkeys(p for _, p in bench.vgg16_layers(16)))
timer = CudaEventTimer("simt", probs, min_ms=3.0)
pm = benchmark_sweep(probs, timer=timer)
write_benchmark_csv(pm, sys.argv[1])
print("wrote", sys.argv[1], pm.n_problems, pm.n_configs)
