"""One (or more) config-3 factorisations at the bench shift x1 (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from paper_0902_0852_b200 import hgpu  # noqa: E402

n, k = 1000, 24576
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
strip = bench.config_strip(n, k)
x = bench.x1_shift(strip, k)
m = hgpu.HankelMatrixGPU(strip, k)
for _ in range(reps):
    r = m.ldlt(x, profile=True)
    print(f"device {r.device_ms:.1f} ms", flush=True)
