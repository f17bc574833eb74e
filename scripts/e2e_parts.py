"""Split of the end-to-end step: matrix construction, first factorisation
(plan + workspace + strip transforms + factorisation), second factorisation."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from paper_0902_0852_b200 import hgpu  # noqa: E402

n, k = 1000, 24576
strip = bench.config_strip(n, k)
x = bench.x1_shift(strip, k)
for rep in range(3):
    t0 = time.perf_counter()
    m = hgpu.HankelMatrixGPU(strip, k)
    t1 = time.perf_counter()
    r = m.ldlt(x)
    t2 = time.perf_counter()
    r2 = m.ldlt(x)
    t3 = time.perf_counter()
    del m
    t4 = time.perf_counter()
    print(f"construct {1e3*(t1-t0):.1f} ms  first {1e3*(t2-t1):.1f} ms (device {r.device_ms:.1f})  "
          f"second {1e3*(t3-t2):.1f} ms (device {r2.device_ms:.1f})  free {1e3*(t4-t3):.1f} ms", flush=True)
