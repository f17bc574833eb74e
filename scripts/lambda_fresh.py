"""Where a fresh-handle time-to-lambda run spends its time (bench.py's
`time_to_lambda_min.seconds` flow): timed steps on one handle, drop it, then
new handle -> start vector -> inverse iteration, each part timed."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from paper_0902_0852_b200 import hgpu  # noqa: E402

n, k = 1000, 24576
strip = bench.config_strip(n, k)
x = bench.x1_shift(strip, k)
m = hgpu.HankelMatrixGPU(strip, k)
for _ in range(3):
    m.ldlt(x)
del m
for rep in range(2):
    t0 = time.perf_counter()
    mm = hgpu.HankelMatrixGPU(strip, k)
    t1 = time.perf_counter()
    u = hgpu.seeded_start_vector(n, k)
    t2 = time.perf_counter()
    rq = hgpu.inverse_iteration(mm, u, 0, 40, digits=40)
    t3 = time.perf_counter()
    print(f"rep {rep}: new handle {t1 - t0:.3f}s  start vector {t2 - t1:.3f}s  inverse iteration {t3 - t2:.3f}s "
          f"(engine-reported {rq['seconds']:.3f}s)  total {t3 - t0:.3f}s", flush=True)
    del mm
