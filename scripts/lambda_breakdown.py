"""Time-to-lambda_min at config 3 after a warm-up factorisation in the same
process (as bench.py measures it); HGPU_RQI_TRACE=1 prints the split."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from paper_0902_0852_b200 import hgpu  # noqa: E402
import pyoracle as po  # noqa: E402

n, k = 1000, 24576
strip = po.exact_strip(n, 1, 1, k)
m = hgpu.HankelMatrixGPU(strip, k)
m.ldlt(-(1 << (k - 16)))
del m
for rep in range(2):
    t = time.perf_counter()
    m = hgpu.HankelMatrixGPU(strip, k)
    t1 = time.perf_counter()
    r = hgpu.inverse_iteration(m, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
    print("rep", rep, "create", round(t1 - t, 3), "total", round(time.perf_counter() - t, 3),
          r["iterations"], r["eigenvalue"], flush=True)
    del m
