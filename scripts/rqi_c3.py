"""Time-to-lambda_min by inverse iteration at BASELINE config 3 (HGPU_RQI_TRACE=1
prints the per-iteration factor / solve split)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from paper_0902_0852_b200 import hgpu  # noqa: E402
import pyoracle as po  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 24576
m = hgpu.HankelMatrixGPU(po.exact_strip(n, 1, 1, k), k)
t = time.time()
r = hgpu.inverse_iteration(m, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
print("wall", time.time() - t, r["iterations"], r["seconds"], r["eigenvalue"])
