"""Config-3 inverse iteration (time to lambda_min): one warm-up factorisation,
then hgpu_inverse_iteration from the seed-0 start vector (HGPU_RQI_TRACE=1
prints the per-step factor / solve split)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from paper_0902_0852_b200 import hgpu  # noqa: E402

n, k = 1000, 24576
strip = bench.config_strip(n, k)
m = hgpu.HankelMatrixGPU(strip, k)
m.ldlt(bench.x1_shift(strip, k))
for rep in range(2):
    t = time.time()
    rq = hgpu.inverse_iteration(m, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
    print(rq["eigenvalue"], rq["iterations"], f"wall {time.time() - t:.3f}s", flush=True)
