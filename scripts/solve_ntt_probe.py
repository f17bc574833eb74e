"""One config-3 factorisation and one solve (HGPU_SOLVE_NTT selects the AXPY),
for launch lists / ncu captures of the solve kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from paper_0902_0852_b200 import hgpu  # noqa: E402
import pyoracle as po  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 24576
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = hgpu.HankelMatrixGPU(po.exact_strip(n, 1, 1, k), k)
print(hgpu.inverse_iteration(m, hgpu.seeded_start_vector(n, k), 0, reps)["iterations"])
