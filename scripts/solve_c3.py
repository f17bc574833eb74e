"""One factorisation + one triangular solve at BASELINE config 3 (for the
ncu launch list of the solve kernels)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from paper_0902_0852_b200 import hgpu  # noqa: E402
import pyoracle as po  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 24576
it = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = hgpu.HankelMatrixGPU(po.exact_strip(n, 1, 1, k), k)
r = hgpu.inverse_iteration(m, hgpu.seeded_start_vector(n, k), 0, it, digits=15)
print(r["iterations"], r["seconds"])
