"""Small end-to-end run for compute-sanitizer: N=96 factorisation at x1 (far
rows, three panels), inverse iteration (solves, Rayleigh-quotient kernels,
register-ladder reciprocal), against the oracle."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from paper_0902_0852_b200 import hgpu  # noqa: E402
import pyoracle as po  # noqa: E402

n, k = 96, 1536
strip = po.exact_strip(n, 1, 1, k)
m = hgpu.HankelMatrixGPU(strip, k)
x = -(1 << (k - 16))
got = m.ldlt(x, capture=True)
want = po.OracleLib().ldlt(strip, x, k, capture=True)
assert got.pivots == want.pivots and got.ratios == want.ratios
u = hgpu.seeded_start_vector(n, k)
r = hgpu.inverse_iteration(m, u, 0, 40, digits=30)
w = po.inverse_iteration_py(strip, k, u, 0, 40)
assert r["rho"] == w, "rho differs"
print("sanity ok", r["eigenvalue"], r["iterations"])
