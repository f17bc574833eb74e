import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'oracle'))
from paper_0902_0852_b200 import hgpu
import pyoracle as po
n, k, digits = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
strip = po.exact_strip(n, 1, 1, k)
m = hgpu.HankelMatrixGPU(strip, k)
t = time.time()
r = hgpu.smallest_eigenvalue(m, digits)
print(f"N={n} K={k} digits={digits}: lambda1={r['eigenvalue']} iterations={r['iterations']} det_s={r['det_seconds']:.2f} wall={time.time()-t:.2f}", flush=True)
