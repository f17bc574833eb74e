import sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'oracle'))
from paper_0902_0852_b200 import hgpu
import pyoracle as po
n, k, bn, bd = map(int, sys.argv[1:5])
strip = po.exact_strip(n, bn, bd, k)
t = time.time(); m = hgpu.HankelMatrixGPU(strip, k); print('upload', round(time.time() - t, 2), m.plan(), flush=True)
t = time.time(); r = m.ldlt(0, profile=True); el = time.time() - t
print(f'N={n} K={k} beta={bn}/{bd}: factor wall {el:.3f}s device {r.device_ms:.1f}ms update {r.update_ms:.1f}ms prod {r.update_products:.3e} launches {r.launches}', flush=True)
