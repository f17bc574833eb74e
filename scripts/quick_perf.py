import sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'oracle'))
from paper_0902_0852_b200 import hgpu
import pyoracle as po
n, k = int(sys.argv[1]), int(sys.argv[2])
strip = po.exact_strip(n, 1, 1, k)
t = time.time(); m = hgpu.HankelMatrixGPU(strip, k); print('upload', time.time() - t, m.plan(), flush=True)
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    t = time.time(); r = m.ldlt(0, profile=True); el = time.time() - t
    print(f'factor wall {el:.3f}s device {r.device_ms:.1f}ms update {r.update_ms:.1f}ms launches {r.update_launches} prod {r.update_products:.3e}', flush=True)
cf = po.closed_form_beta1(n, k)
print('pivots exact:', r.pivots == cf.pivots, flush=True)
