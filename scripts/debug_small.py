import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'oracle'))
from paper_0902_0852_b200 import hgpu
import pyoracle as po
n, k = int(sys.argv[1]), int(sys.argv[2])
strip = po.exact_strip(n, 1, 1, k)
m = hgpu.HankelMatrixGPU(strip, k)
print('plan', m.plan(), flush=True)
r = m.ldlt(0)
print('ok', r.pivots == po.closed_form_beta1(n, k).pivots, flush=True)
