import os, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
from paper_0902_0852_b200 import hgpu
import pyoracle as po
n, k = 1000, 24576
strip = po.exact_strip(n, 1, 1, k)
m = hgpu.HankelMatrixGPU(strip, k); m.ldlt(-(1 << (k - 16))); del m
for i in range(2):
    t = time.perf_counter(); m = hgpu.HankelMatrixGPU(strip, k); r = m.ldlt(-(1 << (k - 16)))
    t1 = time.perf_counter(); r = m.ldlt(-(1 << (k - 16))); t2 = time.perf_counter()
    print("first", round(t1 - t, 3), "second", round(t2 - t1, 3), flush=True); del m
