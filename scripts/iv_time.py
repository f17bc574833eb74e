"""Device time of the interval LDL^T at config 3 (Kv = 49152) and of the
point LDL^T at the same precision."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import bench  # noqa: E402
from paper_0902_0852_b200 import hgpu  # noqa: E402

n, kv = 1000, 49152
strip = bench.config_strip(n, kv)
t = time.time()
m = hgpu.IntervalMatrixGPU(strip, strip, kv)
print("upload", round(time.time() - t, 2), m.plan(), flush=True)
lam_lo = int(1.0892427421041e-52 * 2 ** 200) << (kv - 200)
for i in range(2):
    t = time.time()
    r = m.ldlt_interval(lam_lo, lam_lo)
    print(f"interval wall {time.time() - t:.2f}s device {r['device_ms']:.0f} ms sign {r['det_sign']}", flush=True)
del m
p = hgpu.HankelMatrixGPU(strip, kv)
for i in range(2):
    t = time.time()
    r = p.ldlt(lam_lo)
    print(f"point wall {time.time() - t:.2f}s device {r.device_ms:.0f} ms", flush=True)
