"""One config-3 factorisation (x1) with the chain's phase clocks on:
HGPU_DEBUG=256 prints the reciprocal's Newton levels at p=50, 4096 the
k_pivot phases every 100 stages.  Usage: HGPU_DEBUG=4352 python scripts/probe_chain.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import config_strip, x1_shift  # noqa: E402
from paper_0902_0852_b200 import hgpu  # noqa: E402

n, k = int(os.environ.get("N", "1000")), int(os.environ.get("K", "24576"))
strip = config_strip(n, k)
m = hgpu.HankelMatrixGPU(strip, k)
x = x1_shift(strip, k)
m.ldlt(x)
r = m.ldlt(x)
print(f"device {r.device_ms:.1f} ms, {r.launches} launches")
