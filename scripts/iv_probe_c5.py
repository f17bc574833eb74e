"""Config 5 (N=2000, beta=3/2): where does the interval LDL^T at the lower
probe a = lambda_1 cut to `digits` digits first meet a pivot interval that
contains zero, as a function of Kv?  (How far the certification is from
conclusive at the interval workspaces that fit one B200.)"""
import json
import os
import sys
import time
from fractions import Fraction

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_0902_0852_b200 import hgpu  # noqa: E402

n, bn, bd = 2000, 3, 2
lam = "2.662638424964465055398799214994081026852e-279"
digits = int(sys.argv[1])
for kv in [int(a) for a in sys.argv[2:]]:
    t = time.time()
    lo, hi = hgpu.build_moments(n, bn, bd, kv, interval=True)
    tm = time.time() - t
    mant, ex = lam.split("e")
    a = Fraction(mant[:digits + 1]) * Fraction(10) ** int(ex)  # digits significant digits
    x = int(a * (1 << kv))
    out = {"kv": kv, "digits": digits, "moments_s": round(tm, 1)}
    try:
        im = hgpu.IntervalMatrixGPU(lo, hi, kv)
        t = time.time()
        r = im.ldlt_interval(x, x + 1)
        out.update(det_sign=r["det_sign"], device_ms=r["device_ms"])
        w = [(p, (h - l).bit_length(), max(abs(l), abs(h)).bit_length()) for p, (l, h) in enumerate(r["pivots"])]
        out["width_bits_vs_magnitude_bits"] = [w[i] for i in (0, 500, 1000, 1500, 1900, 1990, 1999)]
        del im
    except hgpu.HgpuError as e:
        out["error"] = str(e)
        out["pivot_index"] = getattr(e, "pivot_index", None)
    out["seconds"] = round(time.time() - t, 1)
    print(json.dumps(out), flush=True)
