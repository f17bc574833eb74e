"""lambda_1 of (n, beta, P) by GPU inverse iteration (40 digits) and its
certification at each Kv given (GPU interval LDL^T).

    python scripts/lambda_run.py n beta_num beta_den P Kv [Kv ...] [--lambda L]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_0902_0852_b200 import hgpu  # noqa: E402

args = sys.argv[1:]
lam = None
if "--lambda" in args:
    i = args.index("--lambda")
    lam = args[i + 1]
    del args[i:i + 2]
n, bn, bd, k = map(int, args[:4])
kvs = [int(a) for a in args[4:]]
out = {"n": n, "beta": f"{bn}/{bd}", "P": k}
if lam is None:
    t = time.time()
    m = hgpu.HankelMatrixGPU(hgpu.build_moments(n, bn, bd, k), k)
    r = hgpu.inverse_iteration(m, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
    lam = r["eigenvalue"]
    out.update(lambda_min=lam, iterations=r["iterations"], seconds=round(time.time() - t, 2))
    del m
else:
    out["lambda_min"] = lam
out["certification"] = []
for kv in kvs:
    t = time.time()
    lo, hi = hgpu.build_moments(n, bn, bd, kv, interval=True)
    try:
        im = hgpu.IntervalMatrixGPU(lo, hi, kv)
        out["certification"].append({"kv": kv, **hgpu.verify_eigenvalue(im, lam, 40),
                                     "seconds": round(time.time() - t, 2)})
        del im
    except hgpu.HgpuError as e:
        out["certification"].append({"kv": kv, "error": str(e)})
print(json.dumps(out), flush=True)
