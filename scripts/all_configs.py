"""lambda_min for every BASELINE config on one B200: moments (host, row f3),
inverse iteration to 40 digits (row a11), certification with the GPU interval
LDL^T (row f1).  Prints one JSON line per config.

    python scripts/all_configs.py [config ...]   (default: 1 2 3 5 4)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_0902_0852_b200 import hgpu  # noqa: E402

CONFIGS = {  # n, beta_num, beta_den, P, Kv (certification), published lambda_1
    1: (64, 1, 1, 1024, 2048, None),
    2: (300, 7, 4, 4096, 12288, "1.4844e-102"),
    3: (1000, 1, 1, 24576, 49152, "1.0892e-52"),
    4: (1500, 1, 2, 65536, 65536, "6.6295e-2"),
    5: (2000, 3, 2, 32768, 65536, None),
}
KV_FALLBACK = {  # certification precision to try when Kv does not fit one GPU
    4: [49152, 32768],
    5: [49152],
}


def run(c: int) -> dict:
    n, bn, bd, k, kv, paper = CONFIGS[c]
    out = {"config": c, "n": n, "beta": f"{bn}/{bd}", "P": k, "paper": paper}
    t = time.time()
    strip = hgpu.build_moments(n, bn, bd, k)
    out["moments_s"] = round(time.time() - t, 2)
    t = time.time()
    m = hgpu.HankelMatrixGPU(strip, k)
    out["plan"] = m.plan()
    r = hgpu.inverse_iteration(m, hgpu.seeded_start_vector(n, k), 0, 40, digits=40)
    out["lambda_min"] = r["eigenvalue"]
    out["iterations"] = r["iterations"]
    out["inverse_iteration_s"] = round(time.time() - t, 2)
    del m
    out["certification"] = []
    for kvt in [kv] + KV_FALLBACK.get(c, []):
        t = time.time()
        lo, hi = hgpu.build_moments(n, bn, bd, kvt, interval=True)
        mom = round(time.time() - t, 2)
        t = time.time()
        try:
            im = hgpu.IntervalMatrixGPU(lo, hi, kvt)
            v = hgpu.verify_eigenvalue(im, r["eigenvalue"], 40)
            out["certification"].append({"kv": kvt, **v, "moments_s": mom,
                                         "seconds": round(time.time() - t, 2)})
            del im
            if v["status"] == "verified":
                break
        except hgpu.HgpuError as e:
            out["certification"].append({"kv": kvt, "error": str(e), "moments_s": mom,
                                         "seconds": round(time.time() - t, 2)})
            im = None
    return out


if __name__ == "__main__":
    cs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 4]
    for c in cs:
        print(json.dumps(run(c)), flush=True)
