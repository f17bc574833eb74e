"""Independent check of config 4's lambda_1 (N=1500, beta=1/2, P=65536) with
the reference's own code, no repo code on the path.

PAPER.md:474 prints 6.6295e-2; the GPU pipeline
certifies 6.52947750188...e-2.  The sign of det(M - xI) settles it:

  x = 6.6e-2      det < 0  <=> an eigenvalue lies below 6.6e-2
                               (contradicts 6.6295e-2, agrees with 6.5295e-2)
  x = 6.5294e-2   det > 0  <=> no eigenvalue below 6.5294e-2

Both determinants run through the reference's ldlt_det_parallel
(ldlt.cpp:315-341, SharedMemoryChannel) at K = 65536 on the strip built by
the reference's build_matrix (hankel_matrix.cpp:13-31), compiled unchanged in
oracle/_ref.  Hours of CPU time: run it in the background

    nice -n 19 python tests/golden/make_config4_sign.py [workers]

Results are appended to tests/golden/config4_sign.json as they arrive.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402

OUT = os.path.join(HERE, "config4_sign.json")
N, BNUM, BDEN, K = 1500, 1, 2, 65536
PROBES = ["6.6e-2", "6.5294e-2"]


def main():
    workers = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    ref = po.RefLib()
    t0 = time.time()
    strip = ref.build_strip(N, BNUM, BDEN, K)
    rec = {"n": N, "beta": f"{BNUM}/{BDEN}", "frac_bits": K, "workers": workers,
           "strip_seconds": round(time.time() - t0, 1), "probes": []}
    if os.path.exists(OUT):
        rec["probes"] = json.load(open(OUT)).get("probes", [])
    done = {p["x"] for p in rec["probes"]}
    for x in PROBES:
        if x in done:
            continue
        r = ref.det_sign_parallel_decimal(strip, K, x, workers)
        rec["probes"].append({"x": x, "det_sign": r["sign"], "det_bits": r["bits"],
                              "seconds": round(r["seconds"], 1)})
        with open(OUT, "w") as f:
            json.dump(rec, f, indent=1)
        print(json.dumps(rec["probes"][-1]), flush=True)


if __name__ == "__main__":
    main()
