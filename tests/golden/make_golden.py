"""Generates the committed golden fixtures from the reference itself.

Run in the build container (needs /root/reference compiled into
oracle/_ref/libheig_ref.so by `make -C oracle`):

    python tests/golden/make_golden.py

Every value below is produced by the reference's own code paths
(hankel_matrix.cpp build_matrix, ldlt.cpp ldlt_det_serial with LdltCapture,
secant.cpp secant_smallest_eigenvalue, decimal.cpp), so the fixtures pin both
the oracle restatements and the GPU path without the reference at run time.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))
import pyoracle as po  # noqa: E402
from helpers import random_pd_hankel  # noqa: E402


def hx(v):
    return po.to_hex(v)


def digest(values):
    h = hashlib.sha256()
    for v in values:
        h.update(hx(v).encode() + b"\n")
    return h.hexdigest()


def main():
    ref = po.RefLib()
    cases = []
    # small LDL^T captures: random PD strips, config 1, beta = 7/4 and 3/2
    specs = [("random_pd_53_6_128", random_pd_hankel(53, 6, 128), 128, [0, -(7 << 124)]),
             ("random_pd_73_24_128", random_pd_hankel(73, 24, 128), 128, [1 << 100]),
             ("config1_n64_beta1_p1024", ref.build_strip(64, 1, 1, 1024), 1024, [0, -(1 << 1008)]),
             ("beta7_4_n20_p512", ref.build_strip(20, 7, 4, 512), 512, [0]),
             ("beta3_2_n16_p512", ref.build_strip(16, 3, 2, 512), 512, [0])]
    for name, strip, k, shifts in specs:
        for x in shifts:
            r = ref.ldlt_serial(strip, x, k, capture=True)
            cases.append({"name": name, "frac_bits": k, "x": hx(x),
                          "strip": [hx(v) for v in strip],
                          "det": hx(r.det), "pivots": [hx(v) for v in r.pivots],
                          "ratios": [[p, rr, hx(v)] for (p, rr), v in sorted(r.ratios.items())]})
    with open(os.path.join(HERE, "ldlt_small.json"), "w") as f:
        json.dump(cases, f)

    # BASELINE config 2 (N=300, beta=7/4, P=4096): strip from the reference's
    # certified Gamma, and digests of its pivots / determinant at x = 0
    n, k = 300, 4096
    strip = ref.build_strip(n, 7, 4, k)
    r = ref.ldlt_serial(strip, 0, k, capture=False)
    pv = ref.ldlt_serial(strip, 0, k, capture=True).pivots
    with open(os.path.join(HERE, "config2_strip.json"), "w") as f:
        json.dump({"n": n, "beta": "7/4", "frac_bits": k, "strip": [hx(v) for v in strip],
                   "det_sha256": digest([r.det]), "pivots_sha256": digest(pv),
                   "pivot_first": hx(pv[0]), "pivot_last": hx(pv[-1])}, f)

    # lambda_1 pins from the reference's secant (15 digits) and iterates
    lam = []
    for n, b, k in [(4, (1, 1), 512), (6, (1, 1), 512), (64, (1, 1), 1024), (100, (1, 1), 832),
                    (40, (7, 4), 1024), (30, (1, 2), 2048)]:
        strip = ref.build_strip(n, b[0], b[1], k)
        sec = ref.secant(strip, k)
        lam.append({"n": n, "beta": f"{b[0]}/{b[1]}", "frac_bits": k,
                    "eigenvalue": sec["eigenvalue"], "iterations": sec["iterations"],
                    "iterates": [[hx(x), hx(d)] for x, d in sec["iterates"]],
                    "strip_sha256": digest(strip)})
    with open(os.path.join(HERE, "lambda_secant.json"), "w") as f:
        json.dump(lam, f)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
