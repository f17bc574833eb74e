"""Reference fixtures for the BASELINE configs' full-size factorisations,
checked on their leading blocks.

The submatrix-order LDL^T of the leading n' x n' block is a prefix of the
full one: ldlt.cpp:65-71 only ever writes W[r][c] with r, c > p, so pivots
p < n' and ratios R_p[r] with p < r < n' depend on the leading block alone.
The GPU runs the whole N x N factorisation (tests/test_gpu_leading_blocks.py)
and compares its leading block with these digests, which the reference's own
ldlt_det_serial with LdltCapture (oracle/_ref, compiled unchanged) produced
here on the leading block:

    python tests/golden/make_leading_blocks.py        # ~5 min, all cores

Shifts: x = 0 and x1, the secant's first probe (secant.cpp:7-16:
-trunc(min(M00, 1) / 2^16), the shift bench.py times).  Strips come from the
reference's build_matrix on n' (anti-diagonal s depends on s and K only, so
they equal the first 2n'-1 entries of the N x N strip).
"""
import hashlib
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402

OUT = os.path.join(HERE, "leading_blocks.json")

# (name, N, beta_num, beta_den, K, n')
CASES = [
    ("config2", 300, 7, 4, 4096, 300),   # the whole matrix
    ("config3", 1000, 1, 1, 24576, 270),
    ("config4", 1500, 1, 2, 65536, 200),
    ("config5", 2000, 3, 2, 32768, 200),
]


def secant_x1(strip0: int, k: int) -> int:
    """initial_points (secant.cpp:7-16): -(min(M00, 1) >> 16), at least 1 ulp."""
    mant = min(strip0, 1 << k) >> 16
    return -(mant if mant else 1)


def digest(values) -> str:
    h = hashlib.sha256()
    for v in values:
        h.update(po.to_hex(v).encode() + b"\n")
    return h.hexdigest()


def one(args):
    name, n, bn, bd, k, nb, which = args
    ref = po.RefLib()
    strip = ref.build_strip(nb, bn, bd, k)
    x = 0 if which == "x0" else secant_x1(strip[0], k)
    r = ref.ldlt_serial(strip, x, k, capture=True)
    ratios = [r.ratios[key] for key in sorted(r.ratios)]
    return {"name": name, "shift": which, "n": n, "beta": f"{bn}/{bd}", "frac_bits": k,
            "n_prime": nb, "x": po.to_hex(x), "strip_sha256": digest(strip),
            "pivots_sha256": digest(r.pivots), "ratios_sha256": digest(ratios),
            "n_ratios": len(ratios), "pivot_first": po.to_hex(r.pivots[0]),
            "pivot_last": po.to_hex(r.pivots[-1]),
            "negative_pivots": sum(1 for v in r.pivots if v < 0)}


def main():
    only = set(sys.argv[1:])  # e.g. config2: regenerate some cases only
    jobs = []
    for name, n, bn, bd, k, nb in CASES:
        shifts = ["x1"] if name == "config3" else ["x0", "x1"]
        if only and name not in only:
            continue
        jobs += [(name, n, bn, bd, k, nb, w) for w in shifts]
    with ProcessPoolExecutor(len(jobs)) as ex:
        out = list(ex.map(one, jobs))
    if only and os.path.exists(OUT):
        keep = [c for c in json.load(open(OUT)) if c["name"] not in only]
        out = sorted(keep + out, key=lambda c: (c["name"], c["shift"]))
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    for o in out:
        print(o["name"], o["shift"], o["n_prime"], o["pivots_sha256"][:12], o["ratios_sha256"][:12])


if __name__ == "__main__":
    main()
