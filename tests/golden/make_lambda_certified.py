"""Generates tests/golden/lambda_certified.json: 40-digit lambda_1 values for
BASELINE configs 1 and 2, computed by the inverse-iteration restatement
(oracle/pyoracle.py:inverse_iteration_py over the C LDL^T restatement) and
CERTIFIED by the reference's own interval LDL^T sign test (verify.cpp:8-42,
via oracle/_ref): the matrix at the value is positive definite and at the
value + 1 ulp (last of 40 digits) it is not.  The GPU tests compare against
these digits (the interval test at N=300 takes minutes, so it runs here).

    python tests/golden/make_lambda_certified.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from fractions import Fraction  # noqa: E402

import pyoracle as po  # noqa: E402


def start_vector(n, k, seed=0):
    out = []
    for v in np.random.default_rng(seed).uniform(-1.0, 1.0, n):
        f = Fraction(float(v)) * (1 << k)
        out.append(int(f) if f >= 0 else -int(-f))
    return out


def main():
    ref, orc = po.RefLib(), po.OracleLib()
    g2 = json.load(open(os.path.join(HERE, "config2_strip.json")))
    cases = [
        ("config1", 64, (1, 1), 1024, po.exact_strip(64, 1, 1, 1024), 2048),
        ("config2", 300, (7, 4), 4096, [int(v, 16) for v in g2["strip"]], 12288),
    ]
    out = []
    for name, n, (bn, bd), k, strip, kv in cases:
        t = time.time()
        rhos = po.inverse_iteration_py(strip, k, start_vector(n, k), 0, 40,
                                       factor=lambda s, x, kk: orc.ldlt(s, x, kk, capture=True))
        lam = ref.truncate_sig_digits(rhos[-1], k, 40)
        lo = ref.interval_sign_decimal(n, bn, bd, kv, lam)
        hi = ref.interval_sign_decimal(n, bn, bd, kv, ref.bump_last_digit(lam))
        assert (lo, hi) == (1, -1), (name, lo, hi)
        out.append({"name": name, "n": n, "beta": f"{bn}/{bd}", "frac_bits": k,
                    "lambda_40": lam, "certified_at_bits": kv,
                    "iterations": len(rhos), "rho_last": po.to_hex(rhos[-1])})
        print(name, lam, f"{time.time() - t:.0f}s", flush=True)
    with open(os.path.join(HERE, "lambda_certified.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
