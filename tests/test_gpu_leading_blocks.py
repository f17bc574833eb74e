"""Full-size BASELINE factorisations pinned to the reference.

* Leading blocks: the GPU factorises the whole N x N matrix (configs 3, 4, 5,
  at x = 0 and at the secant's first probe x1, the shift bench.py times) and
  its leading n' x n' block of pivots and ratio columns must equal the
  reference's ldlt_det_serial with LdltCapture on that block
  (tests/golden/leading_blocks.json, made by the reference itself:
  tests/golden/make_leading_blocks.py).  The leading block of the
  submatrix-order LDL^T depends on the leading block only (ldlt.cpp:65-71).
* Config 3 at x = 0: all 499 500 ratios and all pivots against the beta = 1
  closed form, by digest.
"""
import hashlib
import json
import math
import os

import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def hg():
    from paper_0902_0852_b200 import hgpu
    hgpu.load()
    return hgpu


def digest(values):
    h = hashlib.sha256()
    for v in values:
        h.update(po.to_hex(v).encode() + b"\n")
    return h.hexdigest()


def secant_x1(strip0, k):
    mant = min(strip0, 1 << k) >> 16  # secant.cpp:7-16
    return -(mant if mant else 1)


def cases():
    return json.load(open(os.path.join(GOLDEN, "leading_blocks.json")))


def full_strip(hg, c):
    n, k = c["n"], c["frac_bits"]
    num, den = map(int, c["beta"].split("/"))
    if den == 1 or (num, den) == (1, 2):
        strip = po.exact_strip(n, num, den, k)
    else:
        # the repo's threaded build_matrix, bit-identical to the reference's
        # (tests/test_moments.py, tests/golden/moments_digests.json)
        strip = hg.build_moments(n, num, den, k)
    assert digest(strip[:2 * c["n_prime"] - 1]) == c["strip_sha256"]
    return strip


_strips = {}


@pytest.mark.parametrize("case", cases(), ids=lambda c: f"{c['name']}-{c['shift']}")
def test_full_size_leading_block(hg, case):
    key = case["name"]
    if key not in _strips:
        _strips.clear()
        _strips[key] = full_strip(hg, case)
    strip = _strips[key]
    k, nb = case["frac_bits"], case["n_prime"]
    x = 0 if case["shift"] == "x0" else secant_x1(strip[0], k)
    assert po.to_hex(x) == case["x"]
    m = hg.HankelMatrixGPU(strip, k)
    r = m.ldlt(x, capture_rows=nb, ratio_digest=True)
    m.close()
    assert po.to_hex(r.pivots[0]) == case["pivot_first"]
    assert po.to_hex(r.pivots[nb - 1]) == case["pivot_last"]
    assert digest(r.pivots[:nb]) == case["pivots_sha256"]
    assert r.ratio_sha256 == case["ratios_sha256"]
    # x <= 0 keeps M - xI positive definite (test_ldlt.cpp:171-183)
    assert all(v > 0 for v in r.pivots)


def closed_form_digests(n, k):
    """Streaming digests of the beta = 1, x = 0 closed form: D_p = (p!)^2,
    R_p[r] = C(r, p) r!/p! 2^(K/2), in (p, r) order."""
    k2 = k // 2
    f = [math.factorial(i) for i in range(n)]
    hp, hr = hashlib.sha256(), hashlib.sha256()
    for p in range(n):
        hp.update(po.to_hex((f[p] * f[p]) << k).encode() + b"\n")
    for p in range(n - 1):
        # C(r, p) r!/p! for r = p+1.. by the recurrence
        # t_r = t_{r-1} * r * r / (r - p)   (exact at every step)
        t = 1
        for r in range(p + 1, n):
            t = t * r * r // (r - p)
            hr.update(po.to_hex(t << k2).encode() + b"\n")
    return hp.hexdigest(), hr.hexdigest()


def test_closed_form_recurrence():
    # the streaming recurrence equals the closed form on a small case
    n, k = 12, 64
    cf = po.closed_form_beta1(n, k)
    dp, dr = closed_form_digests(n, k)
    assert dp == digest(cf.pivots)
    assert dr == digest([cf.ratios[key] for key in sorted(cf.ratios)])


def test_config3_all_ratios_closed_form(hg):
    # BASELINE config 3 at x = 0, every pivot and every ratio
    n, k = 1000, 24576
    strip = po.exact_strip(n, 1, 1, k)
    m = hg.HankelMatrixGPU(strip, k)
    r = m.ldlt(0, ratio_digest=True)
    m.close()
    dp, dr = closed_form_digests(n, k)
    assert digest(r.pivots) == dp
    assert r.ratio_sha256 == dr
