"""CPU: the oracle is pinned before it is trusted.

The compiled reference (oracle/_ref) reproduces the reference's own
known-answer tests; the C and Python restatements agree with it bit for bit;
and all of them agree with the committed golden fixtures that the reference
generated (tests/golden/make_golden.py)."""
import hashlib
import json
import math
import os

import pytest

from helpers import random_pd_hankel, strip_from_ints
import pyoracle as po

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ref():
    return po.RefLib()


@pytest.fixture(scope="module")
def orc():
    return po.OracleLib()


def test_reference_two_by_two(ref):
    # tests/test_ldlt.cpp:96-109
    assert ref.ldlt_serial(strip_from_ints([2, 0, 3], 32), 0, 32).det == 6 << 32
    r = ref.ldlt_serial(strip_from_ints([2, 1, 2], 32), 0, 32)
    assert r.det == 3 << 32 and r.pivots == [2 << 32, 3 << 31] and r.ratios == {(0, 1): 1 << 15}


def test_reference_factorial_det_144(ref):
    # tests/test_ldlt.cpp:111-117
    assert ref.ldlt_serial(ref.build_strip(4, 1, 1, 512), 0, 512).det == 144 << 512


def test_reference_zero_pivot_index(ref):
    # tests/test_ldlt.cpp:185-194
    with pytest.raises(po.ZeroPivotError) as e:
        ref.ldlt_serial(strip_from_ints([1, 1, 1], 64), 0, 64)
    assert e.value.pivot_index == 1 and e.value.frac_bits == 64


def test_reference_lambda_pins(ref):
    assert ref.heig_run(4, "1/1")["eigenvalue"] == "5.29002939538683e-2"   # test_verify.cpp:78
    assert ref.heig_run(6, "1/1")["eigenvalue"].startswith("1.0451")      # test_capi.cpp:53
    r = ref.heig_run(100, "1/1")                                            # README.md:110-116
    assert (r["eigenvalue"], r["k_bits"], r["iterations"]) == ("2.10788597588794e-15", 832, 8)


def test_exact_strip_equals_reference_build_matrix(ref):
    for n, b, k in [(10, (1, 1), 512), (12, (1, 2), 640), (64, (1, 1), 1024)]:
        assert ref.build_strip(n, *b, k) == po.exact_strip(n, *b, k)


def test_closed_form_beta1_config1(ref):
    # SURVEY §7 known answer, BASELINE config 1 size
    want = ref.ldlt_serial(ref.build_strip(64, 1, 1, 1024), 0, 1024)
    cf = po.closed_form_beta1(64, 1024)
    assert want.pivots == cf.pivots and want.ratios == cf.ratios and want.det == cf.det


@pytest.mark.parametrize("seed,n,f", [(53, 6, 128), (59, 9, 160), (61, 14, 128), (67, 30, 256)])
def test_restatements_match_reference(ref, orc, seed, n, f):
    strip = random_pd_hankel(seed, n, f)
    for x in (0, -(7 << (f - 4)), 1 << (f // 2)):
        want = ref.ldlt_serial(strip, x, f, capture=True)
        got_c = orc.ldlt(strip, x, f, capture=True)
        assert (got_c.det, got_c.pivots, got_c.ratios) == (want.det, want.pivots, want.ratios)
        if n <= 14:
            got_py = po.ldlt_py(strip, x, f)
            assert (got_py.det, got_py.pivots, got_py.ratios) == (want.det, want.pivots, want.ratios)


def test_reference_parallel_bit_identical_across_workers(ref):
    # tests/test_parallel.cpp:42-55
    for n in (9, 24):
        strip = random_pd_hankel(73 + n, n, 128)
        x = 1 << 100
        serial = ref.ldlt_serial(strip, x, 128, capture=False).det
        for workers in (1, 2, 3, 4, 5, 8):
            assert ref.ldlt_parallel(strip, x, 128, workers)[0] == serial


def test_column_owners_reflected_round_robin(ref):
    # tests/test_ldlt.cpp:73-92
    assert ref.column_owners(8, 4) == [0, 1, 2, 3, 3, 2, 1, 0]
    assert ref.column_owners(13, 3) == [0, 1, 2, 2, 1, 0, 0, 1, 2, 2, 1, 0, 0]
    for n in (7, 40, 101):
        for s in (1, 2, 3, 5, 8):
            assert ref.column_owners(n, s) == po.column_owners(n, s)


def test_golden_ldlt_fixtures(orc):
    cases = json.load(open(os.path.join(GOLDEN, "ldlt_small.json")))
    assert len(cases) >= 6
    for c in cases:
        strip = [int(v, 16) for v in c["strip"]]
        k, x = c["frac_bits"], int(c["x"], 16)
        r = orc.ldlt(strip, x, k, capture=True)
        assert po.to_hex(r.det) == c["det"], c["name"]
        assert [po.to_hex(v) for v in r.pivots] == c["pivots"], c["name"]
        assert [[p, q, po.to_hex(v)] for (p, q), v in sorted(r.ratios.items())] == c["ratios"]


def test_golden_config2_digest(orc):
    g = json.load(open(os.path.join(GOLDEN, "config2_strip.json")))
    strip = [int(v, 16) for v in g["strip"]]
    r = orc.ldlt(strip, 0, g["frac_bits"], capture=True)
    h = hashlib.sha256()
    for v in r.pivots:
        h.update(po.to_hex(v).encode() + b"\n")
    assert h.hexdigest() == g["pivots_sha256"]


def test_golden_lambda_fixture_pins():
    lam = {(d["n"], d["beta"]): d for d in json.load(open(os.path.join(GOLDEN, "lambda_secant.json")))}
    assert lam[(4, "1/1")]["eigenvalue"] == "5.29002939538683e-2"
    assert lam[(100, "1/1")]["eigenvalue"] == "2.10788597588794e-15"
    # mpmath value for config 1: 5.5000214686372010414e-12
    assert lam[(64, "1/1")]["eigenvalue"] == "5.50002146863720e-12"


def test_fold_restatement(orc):
    piv = po.closed_form_beta1(30, 512).pivots
    assert orc.fold(piv, 512) == po.fold_pivots(piv, 512)
    assert po.fold_pivots(piv, 512) == math.prod(math.factorial(k) ** 2 for k in range(30)) << 512


def test_inverse_iteration_restatement_config1(ref):
    """a11 restatement on BASELINE config 1: converges to the reference's
    secant lambda_1 and its 40 digits pass the reference's interval test."""
    import numpy as np
    from fractions import Fraction
    n, k = 64, 1024
    strip = po.exact_strip(n, 1, 1, k)
    u = []
    for v in np.random.default_rng(0).uniform(-1.0, 1.0, n):
        f = Fraction(float(v)) * (1 << k)
        u.append(int(f) if f >= 0 else -int(-f))
    rhos = po.inverse_iteration_py(strip, k, u, 0, 40,
                                   factor=lambda s, x, kk: ref.ldlt_serial(s, x, kk, True))
    assert 4 <= len(rhos) < 40
    lam = ref.truncate_sig_digits(rhos[-1], k, 40)
    assert lam.startswith("5.50002146863720") and lam.endswith("e-12")
    assert ref.interval_sign_decimal(n, 1, 1, 2 * k, lam) == 1
    assert ref.interval_sign_decimal(n, 1, 1, 2 * k, ref.bump_last_digit(lam)) == -1


@pytest.mark.parametrize("seed,n,k", [(111, 6, 256), (113, 20, 512)])
def test_inverse_iteration_restatement_finds_lambda1(orc, seed, n, k):
    strip = random_pd_hankel(seed, n, k)
    u = [((-1) ** i) << (k - 1 - i % 3) for i in range(n)]
    rho = po.inverse_iteration_py(strip, k, u, 0, 40)[-1]
    neg = lambda x: sum(1 for p in orc.ldlt(strip, x, k, capture=True).pivots if p < 0)
    assert neg(rho - (rho >> 40)) == 0 and neg(rho + (rho >> 40)) == 1


@pytest.mark.parametrize("n,bn,bd,k", [(8, 7, 4, 256), (12, 3, 2, 512), (10, 1, 2, 384), (30, 7, 4, 1024)])
def test_interval_restatement_matches_reference(ref, n, bn, bd, k):
    """ldlt_interval_py (row f1's checker) against the reference's own
    ldlt_det_interval on its certified interval strips."""
    lo, hi = ref.build_interval_strip(n, bn, bd, k)
    for dec in ("1e-300", "1e-30", "3.5e-10", "5e-1", "1.2e0"):
        xl, xh = ref.decimal_to_interval(dec, k)
        try:
            want = ref.ldlt_interval(lo, hi, k, xl, xh)
        except po.ZeroPivotError as e:
            with pytest.raises(po.ZeroPivotError) as got:
                po.ldlt_interval_py(lo, hi, k, xl, xh)
            assert got.value.pivot_index == e.pivot_index
            continue
        assert po.ldlt_interval_py(lo, hi, k, xl, xh).det == want
