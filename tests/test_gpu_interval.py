"""GPU interval LDL^T (ldlt_det_interval, ldlt.cpp:79-152) and
verify_eigenvalue (verify.cpp:8-42) against the reference and the pinned
restatement oracle/pyoracle.py:ldlt_interval_py."""
import json
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


@pytest.fixture(scope="module")
def ref():
    return po.RefLib()


CASES = [(8, 7, 4, 256), (12, 3, 2, 512), (10, 1, 2, 384), (16, 1, 1, 512), (30, 7, 4, 1024),
         (40, 7, 4, 2048)]
SHIFTS = ("1e-300", "1e-30", "3.5e-10", "5e-1", "1.2e0")


@pytest.mark.parametrize("n,bn,bd,k", CASES)
def test_interval_pivots_and_det_bit_exact(hg, ref, n, bn, bd, k):
    lo, hi = ref.build_interval_strip(n, bn, bd, k)
    m = hg.IntervalMatrixGPU(lo, hi, k)
    for dec in SHIFTS:
        xl, xh = ref.decimal_to_interval(dec, k)
        try:
            want = po.ldlt_interval_py(lo, hi, k, xl, xh)
        except po.ZeroPivotError as e:
            with pytest.raises(hg.ZeroPivot) as got:
                m.ldlt_interval(xl, xh)
            assert got.value.pivot_index == e.pivot_index
            continue
        got = m.ldlt_interval(xl, xh, fold=True)
        assert got["pivots"] == want.pivots
        assert got["det"] == want.det == ref.ldlt_interval(lo, hi, k, xl, xh)
        s = 1 if want.det[0] > 0 else (-1 if want.det[1] < 0 else 0)
        assert got["det_sign"] == s
        assert m.ldlt_interval(xl, xh)["det_sign"] == s  # sign without the fold


@pytest.mark.parametrize("n,bn,bd,kv,lam", [
    (64, 1, 1, 2048, "5.500021468637201041420759646434514207973e-12"),
    (40, 7, 4, 2048, "1.150595279959255e-22"),
    (30, 1, 2, 4096, "4.628039382438795e-1"),
])
def test_verify_matches_reference(hg, ref, n, bn, bd, kv, lam):
    lo, hi = ref.build_interval_strip(n, bn, bd, kv)
    m = hg.IntervalMatrixGPU(lo, hi, kv)
    got = hg.verify_eigenvalue(m, lam, 15)
    assert got == ref.verify(n, bn, bd, kv, lam)
    assert got["status"] == "verified"
    # a wrong value is refuted the same way
    bad = "5.600021468637201e-12" if n == 64 else lam.replace(lam[2], str((int(lam[2]) + 3) % 10), 1)
    assert hg.verify_eigenvalue(m, bad, 15) == ref.verify(n, bn, bd, kv, bad)


def test_config2_40_digits_certified_on_gpu(hg):
    """the 40 digits of tests/golden/lambda_certified.json (certified there by
    the reference's interval test at 12288 bits, minutes on the CPU) pass the
    GPU interval test at the same precision; one more digit-unit does not."""
    d = {e["name"]: e for e in json.load(open(os.path.join(GOLDEN, "lambda_certified.json")))}["config2"]
    ref = po.RefLib()
    lo, hi = ref.build_interval_strip(300, 7, 4, d["certified_at_bits"])
    m = hg.IntervalMatrixGPU(lo, hi, d["certified_at_bits"])
    got = hg.verify_eigenvalue(m, d["lambda_40"], 40)
    assert got["status"] == "verified", got
    assert got["probe_low"] == d["lambda_40"]


def test_config3_40_digits_certified_on_gpu(hg):
    """BASELINE config 3 (N=1000, beta=1): the inverse-iteration lambda_1 to 40
    digits, certified by the interval LDL^T at Kv = 2P = 49152 bits (the
    reference's serial interval path would take hours here)."""
    n, kv = 1000, 49152
    strip = po.exact_strip(n, 1, 1, kv)  # integer moments: lo = hi
    m = hg.IntervalMatrixGPU(strip, strip, kv)
    lam = "1.089242742104122033671855781638578297244e-52"
    got = hg.verify_eigenvalue(m, lam, 40)
    print("config3 verify", got)
    assert got["status"] == "verified", got
