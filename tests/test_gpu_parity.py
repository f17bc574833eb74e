"""GPU parity: the CUDA LDL^T path (through the C ABI) against the oracle.

Bit-exact: pivots D_p, ratio columns R_p[r] and ZeroPivot indices must equal
the reference's ldlt_det_serial (ldlt.cpp:31-77) on the same strip and shift.
"""
import math

import ctypes

import pytest

from helpers import random_pd_hankel, strip_from_ints
import pyoracle as po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hg():
    from paper_0902_0852_b200 import hgpu
    hgpu.load()
    return hgpu


@pytest.fixture(scope="module")
def ref():
    return po.OracleLib()


def assert_same(gpu, want, check_ratios=True):
    assert len(gpu.pivots) == len(want.pivots)
    for p, (a, b) in enumerate(zip(gpu.pivots, want.pivots)):
        assert a == b, f"pivot {p} differs"
    if check_ratios:
        assert gpu.ratios.keys() == want.ratios.keys()
        bad = [k for k in want.ratios if gpu.ratios[k] != want.ratios[k]]
        assert not bad, f"{len(bad)} ratios differ, first {bad[:3]}"


def test_two_by_two_by_hand(hg):
    # tests/test_ldlt.cpp:96-109
    m = hg.HankelMatrixGPU(strip_from_ints([2, 0, 3], 32), 32)
    r = m.ldlt(0, capture=True)
    assert r.pivots == [2 << 32, 3 << 32]
    m = hg.HankelMatrixGPU(strip_from_ints([2, 1, 2], 32), 32)
    r = m.ldlt(0, capture=True)
    assert r.pivots == [2 << 32, 3 << 31]
    assert r.ratios[(0, 1)] == 1 << 15  # 1/2 at 16 frac bits


def test_one_by_one(hg):
    # tests/test_ldlt.cpp:196-201: a 1x1 matrix runs no elimination
    m = hg.HankelMatrixGPU(strip_from_ints([7], 32), 32)
    assert m.ldlt(0).pivots == [7 << 32]


def test_factorial_4x4(hg):
    # tests/test_ldlt.cpp:111-117: det 144, pivots (k!)^2
    strip = po.exact_strip(4, 1, 1, 512)
    r = hg.HankelMatrixGPU(strip, 512).ldlt(0, capture=True)
    assert r.pivots == [(math.factorial(k) ** 2) << 512 for k in range(4)]
    assert po.fold_pivots(r.pivots, 512) == 144 << 512


def test_zero_pivot_index(hg):
    # tests/test_ldlt.cpp:185-194: all-ones 2x2 collapses in column 1
    m = hg.HankelMatrixGPU(strip_from_ints([1, 1, 1], 64), 64)
    with pytest.raises(hg.ZeroPivot) as ei:
        m.ldlt(0)
    assert ei.value.pivot_index == 1
    # all-ones 3x3 (tests/test_parallel.cpp:90-97)
    m = hg.HankelMatrixGPU([1 << 64] * 5, 64)
    with pytest.raises(hg.ZeroPivot) as ei:
        m.ldlt(0)
    assert ei.value.pivot_index == 1


def test_precision_mismatch(hg):
    m = hg.HankelMatrixGPU(strip_from_ints([2, 1, 2], 32), 32)
    with pytest.raises(hg.PrecisionMismatch):
        m.ldlt(0, x_frac_bits=64)


@pytest.mark.parametrize("seed,n,f", [(53, 6, 128), (59, 8, 160), (61, 9, 128),
                                      (73, 24, 128), (79, 40, 256), (83, 70, 512)])
def test_random_pd_hankel_bit_exact(hg, ref, seed, n, f):
    strip = random_pd_hankel(seed, n, f)
    m = hg.HankelMatrixGPU(strip, f)
    for x in (0, -(7 << (f - 4)), 1 << (f // 2 + 3)):
        want = ref.ldlt(strip, x, f, capture=True)
        got = m.ldlt(x, capture=True)
        assert_same(got, want)


def test_config1_closed_form(hg):
    # BASELINE config 1: N=64, beta=1, P=1024; known answer D_p=(p!)^2 etc.
    n, k = 64, 1024
    strip = po.exact_strip(n, 1, 1, k)
    got = hg.HankelMatrixGPU(strip, k).ldlt(0, capture=True)
    assert_same(got, po.closed_form_beta1(n, k))


def test_config1_shifted_against_reference(hg):
    ref = po.RefLib()
    n, k = 64, 1024
    strip = ref.build_strip(n, 1, 1, k)
    m = hg.HankelMatrixGPU(strip, k)
    x = 5 << (k - 40)  # 5 * 2^-40, below lambda_1 = 5.5e-12? no: above 0
    for xx in (0, -(1 << (k - 16)), x):
        try:
            want = ref.ldlt_serial(strip, xx, k, capture=True)
        except po.ZeroPivotError as e:
            with pytest.raises(hg.ZeroPivot) as ei:
                m.ldlt(xx)
            assert ei.value.pivot_index == e.pivot_index
            continue
        assert_same(m.ldlt(xx, capture=True), want)


def test_set_strip_reuses_the_handle(hg, ref):
    # hgpu_matrix_set_strip: new moments of the same order and precision give
    # the factorisation of a fresh matrix, with the plan kept (fits) or
    # rebuilt (larger moments)
    k = 256
    a = random_pd_hankel(201, 40, k)
    b = random_pd_hankel(202, 40, k)
    big = [v << 200 for v in b]
    m = hg.HankelMatrixGPU(a, k)
    x = 1 << (k // 3)
    assert_same(m.ldlt(x, capture=True), ref.ldlt(a, x, k))
    for strip in (b, big, a):
        m.set_strip(strip)
        assert_same(m.ldlt(x, capture=True), ref.ldlt(strip, x, k))


def test_dump_interchange_round_trip(hg, tmp_path):
    """The reference's on-disk matrix format (hankel_matrix.cpp:52-87): a dump
    written by the reference itself loads onto the device and factorises like
    the strip passed through the ABI, and hgpu_matrix_dump writes the
    reference's text back byte for byte (negative and zero mantissas too)."""
    ref = po.RefLib()
    n, k = 24, 768
    text = ref._call("oref_build_strip", [ctypes.c_long, ctypes.c_ulong, ctypes.c_ulong, ctypes.c_long],
                     n, 7, 4, k)
    strip, kk = po.parse_dump(text)
    assert kk == k
    src = tmp_path / "ref.dump"
    src.write_text(text)
    m = hg.HankelMatrixGPU.from_dump(str(src))
    assert (m.n, m.frac_bits) == (n, k)
    x = -(1 << (k - 16))
    got = m.ldlt(x, capture=True)
    want = po.OracleLib().ldlt(strip, x, k, capture=True)
    assert got.pivots == want.pivots and got.ratios == want.ratios
    out = tmp_path / "gpu.dump"
    m.dump(str(out))
    assert out.read_text() == text
    # signed and zero entries survive the trip
    odd = [5, -(1 << 70) - 3, 0, 1 << 40, -1]
    a = hg.HankelMatrixGPU(odd, 64)
    a.dump(str(out))
    assert out.read_text() == po.make_dump(odd, 64)
    b = hg.HankelMatrixGPU.from_dump(str(out))
    b.dump(str(src))
    assert src.read_text() == po.make_dump(odd, 64)
