"""GPU parity for the determinant fold (ldlt.cpp:22-27) and the smallest
eigenvalue (secant.cpp:27-117 driven by the GPU determinant), against the
reference compiled from its own sources (oracle/_ref) and the C restatement."""
import ctypes
import json
import os

import pytest

from helpers import random_pd_hankel
import pyoracle as po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hg():
    from paper_0902_0852_b200 import hgpu
    hgpu.load()
    return hgpu


@pytest.fixture(scope="module")
def ref():
    return po.RefLib()


@pytest.fixture(scope="module")
def orc():
    return po.OracleLib()


@pytest.mark.parametrize("n,k", [(4, 512), (64, 1024), (100, 832)])
def test_fold_exact_beta1(hg, orc, n, k):
    strip = po.exact_strip(n, 1, 1, k)
    m = hg.HankelMatrixGPU(strip, k)
    for x in (0, -(1 << (k - 16)), 3 << (k - 60)):
        r = m.ldlt(x, fold=True)
        assert r.det == po.fold_pivots(r.pivots, k)
        assert r.det == orc.ldlt(strip, x, k, capture=False).det


def test_fold_random_pd(hg, orc):
    for seed, n, f in [(101, 5, 96), (102, 17, 200), (103, 33, 256)]:
        strip = random_pd_hankel(seed, n, f)
        r = hg.HankelMatrixGPU(strip, f).ldlt(1 << (f // 3), fold=True)
        assert r.det == orc.ldlt(strip, 1 << (f // 3), f, capture=False).det


def test_fold_config3_against_gmp(hg, orc):
    # BASELINE config 3 at full size: pivots from the GPU, fold checked by
    # the GMP fold of the C restatement (det ~ 7.8 Mbit)
    n, k = 1000, 24576
    strip = po.exact_strip(n, 1, 1, k)
    r = hg.HankelMatrixGPU(strip, k).ldlt(0, fold=True)
    cf = po.closed_form_beta1(n, k)
    assert r.pivots == cf.pivots
    assert r.det == orc.fold(r.pivots, k)


@pytest.mark.parametrize("n,k,golden", [
    (4, 512, "5.29002939538683e-2"),    # tests/test_verify.cpp:78
    (6, 512, None),                     # tests/test_capi.cpp:53: starts 1.0451
    (64, 1024, None),                   # BASELINE config 1
    (100, 832, "2.10788597588794e-15"),  # proj/README.md:110-116
])
def test_secant_iterates_bit_identical(hg, ref, n, k, golden):
    strip = ref.build_strip(n, 1, 1, k)
    want = ref.secant(strip, k)
    got = hg.smallest_eigenvalue(hg.HankelMatrixGPU(strip, k), 15)
    assert got["iterates"] == want["iterates"]
    assert got["eigenvalue"] == want["eigenvalue"]
    assert got["iterations"] == want["iterations"]
    if golden:
        assert got["eigenvalue"] == golden
    if n == 6:
        assert got["eigenvalue"].startswith("1.0451")


def test_secant_beta_7_4_against_reference(hg, ref):
    # BASELINE config 2's beta at N=40 (strip from the reference's own
    # certified Gamma, fed identically to both sides)
    n, k = 40, 1024
    strip = ref.build_strip(n, 7, 4, k)
    want = ref.secant(strip, k)
    got = hg.smallest_eigenvalue(hg.HankelMatrixGPU(strip, k), 15)
    assert got["iterates"] == want["iterates"]
    assert got["eigenvalue"] == want["eigenvalue"]


def _heig_run(path, n, beta, k=0, verify=False, workers=1):
    lib = ctypes.CDLL(path)
    lib.heig_config_new.restype = ctypes.c_void_p
    lib.heig_config_set_n.argtypes = [ctypes.c_void_p, ctypes.c_long]
    lib.heig_config_set_beta.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
    lib.heig_config_set_precision_bits.argtypes = [ctypes.c_void_p, ctypes.c_long]
    lib.heig_config_set_verify.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.heig_config_set_workers.argtypes = [ctypes.c_void_p, ctypes.c_long]
    lib.heig_run.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    lib.heig_result_to_json.argtypes = [ctypes.c_void_p]
    lib.heig_result_to_json.restype = ctypes.c_void_p
    lib.heig_string_free.argtypes = [ctypes.c_void_p]
    lib.heig_result_free.argtypes = [ctypes.c_void_p]
    lib.heig_config_free.argtypes = [ctypes.c_void_p]
    lib.heig_last_error.restype = ctypes.c_char_p
    cfg = lib.heig_config_new()
    for st in (lib.heig_config_set_n(cfg, n), lib.heig_config_set_beta(cfg, beta.encode()),
               lib.heig_config_set_precision_bits(cfg, k),
               lib.heig_config_set_verify(cfg, int(verify)),
               lib.heig_config_set_workers(cfg, workers)):
        if st != 0:
            lib.heig_config_free(cfg)
            return st, lib.heig_last_error().decode()
    res = ctypes.c_void_p()
    st = lib.heig_run(cfg, ctypes.byref(res))
    lib.heig_config_free(cfg)
    if st != 0:
        return st, lib.heig_last_error().decode()
    js = lib.heig_result_to_json(res)
    out = json.loads(ctypes.string_at(js).decode())
    lib.heig_string_free(js)
    lib.heig_result_free(res)
    return 0, out


@pytest.mark.parametrize("n,beta", [(4, "1/1"), (100, "1"), (40, "1/2"), (40, "7/4"), (30, "3/2")])
def test_heig_run_c_abi_matches_reference(hg, n, beta):
    ours = _heig_run(hg.LIB_PATH, n, beta)
    theirs = _heig_run(po.REF_SO, n, beta)
    assert ours[0] == 0 and theirs[0] == 0, (ours, theirs)
    for key in ("eigenvalue", "k_bits", "iterations", "n", "beta", "condition_lower_bound"):
        assert ours[1][key] == theirs[1][key], key
    assert set(ours[1]) == set(theirs[1])
    assert set(ours[1]["timing"]) == set(theirs[1]["timing"])


@pytest.mark.parametrize("n,beta", [(4, "1/1"), (100, "1"), (40, "1/2"), (40, "7/4")])
def test_heig_run_verify_matches_reference(hg, n, beta):
    """heig_run with verification (driver.cpp:140-175): the GPU interval LDL^T
    certifies the same value at the same Kv as the reference."""
    ours = _heig_run(hg.LIB_PATH, n, beta, verify=True)
    theirs = _heig_run(po.REF_SO, n, beta, verify=True)
    assert ours[0] == 0 and theirs[0] == 0, (ours, theirs)
    for key in ("eigenvalue", "k_bits", "kv_bits", "verified", "diagnosis"):
        assert ours[1].get(key) == theirs[1].get(key), key
    assert set(ours[1]) == set(theirs[1])
    assert ours[1]["verified"] is True


def test_heig_run_status_codes(hg):
    # decimal beta rejected with status 1 (tests/CMakeLists.txt:38-50 style)
    assert _heig_run(hg.LIB_PATH, 4, "0.5")[0] == 1
    # odd precision rejected
    assert _heig_run(hg.LIB_PATH, 4, "1", k=513)[0] == 1
    # precision cap: a cap below the auto precision -> status 2
    os.environ["HANKEL_EIG_PRECISION_CAP"] = "256"
    try:
        assert _heig_run(hg.LIB_PATH, 4, "1")[0] == 2
    finally:
        del os.environ["HANKEL_EIG_PRECISION_CAP"]


@pytest.mark.parametrize("n,b,k", [(64, (1, 1), 1024), (40, (7, 4), 2048), (30, (1, 2), 2048)])
def test_lambda_40_digits_certified_by_reference(hg, ref, n, b, k):
    """north_star: lambda_min agrees in >= 40 significant decimals.  The GPU
    secant runs to a 40-digit stopping rule; the reference's own interval
    LDL^T (ldlt.cpp:79-152 via verify's probe construction, decimal.cpp)
    at Kv = 2K certifies det(M - aI) > 0 > det(M - bI) for a = trunc40(l),
    b = bump(a), i.e. every one of the 40 digits."""
    strip = ref.build_strip(n, b[0], b[1], k)
    got = hg.smallest_eigenvalue(hg.HankelMatrixGPU(strip, k), 40)
    lam = got["eigenvalue"]
    assert len(lam.split("e")[0].replace(".", "")) == 40
    hi = ref.bump_last_digit(lam)
    assert ref.interval_sign_decimal(n, b[0], b[1], 2 * k, lam) == 1
    assert ref.interval_sign_decimal(n, b[0], b[1], 2 * k, hi) == -1
    # and the 15-digit prefix is the reference's own secant answer
    r15 = ref.secant(strip, k)["eigenvalue"]
    assert lam.split("e")[0][:16] == r15.split("e")[0][:16]
    assert lam.split("e")[1] == r15.split("e")[1]


def test_config2_secant_stalls_like_the_reference(hg, ref):
    """BASELINE config 2 at its own P=4096: det(M) underflows the fixed point,
    and the reference's secant stalls there (its driver escalates precision);
    ours reports the same failure instead of a wrong digit string."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config2_strip.json")))
    strip = [int(v, 16) for v in g["strip"]]
    with pytest.raises(hg.PrecisionExhausted):  # the reference's NoProgress
        hg.smallest_eigenvalue(hg.HankelMatrixGPU(strip, g["frac_bits"]), 15)
    with pytest.raises(RuntimeError, match="stalled"):
        ref.secant(strip, g["frac_bits"])
