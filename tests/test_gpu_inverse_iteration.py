"""GPU inverse iteration (north-star lambda_min step).

The reference has no inverse iteration, so the restatement
oracle/pyoracle.py:inverse_iteration_py defines it; the GPU path must
reproduce every Rayleigh quotient bit for bit, and the eigenvalue it returns
is pinned independently by the reference's own secant (15 digits) and its
interval LDL^T sign test (40 digits, verify.cpp:8-42)."""
import json
import os

import pytest

from helpers import random_pd_hankel
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


def negatives(strip, x, k):
    return sum(1 for p in po.OracleLib().ldlt(strip, x, k, capture=True).pivots if p < 0)


@pytest.mark.parametrize("seed,n,k", [(111, 6, 256), (112, 12, 384), (113, 20, 512), (114, 33, 640)])
def test_rho_iterates_bit_exact_random_pd(hg, seed, n, k):
    strip = random_pd_hankel(seed, n, k)
    u = hg.seeded_start_vector(n, k)
    want = po.inverse_iteration_py(strip, k, u, 0, 40)
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 40)
    assert got["rho"] == want
    assert got["iterations"] == len(want)
    # Sylvester inertia: rho is the SMALLEST eigenvalue
    rho = want[-1]
    assert negatives(strip, rho - (rho >> 40), k) == 0
    assert negatives(strip, rho + (rho >> 40), k) == 1


def test_nonzero_start_shift(hg):
    # phase 1 from a negative shift (the secant's x1 = -2^-16 M00 style)
    strip = random_pd_hankel(115, 16, 512)
    k = 512
    sigma = -(strip[0] >> 16)
    u = hg.seeded_start_vector(16, k, seed=3)
    want = po.inverse_iteration_py(strip, k, u, sigma, 40)
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, sigma, 40)
    assert got["rho"] == want


def test_config1_inverse_iteration(hg, ref):
    # BASELINE config 1 (N=64, beta=1, P=1024) from the seed-0 start vector
    n, k = 64, 1024
    strip = po.exact_strip(n, 1, 1, k)
    u = hg.seeded_start_vector(n, k)
    want = po.inverse_iteration_py(strip, k, u, 0, 40,
                                   factor=lambda s, x, kk: ref.ldlt_serial(s, x, kk, True))
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 40, digits=40)
    assert got["rho"] == want
    lam = got["eigenvalue"]
    fx = {(d["n"], d["beta"]): d for d in json.load(open(os.path.join(GOLDEN, "lambda_secant.json")))}
    sec = fx[(64, "1/1")]["eigenvalue"]  # the reference's secant, 15 digits
    assert lam.split("e")[1] == sec.split("e")[1] and lam[:16] == sec[:16]
    # every one of the 40 digits certified by the reference's interval LDL^T
    assert ref.interval_sign_decimal(n, 1, 1, 2 * k, lam) == 1
    assert ref.interval_sign_decimal(n, 1, 1, 2 * k, ref.bump_last_digit(lam)) == -1


@pytest.mark.parametrize("n,k", [(100, 832), (30, 2048)])
def test_fixture_matrices(hg, ref, n, k):
    d = {(e["n"], e["frac_bits"]): e for e in json.load(open(os.path.join(GOLDEN, "lambda_secant.json")))}[(n, k)]
    num, den = map(int, d["beta"].split("/"))
    strip = po.exact_strip(n, num, den, k)
    u = hg.seeded_start_vector(n, k)
    want = po.inverse_iteration_py(strip, k, u, 0, 40,
                                   factor=lambda s, x, kk: ref.ldlt_serial(s, x, kk, True))
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 40, digits=15)
    assert got["rho"] == want
    assert got["eigenvalue"].split("e")[1] == d["eigenvalue"].split("e")[1]
    assert got["eigenvalue"][:15] == d["eigenvalue"][:15]


def test_config3_time_to_lambda(hg):
    # BASELINE config 3 (N=1000, beta=1, P=24576): agrees with the GPU secant
    # (whose iterates are bit-identical to the reference's, test_gpu_fold_secant)
    n, k = 1000, 24576
    m = hg.HankelMatrixGPU(po.exact_strip(n, 1, 1, k), k)
    got = hg.inverse_iteration(m, hg.seeded_start_vector(n, k), 0, 40, digits=40)
    print("config3 inverse iteration", got["iterations"], "steps", round(got["seconds"], 2), "s",
          got["eigenvalue"])
    assert got["eigenvalue"].startswith("1.0892427421041")
    assert got["eigenvalue"].endswith("e-52")


def test_config2_full_size_certified_digits(hg):
    """BASELINE config 2 (N=300, beta=7/4, P=4096) at its own precision, where
    the secant stalls (test_gpu_fold_secant): the GPU inverse iteration ends on
    the restatement's final Rayleigh quotient bit for bit, and its 40 digits
    are the ones the reference's interval LDL^T certified at 12288 bits
    (tests/golden/make_lambda_certified.py)."""
    fx = {d["name"]: d for d in json.load(open(os.path.join(GOLDEN, "lambda_certified.json")))}
    for name in ("config1", "config2"):
        d = fx[name]
        n, k = d["n"], d["frac_bits"]
        if name == "config1":
            strip = po.exact_strip(n, 1, 1, k)
        else:
            g = json.load(open(os.path.join(GOLDEN, "config2_strip.json")))
            strip = [int(v, 16) for v in g["strip"]]
        got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), hg.seeded_start_vector(n, k), 0, 40,
                                   digits=40)
        assert po.to_hex(got["rho"][-1]) == d["rho_last"]
        assert got["iterations"] == d["iterations"]
        assert got["eigenvalue"] == d["lambda_40"]


@pytest.mark.parametrize("seed,n,k", [(115, 40, 768), (116, 70, 1024)])
def test_tensor_core_solve_bit_exact(hg, seed, n, k, monkeypatch):
    """The opt-in int8 tensor-core AXPY of the triangular solves
    (HGPU_SOLVE_TC=1, solve_kernels.cu) gives the restatement's Rayleigh
    quotients bit for bit; the solves after the first one take that path."""
    monkeypatch.setenv("HGPU_SOLVE_TC", "1")
    monkeypatch.setenv("HGPU_SOLVE_NTT", "0")
    strip = random_pd_hankel(seed, n, k)
    u = hg.seeded_start_vector(n, k)
    want = po.inverse_iteration_py(strip, k, u, 0, 40)
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 40)
    assert got["rho"] == want
    assert got["iterations"] == len(want)


@pytest.mark.parametrize("seed,n,k", [(117, 40, 768), (118, 70, 1024), (119, 130, 2048)])
def test_transform_domain_solve_bit_exact(hg, seed, n, k, monkeypatch):
    """The transform-domain AXPY of the triangular solves (HGPU_SOLVE_NTT=1,
    k_solve_ntt): every accumulator is the same exact integer, so the
    Rayleigh quotients equal the restatement's bit for bit."""
    monkeypatch.setenv("HGPU_SOLVE_NTT", "2")
    strip = random_pd_hankel(seed, n, k)
    u = hg.seeded_start_vector(n, k)
    want = po.inverse_iteration_py(strip, k, u, 0, 40)
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 40)
    assert got["rho"] == want
    assert got["iterations"] == len(want)


@pytest.mark.parametrize("pre", ["0", "1"])
def test_l_entry_transforms_during_or_after_the_factorisation(hg, pre, monkeypatch):
    """HGPU_PRE_LHAT: from the second factorisation of a run on, the L-entry
    transforms are formed panel by panel during the factorisation (1) or all
    at once by the first solve after it (0): the same Rayleigh quotients."""
    monkeypatch.setenv("HGPU_SOLVE_NTT", "2")
    monkeypatch.setenv("HGPU_PRE_LHAT", pre)
    seed, n, k = 121, 90, 1536
    strip = random_pd_hankel(seed, n, k)
    u = hg.seeded_start_vector(n, k)
    want = po.inverse_iteration_py(strip, k, u, 0, 40)
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 40)
    assert got["rho"] == want
    assert got["iterations"] == len(want)


def test_transform_domain_solve_config2(hg, monkeypatch):
    """Config 2 at full size through the transform-domain solve: the final
    Rayleigh quotient and the certified 40 digits of the golden fixture."""
    monkeypatch.setenv("HGPU_SOLVE_NTT", "2")
    d = {e["name"]: e for e in json.load(open(os.path.join(GOLDEN, "lambda_certified.json")))}["config2"]
    g = json.load(open(os.path.join(GOLDEN, "config2_strip.json")))
    strip = [int(v, 16) for v in g["strip"]]
    n, k = d["n"], d["frac_bits"]
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), hg.seeded_start_vector(n, k), 0, 40,
                               digits=40)
    assert po.to_hex(got["rho"][-1]) == d["rho_last"]
    assert got["iterations"] == d["iterations"]
    assert got["eigenvalue"] == d["lambda_40"]


@pytest.mark.parametrize("seed,n,k", [(120, 40, 768), (121, 90, 1536)])
def test_integer_solve_bit_exact(hg, seed, n, k, monkeypatch):
    """The schoolbook AXPY (HGPU_SOLVE_NTT=0, k_solve_axpy), kept as the
    fallback of the transform-domain solve, gives the same quotients."""
    monkeypatch.setenv("HGPU_SOLVE_NTT", "0")
    strip = random_pd_hankel(seed, n, k)
    u = hg.seeded_start_vector(n, k)
    want = po.inverse_iteration_py(strip, k, u, 0, 40)
    got = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 40)
    assert got["rho"] == want
