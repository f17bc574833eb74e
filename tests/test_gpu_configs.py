"""GPU parity at the BASELINE configs' own sizes.

Full-size runs are checked through size-independent properties that pin them
to the reference: the committed reference digest (config 2), the beta=1
closed form (config 3, in test_gpu_fold_secant.py), and leading-block
bit-exactness -- the submatrix-order LDL^T of the leading n' x n' block is a
prefix of the full one (ldlt.cpp:65-71 only touches indices < n' there), so
the first n' pivots and ratio rows of the full GPU run must equal the
oracle's factorisation of the leading block (configs 4 and 5)."""
import hashlib
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


def digest(values):
    h = hashlib.sha256()
    for v in values:
        h.update(po.to_hex(v).encode() + b"\n")
    return h.hexdigest()


def test_config2_full_size_matches_reference_digest(hg):
    # BASELINE config 2: N=300, beta=7/4, P=4096, strip from the reference
    g = json.load(open(os.path.join(GOLDEN, "config2_strip.json")))
    strip = [int(v, 16) for v in g["strip"]]
    m = hg.HankelMatrixGPU(strip, g["frac_bits"])
    r = m.ldlt(0, fold=True)
    assert po.to_hex(r.pivots[0]) == g["pivot_first"]
    assert po.to_hex(r.pivots[-1]) == g["pivot_last"]
    assert digest(r.pivots) == g["pivots_sha256"]
    assert digest([r.det]) == g["det_sha256"]


def test_lambda_fixture_iterates(hg):
    lam = json.load(open(os.path.join(GOLDEN, "lambda_secant.json")))
    for d in lam:
        if d["beta"] not in ("1/1", "1/2"):
            continue
        num, den = map(int, d["beta"].split("/"))
        strip = po.exact_strip(d["n"], num, den, d["frac_bits"])
        assert digest(strip) == d["strip_sha256"]
        got = hg.smallest_eigenvalue(hg.HankelMatrixGPU(strip, d["frac_bits"]), 15)
        assert got["eigenvalue"] == d["eigenvalue"]
        assert [[po.to_hex(x), po.to_hex(y)] for x, y in got["iterates"]] == d["iterates"]


def leading_block_check(hg, full_strip, k, nprime, x=0):
    n = (len(full_strip) + 1) // 2
    got = hg.HankelMatrixGPU(full_strip, k).ldlt(x, capture=True)
    block = full_strip[:2 * nprime - 1]
    want = po.OracleLib().ldlt(block, x, k, capture=True)
    assert got.pivots[:nprime] == want.pivots
    for (p, r), v in want.ratios.items():
        assert got.ratios[(p, r)] == v
    assert all(v > 0 for v in got.pivots)  # PD at x <= 0 (test_ldlt.cpp:171-183)
    return got


@pytest.mark.slow
def test_config4_full_size_leading_block():
    from paper_0902_0852_b200 import hgpu
    # BASELINE config 4: N=1500, beta=1/2, P=65536 (exact moments 2 (2s+1)!)
    n, k = 1500, 65536
    strip = po.exact_strip(n, 1, 2, k)
    m = hgpu.HankelMatrixGPU(strip, k)
    r = m.ldlt(0)
    want = po.OracleLib().ldlt(strip[:2 * 40 - 1], 0, k, capture=True)
    assert r.pivots[:40] == want.pivots
    assert all(v > 0 for v in r.pivots)


def test_config5_leading_block_precision(hg):
    # BASELINE config 5's beta=3/2 and P=32768 on an n'=48 matrix, strip from
    # the reference's certified Gamma (built here, fed to both sides)
    ref = po.RefLib()
    strip = ref.build_strip(48, 3, 2, 32768)
    leading_block_check(hg, strip, 32768, 24)
