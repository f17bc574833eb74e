"""GPU parity of the scheduling variants and opt-in arithmetic paths.

The factorisation's results may not depend on how the panel work is spread
over streams (near/far rows, far lanes, deferred trailing update, SM split)
nor on how the stage's ratios are formed (k_divide or the int8 tensor-core
ratio GEMM), how the trailing update multiplies (IMAD or the tcgen05 int8
update, HGPU_UPDATE_TC) or which reciprocal body runs: every variant must equal the reference's ldlt_det_serial
(ldlt.cpp:31-77) bit for bit.  The knobs are environment variables read when
a matrix is created (engine.cpp).  N is chosen so that the matrix has far
rows (N > 64) and several panels (kb = 32).
"""
import os

import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu

VARIANTS = [
    {},
    {"HGPU_FAR_LANES": "1", "HGPU_DEFER": "0", "HGPU_FUSED_PIVOT": "0"},
    {"HGPU_FAR_LANES": "3", "HGPU_DEFER": "6", "HGPU_NEAR": "40"},
    {"HGPU_RATIO_GEMM": "3"},
    {"HGPU_RATIO_GEMM": "1", "HGPU_FAR_LANES": "1"},
    {"HGPU_SM_SPLIT": "8:b"},
    {"HGPU_UPD_SMS": "96", "HGPU_GRID": "3"},
    {"HGPU_FAR_SUB": "0"},
    {"HGPU_FAR_SUB": "5", "HGPU_FAR_LANES": "3"},
    {"HGPU_FAR_SUB": "16", "HGPU_NEAR": "100"},
    {"HGPU_EDF": "1"},
    {"HGPU_EDF": "3", "HGPU_FAR_LANES": "1"},
    {"HGPU_NEXT_ROW": "1"},
    {"HGPU_NEXT_ROW": "1", "HGPU_PRE_ENTRY": "0", "HGPU_FAR_SUB": "0"},
    {"HGPU_NEXT_ROW": "1", "HGPU_NEAR": "100", "HGPU_EDF": "0"},
    {"HGPU_UPDATE_TC": "1"},
    {"HGPU_UPDATE_TC": "1", "HGPU_EDF": "0", "HGPU_FAR_SUB": "0"},
    {"HGPU_RECIP_FAST": "0"},
    {"HGPU_COL_EXTRACT": "3"},
    {"HGPU_PIVOT_THREADS": "256", "HGPU_COL_EXTRACT": "1"},
    {"HGPU_SM_SPLIT": "4:b", "HGPU_COL_EXTRACT": "1"},
    {"HGPU_LOOKAHEAD": "0"},
    {"HGPU_LOOKAHEAD": "1", "HGPU_FAR_SUB": "4", "HGPU_FAR_LANES": "3"},
    {"HGPU_LOOKAHEAD": "1", "HGPU_NEAR": "64"},
    {"HGPU_RECIP_FAST": "1"},
    {"HGPU_PRE_NEAR": "1"},
    {"HGPU_PRE_NEAR": "1", "HGPU_FAR_LANES": "2", "HGPU_GRID": "2", "HGPU_FAR_PRIO": "1"},
    {"HGPU_PRE_NEAR": "1", "HGPU_NEAR": "100", "HGPU_EDF_RUN": "2"},
    {"HGPU_EDF_RUN": "3", "HGPU_FAR_PRIO": "2"},
    {"HGPU_COL_TR": "16", "HGPU_FAR_SUB": "8"},
    {"HGPU_COL_TR": "8", "HGPU_ROW_THREADS": "128"},
    {"HGPU_COL_TR": "2", "HGPU_COL_THREADS": "64"},
    {"HGPU_KB": "16"},
    {"HGPU_SLOT_SETS": "3"},
    {"HGPU_SLOT_SETS": "4", "HGPU_FLUSH_AHEAD": "0", "HGPU_FLUSH_BATCH": "1"},
    {"HGPU_SLOT_SETS": "4", "HGPU_FLUSH_AHEAD": "3", "HGPU_FLUSH_BATCH": "8"},
    {"HGPU_KB": "64", "HGPU_FAR_SUB": "16"},
    {"HGPU_LAG_FAR": "1"},
    {"HGPU_LAG_FAR": "1", "HGPU_FAR_LANES": "4", "HGPU_PRE_NEAR": "1"},
    {"HGPU_LAG_FAR": "1", "HGPU_FAR_LANES": "2", "HGPU_NEAR": "40", "HGPU_FAR_SUB": "0"},
]


@pytest.fixture(scope="module")
def hg():
    from paper_0902_0852_b200 import hgpu
    hgpu.load()
    return hgpu


@pytest.fixture(scope="module")
def case():
    # config-2 shape at reduced size: beta = 7/4, certified-rounded moments
    n, k = 150, 1024
    strip = po.RefLib().build_strip(n, 7, 4, k)
    x = -(1 << (k - 16))
    want = po.OracleLib().ldlt(strip, x, k, capture=True)
    return n, k, strip, x, want


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_variant_bit_exact(hg, case, env, monkeypatch):
    n, k, strip, x, want = case
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    m = hg.HankelMatrixGPU(strip, k)
    got = m.ldlt(x, capture=True)
    assert got.pivots == want.pivots
    bad = [key for key in want.ratios if got.ratios[key] != want.ratios[key]]
    assert not bad, f"{len(bad)} ratios differ under {env}, first {bad[:3]}"
