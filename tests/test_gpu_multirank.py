"""The column-block-cyclic multi-rank factorisation (ldlt_det_parallel,
ldlt.cpp:154-341) run for real through the engine: an in-process rank group
(hgpu_matrix_new_group) of 2-4 ranks placed on the one GPU a gpurun lease
has.  Every panel's owner publishes it with a CUDA event and the other ranks
read its integers from the owner's memory -- the same code path as one rank
per GPU, ordered by events and host waits only (no kernel waits on another).

Results must be bit-identical to one rank and to the reference, mirroring
tests/test_parallel.cpp:42-55 (determinants bit-identical across worker
counts), tests/acceptance.cpp:251-265 (N=200, K=1400 for 2, 4, 8 workers)
and test_parallel.cpp:90-97 (a zero pivot aborts every worker cleanly)."""
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


def secant_x1(strip0, k):
    mant = min(strip0, 1 << k) >> 16  # secant.cpp:7-16
    return -(mant if mant else 1)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_group_beta_7_4_bit_exact(hg, ref, world):
    # n = 150 > 4 panels of 32 columns, so every rank owns panels and
    # receives the others'; beta = 7/4 moments from the reference
    n, k = 150, 2048
    strip = ref.build_strip(n, 7, 4, k)
    x = secant_x1(strip[0], k)
    want = ref.ldlt_serial(strip, x, k, capture=True)
    m = hg.HankelMatrixGPU(strip, k, devices=[0] * world)
    assert m.world == world
    got = m.ldlt(x, capture=True, fold=True)
    assert got.pivots == want.pivots
    assert got.ratios == want.ratios
    assert got.det == want.det
    assert got.net_ms > 0  # the receivers waited for / pulled panels


def test_group_worker_counts_random_pd(hg, ref):
    # test_parallel.cpp:42-55 at an order that spans several panels
    strip = random_pd_hankel(73, 100, 256)
    x = 1 << 150
    serial = ref.ldlt_serial(strip, x, 256, capture=False).det
    for world in (1, 2, 3, 4, 5):
        m = hg.HankelMatrixGPU(strip, 256, devices=[0] * world)
        assert m.ldlt(x, fold=True).det == serial, f"world {world}"
        m.close()


def test_group_acceptance_n200(hg, ref):
    # acceptance.cpp:251-265: N=200, beta=1, K=1400, workers 2, 4, 8
    n, k = 200, 1400
    strip = po.exact_strip(n, 1, 1, k)
    serial = ref.ldlt_serial(strip, 0, k, capture=False).det
    for world in (2, 4, 8):
        m = hg.HankelMatrixGPU(strip, k, devices=[0] * world)
        r = m.ldlt(0, fold=True)
        assert r.det == serial, f"world {world}"
        m.close()


def test_group_zero_pivot(hg):
    # test_parallel.cpp:90-97: all-ones 3x3 is singular in column 1
    m = hg.HankelMatrixGPU([1 << 64] * 5, 64, devices=[0, 0, 0])
    with pytest.raises(hg.ZeroPivot) as ei:
        m.ldlt(0)
    assert ei.value.pivot_index == 1


def test_group_zero_pivot_in_a_receivers_panel(hg, orc=None):
    # a zero pivot in a panel owned by rank 1: exact integer moments of a
    # 40-node measure make M of order 70 exactly rank 40; the reference's
    # elimination hits its first zero pivot where the C restatement does
    n, k = 70, 64
    nodes = list(range(1, 41))
    strip = [sum(v ** s for v in nodes) << k for s in range(2 * n - 1)]
    want = None
    try:
        po.OracleLib().ldlt(strip, 0, k, capture=False)
    except po.ZeroPivotError as e:
        want = e.pivot_index
    for world in (1, 2, 3):
        m = hg.HankelMatrixGPU(strip, k, devices=[0] * world)
        if want is None:
            m.ldlt(0)
        else:
            with pytest.raises(hg.ZeroPivot) as ei:
                m.ldlt(0)
            assert ei.value.pivot_index == want, f"world {world}"
        m.close()


def test_group_repeated_and_shifted(hg, ref):
    # the same group handle factorises several shifts (event reuse across
    # runs, slot sets recycled within a run: 300 columns = 10 panels)
    n, k = 300, 1024
    strip = po.exact_strip(n, 1, 1, k)
    m = hg.HankelMatrixGPU(strip, k, devices=[0, 0])
    for x in (0, -(1 << (k - 16)), 0):
        got = m.ldlt(x, fold=True)
        want = po.OracleLib().ldlt(strip, x, k, capture=True)
        assert got.pivots == want.pivots
        assert got.det == want.det


def test_group_inverse_iteration(hg):
    # rank 0 keeps the whole L (reading the other ranks' ratio columns in
    # place) and runs the solves: same iterates as one rank
    n, k = 100, 832
    strip = po.exact_strip(n, 1, 1, k)
    u = hg.seeded_start_vector(n, k)
    one = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k), u, 0, 30, digits=15)
    two = hg.inverse_iteration(hg.HankelMatrixGPU(strip, k, devices=[0, 0, 0]), u, 0, 30,
                               digits=15)
    assert two["rho"] == one["rho"]
    assert two["eigenvalue"] == one["eigenvalue"]


def test_heig_run_workers_bit_identical(hg, monkeypatch):
    # heig_run with workers -> ranks (driver.cpp:102-114); on a one-GPU box
    # the rank devices come from HGPU_RANK_DEVICES.  Same iterates, same
    # digits, and the {net} bucket is filled (timing.hpp:7-39)
    from test_gpu_fold_secant import _heig_run
    one = _heig_run(hg.LIB_PATH, 100, "1")
    monkeypatch.setenv("HGPU_RANK_DEVICES", "0,0,0")
    three = _heig_run(hg.LIB_PATH, 100, "1", workers=3)
    theirs = _heig_run(po.REF_SO, 100, "1", workers=3)
    assert one[0] == three[0] == theirs[0] == 0, (one, three, theirs)
    for key in ("eigenvalue", "k_bits", "iterations", "condition_lower_bound"):
        assert three[1][key] == one[1][key] == theirs[1][key], key
    assert three[1]["eigenvalue"] == "2.10788597588794e-15"  # proj/README.md:112
    assert three[1]["workers"] == 3
    assert three[1]["timing"]["net_s"] > 0
    assert three[1]["timing"]["div_s"] == 0
