"""CPU: moment generation in libhgpu.so (host/moments.cpp)
against the reference's build_matrix / build_interval_matrix
(hankel_matrix.cpp:13-50, gamma.cpp:101-230), bit for bit."""
import hashlib
import json
import os

import pytest

import pyoracle as po

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def hg():
    from paper_0902_0852_b200 import hgpu
    hgpu.load()
    return hgpu


@pytest.fixture(scope="module")
def ref():
    return po.RefLib()


@pytest.mark.parametrize("n,bn,bd,k", [
    (8, 7, 4, 256), (20, 3, 2, 512), (10, 1, 2, 384), (16, 1, 1, 512), (40, 7, 4, 1024),
    (30, 2, 3, 2048), (12, 5, 7, 300), (6, 3, 1, 128), (64, 1, 1, 1024), (25, 9, 4, 640),
])
def test_moments_match_reference(hg, ref, n, bn, bd, k):
    assert hg.build_moments(n, bn, bd, k) == ref.build_strip(n, bn, bd, k)
    assert hg.build_moments(n, bn, bd, k, interval=True) == ref.build_interval_strip(n, bn, bd, k)


def test_config2_moments_match_golden(hg):
    g = json.load(open(os.path.join(GOLDEN, "config2_strip.json")))
    assert hg.build_moments(g["n"], 7, 4, g["frac_bits"]) == [int(v, 16) for v in g["strip"]]


def test_moments_bad_arguments(hg):
    with pytest.raises(hg.HgpuError):
        hg.build_moments(0, 1, 1, 64)


def test_config5_moments_digest(hg):
    """BASELINE config 5 (N=2000, beta=3/2, P=32768): 3999 certified Gamma
    moments, digest of the reference's own build_matrix output."""
    d = json.load(open(os.path.join(GOLDEN, "moments_digests.json")))[0]
    num, den = map(int, d["beta"].split("/"))
    strip = hg.build_moments(d["n"], num, den, d["frac_bits"])
    h = hashlib.sha256()
    for v in strip:
        h.update(po.to_hex(v).encode() + b"\n")
    assert h.hexdigest() == d["strip_sha256"]
