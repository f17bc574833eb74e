"""CPU: the C-ABI library loads and exports every symbol include/*.h
declares; host-side logic (ownership map, argument checks) without a GPU."""
import ctypes
import os
import re

import pytest

from paper_0902_0852_b200 import hgpu
import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header: str) -> set:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set()
    for m in re.finditer(r"\b([a-z_][a-z0-9_]*)\s*\(", text):
        name = m.group(1)
        if name.startswith(("hgpu_", "heig_")):
            names.add(name)
    return names


@pytest.mark.parametrize("header", ["hgpu.h", "hankel_eig.h"])
def test_library_exports_every_declared_symbol(header):
    lib = hgpu.load()
    decl = declared_functions(header)
    assert len(decl) > 10
    missing = [n for n in decl if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_lists_all_hgpu_symbols():
    assert declared_functions("hgpu.h") == set(hgpu.EXPORTS)


def test_drop_in_soname_alias():
    path = os.path.join(ROOT, "paper_0902_0852_b200", "libhankeleig.so.1")
    assert os.path.exists(path)
    lib = ctypes.CDLL(path)
    assert hasattr(lib, "heig_run") and hasattr(lib, "heig_result_to_json")


def test_block_owner_is_reference_assignment():
    ref = po.RefLib()
    for world in (1, 2, 3, 4, 8):
        owners = ref.column_owners(50, world)  # assignment.hpp:15-23 over blocks
        assert [hgpu.block_owner(b, world) for b in range(50)] == owners


def test_version_and_errors_without_device():
    lib = hgpu.load()
    assert b"sm_100a" in lib.hgpu_version()
    # no CPU fallback: without a device, creating a matrix fails loudly
    try:
        hgpu.HankelMatrixGPU([1 << 32], 32)
    except hgpu.HgpuError as e:
        assert e.status == 4  # HGPU_ERR_CUDA
    else:
        pytest.skip("a GPU is present")


def test_int_limb_roundtrip():
    for v in (0, 1, -1, 2 ** 32, -(2 ** 200 + 12345), 3 ** 500):
        s, limbs = hgpu.int_to_limbs(v)
        ptr = limbs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        assert hgpu.limbs_to_int(s, ptr) == v


MALFORMED = [
    ("s=0 hex=ff fracbits=32\ns=2 hex=1 fracbits=32\n", "matrix dump out of order at s=2"),
    ("s=0 hex=ff fracbits=32\ns=1 hex=1 fracbits=32\n", "matrix dump must hold 2n-1 anti-diagonals"),
    ("", "matrix dump must hold 2n-1 anti-diagonals"),
    ("s=0 mantissa=ff fracbits=32\n", "matrix dump line: s=0 mantissa=ff fracbits=32"),
    ("s=0 hex=xyz fracbits=32\n", "matrix dump line: s=0 hex=xyz fracbits=32"),
]


@pytest.mark.parametrize("text,message", MALFORMED)
def test_dump_loader_rejects_what_the_reference_rejects(tmp_path, text, message):
    """load_matrix_dump (hankel_matrix.cpp:65-87): MalformedInput cases, same
    messages, checked before any device work (so this runs without a GPU)."""
    path = tmp_path / "m.dump"
    path.write_text(text)
    with pytest.raises(hgpu.HgpuError) as e:
        hgpu.HankelMatrixGPU.from_dump(str(path))
    assert e.value.status == 1  # HGPU_ERR_INVALID_ARGUMENT
    assert message in str(e.value)


def test_dump_loader_missing_file(tmp_path):
    with pytest.raises(hgpu.HgpuError) as e:
        hgpu.HankelMatrixGPU.from_dump(str(tmp_path / "absent.dump"))
    assert e.value.status == 1 and "cannot open dump file" in str(e.value)
