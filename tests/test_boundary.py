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
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    # no CPU fallback: creating a device matrix fails loudly
    with pytest.raises(hgpu.HgpuError) as e:
        hgpu.HankelMatrixGPU([1 << 32], 32)
    assert e.value.status == 4


def test_int_limb_roundtrip():
    for v in (0, 1, -1, 2 ** 32, -(2 ** 200 + 12345), 3 ** 500):
        s, limbs = hgpu.int_to_limbs(v)
        ptr = limbs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        assert hgpu.limbs_to_int(s, ptr) == v
