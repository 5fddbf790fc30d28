"""CPU checks of the C-ABI boundary: the library builds for sm_100a, loads, and exports every
function include/ie_b200.h declares; the binding fails loudly without a GPU (no fallback)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ie_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ie_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2306_17537_b200 import build_lib
    path = build_lib.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ("ie_create", "ie_set_contrast", "ie_set_source", "ie_apply_operator", "ie_solve_subdomain",
                 "ie_solve_dd", "ie_receiver_fields"):
        assert name in d


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    import paper_2306_17537_b200 as pkg
    assert set(pkg.EXPORTED) == set(_declared())


def test_library_is_sm100a(lib):
    import subprocess
    from paper_2306_17537_b200 import build_lib
    out = subprocess.run(["cuobjdump", "--list-elf", build_lib.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2306_17537_b200 as ie
    ie.load_library()
    with pytest.raises(Exception):
        ie.ie_create((8, 8, 8), (0.1, 0.1, 0.1), (0, 0, 0), 1.0, 1e5)
