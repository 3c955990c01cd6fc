"""The C-ABI library loads and exports every symbol include/ss_b200.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ss_b200.h")
LIB = os.path.join(ROOT, "paper_1411_4356_b200", "libss_b200.so")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "paper_1411_4356_b200", "csrc"), "-j8"])
    return ctypes.CDLL(LIB)


def test_header_declares_the_four_calls():
    names = declared()
    for n in ("ss_build", "ss_setup", "ss_solve", "ss_expect"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_signatures_cover_header():
    from paper_1411_4356_b200 import _lib
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared()) == bound


def test_no_device_call_fails_loudly(lib):
    """Without a CUDA device the library refuses to compute (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1411_4356_b200 import _lib
    from workloads import CONFIGS
    with pytest.raises(_lib.SSError) as e:
        _lib.ss_build(CONFIGS["tiny"])
    assert e.value.code == 2
