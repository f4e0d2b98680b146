"""The C ABI: libnskb.so loads on a CPU-only host and exports every function include/nskb.h declares."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nskb.h")
LIB = os.path.join(ROOT, "paper_2409_11600_b200", "libnskb.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(nsk_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ("nsk_gemm", "nsk_conv2d_fprop", "nsk_conv2d_dgrad", "nsk_conv2d_wgrad", "nsk_bn_fwd", "nsk_bn_bwd",
                 "nsk_xent_fwd", "nsk_sgd_multi", "nsk_adamw_multi", "nsk_arena_alloc", "nsk_allreduce",
                 "nsk_augment_crop_flip", "nsk_embedding_fwd"):
        assert must in names


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import sys

        sys.path.insert(0, ROOT)
        from paper_2409_11600_b200 import build

        build.build()
    return ctypes.CDLL(LIB)


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2409_11600_b200 import _lib

    missing = [n for n in declared_functions() if n not in _lib.SIGNATURES]
    assert not missing, missing


def test_abi_version_and_error_string(lib):
    lib.nsk_abi_version.restype = ctypes.c_int
    assert lib.nsk_abi_version() == 1
    lib.nsk_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.nsk_last_error(), bytes)


def test_sass_contains_tcgen05_and_tma():
    """The tensor-core kernels are tcgen05/TMA code for sm_100a (B200_PROFILING.md mnemonics)."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-sass", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UTCHMMA" in out or "UTCMMA" in out or re.search(r"UTC\w*MMA", out)
    assert "UTMALDG" in out
    assert "LDTM" in out
