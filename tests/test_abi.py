"""The C-ABI library builds, loads without a GPU and exports every symbol of include/srht.h."""

import ctypes
import os
import re

import pytest

from tests.conftest import ROOT


@pytest.fixture(scope="module")
def libpath():
    from paper_0812_4547_b200 import build
    return build.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "srht.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(srht_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_boundary():
    names = header_functions()
    for required in ["srht_plan_create", "srht_sketch", "srht_plan_destroy", "srht_plan_create_batched",
                     "srht_sketch_columns", "srht_sketch_batched", "srht_workspace_bytes",
                     "srht_plan_copy_indices", "srht_plan_copy_signs", "srht_status_str"]:
        assert required in names


def test_every_symbol_exported(libpath):
    lib = ctypes.CDLL(libpath)
    for name in header_functions():
        assert hasattr(lib, name), name


def test_binding_declares_every_symbol(libpath):
    from paper_0812_4547_b200 import _lib
    declared = {n for n, _, _ in _lib.SIGNATURES}
    assert set(header_functions()) == declared


def test_status_strings_without_gpu(libpath):
    from paper_0812_4547_b200 import _lib
    lib = _lib.load()
    assert lib.srht_status_str(0) == b"SRHT_OK"
    assert b"invalid" in lib.srht_status_str(1)


def test_argument_validation_without_gpu(libpath):
    # Invalid arguments are rejected before touching the device.
    from paper_0812_4547_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.srht_plan_create(0, 1, 1, 0, ctypes.byref(h)) == _lib.SRHT_EINVAL
    assert lib.srht_plan_create(4, 1, 5, 0, ctypes.byref(h)) == _lib.SRHT_EINVAL
    assert lib.srht_plan_create_batched(4, 1, 1, 0, 0, ctypes.byref(h)) == _lib.SRHT_EINVAL
    assert lib.srht_plan_create(1 << 31, 1, 1, 0, ctypes.byref(h)) == _lib.SRHT_EUNSUPPORTED
    assert lib.srht_plan_destroy(None) == _lib.SRHT_OK
    assert lib.srht_workspace_bytes(None, 5) == 0


def test_no_cpu_fallback_in_product():
    # The product package must not import the oracle.
    pkg = os.path.join(ROOT, "paper_0812_4547_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_sass_is_sm100a(libpath):
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", libpath], capture_output=True, text=True).stdout
    assert "FADD2" in sass or "FFMA2" in sass  # packed FP32 butterflies


def test_new_entry_points_validate_without_gpu(libpath):
    # round-2 entry points reject bad arguments before any device work
    from paper_0812_4547_b200 import _lib
    lib = _lib.load()
    E = _lib.SRHT_EINVAL
    assert lib.srht_rows_finish(None, None, 1, 1, None, 1, None) == E
    assert lib.srht_gram_ex(0, 1, 1, None, 1, 1, None, 1, 1, None, 0, None) == E
    assert lib.srht_gram_ex(8, 4, 1, ctypes.c_void_p(256), 4, 32, ctypes.c_void_p(256), 4, 16, None, 0, None) == E
    assert lib.srht_nnls_gram_bpp(0, 1, None, 1, 1, None, 1, None, None, 0, None) == E
    assert lib.srht_nnls_gram_bpp(4, 1, ctypes.c_void_p(256), 5, 25, ctypes.c_void_p(256), 4, None, None, 0,
                                  None) == E  # no workspace
    assert lib.srht_nnls_gram_bpp(5000, 1, ctypes.c_void_p(256), 5001, 0, ctypes.c_void_p(256), 5000, None,
                                  ctypes.c_void_p(256), 1 << 30, None) == _lib.SRHT_EUNSUPPORTED
    assert lib.srht_nnls_bpp_workspace_bytes(512, 2) == 2 * 512 * 512 * 8
    assert lib.srht_gram_workspace_bytes(8192, 513, 1) > 0       # one problem: K-split partials
    assert lib.srht_gram_workspace_bytes(1024, 101, 3000) == 0   # many problems: no split
