"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/gapsafe_b200.h declares, fails loudly without a GPU, and
the product never reaches into the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gapsafe_b200.h")
PKG = os.path.join(ROOT, "paper_1505_03410_b200")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("gs_tdot", "gs_cd_pass", "gs_screen_sphere", "gs_solver_solve",
                 "gs_solver_seq_screen", "gs_matrix_dense", "gs_matrix_csc", "gs_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1505_03410_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH), "build the extension: __graft_entry__.build()"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding table covers exactly the header
    assert sorted(_lib.SIGNATURES) == _declared()


def test_library_is_sm100a():
    """The cubin inside the .so targets sm_100a (cuobjdump, if available)."""
    import shutil
    import subprocess
    from paper_1505_03410_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _has_gpu():
    from paper_1505_03410_b200 import _lib
    c = ctypes.c_int()
    _lib.load().gs_device_count(ctypes.byref(c))
    return c.value > 0


def test_fails_loudly_without_gpu():
    if _has_gpu():
        pytest.skip("a GPU is present")
    import paper_1505_03410_b200 as gs
    from paper_1505_03410_b200 import _lib
    assert _lib.load().gs_init(0) == _lib.GS_ERR_NODEVICE
    with pytest.raises(_lib.GapSafeDeviceError, match="no CPU fallback"):
        gs.DesignMatrix(np.eye(3))


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "liboracle" not in src, f
