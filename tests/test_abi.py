"""The C-ABI library loads on a CPU-only host and exports every entry point
include/tfft.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "tfft.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(tfft_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2405_02520_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_2405_02520_b200 import _lib
    assert sorted(_lib.SIGNATURES) == _declared()


def test_version_and_error_string_without_gpu():
    from paper_2405_02520_b200 import _lib
    lib = _lib.load()
    assert lib.tfft_version() == 1
    assert isinstance(lib.tfft_last_error(), bytes)
    # argument validation happens before any device work
    h = ctypes.c_void_p()
    dims = (ctypes.c_int64 * 3)(3, 0, 0)
    rc = lib.tfft_plan_create(ctypes.byref(h), 3, 0, 1, dims, 1, 0)
    assert rc == _lib.TFFT_EINVAL


def test_built_for_sm100a():
    import subprocess
    from paper_2405_02520_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
