"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared_functions():
    names = []
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            names += re.findall(r"^[A-Za-z_][\w\s\*]*?\b(fg_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_1603_02526_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    declared = _declared_functions()
    assert len(declared) >= 15
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared) == set(_native.EXPORTS), set(declared) ^ set(_native.EXPORTS)


def test_abi_version_and_error_text():
    from paper_1603_02526_b200 import _native
    lib = _native.load()
    assert lib.fg_abi_version() == 1
    assert isinstance(lib.fg_last_error(), bytes)


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_1603_02526_b200 import _native
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return
    out = subprocess.run([tool, "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
