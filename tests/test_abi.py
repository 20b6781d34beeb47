"""The C-ABI library builds for sm_100a and exports every symbol include/b200rt.h declares.

CPU-only: no compute call is made (there is no GPU in the build container).
"""

import ctypes
import os
import re

from paper_2303_11103_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "b200rt.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(rt_\w+)\(", text, re.M)))


def test_header_declares_the_binding_list():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_builds_and_exports_every_symbol():
    path = _native.build_library()
    lib = ctypes.CDLL(path)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.rt_version() == 1


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.build_library()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out
