"""CPU checks of the boundary: librtucker builds for sm_100a, loads, and exports every
function include/rtucker.h declares (no compute calls without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "rtucker.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:rt_status|const char\*)\s+(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_five_entry_points():
    names = _declared()
    for n in ["rtucker_sketch", "rtucker_qr", "rtucker_core", "rtucker_hosvd", "rtucker_sthosvd"]:
        assert n in names


def test_library_builds_loads_and_exports_all_symbols():
    from paper_2001_07124_b200 import build
    build.build()
    from paper_2001_07124_b200 import _lib
    for n in _declared():
        assert hasattr(_lib.lib, n), n
    assert sorted(_lib.EXPORTS) == _declared()


def test_sass_contains_no_cpu_fallback_and_is_sm100a():
    import subprocess
    from paper_2001_07124_b200 import build
    lib = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
