"""The C-ABI library loads and exports every symbol include/swb.h declares
(no device needed: nothing is called)."""
import ctypes
import re
from pathlib import Path

from paper_1304_5966_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "swb.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(swb_[a-z_0-9]+)\(", text, re.M)))


def test_header_lists_entry_points():
    names = declared_functions()
    for must in ("swb_pass", "swb_crossings", "swb_leaves", "swb_ctx_create", "swb_seq_upload"):
        assert must in names


def test_library_exports_all_header_symbols():
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) == set(declared_functions())


def test_struct_layouts():
    # field sizes mirror the C structs (x86-64 SysV)
    assert ctypes.sizeof(_lib.Subproblem) == 48
    assert ctypes.sizeof(_lib.Crossing) == 40
    assert ctypes.sizeof(_lib.Scheme) == 4 * 68
    assert ctypes.sizeof(_lib.PassOut) == 8 * 9 + 4 * 2


def test_version_without_device():
    assert _lib.load().swb_version() == 1
