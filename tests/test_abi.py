"""The C-ABI library loads and exports every symbol include/swb.h declares
(no device needed: nothing is called)."""
import ctypes
import re
from pathlib import Path

from paper_1304_5966_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "swb.h"


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


STRUCTS = {"Subproblem": "swb_subproblem", "Crossing": "swb_crossing", "Scheme": "swb_scheme",
           "PassOut": "swb_pass_out", "PassDesc": "swb_pass_desc", "IntPeak": "swb_int_peak"}


def test_struct_layouts(tmp_path):
    """ctypes mirrors of include/swb.h: size and every field offset equal what
    the C compiler lays out (compiled here with gcc against the header)."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc") or "/usr/bin/gcc"
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "swb.h"', "int main(void) {"]
    for py, c in STRUCTS.items():
        st = getattr(_lib, py)
        lines.append(f'printf("{py} %zu\\n", sizeof({c}));')
        for name, _ in st._fields_:
            lines.append(f'printf("{py}.{name} %zu\\n", offsetof({c}, {name}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([gcc, "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for py in STRUCTS:
        st = getattr(_lib, py)
        assert int(got[py]) == ctypes.sizeof(st), py
        for name, _ in st._fields_:
            assert int(got[f"{py}.{name}"]) == getattr(st, name).offset, (py, name)


def test_version_without_device():
    assert _lib.load().swb_version() == 1
