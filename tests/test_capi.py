"""CPU-side checks of the C-ABI boundary: the library is built for sm_100a,
loads, exports every entry point include/ftb2.h declares, and the ctypes struct mirrors
match the header's layouts (no compute)."""

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ftb2.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(ftb_\w+)\s*\(", src, re.M)))


def test_library_exports_header():
    from paper_2512_23379_b200 import _capi
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(_capi.lib, n), n
        assert n in _capi.EXPORTS, n
    # and the other way: every entry point the host binds is declared in the public header
    assert set(_capi.EXPORTS) <= set(names), sorted(set(_capi.EXPORTS) - set(names))
    assert _capi.lib.ftb_version() == 1


def test_library_is_sm100a_with_tcgen05():
    from paper_2512_23379_b200 import _capi
    out = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _capi.LIB_PATH], capture_output=True,
                                       text=True).stdout or "sm_100a" in out
    assert "UTCHMMA" in out      # tcgen05.mma
    assert "UTMALDG" in out      # TMA tensor loads
    assert "LDTM" in out         # tcgen05.ld


def test_error_mapping_without_gpu():
    from paper_2512_23379_b200 import _capi
    from paper_2512_23379_b200.errors import ConfigError
    # argument validation happens before any device work
    with pytest.raises(ConfigError):
        _capi.call("ftb_attention_impl", 0, None, 0, None, 0, None, 0, None, 0, 1, 1, 1, 64, 1.0, None, 0, None)


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors in _capi.py (Rope3D, Epilogue, ConvNorm) have the field offsets and
    sizes the C compiler gives the structs of include/ftb2.h (a probe compiled with gcc)."""
    import shutil

    from paper_2512_23379_b200 import _capi as A
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    mirrors = {"ftb_rope3d": A.Rope3D, "ftb_epilogue": A.Epilogue, "ftb_conv_norm": A.ConvNorm}
    lines = ['#include <stdio.h>', '#include "ftb2.h"', "int main(void) {"]
    for cname, py in mirrors.items():
        lines.append('printf("%s sizeof %%zu\\n", sizeof(%s));' % (cname, cname))
        for f, _ in py._fields_:
            lines.append('printf("%s %s %%zu\\n", offsetof(%s, %s));' % (cname, f, cname, f))
    lines += ["return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n"):
        if line:
            cname, f, v = line.split()
            got[(cname, f)] = int(v)
    for cname, py in mirrors.items():
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
