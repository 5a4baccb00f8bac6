"""CPU-side checks of the C-ABI boundary: the library is built for sm_100a,
loads, and exports every entry point include/ftb2.h declares (no compute)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ftb2.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ftb_\w+)\s*\(", src, re.M)))


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
        _capi.call("ftb_attention_impl", 0, None, 0, None, 0, None, 0, None, 0, 1, 1, 1, 64, 1.0, None)
