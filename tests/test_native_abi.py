"""The C-ABI library builds for sm_100a, loads, and exports every entry point
declared in include/dictamux_b200.h (no compute calls: CPU container)."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    hdr = (ROOT / "include" / "dictamux_b200.h").read_text()
    return sorted(set(re.findall(r"DM_API\s+[\w\s\*]+?\b(dm_\w+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol(native_lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(native_lib, s), s
    from paper_2507_01021_b200 import _native
    assert set(_native.EXPORTS) == set(syms)
    assert native_lib.dm_version() >= 1


def test_library_is_sm100a_with_tcgen05_and_tma(native_lib):
    lib = ROOT / "paper_2507_01021_b200" / "_lib" / "libdictamux_b200.so"
    out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(lib)], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out


def test_errors_surface_through_last_error(native_lib):
    import ctypes as C
    rc = native_lib.dm_logmel(None, None, None, 1, 81, None, None)
    assert rc == 1
    assert b"n_mels" in native_lib.dm_last_error()
