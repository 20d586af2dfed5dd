"""The C-ABI library loads and exports every symbol include/lfb_volume.h
declares; argument validation paths (host-only, no kernel launch) return
the documented codes. No compute calls: these run without a GPU."""

from __future__ import annotations

import ctypes
import pathlib
import re

import pytest

from paper_1604_08501_b200 import _native
from paper_1604_08501_b200.diagnostics import ExecutionError

HEADER = pathlib.Path(__file__).resolve().parents[1] / "include" / "lfb_volume.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"LFB_API\s+[\w\s\*]*?\b(lfb_\w+)\s*\(", text)))


def test_header_declares_what_python_binds():
    assert declared_symbols() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_every_header_is_exported_by_its_library():
    """include/lfb_emitted.h -> liblfb_emitted.so (the emitted-kernel backend)."""
    from paper_1604_08501_b200 import emitted
    text = (HEADER.parent / "lfb_emitted.h").read_text()
    syms = sorted(set(re.findall(r"LFB_API\s+[\w\s\*]*?\b(lfb_\w+)\s*\(", text)))
    assert syms == sorted(emitted.EXPORTED_SYMBOLS)
    L = emitted.lib()
    for name in syms:
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_version_and_strings():
    L = _native.lib()
    assert L.lfb_version() >> 16 == 1
    assert _native.error_string(0) == "ok"
    assert "Nq" in _native.error_string(_native.LFB_ERR_BAD_NQ)
    assert L.lfb_variant_name(_native.VARIANT_BASIC) == b"basic"
    assert _native.variant_available("basic", 8, 8)
    assert not _native.variant_available("basic", 8, 17)
    assert not _native.variant_available(99, 8, 8)


@pytest.mark.parametrize("fn_name", ["lfb_volume_rhs_f64", "lfb_volume_rhs_f32"])
def test_validation_codes(fn_name):
    L = _native.lib()
    fn = getattr(L, fn_name)
    p = 4096  # fake, aligned, never dereferenced: validation rejects first
    assert fn(0, 1, 1e5, 287.0, 1.4, p, p, p, p, p, None) == _native.LFB_ERR_BAD_NQ
    assert fn(17, 1, 1e5, 287.0, 1.4, p, p, p, p, p, None) == _native.LFB_ERR_BAD_NQ
    assert fn(4, -1, 1e5, 287.0, 1.4, p, p, p, p, p, None) == _native.LFB_ERR_BAD_NE
    assert fn(4, 1, 1e5, 287.0, 0.9, p, p, p, p, p, None) == _native.LFB_ERR_BAD_CONSTANTS
    assert fn(4, 1, 1e5, 287.0, 1.4, None, p, p, p, p, None) == _native.LFB_ERR_NULL
    assert fn(4, 1, 1e5, 287.0, 1.4, p + 2, p, p, p, p, None) == _native.LFB_ERR_MISALIGNED
    # Ne == 0 is a no-op that never touches the pointers or the device
    assert fn(4, 0, 1e5, 287.0, 1.4, None, None, None, None, None, None) == 0


def test_bad_variant_code():
    L = _native.lib()
    p = 4096
    rc = L.lfb_volume_rhs_variant_f64(42, 4, 1, 1e5, 287.0, 1.4, p, p, p, p, p, None)
    assert rc == _native.LFB_ERR_BAD_VARIANT


def test_error_mapping_raises_reference_style_exceptions():
    with pytest.raises(ExecutionError, match="Nq"):
        _native.check(_native.LFB_ERR_BAD_NQ)
    with pytest.raises(ExecutionError):
        _native.variant_id("no-such-variant")


# LFB_VARIANT_AUTO per (dtype, Nq): the measured winners of the config-5 sweep
# (profiles/r02_sweep_*.jsonl, DESIGN.md §4 results table)
AUTO_F64 = {2: "tc", 3: "col", 4: "tc", 5: "col", 6: "tc", 7: "tc", 8: "tc", 9: "lo",
            10: "lo", 11: "lt", 12: "lt", 13: "lines"}
AUTO_F32 = {4: "tc", 5: "col", 6: "tc", 7: "tc", 8: "tc", 9: "lo", 10: "lo", 11: "lo",
            12: "lt", 13: "tc", 16: "tc"}


@pytest.mark.parametrize("nbytes,table", [(8, AUTO_F64), (4, AUTO_F32)])
def test_auto_resolution_table(nbytes, table):
    got = {nq: _native.resolve_variant(nbytes, nq) for nq in table}
    assert got == table
    for nq, v in table.items():
        assert _native.variant_available(v, nbytes, nq), (nbytes, nq, v)
