"""libtsb.so loads and exports every symbol include/tsb.h declares (no GPU calls)."""

import re
from pathlib import Path

from paper_2306_05893_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "tsb.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(tsb_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_bound_symbols():
    assert declared_symbols() == sorted(_lib.exported_symbols())


def test_library_loads_and_exports_all_symbols():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tsb_abi_version() == 3


def test_error_message_roundtrip():
    lib = _lib.load()
    assert lib.tsb_ldlt_create(None, None) == _lib.TSB_E_ARG
    assert "null" in _lib.last_error()


def test_struct_layouts_match_the_header():
    from paper_2306_05893_b200 import _ldlt_pack

    lib = _lib.load()
    assert lib.tsb_struct_size(0) == _lib.C.sizeof(_lib.AsmPlan)
    assert lib.tsb_struct_size(1) == _lib.C.sizeof(_lib.AsmCoeffs)
    assert lib.tsb_struct_size(2) == _ldlt_pack.BLOCK_DTYPE.itemsize
    assert lib.tsb_struct_size(3) == _lib.C.sizeof(_lib.LdltDesc)
    assert lib.tsb_struct_size(4) == _lib.C.sizeof(_lib.Report)
    assert lib.tsb_struct_size(5) == _ldlt_pack.TILE_DTYPE.itemsize
    from paper_2306_05893_b200 import refactor

    assert lib.tsb_struct_size(6) == refactor.FRONT_DTYPE.itemsize
    assert lib.tsb_struct_size(7) == refactor.PAIR_DTYPE.itemsize
    assert lib.tsb_struct_size(8) == _lib.C.sizeof(_lib.RefactorDesc)
    assert lib.tsb_struct_size(9) == _lib.C.sizeof(_lib.PatternDesc)
