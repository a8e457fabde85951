"""CPU-side checks of the C ABI: libhs.so loads (no GPU needed to dlopen) and
exports exactly the functions include/hs.h declares."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared() -> set[str]:
    names = set()
    for hdr in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", hdr.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_entry_points():
    names = _declared()
    assert "hs_op_gemm_bf16" in names and "hs_op_decode_attention" in names
    assert len(names) >= 15


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2603_12831_b200 import _lib

    if not _lib.lib_path().exists():
        pytest.fail("libhs.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_lib.lib_path()))
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, f"declared in include/*.h but not exported: {missing}"
    # the ctypes binding covers every declared symbol too
    bound = set(_lib.exported_symbols())
    assert _declared() <= bound, sorted(_declared() - bound)


def test_version_string_without_gpu():
    from paper_2603_12831_b200 import _lib

    lib = _lib.load()
    assert b"sm_100a" in lib.hs_version()
