"""The C-ABI library loads without a GPU and exports every symbol include/spamm_b200.h declares."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "spamm_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spamm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1203_1692_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH), "build the library first (__graft_entry__.build())"
    handle = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(handle, n)]
    assert not missing, f"declared in the header but not exported: {missing}"
    # and the Python binding knows every one of them
    unbound = [n for n in names if n not in _lib.SIGNATURES]
    assert not unbound, f"declared in the header but not bound in _lib.SIGNATURES: {unbound}"


def test_version_and_level_offsets_without_a_gpu():
    from paper_1203_1692_b200 import _lib
    lib = _lib.lib()
    assert lib.spamm_abi_version() == 2
    for t in range(12):
        assert lib.spamm_level_offset_of(t) == _lib.level_offset(t)
        assert _lib.level_offset(t) % 4 == 0 or t == 0
    assert lib.spamm_error_string(1) == b"invalid argument"
    lay = _lib.ArenaLayout()
    assert lib.spamm_multiply_arena_layout(8, 8, 10000, 20000, ctypes.byref(lay)) == 0
    offs = [getattr(lay, f) for f, _ in _lib.ArenaLayout._fields_ if f not in ("plan_ws_bytes", "total", "chain")]
    assert offs == sorted(offs) and all(o % 256 == 0 for o in offs) and lay.total > offs[-1]
    # the chain flags follow the work units inside the tile_order region
    assert lay.chain == lay.tile_order + 4 * (20000 + _lib.UNIT_EXTRA) and lay.chain + 4 * 20000 <= lay.values and lay.plan_ws_bytes > 0


def test_missing_library_fails_loudly(monkeypatch):
    from paper_1203_1692_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libspamm_b200.so")
    with pytest.raises(RuntimeError, match="no CPU or PyTorch fallback"):
        _lib.lib()
