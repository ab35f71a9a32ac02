"""SPAMMQT1 tree files: header and record validation (no GPU needed: every check fires before any
device work), mirroring the error cases of the reference's `tests/test_io.py`."""

import struct

import numpy as np
import pytest


def _file(tmp_path, m, n, nb, depth, records, name="t.qt", magic=b"SPAMMQT1", count=None):
    raw = magic + struct.pack("<5Q", m, n, nb, depth, len(records) if count is None else count)
    for key, vals in records:
        raw += struct.pack("<Q", key) + np.asarray(vals, "<f4").tobytes()
    p = tmp_path / name
    p.write_bytes(raw)
    return p


def test_rejects_malformed_files(tmp_path):
    from paper_1203_1692_b200.io import MatrixFormatError, load_quadtree
    one = np.ones((16, 16), np.float32)
    cases = {
        "truncated header": (tmp_path / "a.qt", b"SPAMMQT1" + b"\0" * 10),
        "bad magic": (tmp_path / "b.qt", b"SPAMMQT2" + struct.pack("<5Q", 16, 16, 16, 0, 0)),
    }
    for what, (p, raw) in cases.items():
        p.write_bytes(raw)
        with pytest.raises(MatrixFormatError, match=what):
            load_quadtree(p)
    with pytest.raises(MatrixFormatError, match="depth"):
        load_quadtree(_file(tmp_path, 40, 40, 16, 1, []))                       # 40 x 40 needs depth 2
    with pytest.raises(MatrixFormatError, match="bad header"):
        load_quadtree(_file(tmp_path, 0, 40, 16, 2, []))
    with pytest.raises(MatrixFormatError, match="expected 2 leaf records"):
        load_quadtree(_file(tmp_path, 32, 32, 16, 1, [(0, one)], count=2))
    with pytest.raises(MatrixFormatError, match="not strictly ascending at record 1"):
        load_quadtree(_file(tmp_path, 32, 32, 16, 1, [(2, one), (2, one)]))
    with pytest.raises(MatrixFormatError, match="out of range"):
        load_quadtree(_file(tmp_path, 32, 32, 16, 1, [(0, one), (4, one)]))
    bad = one.copy()
    bad[3, 3] = np.inf
    with pytest.raises(MatrixFormatError, match="non-finite values in leaf 1"):
        load_quadtree(_file(tmp_path, 32, 32, 16, 1, [(0, one), (1, bad)]))
    with pytest.raises(OSError):
        load_quadtree(tmp_path / "missing.qt")


def test_drop_tolerance_pins():
    # tests/test_core.py:49-61 of the reference
    from paper_1203_1692_b200 import drop_tolerance
    assert drop_tolerance(1e-8, 100.0, 10.0) == 1e-10
    assert drop_tolerance(1e-6, 2.0, 2.0) == 5e-7
    assert drop_tolerance(0.0, 1.0, 1.0) == 0.0
    for args in ((-1e-9, 1.0, 1.0), (1e-9, -1.0, 1.0), (1e-9, 0.0, 0.0)):
        with pytest.raises(ValueError):
            drop_tolerance(*args)
