"""Binary tree files (`SPAMMQT1`) straight to and from the packed device store.

Same file layout as the reference's `save_quadtree` / `load_quadtree`
(`pkg/src/spamm/io.py:99-149`, pinned by `tests/test_io.py:136-154`): the 8-byte magic, five
little-endian u64 words (m, n, n_b, depth, leaf count), then one record per stored leaf in ascending
key order: the u64 Morton key and the 16 x 16 float32 values row-major.  Norms are not stored; on
load they are recomputed on the device in `compute_norms` order, so a saved and reloaded tree is
bit-identical to the original.  The leaf records are the packed leaf arrays of the device tree, so
a file is read with one vectorised pass and one host-to-device copy (no per-leaf objects).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .tree import QuadtreeMatrix, tree_depth

QUADTREE_MAGIC = b"SPAMMQT1"
_HEADER = np.dtype("<u8")
_RECORD = np.dtype([("key", "<u8"), ("values", "<f4", (256,))])     # 8 + 1024 bytes, no padding


class MatrixFormatError(Exception):
    """A tree file exists but its contents are not usable."""


def save_quadtree(path, tree: QuadtreeMatrix) -> None:
    """Write the leaf dump of `tree` (one device-to-host copy of its packed leaves)."""
    keys, values, _ = tree.packed_leaves()
    rec = np.empty(keys.shape[0], _RECORD)
    rec["key"] = keys
    rec["values"] = values.reshape(-1, 256)
    with open(path, "wb") as fh:
        fh.write(QUADTREE_MAGIC)
        fh.write(np.array([tree.m, tree.n, tree.n_b, tree.depth, keys.shape[0]], _HEADER).tobytes())
        fh.write(rec.tobytes())


def load_quadtree(path, device=None) -> QuadtreeMatrix:
    """Read a leaf dump into a device tree, rebuilding every norm."""
    with open(path, "rb") as fh:
        raw = fh.read()
    head = len(QUADTREE_MAGIC) + 5 * _HEADER.itemsize
    if len(raw) < head:
        raise MatrixFormatError(f"{path}: truncated header")
    if raw[: len(QUADTREE_MAGIC)] != QUADTREE_MAGIC:
        raise MatrixFormatError(f"{path}: bad magic {raw[:8]!r}")
    m, n, n_b, depth, count = (int(x) for x in np.frombuffer(raw, _HEADER, 5, len(QUADTREE_MAGIC)))
    try:
        tree = QuadtreeMatrix(m, n, n_b, device=device)
    except ValueError as exc:
        raise MatrixFormatError(f"{path}: bad header: {exc}") from exc
    if tree.depth != depth:
        raise MatrixFormatError(f"{path}: header depth {depth} does not match {tree_depth(m, n, n_b)} for a "
                                f"{m}x{n} matrix at block size {n_b}")
    if n_b != 16:
        raise MatrixFormatError(f"{path}: block size {n_b}; the GPU path stores 16 x 16 leaves")
    if len(raw) != head + count * _RECORD.itemsize:
        raise MatrixFormatError(f"{path}: expected {count} leaf records ({head + count * _RECORD.itemsize} bytes), "
                                f"file has {len(raw)}")
    if count == 0:
        return tree
    rec = np.frombuffer(raw, _RECORD, count, head)
    keys = rec["key"]
    if count > 1 and not np.all(keys[1:] > keys[:-1]):
        bad = int(np.flatnonzero(keys[1:] <= keys[:-1])[0]) + 1
        raise MatrixFormatError(f"{path}: leaf keys not strictly ascending at record {bad}")
    if int(keys[-1]) >= 4 ** depth:
        raise MatrixFormatError(f"{path}: leaf key {int(keys[-1])} out of range for depth {depth}")
    finite = np.isfinite(rec["values"]).all(axis=1)
    if not finite.all():
        raise MatrixFormatError(f"{path}: non-finite values in leaf {int(keys[np.flatnonzero(~finite)[0]])}")
    records = np.zeros((count, _lib.REC), np.float32)
    records[:, :256] = rec["values"]
    tree._set_packed_values(torch.from_numpy(keys.astype(np.int64).astype(np.int32)).to(tree.device),
                            torch.from_numpy(records).to(tree.device))
    return tree
