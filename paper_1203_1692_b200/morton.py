"""Z-order leaf keys at the boundary of the device path.

On the device every kernel works in plain block coordinates ``(i, k, j)``;
Morton keys only appear where the reference's API shows them: the key of a
packed leaf, the ``a``/``b``/``c_key`` handles of a ``ProductTask`` and the
order of ``packed_leaves()``.  The convention is the reference's
(`pkg/src/spamm/morton.py:22-23`, `:57-61`): row bit above column bit in
every bit pair, so ``key = spread(i) << 1 | spread(j)``.

Only numpy arrays are handled here (the scalar forms are thin wrappers); the
device kernels carry their own copy of the bit tricks in ``csrc/common.cuh``.
"""

from __future__ import annotations

import numpy as np

COL_LANE = 0x5555555555555555   # j bits, and k of an A leaf  (reference ODD_MASK)
ROW_LANE = 0xAAAAAAAAAAAAAAAA   # i bits, and k of a B leaf  (reference EVEN_MASK)
ODD_MASK = COL_LANE
EVEN_MASK = ROW_LANE
COORD_LIMIT = 1 << 31

_STAGES = (
    (16, 0x0000FFFF0000FFFF),
    (8, 0x00FF00FF00FF00FF),
    (4, 0x0F0F0F0F0F0F0F0F),
    (2, 0x3333333333333333),
    (1, 0x5555555555555555),
)


def spread_bits(x) -> np.ndarray:
    """Move bit m of each 32-bit coordinate to bit 2m (uint64 result)."""
    v = np.asarray(x).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    for shift, mask in _STAGES:
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def squeeze_bits(x) -> np.ndarray:
    """Inverse of :func:`spread_bits` on the column lane of ``x``."""
    v = np.asarray(x).astype(np.uint64) & np.uint64(COL_LANE)
    for shift, mask in (
        (1, 0x3333333333333333),
        (2, 0x0F0F0F0F0F0F0F0F),
        (4, 0x00FF00FF00FF00FF),
        (8, 0x0000FFFF0000FFFF),
        (16, 0x00000000FFFFFFFF),
    ):
        v = (v | (v >> np.uint64(shift))) & np.uint64(mask)
    return v


def encode_array(i, j) -> np.ndarray:
    return (spread_bits(i) << np.uint64(1)) | spread_bits(j)


def decode_array(keys) -> tuple[np.ndarray, np.ndarray]:
    k = np.asarray(keys).astype(np.uint64)
    return squeeze_bits(k >> np.uint64(1)), squeeze_bits(k)


def encode(i: int, j: int) -> int:
    if not (0 <= i < COORD_LIMIT and 0 <= j < COORD_LIMIT):
        raise ValueError(f"block coordinates ({i}, {j}) outside [0, 2^31)")
    return int(encode_array(np.uint64(i), np.uint64(j)))


def decode(key: int) -> tuple[int, int]:
    if key < 0 or key >> 62:
        raise ValueError(f"key {key} outside the 62 bit interleave range")
    i, j = decode_array(np.uint64(key))
    return int(i), int(j)


def k_of_a(key: int) -> int:
    return key & COL_LANE


def k_of_b(key: int) -> int:
    return key & ROW_LANE


def k_match(key_a: int, key_b: int) -> bool:
    return (key_b & ROW_LANE) >> 1 == (key_a & COL_LANE)


def c_index(key_a: int, key_b: int) -> int:
    """Key of the product leaf: rows of A, columns of B (`morton.py:98-100`)."""
    return (key_a & ROW_LANE) | (key_b & COL_LANE)
