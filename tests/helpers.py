"""Shared test helpers: golden fixture access and oracle-side records."""

from __future__ import annotations

import json
import os

import numpy as np

from cases import CASES, FULL_LIMIT, build_inputs, case_by_name, digest  # noqa: F401
from oracle import oracle as O

_GOLDEN = None


class Golden:
    def __init__(self, path):
        self.z = np.load(path)
        self.meta = json.loads(bytes(self.z["__meta__"]).decode())

    def get(self, case: str, key: str):
        full = f"{case}/{key}"
        if full in self.z.files:
            return self.z[full]
        return self.meta["cases"][case][key]

    def has(self, case: str, key: str) -> bool:
        return f"{case}/{key}" in self.z.files or key in self.meta["cases"][case]


def golden() -> Golden:
    global _GOLDEN
    if _GOLDEN is None:
        _GOLDEN = Golden(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    return _GOLDEN


def tiers_blob(norm_levels, depth: int) -> np.ndarray:
    """Every tier's (sorted keys, norms) as bytes, as make_golden.tree_record does.
    `norm_levels` is the oracle's flat level buffer or a callable tier -> grid."""
    parts = []
    for t in range(depth + 1):
        s = 1 << t
        if callable(norm_levels):
            g = norm_levels(t)
        else:
            off = O.level_offset(t)
            g = norm_levels[off:off + s * s].reshape(s, s)
        ii, jj = np.nonzero(g >= 0)
        keys = O.encode(ii, jj)
        order = np.argsort(keys, kind="stable")
        parts.append(np.concatenate([keys[order].astype(np.uint64).view(np.uint8),
                                     g[ii, jj][order].astype(np.float32).view(np.uint8)]))
    return np.concatenate(parts) if parts else np.zeros(0, np.uint8)


def oracle_operands(case: dict):
    """(A, B, C0) oracle trees of a golden case, including the `chain` construction."""
    a_d, b_d, c_d = build_inputs(case)
    qa = O.tree_from_dense(a_d)
    qb = qa if b_d is None else O.tree_from_dense(b_d)
    if case.get("chain"):
        prod, _, _ = O.multiply(qa, qb, 0.0)
        qa = qb = prod
    c0 = O.tree_from_dense(c_d) if c_d is not None else None
    return qa, qb, c0, (a_d, b_d, c_d)


def check_tree(g: Golden, case: str, prefix: str, keys, values, subnorms, leaf_norm, tiers,
               m=None, n=None, depth=None):
    """Compare a packed tree (any implementation) against the reference's record."""
    assert np.array_equal(np.asarray(keys, np.uint64), g.get(case, f"{prefix}keys")), f"{prefix} keys"
    if m is not None:
        assert (m, n, depth) == (g.get(case, f"{prefix}m"), g.get(case, f"{prefix}n"),
                                 g.get(case, f"{prefix}depth"))
    assert digest(np.asarray(values, np.float32).reshape(-1, 16, 16)) == g.get(case, f"{prefix}values_sha"), f"{prefix} values"
    assert digest(np.asarray(subnorms, np.float32).reshape(-1, 4, 4)) == g.get(case, f"{prefix}subnorms_sha"), f"{prefix} subnorms"
    assert digest(np.asarray(leaf_norm, np.float32)) == g.get(case, f"{prefix}leaf_norm_sha"), f"{prefix} leaf norms"
    assert digest(tiers) == g.get(case, f"{prefix}tiers_sha"), f"{prefix} interior norms"
    if g.has(case, f"{prefix}values"):
        assert np.array_equal(values.reshape(-1, 16, 16), g.get(case, f"{prefix}values"))
        assert np.array_equal(subnorms.reshape(-1, 4, 4), g.get(case, f"{prefix}subnorms"))


def check_oracle_tree(g: Golden, case: str, prefix: str, t: O.OracleTree):
    ii, jj = np.nonzero(t.slot >= 0)
    order = np.argsort(O.encode(ii, jj), kind="stable")
    leaf_norm = t.leaf_norm[ii, jj][order]
    check_tree(g, case, prefix, t.keys, t.values, t.subnorms, leaf_norm,
               tiers_blob(t.norm_levels, t.depth), t.m, t.n, t.depth)


def check_device_tree(g: Golden, case: str, prefix: str, q):
    """Device QuadtreeMatrix against the reference's record (bit for bit)."""
    keys, values, subs = q.packed_leaves()
    from paper_1203_1692_b200 import morton
    i, j = morton.decode_array(keys)
    leaf_norm = q.level_norms(q.depth)[i.astype(np.int64), j.astype(np.int64)] if keys.size else np.zeros(0, np.float32)
    check_tree(g, case, prefix, keys, values, subs, leaf_norm, tiers_blob(q.level_norms, q.depth), q.m, q.n, q.depth)


def assert_trees_equal(q, t: O.OracleTree, what: str = ""):
    """Device tree == oracle tree: leaves, sub-norms and every tier's norms, bit for bit."""
    keys, values, subs = q.packed_leaves()
    assert np.array_equal(keys, t.keys.astype(np.uint64)), f"{what}: leaf keys"
    assert np.array_equal(values.view(np.uint32), t.values.view(np.uint32)), f"{what}: leaf values"
    assert np.array_equal(subs.view(np.uint32), t.subnorms.view(np.uint32)), f"{what}: sub-norms"
    assert (q.m, q.n, q.depth) == (t.m, t.n, t.depth)
    for tier in range(t.depth + 1):
        assert np.array_equal(q.level_norms(tier), t.level_norm(tier)), f"{what}: tier {tier} norms"
