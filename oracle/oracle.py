"""numpy front end of the CPU oracle (``spamm_oracle.c``).

TEST INFRASTRUCTURE ONLY -- imported by ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``; the shipped
package never imports it.  Parity status: pinned against vectors produced by
the unmodified reference (``tests/golden/make_golden.py``).

The functions mirror the reference calls that form the oracle:

    tree_from_dense   <- QuadtreeMatrix.from_dense            core.py:213-266
    tree_from_packed  <- put_leaf ... compute_norms           core.py:315-345
    build_plan        <- symbolic.build_plan                  symbolic.py:151-159
    recursive_tasks   <- reference.recursive_spamm (visits)   reference.py:72-129
    task_masks        <- the fine4 gate                       numeric.py:232-238
    execute_plan      <- numeric.execute_plan                 numeric.py:138-181
    multiply          <- numeric.multiply                     numeric.py:302-313
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libspamm_oracle.so")

NB = 16


def build(force: bool = False) -> str:
    """Compile the C oracle with the committed Makefile (gcc, seconds)."""
    src = os.path.join(_HERE, "spamm_oracle.c")
    stale = (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src)
    if force or stale:
        subprocess.run(["make", "-C", _HERE, "-s"] + (["-B"] if force else []), check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, f64, vp = C.c_int64, C.c_double, C.c_void_p
        _lib.oracle_plan.restype = i64
        _lib.oracle_plan.argtypes = [vp, i64, i64, vp, i64, i64, i64, f64, vp, vp, vp, vp, i64, vp]
        _lib.oracle_recursive_tasks.restype = i64
        _lib.oracle_recursive_tasks.argtypes = [vp, vp, C.c_int, f64, vp, vp, vp, i64]
        _lib.oracle_execute.restype = i64
        _lib.oracle_execute.argtypes = [vp, vp, vp, i64, vp, vp, vp, i64, i64, i64,
                                        vp, vp, vp, i64, f64, C.c_int, vp, vp, i64, vp]
        _lib.oracle_leaf_norms_from_dense.restype = None
        _lib.oracle_leaf_norms_from_dense.argtypes = [vp, i64, i64, i64, vp, vp, vp]
        _lib.oracle_leaf_norms_refresh.restype = None
        _lib.oracle_leaf_norms_refresh.argtypes = [vp, i64, vp, vp, vp]
        _lib.oracle_pyramid.restype = None
        _lib.oracle_pyramid.argtypes = [vp, vp, C.c_int, vp, vp]
        _lib.oracle_task_masks.restype = None
        _lib.oracle_task_masks.argtypes = [vp, vp, vp, vp, i64, i64, vp, vp, vp, i64, f64, vp]
        _lib.oracle_compose_leaf.restype = None
        _lib.oracle_compose_leaf.argtypes = [vp, vp, f64, f64, vp]
        _lib.oracle_dense_single.restype = None
        _lib.oracle_dense_single.argtypes = [vp, vp, i64, i64, i64, vp]
        _lib.oracle_num_threads.restype = C.c_int
        _lib.oracle_set_threads.argtypes = [C.c_int]
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


# -- key algebra (morton.py:57-68), numpy only ---------------------------------

def _spread(x):
    v = np.asarray(x).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    for s, m in ((16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF), (4, 0x0F0F0F0F0F0F0F0F),
                 (2, 0x3333333333333333), (1, 0x5555555555555555)):
        v = (v | (v << np.uint64(s))) & np.uint64(m)
    return v


def encode(i, j):
    return (_spread(i) << np.uint64(1)) | _spread(j)


def tree_depth(m: int, n: int) -> int:
    """core.py:33-39 with n_b = 16."""
    q = -(-max(m, n) // NB)
    return (q - 1).bit_length()


def level_offset(t: int) -> int:
    return ((1 << (2 * t)) - 1) // 3


# -- trees ---------------------------------------------------------------------

@dataclass
class OracleTree:
    """What the reference's QuadtreeMatrix holds, as flat arrays.

    keys/values/subnorms are ``packed_leaves()`` (core.py:387-405): ascending
    Morton key.  ``slot`` maps leaf (i, j) of the 2^depth grid to its packed
    index, -1 where no leaf is stored.  ``norm_levels`` / ``sq_levels`` hold
    every tier's norm grid back to back (tier t at ``level_offset(t)``).
    """

    m: int
    n: int
    depth: int
    keys: np.ndarray
    values: np.ndarray
    subnorms: np.ndarray
    slot: np.ndarray
    norm_levels: np.ndarray
    sq_levels: np.ndarray
    n_b: int = NB

    @property
    def L(self) -> int:
        return 1 << self.depth

    @property
    def leaf_norm(self) -> np.ndarray:
        L = self.L
        return self.norm_levels[level_offset(self.depth):].reshape(L, L)

    def level_norm(self, t: int) -> np.ndarray:
        s = 1 << t
        return self.norm_levels[level_offset(t):level_offset(t) + s * s].reshape(s, s)

    @property
    def norm(self) -> float:
        r = float(self.norm_levels[0])
        return r if r >= 0 else 0.0

    def to_dense(self) -> np.ndarray:
        """core.py:268-276."""
        L = self.L
        out = np.zeros((L, NB, L, NB), np.float32)
        ii, jj = np.nonzero(self.slot >= 0)
        out[ii, :, jj, :] = self.values[self.slot[ii, jj]]
        return np.ascontiguousarray(out.reshape(L * NB, L * NB)[: self.m, : self.n])


def _finish_tree(m, n, depth, present, leafsq_grid, keys, values, subnorms, slot) -> OracleTree:
    L = 1 << depth
    total = level_offset(depth + 1)
    norm_levels = np.empty(total, np.float32)
    sq_levels = np.empty(total, np.float64)
    pres = np.ascontiguousarray(present.astype(np.uint8))
    lsq = np.ascontiguousarray(leafsq_grid, np.float64)
    lib().oracle_pyramid(_p(pres), _p(lsq), depth, _p(norm_levels), _p(sq_levels))
    return OracleTree(m, n, depth, keys, values, subnorms, slot, norm_levels, sq_levels)


def tree_from_dense(dense: np.ndarray) -> OracleTree:
    """QuadtreeMatrix.from_dense(dense, 16) (core.py:213-266)."""
    a = np.ascontiguousarray(dense, np.float32)
    m, n = a.shape
    depth = tree_depth(m, n)
    L = 1 << depth
    br, bc = -(-m // NB), -(-n // NB)
    sub = np.empty((br * bc, 16), np.float32)
    lsq = np.empty(br * bc, np.float64)
    lnorm = np.empty(br * bc, np.float32)
    lib().oracle_leaf_norms_from_dense(_p(a), m, n, n, _p(sub), _p(lsq), _p(lnorm))
    present = np.zeros((L, L), bool)
    present[:br, :bc] = lsq.reshape(br, bc) != 0.0
    sq_grid = np.zeros((L, L), np.float64)
    sq_grid[:br, :bc] = lsq.reshape(br, bc)
    bi, bj = np.nonzero(present)
    keys = encode(bi, bj)
    order = np.argsort(keys, kind="stable")
    bi, bj, keys = bi[order], bj[order], keys[order]
    padded = np.zeros((br * NB, bc * NB), np.float32)
    padded[:m, :n] = a
    tiles = padded.reshape(br, NB, bc, NB)
    values = np.ascontiguousarray(tiles[bi, :, bj, :])
    subnorms = np.ascontiguousarray(sub.reshape(br, bc, 4, 4)[bi, bj])
    slot = np.full((L, L), -1, np.int32)
    slot[bi, bj] = np.arange(keys.size, dtype=np.int32)
    return _finish_tree(m, n, depth, present, sq_grid, keys, values, subnorms, slot)


def tree_from_packed(m: int, n: int, bi: np.ndarray, bj: np.ndarray, values: np.ndarray) -> OracleTree:
    """put_leaf for every (bi, bj) then compute_norms (core.py:315-345)."""
    depth = tree_depth(m, n)
    L = 1 << depth
    keys = encode(bi, bj)
    order = np.argsort(keys, kind="stable")
    bi, bj, keys = np.asarray(bi)[order], np.asarray(bj)[order], keys[order]
    values = np.ascontiguousarray(np.asarray(values, np.float32).reshape(-1, NB, NB)[order])
    nl = keys.size
    sub = np.empty((nl, 4, 4), np.float32)
    lsq = np.empty(nl, np.float64)
    lnorm = np.empty(nl, np.float32)
    lib().oracle_leaf_norms_refresh(_p(values), nl, _p(sub), _p(lsq), _p(lnorm))
    present = np.zeros((L, L), bool)
    present[bi, bj] = True
    sq_grid = np.zeros((L, L), np.float64)
    sq_grid[bi, bj] = lsq
    slot = np.full((L, L), -1, np.int32)
    slot[bi, bj] = np.arange(nl, dtype=np.int32)
    return _finish_tree(m, n, depth, present, sq_grid, keys, values, sub, slot)


def empty_tree(m: int, n: int) -> OracleTree:
    return tree_from_packed(m, n, np.zeros(0, np.int64), np.zeros(0, np.int64),
                            np.zeros((0, NB, NB), np.float32))


# -- symbolic phase --------------------------------------------------------------

@dataclass
class OraclePlan:
    """Tasks in the reference's plan order as (i, k, j) leaf coordinates."""

    ti: np.ndarray
    tk: np.ndarray
    tj: np.ndarray
    norm_product: np.ndarray
    tau: float
    emitted: int = 0
    examined: int = 0
    pruned: int = 0

    def __len__(self) -> int:
        return int(self.ti.size)

    @property
    def a_keys(self):
        return encode(self.ti, self.tk)

    @property
    def b_keys(self):
        return encode(self.tk, self.tj)

    @property
    def c_keys(self):
        return encode(self.ti, self.tj)

    def pair_set(self) -> set:
        return set(zip(self.a_keys.tolist(), self.b_keys.tolist()))

    def dump(self) -> str:
        """plan_dump (symbolic.py:139-148)."""
        if len(self) == 0:
            return ""
        rows = zip(self.a_keys.tolist(), self.b_keys.tolist(), self.c_keys.tolist(),
                   self.norm_product.tolist())
        return "\n".join(f"{a} {b} {c} {p:.9e}" for a, b, c, p in rows) + "\n"


def _check_tau(tau: float) -> None:
    if np.isnan(tau) or tau < 0:
        raise ValueError(f"tau must be nonnegative, got {tau}")


def build_plan(a: OracleTree, b: OracleTree, tau: float) -> OraclePlan:
    """symbolic.build_plan (symbolic.py:151-159)."""
    if a.n_b != b.n_b:
        raise ValueError(f"block sizes differ: {a.n_b} vs {b.n_b}")
    if a.n != b.m:
        raise ValueError(f"inner dimensions differ: {a.m}x{a.n} times {b.m}x{b.n}")
    _check_tau(tau)
    na, nb = a.leaf_norm, b.leaf_norm
    rows_a, cols_b = -(-a.m // NB), -(-b.n // NB)
    K = -(-a.n // NB)
    stats = np.zeros(3, np.int64)
    args = (_p(na), rows_a, a.L, _p(nb), cols_b, b.L, K, float(tau))
    T = lib().oracle_plan(*args, None, None, None, None, 0, _p(stats))
    ti = np.empty(T, np.int32)
    tk = np.empty(T, np.int32)
    tj = np.empty(T, np.int32)
    pr = np.empty(T, np.float64)
    lib().oracle_plan(*args, _p(ti), _p(tk), _p(tj), _p(pr), T, _p(stats))
    return OraclePlan(ti, tk, tj, pr, float(tau), int(stats[0]), int(stats[1]), int(stats[2]))


def recursive_tasks(a: OracleTree, b: OracleTree, tau: float) -> np.ndarray:
    """Leaf pairs visited by reference.recursive_spamm, as sorted (i,k,j) rows."""
    if a.depth != b.depth:
        raise ValueError(f"mismatched depths: {a.depth} vs {b.depth}")
    _check_tau(tau)
    args = (_p(a.norm_levels), _p(b.norm_levels), a.depth, float(tau))
    T = lib().oracle_recursive_tasks(*args, None, None, None, 0)
    ti = np.empty(T, np.int32)
    tk = np.empty(T, np.int32)
    tj = np.empty(T, np.int32)
    lib().oracle_recursive_tasks(*args, _p(ti), _p(tk), _p(tj), T)
    out = np.stack([ti, tk, tj], axis=1)
    return out[np.lexsort((tk, tj, ti))]


def task_masks(a: OracleTree, b: OracleTree, plan: OraclePlan, tau: float) -> np.ndarray:
    """fine4 live bits per task: bit r*16 + p*4 + q (numeric.py:232-238)."""
    T = len(plan)
    out = np.empty(T, np.uint64)
    lib().oracle_task_masks(_p(a.slot), _p(a.subnorms), _p(b.slot), _p(b.subnorms), a.L, b.L,
                            _p(plan.ti), _p(plan.tk), _p(plan.tj), T, float(tau), _p(out))
    return out


# -- numeric phase ---------------------------------------------------------------

GRANULARITIES = ("fine4", "coarse16")


@dataclass
class OracleCounters:
    products4: int = 0
    skipped4: int = 0
    seconds: float = 0.0

    @property
    def flops(self) -> int:
        return self.products4 * 128


def execute_plan(plan: OraclePlan, a: OracleTree, b: OracleTree, c: OracleTree | None,
                 tau: float, granularity: str = "fine4", alpha: float = 1.0,
                 beta: float = 0.0) -> tuple[OracleTree, OracleCounters]:
    """numeric.execute_plan (numeric.py:138-181, :268-284)."""
    if granularity not in GRANULARITIES:
        raise ValueError(f"granularity must be one of {GRANULARITIES}, got {granularity!r}")
    _check_tau(tau)
    if not (np.isfinite(alpha) and np.isfinite(beta)):
        raise ValueError("alpha and beta must be finite")
    if plan.tau != tau:
        raise ValueError(f"plan built for tau={plan.tau}, config has tau={tau}")
    if a.n != b.m:
        raise ValueError(f"inner dimensions differ: {a.m}x{a.n} times {b.m}x{b.n}")
    if c is not None and (c.m, c.n) != (a.m, b.n):
        raise ValueError(f"accumulator is {c.m}x{c.n} (n_b={c.n_b}), product needs {a.m}x{b.n} (n_b={NB})")
    m, n = a.m, b.n
    depth = tree_depth(m, n)
    Lc = 1 << depth
    counters = OracleCounters()
    T = len(plan)
    prod_ij = np.zeros((0, 2), np.int64)
    prod_vals = np.zeros((0, NB, NB), np.float32)
    if T and alpha != 0:
        rows_c, cols_c = -(-m // NB), -(-n // NB)
        cslot = np.empty(rows_c * cols_c, np.int32)
        ncap = int(np.unique(plan.ti.astype(np.int64) * cols_c + plan.tj).size)
        cvals = np.empty((ncap, NB, NB), np.float32)
        cnt = np.zeros(2, np.int64)
        nc = lib().oracle_execute(_p(a.slot), _p(a.values), _p(a.subnorms), a.L,
                                  _p(b.slot), _p(b.values), _p(b.subnorms), b.L,
                                  rows_c, cols_c, _p(plan.ti), _p(plan.tk), _p(plan.tj), T,
                                  float(tau), 1 if granularity == "fine4" else 0,
                                  _p(cslot), _p(cvals), ncap, _p(cnt))
        if nc == -1:
            raise ValueError("plan references leaves not stored in an operand (stale handles)")
        if nc < 0:
            raise RuntimeError("oracle_execute: capacity")
        counters.products4, counters.skipped4 = int(cnt[0]), int(cnt[1])
        g = cslot.reshape(rows_c, cols_c)
        pi, pj = np.nonzero(g >= 0)
        prod_ij = np.stack([pi, pj], axis=1)
        prod_vals = cvals[g[pi, pj]]
    # _compose (numeric.py:268-284); the float32 expressions are the reference's own
    a32, b32 = np.float32(alpha), np.float32(beta)
    scaled_prod = a32 * prod_vals if alpha != 1 else prod_vals
    cols = 1 << depth
    lin_p = prod_ij[:, 0] * cols + prod_ij[:, 1]
    if beta == 0 or c is None or c.keys.size == 0:
        out_ij, out_vals = prod_ij, scaled_prod
    else:
        ci, cj = np.nonzero(c.slot >= 0)
        lin_c = ci.astype(np.int64) * cols + cj
        old = c.values[c.slot[ci, cj]]
        old = old * b32 if beta != 1 else old
        pos = {int(v): x for x, v in enumerate(lin_c.tolist())}
        hit = np.array([pos.get(int(v), -1) for v in lin_p.tolist()], np.int64)
        both = hit >= 0
        merged = old.copy()
        if both.any():
            merged[hit[both]] = scaled_prod[both] + old[hit[both]]
        out_ij = np.concatenate([np.stack([ci, cj], axis=1), prod_ij[~both]])
        out_vals = np.concatenate([merged, scaled_prod[~both]])
    if out_ij.shape[0]:
        tree = tree_from_packed(m, n, out_ij[:, 0], out_ij[:, 1], out_vals)
    else:
        tree = empty_tree(m, n)
    assert tree.depth == depth and tree.L == Lc
    return tree, counters


def multiply(a: OracleTree, b: OracleTree, tau: float = 0.0, granularity: str = "fine4",
             alpha: float = 1.0, beta: float = 0.0, c: OracleTree | None = None):
    """numeric.multiply (numeric.py:302-313)."""
    plan = build_plan(a, b, tau)
    out, counters = execute_plan(plan, a, b, c, tau, granularity, alpha, beta)
    return out, plan, counters


def dense_multiply_single(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """reference.dense_multiply_single (reference.py:58-69)."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    out = np.empty((a.shape[0], b.shape[1]), np.float32)
    lib().oracle_dense_single(_p(a), _p(b), a.shape[0], a.shape[1], b.shape[1], _p(out))
    return out
