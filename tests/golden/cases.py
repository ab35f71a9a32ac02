"""Parity cases shared by make_golden.py (reference side) and the tests (oracle and
device side).  Inputs are rebuilt from seeds; the fixture stores digests of them so
generator drift is caught rather than silently compared against stale goldens."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

from paper_1203_1692_b200 import inputs  # noqa: E402

FULL_LIMIT = 128   # cases no larger than this keep full arrays in golden.npz


def digest(a: np.ndarray | None) -> str:
    if a is None:
        return ""
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(f"{a.dtype.str}{a.shape}".encode())
    h.update(a.tobytes())
    return h.hexdigest()


def uniform(m: int, n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return ((rng.random((m, n)) * 2.0 - 1.0) * scale).astype(np.float32)


def block_sparse(n: int, seed: int, fill: float = 0.4) -> np.ndarray:
    """Random 16x16 blocks at three magnitudes, 60 % of blocks empty."""
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n), np.float32)
    for bi in range(n // 16):
        for bj in range(n // 16):
            if rng.random() < fill:
                a[16 * bi:16 * bi + 16, 16 * bj:16 * bj + 16] = (
                    rng.random((16, 16)) * rng.choice([1e-6, 1e-3, 1.0]))
    return a


def zero_product_pair() -> tuple[np.ndarray, np.ndarray]:
    """32x32 operands whose product has a stored leaf that is exactly zero:
    A's leaf (0,0) only has column 0, B's leaf (0,1) only has row 1."""
    a = np.zeros((32, 32), np.float32)
    b = np.zeros((32, 32), np.float32)
    a[:16, 0] = np.arange(1, 17, dtype=np.float32)
    a[16:, 16:] = uniform(16, 16, 3)
    b[1, 16:] = np.arange(1, 17, dtype=np.float32) * 0.5
    b[:16, :16] = uniform(16, 16, 4)
    b[16:, 16:] = uniform(16, 16, 5)
    return a, b


_TAUS4 = (1e-4, 1e-6, 1e-8, 1e-10)

CASES = [
    dict(name="rand64", kind="uniform", shape=(64, 64, 64), seeds=(13, 14), runs=[
        dict(tag="t0", tau=0.0, recursive=True),
        dict(tag="t0c", tau=0.0, granularity="coarse16"),
    ]),
    dict(name="exp96", kind="exp", n=96, lam=0.7, seeds=(11, 12), runs=[
        dict(tag="t0", tau=0.0, recursive=True),
        dict(tag="t1e-6", tau=1e-6, recursive=True),
        dict(tag="t1e-6c", tau=1e-6, granularity="coarse16"),
        dict(tag="t1e-3", tau=1e-3, recursive=True),
        dict(tag="t10", tau=10.0, recursive=True),
    ]),
    dict(name="rect", kind="uniform", shape=(40, 72, 24), seeds=(15, 16), runs=[
        dict(tag="t0", tau=0.0),
        dict(tag="t3", tau=3.0),
    ]),
    dict(name="alphabeta64", kind="exp", n=64, lam=0.6, seeds=(21, None), c_seed=22, runs=[
        dict(tag="a2", tau=0.0, alpha=2.0),
        dict(tag="a2b05", tau=0.0, alpha=2.0, beta=0.5, use_c=True),
        dict(tag="a0b1", tau=0.0, alpha=0.0, beta=1.0, use_c=True),
        dict(tag="b0", tau=1e-4, beta=0.0, use_c=True),
        dict(tag="am15b1", tau=1e-4, alpha=-1.5, beta=1.0, use_c=True),
        dict(tag="b3noC", tau=1e-4, alpha=1.0, beta=3.0),
    ]),
    dict(name="zeroleaf", kind="zero_product", chain=True, runs=[
        dict(tag="t0", tau=0.0, recursive=True),
        dict(tag="t1e-30", tau=1e-30),
    ]),
    dict(name="blocksparse128", kind="block_sparse", n=128, seeds=(23, 24), runs=[
        dict(tag="t0", tau=0.0, recursive=True),
        dict(tag="t1e-9", tau=1e-9, recursive=True),
        dict(tag="t1e-4", tau=1e-4, recursive=True),
        dict(tag="t1", tau=1.0),
        dict(tag="t1e6", tau=1e6, recursive=True),
    ]),
    dict(name="cfg1", kind="workload", workload="cfg1", runs=[
        dict(tag="t1e-6", tau=1e-6, recursive=True),
        dict(tag="t1e-6c", tau=1e-6, granularity="coarse16"),
    ]),
    dict(name="cfg2_512", kind="workload", workload="cfg2", n=512, runs=[
        dict(tag=f"t{t:g}", tau=t, recursive=(t == 1e-8)) for t in _TAUS4
    ]),
    dict(name="cfg3_512", kind="workload", workload="cfg3", n=512, runs=[
        dict(tag="t1e-8", tau=1e-8, recursive=True),
        dict(tag="t1e-8c", tau=1e-8, granularity="coarse16"),
    ]),
    dict(name="cfg4_500", kind="workload", workload="cfg4", n=500, runs=[
        dict(tag="t1e-6", tau=1e-6),
        dict(tag="t1e-8", tau=1e-8, recursive=True),
    ]),
    dict(name="cfg5_1024", kind="workload", workload="cfg5", n=1024, runs=[
        dict(tag="t1e-8", tau=1e-8),
    ]),
]


def build_inputs(case: dict):
    """Dense fp32 (A, B or None when B is A, C0 or None)."""
    kind = case["kind"]
    c0 = None
    if kind == "uniform":
        m, k, n = case["shape"]
        a, b = uniform(m, k, case["seeds"][0]), uniform(k, n, case["seeds"][1])
    elif kind == "exp":
        n = case["n"]
        a = inputs.exponential_decay(n, case["lam"], seed=case["seeds"][0], symmetric=False)
        b = None if case["seeds"][1] is None else inputs.exponential_decay(
            n, case["lam"] * 0.9, seed=case["seeds"][1], symmetric=False)
        if case.get("c_seed") is not None:
            c0 = uniform(n, n, case["c_seed"])
    elif kind == "block_sparse":
        a, b = block_sparse(case["n"], case["seeds"][0]), block_sparse(case["n"], case["seeds"][1])
    elif kind == "zero_product":
        a, b = zero_product_pair()
    elif kind == "workload":
        a, b = inputs.make_operands(case["workload"], case.get("n"))
    else:
        raise ValueError(kind)
    return a, b, c0


def case_by_name(name: str) -> dict:
    for c in CASES:
        if c["name"] == name:
            return c
    raise KeyError(name)
