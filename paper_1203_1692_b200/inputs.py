"""Seeded synthetic operands for the five BASELINE.json configurations.

These follow the laws written in BASELINE.json (amplitude ``u ~ U[0.5, 1)``,
seeded signs, the stated envelopes), not the reference package's own
generator (`pkg/src/spamm/generators.py:5`, `:95`, `:111` use ``0.05+0.9u`` and
``|i-j|**lam``).  The paper's real inputs (FreeON density matrices,
`PAPER.md:733-746`) are not available; these matrices stand in for them.

Draw order is part of the definition and frozen here: rows are produced in
chunks of ``CHUNK`` rows; for each chunk first the amplitudes, then the signs,
from one ``np.random.default_rng(seed)``.  "Symmetric" copies the upper
triangle (diagonal included) onto the lower one, the reference's convention
(`generators.py:117-127`).

Everything here is host-side numpy: the same arrays feed the oracle and the
device path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CHUNK = 1024


def _draw(n: int, seed: int, env_rows) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.empty((n, n), np.float32)
    for r0 in range(0, n, CHUNK):
        r1 = min(n, r0 + CHUNK)
        u = rng.uniform(0.5, 1.0, (r1 - r0, n))
        s = rng.integers(0, 2, (r1 - r0, n)).astype(np.float64) * 2.0 - 1.0
        out[r0:r1] = (s * u * env_rows(r0, r1)).astype(np.float32)
    return out


def symmetrise(a: np.ndarray) -> np.ndarray:
    """Mirror the upper triangle onto the lower one, in place, by row chunks."""
    n = a.shape[0]
    for r0 in range(0, n, CHUNK):
        r1 = min(n, r0 + CHUNK)
        a[r0:r1, :r0] = a[:r0, r0:r1].T
        blk = a[r0:r1, r0:r1]
        iu, ju = np.triu_indices(r1 - r0, 1)
        blk[ju, iu] = blk[iu, ju]
    return a


def exponential_decay(n: int, lam: float, seed: int = 0, symmetric: bool = True) -> np.ndarray:
    """``a_ij = s_ij u_ij lam**|i-j|`` (configs 1, 2, 5)."""
    cols = np.arange(n, dtype=np.int64)[None, :]

    def env(r0, r1):
        rows = np.arange(r0, r1, dtype=np.int64)[:, None]
        return np.power(float(lam), np.abs(rows - cols).astype(np.float64))

    a = _draw(n, seed, env)
    return symmetrise(a) if symmetric else a


def algebraic_decay(n: int, seed: int = 0, power: int = 3, symmetric: bool = True) -> np.ndarray:
    """``a_ij = s_ij u_ij / (|i-j|**power + 1)`` (config 3)."""
    cols = np.arange(n, dtype=np.int64)[None, :]

    def env(r0, r1):
        rows = np.arange(r0, r1, dtype=np.int64)[:, None]
        return 1.0 / (np.abs(rows - cols).astype(np.float64) ** power + 1.0)

    a = _draw(n, seed, env)
    return symmetrise(a) if symmetric else a


def _hilbert_index_3d(q: np.ndarray, bits: int) -> np.ndarray:
    """Hilbert-curve rank of integer points ``q`` (N, 3) on a ``2**bits`` grid.

    Skilling's transpose algorithm ("Programming the Hilbert curve", 2004):
    axes are Gray-decoded in place, then the transposed bits are interleaved.
    """
    x = q.astype(np.uint64).copy()
    n_pts, dims = x.shape
    m = np.uint64(1) << np.uint64(bits - 1)
    # inverse undo
    qq = m
    while qq > 1:
        p = qq - np.uint64(1)
        for d in range(dims):
            hit = (x[:, d] & qq) != 0
            x[hit, 0] ^= p
            t = (x[:, 0] ^ x[:, d]) & p
            t[hit] = 0
            x[:, 0] ^= t
            x[:, d] ^= t
        qq >>= np.uint64(1)
    # Gray encode
    for d in range(1, dims):
        x[:, d] ^= x[:, d - 1]
    t = np.zeros(n_pts, np.uint64)
    qq = m
    while qq > 1:
        hit = (x[:, dims - 1] & qq) != 0
        t[hit] ^= qq - np.uint64(1)
        qq >>= np.uint64(1)
    for d in range(dims):
        x[:, d] ^= t
    # interleave: bit b of axis d lands at position b*dims + (dims-1-d)
    h = np.zeros(n_pts, np.uint64)
    for b in range(bits):
        for d in range(dims):
            bit = (x[:, d] >> np.uint64(b)) & np.uint64(1)
            h |= bit << np.uint64(b * dims + (dims - 1 - d))
    return h


def molecule_decay(
    centres: int = 300,
    per_centre: int = 25,
    side: float = 21.0,
    length: float = 1.5,
    seed: int = 0,
) -> np.ndarray:
    """Config 4: Hilbert-ordered molecule centres, ``exp(-r_IJ / length)`` envelope.

    Returns the ``n = centres * per_centre`` square matrix (7500 for the
    defaults); the tree pads it to 8192 itself (`core.py:156-166`,
    ``tree_depth(7500, 7500, 16) == 9``, `tests/test_core.py:22`).
    """
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, side, (centres, 3))
    grid = np.minimum((pos / side * 1024.0).astype(np.int64), 1023)
    order = np.argsort(_hilbert_index_3d(grid, 10), kind="stable")
    pos = pos[order]
    dist = np.sqrt(((pos[:, None, :] - pos[None, :, :]) ** 2).sum(axis=2))
    env_c = np.exp(-dist / length)
    n = centres * per_centre
    owner = np.arange(n) // per_centre

    def env(r0, r1):
        return env_c[owner[r0:r1]][:, owner]

    # draws continue on the same generator, after the centre positions
    out = np.empty((n, n), np.float32)
    for r0 in range(0, n, CHUNK):
        r1 = min(n, r0 + CHUNK)
        u = rng.uniform(0.5, 1.0, (r1 - r0, n))
        s = rng.integers(0, 2, (r1 - r0, n)).astype(np.float64) * 2.0 - 1.0
        out[r0:r1] = (s * u * env(r0, r1)).astype(np.float32)
    return symmetrise(out)


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    taus: tuple[float, ...]
    square: bool          # C = A A when True, C = A B otherwise
    description: str


WORKLOADS = {
    "cfg1": Workload("cfg1", 1024, (1e-6,), True, "exp decay lam=0.9 n=1024 sym, C=A*A"),
    "cfg2": Workload("cfg2", 4096, (1e-4, 1e-6, 1e-8, 1e-10), True,
                     "exp decay lam=0.95 n=4096 sym, C=A*A"),
    "cfg3": Workload("cfg3", 8192, (1e-8,), False,
                     "algebraic 1/(d^3+1) n=8192 sym, C=A*B (seeds 0,1)"),
    "cfg4": Workload("cfg4", 7500, (1e-6, 1e-8), True,
                     "300 Hilbert-ordered centres x 25, exp(-r/1.5A), n=7500->8192, C=A*A"),
    "cfg5": Workload("cfg5", 32768, (1e-8,), True, "exp decay lam=0.97 n=32768 sym, C=A*A"),
}


def make_operands(name: str, n: int | None = None) -> tuple[np.ndarray, np.ndarray | None]:
    """Dense fp32 operands ``(A, B)`` of a named workload; ``B is None`` means C = A A.

    ``n`` overrides the size for scaled-down parity cases of the same law
    (for cfg4 it scales the number of centres, 25 indices each).
    """
    if name == "cfg1":
        return exponential_decay(n or 1024, 0.9, seed=0), None
    if name == "cfg2":
        return exponential_decay(n or 4096, 0.95, seed=0), None
    if name == "cfg3":
        m = n or 8192
        return algebraic_decay(m, seed=0), algebraic_decay(m, seed=1)
    if name == "cfg4":
        centres = 300 if n is None else max(1, n // 25)
        return molecule_decay(centres=centres), None
    if name == "cfg5":
        return exponential_decay(n or 32768, 0.97, seed=0), None
    raise ValueError(f"unknown workload {name!r}")
