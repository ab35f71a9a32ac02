"""Symbolic multiply phase on the device: ``build_plan``.

Drop-in for `pkg/src/spamm/symbolic.py:151-159`.  The plan lives in HBM as the CSR task list
the numeric kernel consumes (product leaves in Morton order, tasks in ascending k); the
reference's host view -- ``plan.tasks`` as ``ProductTask`` objects in the reference's plan
order, ``plan.stats`` and ``plan_dump`` -- is materialised lazily from it.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, morton
from .tree import QuadtreeMatrix, _stream


@dataclass(slots=True)
class ProductTask:
    a: int                  # leaf key handle into A
    b: int                  # leaf key handle into B
    c_key: int              # product leaf key
    norm_product: float


@dataclass(slots=True)
class PlanStats:
    emitted: int = 0
    examined: int = 0
    pruned: int = 0


# capacity that worked last time for a (depth, leaves of A, leaves of B) shape
_capacity_hint: dict[tuple, tuple[int, int]] = {}


class MultiplyPlan:
    """Surviving block products for one (A, B, tau) (`symbolic.py:49-56`), device resident.

    Device arrays (see ``spamm_plan_buffers``): ``c_keys[nC]``, ``c_off[nC+1]``, ``task_k/a/b[T]``,
    ``task_mask[T]``.  ``len(plan)`` is the task count; ``plan.tasks`` builds the reference's
    host list on demand.
    """

    def __init__(self, tau, granularity, depth, n_tasks, n_cleaves, buffers, a, b, row_range):
        self.tau = float(tau)
        self.granularity = granularity
        self.depth = depth
        self.n_tasks = int(n_tasks)
        self.n_cleaves = int(n_cleaves)
        self.c_keys, self.c_off, self.task_k, self.task_a, self.task_b, self.task_mask = buffers
        self._a, self._b = a, b
        self._tokens = (id(a), a._rev, id(b), b._rev)
        self.row_range = row_range
        self._tasks = None
        self._stats = None

    def __len__(self) -> int:
        return self.n_tasks

    # -- host views ---------------------------------------------------------------------------
    def ikj(self) -> np.ndarray:
        """(T, 3) int64 array of (i, k, j) leaf coordinates in device order."""
        T, nC = self.n_tasks, self.n_cleaves
        if T == 0:
            return np.zeros((0, 3), np.int64)
        keys = self.c_keys[:nC].cpu().numpy().astype(np.uint64)
        off = self.c_off[:nC + 1].cpu().numpy().astype(np.int64)
        ci, cj = morton.decode_array(keys)
        rep = np.diff(off)
        k = self.task_k[:T].cpu().numpy().astype(np.int64)
        return np.stack([np.repeat(ci.astype(np.int64), rep), k, np.repeat(cj.astype(np.int64), rep)], axis=1)

    def masks(self) -> np.ndarray:
        return self.task_mask[: self.n_tasks].cpu().numpy().view(np.uint64)

    def pair_keys(self) -> tuple[np.ndarray, np.ndarray]:
        t = self.ikj()
        return morton.encode_array(t[:, 0], t[:, 1]), morton.encode_array(t[:, 1], t[:, 2])

    def _reference_order(self):
        """Tasks in the reference's plan order with their norm products, and the loop
        statistics of `symbolic.py:92-132` (ascending k; A then B by descending norm, ties on
        ascending key; examined counts the first failing B entry of each A entry, and the
        A entry that emits nothing ends its k block)."""
        t = self.ikj()
        na = self._a.level_norms(self._a.depth).astype(np.float64)
        nb = self._b.level_norms(self._b.depth).astype(np.float64)
        if t.shape[0]:
            i, k, j = t[:, 0], t[:, 1], t[:, 2]
            va, vb = na[i, k], nb[k, j]
            ka, kb = morton.encode_array(i, k), morton.encode_array(k, j)
            order = np.lexsort((kb, -vb, ka, -va, k))
            tasks = (ka[order], kb[order], morton.encode_array(i, j)[order], (va * vb)[order])
        else:
            tasks = (np.zeros(0, np.uint64),) * 3 + (np.zeros(0, np.float64),)
        # statistics: per k block, walk A entries by descending norm
        examined = pruned = 0
        rows_a, cols_b = -(-self._a.m // 16), -(-self._b.n // 16)
        r0, r1 = self.row_range
        K = min(-(-self._a.n // 16), na.shape[1], nb.shape[0])
        for k in range(K):
            a_col = na[r0:min(r1, rows_a), k]
            b_row = nb[k, :cols_b]
            a_col = np.sort(a_col[a_col >= 0])[::-1]
            b_row = np.sort(b_row[b_row >= 0])[::-1]
            if a_col.size == 0 or b_row.size == 0:
                continue
            for v in a_col:
                cnt = int(np.count_nonzero(v * b_row >= self.tau))
                examined += cnt + (1 if cnt < b_row.size else 0)
                pruned += 1 if cnt < b_row.size else 0
                if cnt == 0:
                    break
        return tasks, PlanStats(self.n_tasks, examined, pruned)

    @property
    def tasks(self) -> list[ProductTask]:
        if self._tasks is None:
            (ka, kb, kc, pr), self._stats = self._reference_order()
            self._tasks = [ProductTask(int(a), int(b), int(c), float(p))
                           for a, b, c, p in zip(ka.tolist(), kb.tolist(), kc.tolist(), pr.tolist())]
        return self._tasks

    @property
    def stats(self) -> PlanStats:
        if self._stats is None:
            _, self._stats = self._reference_order()
        return self._stats


def plan_stats(plan: MultiplyPlan) -> PlanStats:
    return plan.stats


def plan_dump(plan: MultiplyPlan) -> str:
    """Plan as text lines 'a_key b_key c_key norm_product', plan order (`symbolic.py:139-148`)."""
    if not len(plan):
        return ""
    return "\n".join(f"{t.a} {t.b} {t.c_key} {t.norm_product:.9e}" for t in plan.tasks) + "\n"


def _check_tau(tau) -> None:
    if np.isnan(tau) or tau < 0:
        raise ValueError(f"tau must be nonnegative, got {tau}")


def build_plan(a: QuadtreeMatrix, b: QuadtreeMatrix, tau: float, granularity: str = "fine4",
               row_range: tuple[int, int] | None = None) -> MultiplyPlan:
    """Full symbolic pipeline for C = A B on the device (`symbolic.py:151-159`).

    ``granularity`` only selects which fine4 masks are attached to the tasks (the task set does
    not depend on it); ``row_range`` restricts the plan to product leaf rows [r0, r1) for the
    row-block sharding across GPUs.
    """
    if a.n_b != b.n_b:
        raise ValueError(f"block sizes differ: {a.n_b} vs {b.n_b}")
    if a.n != b.m:
        raise ValueError(f"inner dimensions differ: {a.m}x{a.n} times {b.m}x{b.n}")
    _check_tau(tau)
    a._require_16()
    lib = _lib.lib()
    depth = max(a.depth, b.depth)
    L = 1 << depth
    r0, r1 = (0, L) if row_range is None else (int(row_range[0]), int(row_range[1]))
    dev = a.device
    gran = _lib.FINE4 if granularity == "fine4" else _lib.COARSE16
    if a.nleaf == 0 or b.nleaf == 0:
        empty = torch.empty((1,), dtype=torch.int32, device=dev)
        return MultiplyPlan(tau, granularity, depth, 0, 0, (empty,) * 5 + (torch.empty((1,), dtype=torch.int64, device=dev),),
                            a, b, (r0, r1))
    va, vb = a.view(depth), b.view(depth)
    hint_key = (depth, a.nleaf, b.nleaf, float(tau), r0, r1)
    task_cap, leaf_cap = _capacity_hint.get(hint_key, (max(4096, 24 * (a.nleaf + b.nleaf)),
                                                       min(L * L, max(1024, 2 * (a.nleaf + b.nleaf)))))
    max_tasks = min((1 << 31) - 128, L * L * L)
    while True:
        c_keys = torch.empty((leaf_cap + 1,), dtype=torch.int32, device=dev)
        c_off = torch.empty((leaf_cap + 2,), dtype=torch.int32, device=dev)
        task_k = torch.empty((task_cap + 1,), dtype=torch.int32, device=dev)
        task_a = torch.empty((task_cap + 1,), dtype=torch.int32, device=dev)
        task_b = torch.empty((task_cap + 1,), dtype=torch.int32, device=dev)
        task_mask = torch.empty((task_cap + 1,), dtype=torch.int64, device=dev)
        counts = torch.empty((4,), dtype=torch.int32, device=dev)
        ws_bytes = lib.spamm_plan_workspace_bytes(depth, task_cap, leaf_cap)
        ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=dev)
        bufs = _lib.PlanBuffers(c_keys.data_ptr(), c_off.data_ptr(), task_k.data_ptr(), task_a.data_ptr(),
                                task_b.data_ptr(), task_mask.data_ptr(), task_cap, leaf_cap, counts.data_ptr())
        _lib.check(lib.spamm_plan(C.byref(va), C.byref(vb), float(tau), gran, r0, r1, C.byref(bufs), ws.data_ptr(),
                                  ws_bytes, _stream()), "plan")
        n_c, n_t, overflow, max_list = counts.tolist()
        if not overflow:
            break
        if task_cap >= max_tasks and leaf_cap >= L * L:
            raise RuntimeError("plan does not fit the 2^31 task limit")
        task_cap = min(max_tasks, max(2 * task_cap, int(1.25 * max_list) + 1024))
        leaf_cap = min(L * L, 4 * leaf_cap)
    _capacity_hint[hint_key] = (task_cap, leaf_cap)
    return MultiplyPlan(tau, granularity, depth, n_t, n_c, (c_keys, c_off, task_k, task_a, task_b, task_mask),
                        a, b, (r0, r1))
