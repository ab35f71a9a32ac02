"""Symbolic multiply phase on the device: ``build_plan``.

Drop-in for `pkg/src/spamm/symbolic.py:151-159`.  The plan lives in HBM as the step records the
numeric kernel consumes (``spamm_step`` in ``include/spamm_b200.h``: per 4x4 super-tile of
product leaves and per k, the 16 live-task bits and the operand leaf slots).  The reference's host
view -- ``plan.tasks`` as ``ProductTask`` objects in the reference's plan order, ``plan.stats``
and ``plan_dump`` -- is decoded from it on demand.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, morton
from .tree import QuadtreeMatrix, _lazy_tensor, _ptr, _stream


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


# capacities that worked last time for a (depth, leaves of A, leaves of B, tau, rows) shape
_capacity_hint: dict[tuple, tuple[int, int]] = {}

_POS_DI = np.array([((p >> 3) & 1) << 1 | ((p >> 1) & 1) for p in range(16)], np.int64)
_POS_DJ = np.array([((p >> 2) & 1) << 1 | (p & 1) for p in range(16)], np.int64)


class MultiplyPlan:
    """Surviving block products for one (A, B, tau) (`symbolic.py:49-56`), device resident.

    ``len(plan)`` is the task count; ``plan.tasks`` builds the reference's host list on demand.
    """

    def __init__(self, tau, depth, n_tasks, n_cleaves, n_steps, steps, c_keys, tile_off, tile_order, counts, a, b,
                 row_range):
        self.tau = float(tau)
        self.depth = depth
        # None = still on the device (asynchronous multiply): resolved on first use
        self._n_tasks = None if n_tasks is None else int(n_tasks)
        self._n_cleaves = None if n_cleaves is None else int(n_cleaves)
        self._n_steps = None if n_steps is None else int(n_steps)
        self._async = None            # set by the asynchronous multiply (numeric._AsyncProduct)
        self.steps, self.c_keys, self.tile_off, self.tile_order, self.counts = steps, c_keys, tile_off, tile_order, counts
        self._a, self._b = a, b
        self._tokens = (id(a), a._rev, id(b), b._rev)
        self.row_range = row_range
        self._tasks = None
        self._stats = None
        self._ikj = None

    def _resolve(self) -> None:
        """Read the counts back (one synchronisation); repeat the multiply if a buffer overflowed."""
        if self._n_tasks is not None:
            return
        cnt = self.counts.tolist()
        if cnt[2] and self._async is not None:
            self._async.on_overflow(cnt)      # replaces the buffers of this plan (and of C) in place
            cnt = self.counts.tolist()
        if cnt[2]:
            raise RuntimeError("plan buffers overflowed")
        if cnt[15]:
            raise RuntimeError("the numeric kernel gave up waiting for a chained segment (scheduling bug): results invalid")
        self._n_cleaves, self._n_steps = cnt[0], cnt[4]
        self._n_tasks = (cnt[6] & 0xFFFFFFFF) | ((cnt[7] & 0xFFFFFFFF) << 32)
        self._products4 = (cnt[8] & 0xFFFFFFFF) | ((cnt[9] & 0xFFFFFFFF) << 32)   # spamm_multiply only
        if self._async is not None:
            self._async.on_resolved(cnt)
            self._async = None

    def _count_leaves(self) -> int:
        return self.n_cleaves

    @property
    def n_tasks(self) -> int:
        self._resolve()
        return self._n_tasks

    @property
    def n_cleaves(self) -> int:
        self._resolve()
        return self._n_cleaves

    @property
    def n_steps(self) -> int:
        self._resolve()
        return self._n_steps

    def __len__(self) -> int:
        return self.n_tasks

    def buffers(self) -> _lib.PlanBuffers:
        leaf_cap = self._c_keys.shape[0]       # tile_order tensor: units, then the chain flags
        order = _ptr(self._tile_order)
        return _lib.PlanBuffers(_ptr(self._steps), _ptr(self._c_keys), _ptr(self._tile_off), order,
                                order + 4 * (leaf_cap + _lib.UNIT_EXTRA), self._steps.shape[0], leaf_cap,
                                _ptr(self._counts))

    # device arrays; after an asynchronous multiply they are regions of its arena (tree._Span)
    steps = _lazy_tensor("steps")
    c_keys = _lazy_tensor("c_keys")
    tile_off = _lazy_tensor("tile_off")
    tile_order = _lazy_tensor("tile_order")
    counts = _lazy_tensor("counts")

    # -- host views ---------------------------------------------------------------------------
    def step_records(self) -> np.ndarray:
        """(n_steps, 16) uint32 host copy of the step records."""
        return self.steps[: self.n_steps].cpu().numpy().view(np.uint32).reshape(-1, _lib.STEP_WORDS)

    def ikj(self) -> np.ndarray:
        """(T, 3) int64 array of task coordinates (i, k, j), sorted by product leaf key then k."""
        if self._ikj is not None:
            return self._ikj
        if self.n_tasks == 0:
            self._ikj = np.zeros((0, 3), np.int64)
            return self._ikj
        rec = self.step_records()
        sub_shift = min(2, self.depth)               # super-tiles are 4x4 leaves (2x2, 1x1 for tiny trees)
        kblock = rec[:, 0].astype(np.int64)
        live = rec[:, 8:12].astype(np.int64) & 0xFFFF                     # (steps, kk)
        ti, tj = morton.decode_array(rec[:, 3].astype(np.uint64))
        bits = (live[:, :, None] >> np.arange(16)[None, None, :]) & 1
        s_idx, kk, pos = np.nonzero(bits)
        i = (ti[s_idx].astype(np.int64) << sub_shift) + _POS_DI[pos]
        j = (tj[s_idx].astype(np.int64) << sub_shift) + _POS_DJ[pos]
        t = np.stack([i, (kblock[s_idx] << sub_shift) + kk, j], axis=1)
        ck = morton.encode_array(t[:, 0], t[:, 2])
        order = np.lexsort((t[:, 1], ck))
        self._ikj = t[order]
        assert self._ikj.shape[0] == self.n_tasks
        return self._ikj

    def pair_keys(self) -> tuple[np.ndarray, np.ndarray]:
        t = self.ikj()
        return morton.encode_array(t[:, 0], t[:, 1]), morton.encode_array(t[:, 1], t[:, 2])

    def masks(self) -> np.ndarray:
        """fine4 live bits per task of ``ikj()`` (bit r*16 + p*4 + q, `numeric.py:232-238`),
        evaluated on the host from the operands' sub-block norms; the device evaluates the same
        products inside the numeric kernel."""
        t = self.ikj()
        out = np.zeros(t.shape[0], np.uint64)
        if t.shape[0] == 0:
            return out
        ka, _, sa = self._a.packed_leaves()
        kb, _, sb = self._b.packed_leaves()
        an = sa[np.searchsorted(ka, morton.encode_array(t[:, 0], t[:, 1]))].astype(np.float64)
        bn = sb[np.searchsorted(kb, morton.encode_array(t[:, 1], t[:, 2]))].astype(np.float64)
        for r in range(4):
            live = an[:, :, r][:, :, None] * bn[:, r, :][:, None, :] >= self.tau
            for p in range(4):
                for q in range(4):
                    out |= live[:, p, q].astype(np.uint64) << np.uint64(r * 16 + p * 4 + q)
        return out

    def device_masks(self) -> np.ndarray:
        """The same bits as ``masks()``, but as evaluated ON THE DEVICE by the numeric kernel's own gate
        (planner classification + per-lane products, ``spamm_execute_gates``): one fine4 run into
        scratch product buffers that records which micro products it executed."""
        import ctypes as C
        import torch
        from .tree import _stream
        t = self.ikj()
        if t.shape[0] == 0:
            return np.zeros(0, np.uint64)
        a, b = self._a, self._b
        dev = a.device
        nC, ns = self.n_cleaves, self.n_steps
        va, vb = a.view(self.depth), b.view(self.depth, left=False)
        vals = torch.empty((nC, _lib.REC), dtype=torch.float32, device=dev)
        vals_t = torch.empty((nC, _lib.REC), dtype=torch.float32, device=dev)
        leaf_sq = torch.empty((nC,), dtype=torch.float64, device=dev)
        counters = torch.zeros((2,), dtype=torch.int64, device=dev)
        gates = torch.zeros((ns * 64,), dtype=torch.int64, device=dev)
        bufs = self.buffers()
        _lib.check(_lib.lib().spamm_execute_gates(C.byref(va), C.byref(vb), C.byref(bufs), ns, nC, float(self.tau),
                                                  vals.data_ptr(), vals_t.data_ptr(), leaf_sq.data_ptr(),
                                                  counters.data_ptr(), gates.data_ptr(), _stream()), "execute_gates")
        gh = gates.cpu().numpy().view(np.uint64).reshape(ns, 4, 16)
        rec = self.step_records()
        live = rec[:, 8:12].astype(np.int64) & 0xFFFF
        bits = (live[:, :, None] >> np.arange(16)[None, None, :]) & 1
        s_idx, kk, pos = np.nonzero(bits)                  # same enumeration as ikj()
        sub_shift = min(2, self.depth)
        ti, tj = morton.decode_array(rec[:, 3].astype(np.uint64))
        i = (ti[s_idx].astype(np.int64) << sub_shift) + _POS_DI[pos]
        j = (tj[s_idx].astype(np.int64) << sub_shift) + _POS_DJ[pos]
        k = (rec[:, 0].astype(np.int64)[s_idx] << sub_shift) + kk
        order = np.lexsort((k, morton.encode_array(i, j)))
        assert int(counters[0].item()) == int(sum(bin(int(x)).count("1") for x in gh[s_idx, kk, pos]))
        return gh[s_idx, kk, pos][order]

    def classification(self) -> tuple[np.ndarray, np.ndarray]:
        """(full, dead) flags per task of ``ikj()``: what the planner decided from the sub-norm ranges
        (spamm_step.live bits 16..31 and spamm_step.dead)."""
        rec = self.step_records()
        live = rec[:, 8:12].astype(np.int64) & 0xFFFF
        full = (rec[:, 8:12].astype(np.int64) >> 16) & 0xFFFF
        dead = np.stack([rec[:, 13] & 0xFFFF, rec[:, 13] >> 16, rec[:, 14] & 0xFFFF, rec[:, 14] >> 16], axis=1).astype(np.int64)
        bits = (live[:, :, None] >> np.arange(16)[None, None, :]) & 1
        s_idx, kk, pos = np.nonzero(bits)
        sub_shift = min(2, self.depth)
        ti, tj = morton.decode_array(rec[:, 3].astype(np.uint64))
        i = (ti[s_idx].astype(np.int64) << sub_shift) + _POS_DI[pos]
        j = (tj[s_idx].astype(np.int64) << sub_shift) + _POS_DJ[pos]
        k = (rec[:, 0].astype(np.int64)[s_idx] << sub_shift) + kk
        order = np.lexsort((k, morton.encode_array(i, j)))
        f = ((full[s_idx, kk] >> pos) & 1).astype(bool)[order]
        d = ((dead[s_idx, kk] >> pos) & 1).astype(bool)[order]
        return f, d

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


def build_plan(a: QuadtreeMatrix, b: QuadtreeMatrix, tau: float,
               row_range: tuple[int, int] | None = None) -> MultiplyPlan:
    """Full symbolic pipeline for C = A B on the device (`symbolic.py:151-159`).

    ``row_range`` restricts the plan to product leaf rows [r0, r1): the row-block sharding
    across GPUs.
    """
    if a.n_b != b.n_b:
        raise ValueError(f"block sizes differ: {a.n_b} vs {b.n_b}")
    if a.n != b.m:
        raise ValueError(f"inner dimensions differ: {a.m}x{a.n} times {b.m}x{b.n}")
    _check_tau(tau)
    from .tree import as_device_tree
    a, b = as_device_tree(a), as_device_tree(b)      # trees of the reference package are copied once per revision
    a._require_16()
    lib = _lib.lib()
    depth = max(a.depth, b.depth)
    L = 1 << depth
    r0, r1 = (0, L) if row_range is None else (int(row_range[0]), int(row_range[1]))
    dev = a.device
    if a.nleaf == 0 or b.nleaf == 0:
        z = torch.zeros((1, _lib.STEP_WORDS), dtype=torch.int32, device=dev)
        e = torch.zeros((_lib.PLAN_COUNTS,), dtype=torch.int32, device=dev)
        return MultiplyPlan(tau, depth, 0, 0, 0, z, e, e, e, e, a, b, (r0, r1))
    va, vb = a.view(depth), b.view(depth, left=False)
    hint_key, (step_cap, leaf_cap) = plan_capacity(a, b, tau, depth, r0, r1)
    while True:
        pb = PlanAlloc(dev, depth, step_cap, leaf_cap)
        _lib.check(lib.spamm_plan(C.byref(va), C.byref(vb), float(tau), r0, r1, C.byref(pb.struct), pb.ws.data_ptr(),
                                  pb.ws_bytes, _stream()), "plan")
        cnt = pb.counts.tolist()
        n_c, overflow, n_steps = cnt[0], cnt[2], cnt[4]
        n_t = (cnt[6] & 0xFFFFFFFF) | ((cnt[7] & 0xFFFFFFFF) << 32)
        if not overflow:
            break
        step_cap, leaf_cap = grow_capacity(depth, step_cap, leaf_cap, cnt)
    remember_capacity(hint_key, max(n_steps, cnt[3]), n_c, depth)
    return MultiplyPlan(tau, depth, n_t, n_c, n_steps, pb.steps, pb.c_keys, pb.tile_off, pb.tile_order, pb.counts,
                        a, b, (r0, r1))


class PlanAlloc:
    """Device buffers of one plan (``spamm_plan_buffers``) plus the planner's workspace."""

    def __init__(self, dev, depth: int, step_cap: int, leaf_cap: int):
        tl = max(depth - 2, 0)
        if tl <= 7:     # room for every super-tile node: lets the planner start densely at that level
            leaf_cap = max(leaf_cap, 1 << (2 * tl))
        self.step_cap, self.leaf_cap = step_cap, leaf_cap
        self.steps = torch.empty((step_cap, _lib.STEP_WORDS), dtype=torch.int32, device=dev)
        self.c_keys = torch.empty((leaf_cap,), dtype=torch.int32, device=dev)
        self.tile_off = torch.empty((leaf_cap + 1,), dtype=torch.int32, device=dev)
        self.tile_order = torch.empty((2 * leaf_cap + _lib.UNIT_EXTRA,), dtype=torch.int32, device=dev)
        self.counts = torch.empty((_lib.PLAN_COUNTS,), dtype=torch.int32, device=dev)
        self.ws_bytes = _lib.lib().spamm_plan_workspace_bytes(depth, step_cap, leaf_cap)
        self.ws = torch.empty((self.ws_bytes,), dtype=torch.uint8, device=dev)
        self.struct = _lib.PlanBuffers(self.steps.data_ptr(), self.c_keys.data_ptr(), self.tile_off.data_ptr(),
                                       self.tile_order.data_ptr(),
                                       self.tile_order.data_ptr() + 4 * (leaf_cap + _lib.UNIT_EXTRA), step_cap, leaf_cap,
                                       self.counts.data_ptr())


def plan_capacity(a: QuadtreeMatrix, b: QuadtreeMatrix, tau: float, depth: int, r0: int, r1: int):
    """(hint key, (step capacity, leaf capacity)): what worked last time for this shape, else a guess."""
    L = 1 << depth
    na, nb = a._leaf_bound(), b._leaf_bound()
    key = (depth, na, nb, float(tau), r0, r1)
    guess = (max(4096, na + nb), min(L * L, max(1024, 2 * (na + nb))))
    return key, _capacity_hint.get(key, guess)


def grow_capacity(depth: int, step_cap: int, leaf_cap: int, cnt) -> tuple[int, int]:
    L = 1 << depth
    max_steps = min((1 << 31) - 128, max(1, (L * L * L) // 16 + L * L))
    if step_cap >= max_steps and leaf_cap >= L * L:
        raise RuntimeError("plan does not fit the 2^31 step limit")
    step_cap = min(max_steps, max(2 * step_cap, int(1.25 * max(cnt[3], cnt[4])) + 1024))
    leaf_cap = min(L * L, max(4 * leaf_cap, int(1.25 * cnt[0]) + 1024))
    return step_cap, leaf_cap


def remember_capacity(key, n_steps: int, n_cleaves: int, depth: int) -> None:
    """Next time, size the buffers just above what this shape needed."""
    L = 1 << depth
    # (the step capacity also bounds the candidate lists of the coarser levels; the start level
    # alone can hold 1024 nodes x 32 candidates; an overflow there just repeats the plan)
    _capacity_hint[key] = (max(8192, int(1.1 * n_steps) + 256), min(L * L, max(320, int(1.1 * n_cleaves) + 64)))
