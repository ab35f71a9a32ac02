"""Numeric multiply phase on the device: ``execute_plan`` and ``multiply``.

Drop-in for `pkg/src/spamm/numeric.py` (``MultiplyConfig`` :32-47, ``ExecCounters`` :50-72,
``execute_plan`` :138-181, ``multiply`` :302-313): same names, arguments, return values and
ValueError conditions.  Work is counted in 4x4x4 micro products exactly as the reference does.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .symbolic import MultiplyPlan, build_plan
from .tree import QuadtreeMatrix, _stream

GRANULARITIES = ("fine4", "coarse16")

# Modeled flops of one 4x4x4 micro product (`numeric.py:28-29`).
MICRO_FLOPS = 128


@dataclass
class MultiplyConfig:
    tau: float = 0.0
    granularity: str = "fine4"
    alpha: float = 1.0
    beta: float = 0.0
    # B200 extension: True rounds every product and sum separately (bit-identical to the
    # reference); False (default) uses fused multiply-add, within the 1e-5 budget.
    exact: bool = False

    def __post_init__(self):
        if self.granularity not in GRANULARITIES:
            raise ValueError(f"granularity must be one of {GRANULARITIES}, got {self.granularity!r}")
        if np.isnan(self.tau) or self.tau < 0:
            raise ValueError(f"tau must be nonnegative, got {self.tau}")
        if not (np.isfinite(self.alpha) and np.isfinite(self.beta)):
            raise ValueError("alpha and beta must be finite")


class ExecCounters:
    """Work counters of one numeric pass (`numeric.py:50-72`).

    ``products4`` is read back from the device on first access, so a caller that only wants C
    does not pay a synchronisation."""

    def __init__(self, products4=0, skipped4=0, seconds=0.0, _dev=None, _total=0, _fine=True, _events=None, _plan=None):
        self._products4, self._skipped4, self.seconds = products4, skipped4, seconds
        self._dev, self._total, self._fine, self._events, self._plan = _dev, _total, _fine, _events, _plan

    def _fetch(self):
        if self._plan is not None:                 # asynchronous multiply: the task count arrives with the plan
            plan, self._plan = self._plan, None
            self._total = 64 * plan.n_tasks        # (resolving the plan may swap self._dev after an overflow)
            if not self._fine:
                self._products4, self._dev = self._total, None
        if self._dev is not None:
            self._products4 = int(self._dev[0].item())
            self._skipped4 = self._total - self._products4 if self._fine else 0
            self._dev = None
        if self._events is not None:
            e0, e1 = self._events
            e1.synchronize()
            self.seconds = e0.elapsed_time(e1) * 1e-3
            self._events = None

    @property
    def products4(self) -> int:
        self._fetch()
        return self._products4

    @property
    def skipped4(self) -> int:
        self._fetch()
        return self._skipped4

    @property
    def complexity(self) -> int:
        return self.products4

    @property
    def flops(self) -> int:
        return self.products4 * MICRO_FLOPS

    def merge(self, other: "ExecCounters") -> "ExecCounters":
        return ExecCounters(self.products4 + other.products4, self.skipped4 + other.skipped4,
                            self.seconds + other.seconds)

    def __repr__(self):
        return f"ExecCounters(products4={self.products4}, skipped4={self.skipped4}, seconds={self.seconds:.6g})"


def _check_plan_handles(plan: MultiplyPlan, a: QuadtreeMatrix, b: QuadtreeMatrix) -> None:
    """The plan addresses leaves by packed slot; it is only valid for the tree revisions it was
    built from (the reference checks the same thing by key lookup, `numeric.py:128-135`)."""
    if plan.n_tasks == 0:
        return
    if plan._tokens != (id(a), a._rev, id(b), b._rev):
        for side, q, (ka, kb) in (("A", a, (0, 1)), ("B", b, (1, 2))):
            have = set(q.leaf_keys().tolist()) if q.nleaf else set()
            if not have:
                raise ValueError(f"plan references leaves but {side} has none (stale handles)")
        raise ValueError("plan was built for other operand revisions (stale handles); rebuild it with build_plan")


def execute_plan(plan: MultiplyPlan, a: QuadtreeMatrix, b: QuadtreeMatrix, c: QuadtreeMatrix | None,
                 cfg: MultiplyConfig) -> tuple[QuadtreeMatrix, ExecCounters]:
    """Run the numeric phase: C = alpha * (planned products) + beta * C (`numeric.py:138-181`)."""
    if plan.tau != cfg.tau:
        raise ValueError(f"plan built for tau={plan.tau}, config has tau={cfg.tau}")
    if a.n_b != b.n_b:
        raise ValueError(f"block sizes differ: {a.n_b} vs {b.n_b}")
    if a.n != b.m:
        raise ValueError(f"inner dimensions differ: {a.m}x{a.n} times {b.m}x{b.n}")
    nb = a.n_b
    if nb % 4:
        raise ValueError(f"numeric phase needs 4 | n_b, got n_b = {nb}")
    a._require_16()
    if c is None:
        c = QuadtreeMatrix(a.m, b.n, nb, device=a.device)
    elif (c.m, c.n) != (a.m, b.n) or c.n_b != nb:
        raise ValueError(f"accumulator is {c.m}x{c.n} (n_b={c.n_b}), product needs {a.m}x{b.n} (n_b={nb})")
    _check_plan_handles(plan, a, b)
    lib = _lib.lib()
    st = _stream()
    dev = a.device
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    T, nC = plan.n_tasks, plan.n_cleaves
    run = T > 0 and cfg.alpha != 0
    counters_dev = torch.zeros((2,), dtype=torch.int64, device=dev)
    fine = cfg.granularity == "fine4"
    keep_old = cfg.beta != 0 and c.nleaf > 0
    prod = None
    if run:
        va, vb = a.view(plan.depth), b.view(plan.depth)
        vals = torch.empty((nC, _lib.REC), dtype=torch.float32, device=dev)
        vals_t = torch.empty((nC, _lib.REC), dtype=torch.float32, device=dev)
        leaf_sq = torch.empty((nC,), dtype=torch.float64, device=dev)
        bufs = plan.buffers()
        # with an accumulator to merge, the kernel leaves alpha to the compose step
        alpha_k = 1.0 if keep_old else float(np.float32(cfg.alpha))
        gran = _lib.FINE4 if fine else _lib.COARSE16
        _lib.check(lib.spamm_execute(C.byref(va), C.byref(vb), C.byref(bufs), plan.n_steps, nC, float(cfg.tau), alpha_k,
                                     gran, int(cfg.exact), vals.data_ptr(), vals_t.data_ptr(), leaf_sq.data_ptr(),
                                     counters_dev.data_ptr(), st), "execute")
        prod = (plan.c_keys[:nC], vals, vals_t, leaf_sq)
    # _compose (`numeric.py:268-284`)
    if not keep_old:
        if prod is None:
            if cfg.beta == 0 or c.nleaf == 0:
                c.clear()
        else:
            keys, vals, vals_t, leaf_sq = prod
            c._adopt_packed(keys.clone(), vals, vals_t, leaf_sq, nC)
    else:
        _compose_with_accumulator(c, prod, cfg)
    e1.record()
    total = 64 * T if run else 0
    if not run:
        counters = ExecCounters(0, 0, 0.0, _events=(e0, e1))
    elif fine:
        counters = ExecCounters(_dev=counters_dev, _total=total, _fine=True, _events=(e0, e1))
    else:
        counters = ExecCounters(total, 0, 0.0, _events=(e0, e1))
    return c, counters


def _compose_with_accumulator(c: QuadtreeMatrix, prod, cfg: MultiplyConfig) -> None:
    """beta != 0 and C has leaves: leaf-set union, alpha/beta combine, norms rebuilt."""
    lib = _lib.lib()
    st = _stream()
    dev = c.device
    depth, L = c.depth, 1 << c.depth
    cells = L * L
    g = c.grids()
    if prod is None:
        nprod, pk, pv = 0, None, None
    else:
        pk, pv = prod[0], prod[1]
        nprod = int(pk.numel())
    scratch = torch.empty((cells,), dtype=torch.int32, device=dev)
    cap = min(cells, c.nleaf + nprod)
    out_keys = torch.empty((cap,), dtype=torch.int32, device=dev)
    idx_old = torch.empty((cap,), dtype=torch.int32, device=dev)
    idx_prod = torch.empty((cap,), dtype=torch.int32, device=dev)
    nout_dev = torch.empty((1,), dtype=torch.int32, device=dev)
    ws_bytes = lib.spamm_scan_workspace_bytes(cells)
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=dev)
    _lib.check(lib.spamm_union_leaves(g.slot.data_ptr(), None if pk is None else pk.data_ptr(), nprod, depth,
                                      scratch.data_ptr(), out_keys.data_ptr(), idx_old.data_ptr(), idx_prod.data_ptr(),
                                      nout_dev.data_ptr(), ws.data_ptr(), ws_bytes, st), "union_leaves")
    nout = int(nout_dev.item())
    out_vals = torch.empty((nout, _lib.REC), dtype=torch.float32, device=dev)
    _lib.check(lib.spamm_compose(None if pv is None else pv.data_ptr(), c.values.data_ptr(), idx_prod.data_ptr(),
                                 idx_old.data_ptr(), nout, float(np.float32(cfg.alpha)), float(np.float32(cfg.beta)),
                                 int(cfg.alpha == 1), int(cfg.beta == 1), out_vals.data_ptr(), st), "compose")
    c._set_packed_values(out_keys[:nout].clone(), out_vals)


def multiply(a: QuadtreeMatrix, b: QuadtreeMatrix, cfg: MultiplyConfig | None = None,
             c: QuadtreeMatrix | None = None) -> tuple[QuadtreeMatrix, MultiplyPlan, ExecCounters]:
    """Symbolic plus numeric phases in one call (`numeric.py:302-313`).

    When no accumulator content has to be merged (``beta == 0`` or ``c`` empty) the whole multiply
    -- plan, leaf products, norms of C -- is enqueued on the current stream without a host
    synchronisation; the task and leaf counts are read back when first asked for."""
    if cfg is None:
        cfg = MultiplyConfig()
    merge_old = c is not None and cfg.beta != 0 and c._leaf_bound() > 0
    if not merge_old and cfg.alpha != 0 and a._leaf_bound() > 0 and b._leaf_bound() > 0:
        from .symbolic import _capacity_hint, plan_capacity
        depth = max(a.depth, b.depth)
        key, _ = plan_capacity(a, b, cfg.tau, depth, 0, 1 << depth)
        if key in _capacity_hint:        # sizes known from an earlier product of this shape
            return multiply_async(a, b, cfg, c)
    plan = build_plan(a, b, cfg.tau)
    out, counters = execute_plan(plan, a, b, c, cfg)
    return out, plan, counters


def multiply_async(a: QuadtreeMatrix, b: QuadtreeMatrix, cfg: MultiplyConfig, c: QuadtreeMatrix | None = None,
                   row_range: tuple[int, int] | None = None) -> tuple[QuadtreeMatrix, MultiplyPlan, ExecCounters]:
    """C = alpha A B through ``spamm_multiply``: one C call, no host synchronisation."""
    from .symbolic import PlanAlloc, grow_capacity, plan_capacity, remember_capacity
    from .tree import _Grids

    if a.n_b != b.n_b:
        raise ValueError(f"block sizes differ: {a.n_b} vs {b.n_b}")
    if a.n != b.m:
        raise ValueError(f"inner dimensions differ: {a.m}x{a.n} times {b.m}x{b.n}")
    a._require_16()
    if c is None:
        c = QuadtreeMatrix(a.m, b.n, a.n_b, device=a.device)
    elif (c.m, c.n) != (a.m, b.n) or c.n_b != a.n_b:
        raise ValueError(f"accumulator is {c.m}x{c.n} (n_b={c.n_b}), product needs {a.m}x{b.n} (n_b={a.n_b})")
    lib = _lib.lib()
    dev = a.device
    depth = max(a.depth, b.depth)
    L = 1 << depth
    r0, r1 = (0, L) if row_range is None else (int(row_range[0]), int(row_range[1]))
    fine = cfg.granularity == "fine4"
    gran = _lib.FINE4 if fine else _lib.COARSE16
    alpha32 = float(np.float32(cfg.alpha))
    hint_key, caps = plan_capacity(a, b, cfg.tau, depth, r0, r1)
    cd, cells, total = c.depth, 1 << (2 * c.depth), _lib.level_total(c.depth)

    def launch(step_cap: int, leaf_cap: int):
        va, vb = a.view(depth), b.view(depth)
        pb = PlanAlloc(dev, depth, step_cap, leaf_cap)
        vals = torch.empty((leaf_cap, _lib.REC), dtype=torch.float32, device=dev)
        vals_t = torch.empty((leaf_cap, _lib.REC), dtype=torch.float32, device=dev)
        leaf_sq = torch.empty((leaf_cap,), dtype=torch.float64, device=dev)
        grids = _Grids(cd, torch.empty((cells,), dtype=torch.int32, device=dev),
                       torch.empty((cells,), dtype=torch.int32, device=dev),
                       torch.empty((total,), dtype=torch.float32, device=dev),
                       torch.empty((total,), dtype=torch.float32, device=dev))
        sq_grid = torch.empty((cells,), dtype=torch.float64, device=dev)
        sq_levels = torch.empty((total,), dtype=torch.float64, device=dev)
        counters_dev = torch.zeros((2,), dtype=torch.int64, device=dev)
        prod = _lib.ProductBuffers(vals.data_ptr(), vals_t.data_ptr(), leaf_sq.data_ptr(), grids.slot.data_ptr(),
                                   grids.slot_t.data_ptr(), grids.norm.data_ptr(), grids.norm_t.data_ptr(),
                                   sq_grid.data_ptr(), sq_levels.data_ptr(), cd)
        _lib.check(lib.spamm_multiply(C.byref(va), C.byref(vb), float(cfg.tau), gran, int(cfg.exact), alpha32, r0, r1,
                                      C.byref(pb.struct), pb.ws.data_ptr(), pb.ws_bytes, C.byref(prod),
                                      counters_dev.data_ptr(), _stream()), "multiply")
        return pb, vals, vals_t, leaf_sq, grids, counters_dev

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pb, vals, vals_t, leaf_sq, grids, counters_dev = launch(*caps)
    e1.record()
    plan = MultiplyPlan(cfg.tau, depth, None, None, None, pb.steps, pb.c_keys, pb.tile_off, pb.tile_order, pb.counts,
                        a, b, (r0, r1))
    counters = ExecCounters(_dev=counters_dev, _fine=fine, _events=(e0, e1), _plan=plan)
    c._adopt_product(pb.c_keys, vals, vals_t, leaf_sq, grids, plan._count_leaves)
    plan._tokens = (id(a), a._rev, id(b), b._rev)
    plan._async = _AsyncProduct(launch, depth, hint_key, (pb.step_cap, pb.leaf_cap), plan, c, counters)
    return c, plan, counters


class _AsyncProduct:
    """What a lazily resolved plan needs to repeat its multiply after a buffer overflow.  Holds the
    plan, the product tree and the counters weakly, so nothing here keeps device memory alive."""

    def __init__(self, launch, depth, hint_key, caps, plan, c, counters):
        import weakref
        self.launch, self.depth, self.hint_key, self.caps = launch, depth, hint_key, caps
        self.plan, self.c, self.counters = weakref.ref(plan), weakref.ref(c), weakref.ref(counters)

    def on_overflow(self, cnt) -> None:
        """A capacity was too small: repeat, synchronously, until the buffers fit."""
        from .symbolic import grow_capacity
        step_cap, leaf_cap = self.caps
        while True:
            step_cap, leaf_cap = grow_capacity(self.depth, step_cap, leaf_cap, cnt)
            npb, nvals, nvals_t, nleaf_sq, ngrids, ncounters = self.launch(step_cap, leaf_cap)
            cnt = npb.counts.tolist()
            if not cnt[2]:
                break
        plan, c, counters = self.plan(), self.c(), self.counters()
        if plan is not None:
            plan.steps, plan.c_keys, plan.tile_off, plan.tile_order, plan.counts = (
                npb.steps, npb.c_keys, npb.tile_off, npb.tile_order, npb.counts)
        if c is not None and plan is not None:
            rev = c._rev
            c._adopt_product(npb.c_keys, nvals, nvals_t, nleaf_sq, ngrids, plan._count_leaves)
            c._rev = rev
        if counters is not None:
            counters._dev = ncounters

    def on_resolved(self, cnt) -> None:
        from .symbolic import remember_capacity
        remember_capacity(self.hint_key, max(cnt[4], cnt[3]), cnt[0], self.depth)
