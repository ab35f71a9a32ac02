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
from .tree import QuadtreeMatrix, _Span, _stream, as_device_tree, write_back

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
        if self._plan is not None:                 # asynchronous multiply: everything arrives with the plan counts
            plan, self._plan = self._plan, None
            self._total = 64 * plan.n_tasks
            self._products4 = plan._products4 if self._fine else self._total
            self._skipped4 = self._total - self._products4 if self._fine else 0
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
        for side, q in (("A", a), ("B", b)):
            if q.nleaf == 0:
                raise ValueError(f"plan references leaves but {side} has none (stale handles)")
        raise ValueError("plan was built for other operand revisions (stale handles); rebuild it with build_plan")


def execute_plan(plan: MultiplyPlan, a: QuadtreeMatrix, b: QuadtreeMatrix, c: QuadtreeMatrix | None,
                 cfg: MultiplyConfig) -> tuple[QuadtreeMatrix, ExecCounters]:
    """Run the numeric phase: C = alpha * (planned products) + beta * C (`numeric.py:138-181`).
    Operands and accumulator may be trees of the reference package (copied to the device once per
    revision; a reference accumulator gets the result written back in place)."""
    if not isinstance(c, (QuadtreeMatrix, type(None))):
        dc, counters = execute_plan(plan, a, b, as_device_tree(c), cfg)
        return write_back(c, dc), counters
    a, b = as_device_tree(a), as_device_tree(b)
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
        va, vb = a.view(plan.depth), b.view(plan.depth, left=False)
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
    if not isinstance(c, (QuadtreeMatrix, type(None))):      # a reference tree as accumulator: mutate it in place
        dc, plan, counters = multiply(a, b, cfg, as_device_tree(c))
        return write_back(c, dc), plan, counters
    a, b = as_device_tree(a), as_device_tree(b)
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


_planner_ws: dict = {}


def _planner_workspace(dev, nbytes: int, stream: int | None = None) -> torch.Tensor:
    """The planner's workspace, one per (device, stream): the library needs it all zero when a
    multiply is enqueued and leaves it all zero, so it is cleared only when it is (re)allocated."""
    key = (dev.index, _stream() if stream is None else stream)
    ws = _planner_ws.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros((max(nbytes, 1 << 20),), dtype=torch.uint8, device=dev)
        _planner_ws[key] = ws
    return ws


def multiply_async(a: QuadtreeMatrix, b: QuadtreeMatrix, cfg: MultiplyConfig, c: QuadtreeMatrix | None = None,
                   row_range: tuple[int, int] | None = None, host=None) -> tuple[QuadtreeMatrix, MultiplyPlan, ExecCounters]:
    """C = alpha A B through ``spamm_multiply``: one C call, no host synchronisation.
    ``host``: a ``_lib.HostOperands`` when the operands' leaf values are still in host memory (hosttree.py)."""
    from .symbolic import plan_capacity
    from .tree import _Grids

    if a.n_b != b.n_b:
        raise ValueError(f"block sizes differ: {a.n_b} vs {b.n_b}")
    if a.n != b.m:
        raise ValueError(f"inner dimensions differ: {a.m}x{a.n} times {b.m}x{b.n}")
    a._require_16()
    if cfg.beta != 0 and c is not None and c._leaf_bound() > 0:
        raise ValueError("multiply_async computes C = alpha A B; use multiply() to merge an accumulator (beta != 0)")
    if c is None:
        c = QuadtreeMatrix(a.m, b.n, a.n_b, device=a.device)
    elif (c.m, c.n) != (a.m, b.n) or c.n_b != a.n_b:
        raise ValueError(f"accumulator is {c.m}x{c.n} (n_b={c.n_b}), product needs {a.m}x{b.n} (n_b={a.n_b})")
    # An operand that is itself the product of a multiply still in flight: its buffers are only final
    # once its plan is known not to have overflowed (an overflowed multiply computes nothing and is
    # repeated into new buffers).  Resolve it first -- one read-back -- instead of planning against
    # storage that may be replaced.
    for q in (a, b):
        if q._nleaf is None:
            q.nleaf
    if cfg.alpha == 0 or a.nleaf == 0 or b.nleaf == 0:
        # the reference skips the product pass (numeric.py:173-177): C comes out empty
        c.clear()
        return c, build_plan(a, b, cfg.tau, row_range), ExecCounters(0, 0, 0.0)
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

    tl = max(depth - 2, 0)
    i32t, f32t, f64t = torch.int32, torch.float32, torch.float64

    def launch(step_cap: int, leaf_cap: int):
        """One allocation, one C call; returns the arena and its layout."""
        if tl <= 7:     # room for every super-tile node: lets the planner start densely at that level
            leaf_cap = max(leaf_cap, 1 << (2 * tl))
        lay = _arena_layout(depth, cd, step_cap, leaf_cap)
        arena = torch.empty((lay.total,), dtype=torch.uint8, device=dev)
        st = _stream()
        ws = _planner_workspace(dev, lay.plan_ws_bytes, st)
        va, vb = a.view(depth), b.view(depth, left=False)
        try:
            if host is None:
                _lib.check(lib.spamm_multiply_arena(C.byref(va), C.byref(vb), float(cfg.tau), gran, int(cfg.exact), alpha32,
                                                    r0, r1, cd, step_cap, leaf_cap, arena.data_ptr(), lay.total,
                                                    ws.data_ptr(), ws.numel(), st), "multiply")
            else:
                _lib.check(lib.spamm_multiply_arena_host(C.byref(va), C.byref(vb), float(cfg.tau), gran, int(cfg.exact),
                                                         alpha32, r0, r1, cd, step_cap, leaf_cap, arena.data_ptr(), lay.total,
                                                         ws.data_ptr(), ws.numel(), C.byref(host), st), "multiply_host")
        except Exception:
            _planner_ws.clear()         # a failed enqueue may leave the workspace dirty: start from a fresh one
            raise
        return arena, lay, step_cap, leaf_cap

    def bind(plan: MultiplyPlan, c: QuadtreeMatrix, arena, lay, step_cap: int, leaf_cap: int) -> None:
        """Point the plan and the product tree at their regions of the arena (views made on demand)."""
        plan.steps = _Span(arena, lay.steps, (step_cap, _lib.STEP_WORDS), i32t)
        plan.c_keys = _Span(arena, lay.c_keys, (leaf_cap,), i32t)
        plan.tile_off = _Span(arena, lay.tile_off, (leaf_cap + 1,), i32t)
        # units followed by the chain flags, as in symbolic.PlanAlloc (the arena keeps them adjacent)
        plan.tile_order = _Span(arena, lay.tile_order, (2 * leaf_cap + _lib.UNIT_EXTRA,), i32t)
        plan.counts = _Span(arena, lay.counts, (_lib.PLAN_COUNTS,), i32t)
        grids = _Grids(cd, _Span(arena, lay.slot, (cells,), i32t), _Span(arena, lay.slot_t, (cells,), i32t),
                       _Span(arena, lay.norm, (total,), f32t), _Span(arena, lay.norm_t, (total,), f32t))
        c._adopt_product(plan._c_keys, _Span(arena, lay.values, (leaf_cap, _lib.REC), f32t),
                         _Span(arena, lay.values_t, (leaf_cap, _lib.REC), f32t),
                         _Span(arena, lay.leaf_sq, (leaf_cap,), f64t), grids, plan._count_leaves)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    arena, lay, step_cap, leaf_cap = launch(*caps)
    e1.record()
    plan = MultiplyPlan(cfg.tau, depth, None, None, None, None, None, None, None, None, a, b, (r0, r1))
    bind(plan, c, arena, lay, step_cap, leaf_cap)
    counters = ExecCounters(_fine=fine, _events=(e0, e1), _plan=plan)
    plan._async = _AsyncProduct(launch, bind, depth, hint_key, (step_cap, leaf_cap), plan, c)
    return c, plan, counters


_layouts: dict[tuple, "_lib.ArenaLayout"] = {}


def _arena_layout(depth: int, c_depth: int, step_cap: int, leaf_cap: int):
    key = (depth, c_depth, step_cap, leaf_cap)
    lay = _layouts.get(key)
    if lay is None:
        lay = _lib.ArenaLayout()
        _lib.check(_lib.lib().spamm_multiply_arena_layout(depth, c_depth, step_cap, leaf_cap, C.byref(lay)), "layout")
        _layouts[key] = lay
    return lay


class _AsyncProduct:
    """What a lazily resolved plan needs to repeat its multiply after a buffer overflow.  Holds the
    plan, the product tree and the counters weakly, so nothing here keeps device memory alive."""

    def __init__(self, launch, bind, depth, hint_key, caps, plan, c):
        import weakref
        self.launch, self.bind, self.depth, self.hint_key, self.caps = launch, bind, depth, hint_key, caps
        self.plan, self.c = weakref.ref(plan), weakref.ref(c)

    def on_overflow(self, cnt) -> None:
        """A capacity was too small: repeat, synchronously, until the buffers fit."""
        from .symbolic import grow_capacity
        step_cap, leaf_cap = self.caps
        while True:
            step_cap, leaf_cap = grow_capacity(self.depth, step_cap, leaf_cap, cnt)
            arena, lay, step_cap, leaf_cap = self.launch(step_cap, leaf_cap)
            cnt = _Span(arena, lay.counts, (_lib.PLAN_COUNTS,), torch.int32).tensor().tolist()
            if not cnt[2]:
                break
        plan, c = self.plan(), self.c()
        if plan is not None:
            target = c if c is not None else QuadtreeMatrix(plan._a.m, plan._b.n, 16, device=plan._a.device)
            # the product moved to new buffers: its revision advances, so a plan built from the
            # old (empty) storage is recognised as stale
            self.bind(plan, target, arena, lay, step_cap, leaf_cap)

    def on_resolved(self, cnt) -> None:
        from .symbolic import remember_capacity
        remember_capacity(self.hint_key, max(cnt[4], cnt[3]), cnt[0], self.depth)
