"""Products of trees that live in host memory: only the leaves a product touches cross PCIe.

The reference's trees are host objects (`pkg/src/spamm/core.py:146-405`).  A drop-in that first copies a
whole operand to the GPU moves every stored leaf -- 50 MB for BASELINE config 2 -- although the product
at tau = 1e-8 reads 28 % of them.  ``HostTree`` keeps the leaf VALUES in pinned host memory and puts only
what the symbolic phase needs on the device (keys, leaf norms, sub-block norms: 76 bytes per leaf);
``multiply_host`` then plans, marks the leaves that occur in a surviving task, lets the GPU fetch exactly
those 1 KB blocks from host memory (`spamm_mark_touched`, `spamm_gather_blocks`) and runs the numeric
phase.  The result equals ``multiply`` on fully resident trees: task set, gates and arithmetic are the same.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .numeric import ExecCounters, MultiplyConfig, execute_plan
from .symbolic import MultiplyPlan, build_plan
from .tree import DEFAULT_BLOCK, QuadtreeMatrix, _stream


def _pinned(x, dtype) -> torch.Tensor:
    t = torch.as_tensor(x)
    if t.dtype != dtype:
        t = t.to(dtype)
    t = t.contiguous()
    return t if t.is_pinned() else t.pin_memory()


class HostTree:
    """A quadtree matrix whose leaf values stay on the host: the arrays of the reference's
    ``packed_leaves()`` (`core.py:387-405`: ascending Morton keys, 16x16 blocks, 4x4 sub-block norms) plus
    the leaf norms (``node.norm`` of `core.py:176-182`), all kept as pinned tensors."""

    def __init__(self, m: int, n: int, keys, blocks, subnorms, norms):
        self.m, self.n, self.n_b = int(m), int(n), DEFAULT_BLOCK
        self.keys = _pinned(np.asarray(keys).astype(np.int64).astype(np.int32) if not isinstance(keys, torch.Tensor) else keys, torch.int32)
        nl = int(self.keys.numel())
        self.blocks = _pinned(blocks, torch.float32).reshape(nl, 256)
        self.subnorms = _pinned(subnorms, torch.float32).reshape(nl, 16)
        self.norms = _pinned(norms, torch.float32).reshape(nl)
        self.nleaf = nl

    @classmethod
    def from_reference(cls, tree) -> "HostTree":
        """From a tree of the reference package (anything with ``m, n, packed_leaves(), leaf_items()``)."""
        keys, vals, subs = tree.packed_leaves()
        norms = np.fromiter((nd.norm for _, nd in tree.leaf_items()), np.float32, int(keys.shape[0]))
        return cls(tree.m, tree.n, keys, vals, subs, norms)

    @classmethod
    def from_device(cls, q: QuadtreeMatrix) -> "HostTree":
        """Host copy of a device tree (set-up, e.g. for benchmarks)."""
        keys, vals, subs = q.packed_leaves()
        from . import morton
        ii, jj = morton.decode_array(keys.astype(np.uint64))
        norms = q.level_norms(q.depth)[ii, jj].astype(np.float32)
        return cls(q.m, q.n, keys, vals, subs, norms)

    def skeleton(self, device=None) -> QuadtreeMatrix:
        """The device tree without leaf values: keys, norm pyramid, slot grids and the sub-norm tails of the
        leaf records (what the symbolic phase and the fine4 classification read).  The leaf square sums are
        float64(norm)^2, as for ``QuadtreeMatrix.from_reference``."""
        q = QuadtreeMatrix(self.m, self.n, DEFAULT_BLOCK, device)
        nl = self.nleaf
        if nl == 0:
            return q
        dev = q.device
        keys = self.keys.to(dev, non_blocking=True)
        subs = self.subnorms.to(dev, non_blocking=True)
        leaf_sq = self.norms.to(dev, non_blocking=True).double().square()
        values = torch.empty((nl, _lib.REC), dtype=torch.float32, device=dev)
        values_t = torch.empty((nl, _lib.REC), dtype=torch.float32, device=dev)
        _lib.check(_lib.lib().spamm_subnorm_tails(subs.data_ptr(), nl, values.data_ptr(), values_t.data_ptr(), _stream()),
                   "subnorm_tails")
        q._adopt_packed(keys, values, values_t, leaf_sq, nl)
        return q

    def skeleton_bytes(self) -> int:
        return self.nleaf * (4 + 4 + 64)


def multiply_host(a: HostTree, b: HostTree | None, cfg: MultiplyConfig | None = None):
    """C = alpha A B for operands in host memory (``b is None``: B is A).  Returns ``(c, plan, counters,
    fetched)``: the product tree on the device, its plan and counters as from ``multiply``, and the number of
    operand leaves whose values were fetched from the host (left, right; a device tensor)."""
    (rows, c, plan, counters, fetched), = multiply_host_parts(a, b, cfg, parts=1)
    return c, plan, counters, fetched


def multiply_host_parts(a: HostTree, b: HostTree | None, cfg: MultiplyConfig | None = None, parts: int = 2, on_part=None):
    """The same product in ``parts`` blocks of leaf rows of C, enqueued one after the other on the current stream:
    while block r+1 is planned, fetched and multiplied, the caller can already copy block r back (``on_part(part)``
    is called right after a block has been enqueued) -- PCIe is used in both directions at once.  Returns the list of
    ``((row0, row1), c, plan, counters, fetched)``; every ``c`` has the global shape and holds its rows only, and each
    product leaf is computed in one pass in ascending k, as in ``parallel.ShardedMultiply``."""
    if cfg is None:
        cfg = MultiplyConfig()
    if cfg.beta != 0:
        raise ValueError("multiply_host computes C = alpha A B; merge an accumulator with multiply() (beta != 0)")
    if parts < 1:
        raise ValueError(f"parts must be positive, got {parts}")
    lib = _lib.lib()
    qa = a.skeleton()
    same = b is None or b is a
    qb = qa if same else b.skeleton()
    dev = qa.device
    st = _stream()
    depth = max(qa.depth, qb.depth)
    nrows = 1 << depth
    # blocks of rows cut at multiples of 4 leaf rows (a super-tile has one owner)
    cuts = sorted({min(nrows, ((nrows * i // parts + 3) // 4) * 4) for i in range(parts + 1)} | {0, nrows})
    out = []
    from .symbolic import _capacity_hint, plan_capacity
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        copied = torch.zeros((2,), dtype=torch.int64, device=dev)
        rr = None if (r0, r1) == (0, nrows) else (r0, r1)
        if a.nleaf == 0 or (not same and b.nleaf == 0) or cfg.alpha == 0:
            plan = build_plan(qa, qb, cfg.tau, rr)
            c, counters = execute_plan(plan, qa, qb, None, cfg)
        else:
            fa = torch.empty((a.nleaf,), dtype=torch.uint8, device=dev)
            fb = fa if same else torch.empty((b.nleaf,), dtype=torch.uint8, device=dev)
            key, _ = plan_capacity(qa, qb, cfg.tau, depth, r0, r1)
            if key in _capacity_hint:
                # buffer sizes known from an earlier product of this shape: plan, mark, fetch, leaf products and norms
                # of C in ONE C call, no host synchronisation
                from .numeric import multiply_async
                host = _lib.HostOperands(a.blocks.data_ptr(), a.nleaf, fa.data_ptr(), None if same else b.blocks.data_ptr(),
                                         0 if same else b.nleaf, None if same else fb.data_ptr(), copied.data_ptr())
                c, plan, counters = multiply_async(qa, qb, cfg, None, row_range=rr, host=host)
                plan._host_keepalive = (a, b, fa, fb, copied)       # a repeat after an overflow fetches again
            else:
                plan = build_plan(qa, qb, cfg.tau, rr)
                if len(plan):
                    fa.zero_()
                    if not same:
                        fb.zero_()
                    bufs = plan.buffers()
                    import ctypes as C
                    _lib.check(lib.spamm_mark_touched(C.byref(bufs), fa.data_ptr(), fb.data_ptr(), st), "mark_touched")
                    if same:
                        _lib.check(lib.spamm_gather_blocks(a.blocks.data_ptr(), fa.data_ptr(), a.nleaf, 3, qa.values.data_ptr(),
                                                           qa.values_t.data_ptr(), copied.data_ptr(), st), "gather_blocks")
                    else:
                        # the left operand is read through its transposed records, the right one through the plain ones
                        _lib.check(lib.spamm_gather_blocks(a.blocks.data_ptr(), fa.data_ptr(), a.nleaf, 2, qa.values.data_ptr(),
                                                           qa.values_t.data_ptr(), copied.data_ptr(), st), "gather_blocks")
                        _lib.check(lib.spamm_gather_blocks(b.blocks.data_ptr(), fb.data_ptr(), b.nleaf, 1, qb.values.data_ptr(),
                                                           qb.values_t.data_ptr(), copied.data_ptr() + 8, st), "gather_blocks")
                c, counters = execute_plan(plan, qa, qb, None, cfg)
        part = ((r0, r1), c, plan, counters, copied)
        out.append(part)
        if on_part is not None:
            on_part(part)
    return out
