"""Device-resident quadtree matrix: the operand type of the multiply.

Mirrors the part of the reference's ``QuadtreeMatrix`` the multiply path touches
(`pkg/src/spamm/core.py:146-405`): ``from_dense``, ``to_dense``, ``packed_leaves``,
``put_leaf`` / ``clear`` / ``compute_norms``, ``norm``, ``leaf_count``, ``node``, plus
``sparsify`` / ``drop_tolerance`` and the host-side accessors ``leaf_items``, ``node_count``,
``get_element``.  Not provided (outside the path): ``set_element``
(raises ``NotImplementedError``), ``DenseMatrix``'s precision handling (``precision``,
``to_single`` / ``to_double``, ``frobenius``), ``n_b != 16`` and the dense-leaf foil
``execute_plan_dense_leaf``.  Added: ``from_packed`` (host or device packed leaves) and
``from_reference`` (a tree of the reference package).

Layout in HBM (see ``include/spamm_b200.h``): stored 16x16 leaves packed in ascending
Morton-key order -- row-major (``values``) and transposed (``values_t``, the staging layout of
an A operand) -- their 4x4 sub-block norms, a leaf-slot grid and the norm pyramid, each also
kept transposed so a B operand is read along k.  PyTorch only owns the memory.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import morton

DEFAULT_BLOCK = 16


def _validate_block_size(n_b) -> None:
    if not isinstance(n_b, (int, np.integer)) or n_b < 1 or n_b & (n_b - 1):
        raise ValueError(f"block size must be a positive power of two, got {n_b}")


def tree_depth(m: int, n: int, n_b: int = DEFAULT_BLOCK) -> int:
    """Smallest d with n_b * 2^d >= max(m, n) (`core.py:33-39`)."""
    _validate_block_size(n_b)
    if m < 1 or n < 1:
        raise ValueError(f"matrix dimensions must be positive, got {m} x {n}")
    q = -(-max(m, n) // n_b)
    return (q - 1).bit_length()


def drop_tolerance(tau: float, norm_a: float, norm_b: float) -> float:
    """Element-wise drop threshold that goes with a product tolerance tau: tau over the larger
    operand norm (`core.py:42-51`); the eps to hand to ``QuadtreeMatrix.sparsify``."""
    if not tau >= 0:
        raise ValueError(f"tau must be nonnegative, got {tau}")
    if norm_a < 0 or norm_b < 0:
        raise ValueError("operand norms must be nonnegative")
    largest = max(norm_a, norm_b)
    if largest == 0:
        raise ValueError("both operand norms are zero, drop tolerance undefined")
    return tau / largest


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def pack_reference_leaves(tree) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Host side of ``QuadtreeMatrix.from_reference``: (int32 keys, (n, 272) float32 leaf records,
    float64 leaf square sums) of a reference-package tree, in ascending key order.  A record is the
    256 row-major values followed by the sub-block norms transposed, tail[q*4+p] = sub[p][q]
    (include/spamm_b200.h); the square sum is float64(leaf norm)^2, whose correctly rounded root is
    the reference's float32 leaf norm again."""
    if tree.n_b != DEFAULT_BLOCK:
        raise ValueError(f"the B200 path stores 16x16 leaves (n_b = 16), got n_b = {tree.n_b}")
    keys, vals, subs = tree.packed_leaves()
    n = int(keys.shape[0])
    rec = np.empty((n, _lib.REC), np.float32)
    if n == 0:
        return np.zeros(0, np.int32), rec, np.zeros(0, np.float64)
    if int(keys.max()) >> 31:
        raise ValueError("leaf keys beyond 31 bits are not supported (depth <= 15)")
    norms = np.fromiter((nd.norm for _, nd in tree.leaf_items()), np.float64, n)   # ascending key, as packed_leaves
    rec[:, :256] = vals.reshape(n, 256)
    rec[:, 256:] = subs.transpose(0, 2, 1).reshape(n, 16)
    leaf_sq = norms.astype(np.float32).astype(np.float64) ** 2
    return keys.astype(np.int64).astype(np.int32), rec, leaf_sq


_ingested = None      # reference tree -> (its revision, device copy); weak keys


def as_device_tree(x, device=None):
    """Operands of ``build_plan`` / ``execute_plan`` / ``multiply`` may be trees of the reference
    package (duck-typed: ``packed_leaves()`` plus ``m, n, n_b``); they are copied to the device once
    per revision, as `core.py:391-404` caches the packed view by ``_rev``."""
    global _ingested
    if x is None or isinstance(x, QuadtreeMatrix):
        return x
    if not (hasattr(x, "packed_leaves") and hasattr(x, "leaf_items") and hasattr(x, "n_b")):
        raise TypeError(f"expected a QuadtreeMatrix, got {type(x).__name__}")
    if _ingested is None:
        import weakref
        _ingested = weakref.WeakKeyDictionary()
    rev = getattr(x, "_rev", None)
    hit = _ingested.get(x)
    if hit is not None and rev is not None and hit[0] == rev:
        return hit[1]
    q = QuadtreeMatrix.from_reference(x, device)
    _ingested[x] = (rev, q)
    return q


def write_back(dst, src: "QuadtreeMatrix"):
    """Store the leaves of a device tree into a reference-package tree (the accumulator a caller
    passed in is mutated in place, `numeric.py:165-181`): ``clear`` / ``put_leaf`` / ``compute_norms``."""
    keys, vals, _ = src.packed_leaves()
    dst.clear()
    for k, v in zip(keys.tolist(), vals):
        dst.put_leaf(int(k), v)
    dst.compute_norms()
    return dst


class _Span:
    """A typed region of one arena tensor (the single allocation of an asynchronous multiply).
    The kernels only need its address; the tensor view is made when the host first touches it."""

    __slots__ = ("arena", "off", "shape", "dtype", "_t")

    def __init__(self, arena: torch.Tensor, off: int, shape: tuple, dtype: torch.dtype):
        self.arena, self.off, self.shape, self.dtype, self._t = arena, int(off), shape, dtype, None

    def ptr(self) -> int:
        return self.arena.data_ptr() + self.off

    def tensor(self) -> torch.Tensor:
        if self._t is None:
            n = int(np.prod(self.shape)) * torch.empty((), dtype=self.dtype).element_size()
            self._t = self.arena[self.off:self.off + n].view(self.dtype).view(self.shape)
        return self._t


def _tensor(x):
    return x.tensor() if isinstance(x, _Span) else x


def _ptr(x) -> int | None:
    if x is None:
        return None
    return x.ptr() if isinstance(x, _Span) else x.data_ptr()


def _lazy_tensor(name: str):
    """Attribute that may hold a tensor or a _Span; reads always give a tensor."""
    slot = "_" + name

    def get(self):
        return _tensor(getattr(self, slot))

    def put(self, value):
        setattr(self, slot, value)

    return property(get, put)


class DenseMatrix:
    """Host dense matrix as returned by ``to_dense`` (`core.py:54-105`, data only)."""

    __slots__ = ("data",)

    def __init__(self, data):
        self.data = np.ascontiguousarray(data)

    @property
    def m(self) -> int:
        return self.data.shape[0]

    @property
    def n(self) -> int:
        return self.data.shape[1]


@dataclass
class TreeNode:
    tier: int
    index: int
    norm: float


class _Grids:
    """Slot grids and norm pyramid of a tree indexed at one depth."""

    __slots__ = ("depth", "_slot", "_slot_t", "_norm", "_norm_t", "_sub", "_sub_t")

    def __init__(self, depth, slot, slot_t, norm, norm_t):
        self.depth, self._slot, self._slot_t, self._norm, self._norm_t = depth, slot, slot_t, norm, norm_t
        self._sub = self._sub_t = None      # sub-norm range grids, made on the first use as an operand

    slot = _lazy_tensor("slot")
    slot_t = _lazy_tensor("slot_t")
    norm = _lazy_tensor("norm")
    norm_t = _lazy_tensor("norm_t")


class QuadtreeMatrix:
    """Quadtree of 16x16 single-precision leaves with per-node Frobenius norms, in HBM."""

    def __init__(self, m: int, n: int, n_b: int = DEFAULT_BLOCK, device=None):
        _validate_block_size(n_b)
        if m < 1 or n < 1:
            raise ValueError(f"matrix dimensions must be positive, got {m} x {n}")
        self.m, self.n, self.n_b = int(m), int(n), int(n_b)
        self.depth = tree_depth(m, n, n_b)
        self.padded = n_b << self.depth
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self._rev = 0
        self._pending: dict[int, np.ndarray] = {}   # put_leaf staging (host) until compute_norms
        self._set_empty()

    # -- storage -------------------------------------------------------------------------------
    # The leaf count of a multiply result is produced on the device; it is read back (one
    # synchronisation) only when something on the host first asks for it.
    @property
    def nleaf(self) -> int:
        if self._nleaf is None:
            self._nleaf = int(self._nleaf_source())
            self._nleaf_source = None
        return self._nleaf

    @nleaf.setter
    def nleaf(self, value: int) -> None:
        self._nleaf = int(value)
        self._nleaf_source = None

    keys = _lazy_tensor("keys")
    values = _lazy_tensor("values")
    values_t = _lazy_tensor("values_t")
    leaf_sq = _lazy_tensor("leaf_sq")

    def _leaf_bound(self) -> int:
        """Stored leaves, or their upper bound while the count is still on the device."""
        return self._nleaf if self._nleaf is not None else int(self._keys.shape[0])

    def _adopt_product(self, keys, values, values_t, leaf_sq, grids: "_Grids", count_source) -> None:
        """Take over the buffers an asynchronous multiply is filling (capacity sized)."""
        self._pending.clear()
        self.keys, self.values, self.values_t, self.leaf_sq = keys, values, values_t, leaf_sq
        self._leaf_sq_grid = None
        self._grids = {grids.depth: grids}
        self._nleaf = None
        self._nleaf_source = count_source
        self._rev += 1

    def _set_empty(self) -> None:
        self.nleaf = 0
        self.keys = self.values = self.values_t = None
        self.leaf_sq = None          # double square sum per packed leaf
        self._leaf_sq_grid = None    # the same on the leaf grid (from_dense keeps this form)
        self._grids: dict[int, _Grids] = {}

    def _require_16(self) -> None:
        if self.n_b != 16:
            raise ValueError(f"the B200 path stores 16x16 leaves (n_b = 16), got n_b = {self.n_b}")

    def _alloc(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)

    @property
    def leaf_count(self) -> int:
        return self.nleaf + len(self._pending)

    @property
    def norm(self) -> float:
        if self.nleaf == 0:
            return 0.0
        v = float(self.grids().norm[0].item())
        return v if v >= 0 else 0.0

    # -- construction ----------------------------------------------------------------------------
    @classmethod
    def from_dense(cls, dense, n_b: int = DEFAULT_BLOCK, device=None) -> "QuadtreeMatrix":
        """Build the tree from a dense matrix (numpy or torch, host or device), skipping
        all-zero blocks (`core.py:213-250`): leaf pass, Z-order slot scan, leaf packing,
        interior norms -- four kernels, one small read-back (the leaf count)."""
        if isinstance(dense, DenseMatrix):
            dense = dense.data
        if isinstance(dense, np.ndarray):
            if dense.ndim != 2 or dense.shape[0] < 1 or dense.shape[1] < 1:
                raise ValueError(f"expected a nonempty 2-D matrix, got shape {dense.shape}")
            if not np.isfinite(dense).all():
                raise ValueError("matrix elements must be finite")
            dense = torch.from_numpy(np.ascontiguousarray(dense, dtype=np.float32))
        q = cls(dense.shape[0], dense.shape[1], n_b, device)
        q._require_16()
        d = dense.to(device=q.device, dtype=torch.float32, non_blocking=True).contiguous()
        q._build_from_device_dense(d)
        return q

    @classmethod
    def from_reference(cls, tree, device=None) -> "QuadtreeMatrix":
        """Device copy of a tree of the reference package (anything with ``m, n, n_b``,
        ``packed_leaves()`` and ``leaf_items()``, `core.py:146-405`): the reference's own leaf values,
        sub-block norms and leaf norms are taken as they are (`core.py:387-405`), so the task set and
        the gates come out exactly as the reference computes them from that tree.  Interior norms are
        rebuilt on the device from the leaf norms (they only steer the pruned walk; a parent rebuilt
        from its children's norms still bounds them, so the task set is the flat rule's)."""
        q = cls(tree.m, tree.n, tree.n_b, device)
        keys, rec, leaf_sq = pack_reference_leaves(tree)
        n = int(keys.shape[0])
        if n == 0:
            return q
        values = torch.from_numpy(rec).to(q.device)
        values_t = torch.empty_like(values)
        _lib.check(_lib.lib().spamm_transpose_records(values.data_ptr(), n, values_t.data_ptr(), _stream()),
                   "transpose_records")
        q._adopt_packed(torch.from_numpy(keys).to(q.device), values, values_t, torch.from_numpy(leaf_sq).to(q.device), n)
        return q

    @classmethod
    def from_packed(cls, m: int, n: int, keys, blocks, device=None) -> "QuadtreeMatrix":
        """Tree from packed leaves: ``keys`` = ascending Morton keys of the stored leaves, ``blocks`` =
        their 16x16 values, shape (nleaf, 16, 16) or (nleaf, 256) float32 -- the first two arrays of
        the reference's ``packed_leaves()`` (`core.py:387-405`).  Host arrays (numpy, or torch tensors,
        pinned for an asynchronous copy) or device tensors.  Equivalent to ``put_leaf`` for every
        leaf followed by ``compute_norms`` (`core.py:315-345`): all norms are recomputed on the device."""
        q = cls(m, n, DEFAULT_BLOCK, device)
        keys_t = torch.as_tensor(keys)
        blocks_t = torch.as_tensor(blocks)
        nl = int(keys_t.numel())
        if blocks_t.dtype != torch.float32 or blocks_t.numel() != nl * 256:
            raise ValueError("blocks must hold one float32 16x16 block per key")
        if nl == 0:
            return q
        if nl > (1 << (2 * q.depth)):
            raise ValueError("more leaves than the tree has")
        dev_blocks = blocks_t.reshape(nl, 256).to(q.device, non_blocking=True).contiguous()
        dev_keys = keys_t.to(q.device, non_blocking=True).to(torch.int32)
        values = q._alloc((nl, _lib.REC), torch.float32)
        values_t = q._alloc((nl, _lib.REC), torch.float32)
        leaf_sq = q._alloc((nl,), torch.float64)
        _lib.check(_lib.lib().spamm_leaves_from_blocks(dev_blocks.data_ptr(), nl, values.data_ptr(), values_t.data_ptr(),
                                                      leaf_sq.data_ptr(), _stream()), "leaves_from_blocks")
        q._adopt_packed(dev_keys, values, values_t, leaf_sq, nl)
        return q

    def _build_from_device_dense(self, d: torch.Tensor) -> None:
        lib = _lib.lib()
        st = _stream()
        depth, L = self.depth, 1 << self.depth
        cells = L * L
        sub4_grid = self._alloc((cells, 16), torch.float32)
        leaf_sq_grid = self._alloc((cells,), torch.float64)
        norm = self._alloc((_lib.level_total(depth),), torch.float32)
        norm_t = self._alloc((_lib.level_total(depth),), torch.float32)
        off = _lib.level_offset(depth)
        leaf_norm = norm[off:off + cells]
        _lib.check(lib.spamm_leaf_norms_dense(d.data_ptr(), self.m, self.n, d.stride(0), depth, sub4_grid.data_ptr(),
                                              leaf_sq_grid.data_ptr(), leaf_norm.data_ptr(), st), "leaf_norms_dense")
        slot = self._alloc((cells,), torch.int32)
        slot_t = self._alloc((cells,), torch.int32)
        keys = self._alloc((cells,), torch.int32)
        nleaf_dev = self._alloc((1,), torch.int32)
        ws_bytes = lib.spamm_scan_workspace_bytes(cells)
        ws = self._alloc((ws_bytes,), torch.uint8)
        _lib.check(lib.spamm_assign_slots(leaf_norm.data_ptr(), depth, slot.data_ptr(), slot_t.data_ptr(), keys.data_ptr(),
                                          nleaf_dev.data_ptr(), ws.data_ptr(), ws_bytes, st), "assign_slots")
        nleaf = int(nleaf_dev.item())
        self.nleaf = nleaf
        self.keys = keys[:nleaf].clone()
        self.values = self._alloc((max(nleaf, 1), _lib.REC), torch.float32)
        self.values_t = self._alloc((max(nleaf, 1), _lib.REC), torch.float32)
        _lib.check(lib.spamm_pack_leaves(d.data_ptr(), self.m, self.n, d.stride(0), depth, self.keys.data_ptr(), nleaf,
                                         sub4_grid.data_ptr(), self.values.data_ptr(), self.values_t.data_ptr(), st),
                   "pack_leaves")
        sq_levels = self._alloc((_lib.level_total(depth),), torch.float64)
        _lib.check(lib.spamm_build_interior(leaf_sq_grid.data_ptr(), depth, norm.data_ptr(), norm_t.data_ptr(),
                                            sq_levels.data_ptr(), 1, st), "build_interior")
        self._leaf_sq_grid = leaf_sq_grid
        self.leaf_sq = None
        self._grids = {depth: _Grids(depth, slot, slot_t, norm, norm_t)}
        self._rev += 1

    def _adopt_packed(self, keys: torch.Tensor, values: torch.Tensor, values_t: torch.Tensor,
                      leaf_sq: torch.Tensor, nleaf: int) -> None:
        """Take ownership of packed leaves whose norms are already known (a multiply result)."""
        self._pending.clear()
        self.nleaf = int(nleaf)
        self.keys, self.values, self.values_t, self.leaf_sq = keys, values, values_t, leaf_sq
        self._leaf_sq_grid = None
        self._grids = {}
        self._index(self.depth)
        self._rev += 1

    def _packed_leaf_sq(self) -> torch.Tensor:
        if self.nleaf == 0:
            return torch.zeros((1,), dtype=torch.float64, device=self.device)
        if self.leaf_sq is None:
            i, j = morton.decode_array(self.keys.cpu().numpy().astype(np.uint64))
            idx = torch.from_numpy((i.astype(np.int64) << self.depth) + j.astype(np.int64)).to(self.device)
            self.leaf_sq = self._leaf_sq_grid[idx].contiguous() if self.nleaf else self._alloc((1,), torch.float64)
        return self.leaf_sq

    def _index(self, depth: int) -> _Grids:
        """Slot grids and norm pyramid at `depth` >= self.depth (`core.py:252-266`)."""
        lib = _lib.lib()
        st = _stream()
        L = 1 << depth
        cells = L * L
        total = _lib.level_total(depth)
        slot = self._alloc((cells,), torch.int32)
        slot_t = self._alloc((cells,), torch.int32)
        norm = self._alloc((total,), torch.float32)
        norm_t = self._alloc((total,), torch.float32)
        sq_grid = self._alloc((cells,), torch.float64)
        sq_levels = self._alloc((total,), torch.float64)
        leaf_sq = self._packed_leaf_sq()
        keys_ptr = self.keys.data_ptr() if self.nleaf else None
        _lib.check(lib.spamm_index_leaves(keys_ptr, leaf_sq.data_ptr() if self.nleaf else None, self.nleaf, depth,
                                          slot.data_ptr(), slot_t.data_ptr(), norm.data_ptr(), norm_t.data_ptr(),
                                          sq_grid.data_ptr(), st), "index_leaves")
        _lib.check(lib.spamm_build_interior(sq_grid.data_ptr(), depth, norm.data_ptr(), norm_t.data_ptr(),
                                            sq_levels.data_ptr(), 0, st), "build_interior")
        g = _Grids(depth, slot, slot_t, norm, norm_t)
        self._grids[depth] = g
        return g

    def grids(self, depth: int | None = None) -> _Grids:
        depth = self.depth if depth is None else depth
        if depth < self.depth:
            raise ValueError("cannot index a tree above its own depth")
        self._flush_guard()
        g = self._grids.get(depth)
        return g if g is not None else self._index(depth)

    def view(self, depth: int | None = None, left: bool = True) -> _lib.TreeView:
        """ctypes view for the kernels, indexed at a (possibly larger) common depth.  A tree built
        without transposed leaf copies (a gathered right-hand operand, parallel.tree_from_shard)
        gets them on its first use as a left-hand operand."""
        g = self.grids(depth)
        nz = self._nleaf is None or self._nleaf > 0        # do not force a pending count to the host
        if left and nz and self._values_t is None and self._values is not None:
            vt = torch.empty_like(self.values)
            _lib.check(_lib.lib().spamm_transpose_records(self.values.data_ptr(), self.values.shape[0], vt.data_ptr(),
                                                          _stream()), "transpose_records")
            self.values_t = vt
        if nz and g._sub is None and self._values is not None:
            # range of every leaf's sub-block norms: lets the planner classify fine4 tasks (device only,
            # from the record tails through the slot grid; no host synchronisation)
            cells = 1 << (2 * g.depth)
            g._sub = self._alloc((cells,), torch.int32)
            g._sub_t = self._alloc((cells,), torch.int32)
            _lib.check(_lib.lib().spamm_subrange_grids(_ptr(self._values), _ptr(g._slot), g.depth, g._sub.data_ptr(),
                                                       g._sub_t.data_ptr(), _stream()), "subrange_grids")
        return _lib.TreeView(self.m, self.n, g.depth, self._leaf_bound() if nz else 0,
                             _ptr(self._keys) if nz else None, _ptr(self._values) if nz else None,
                             _ptr(self._values_t) if nz else None,
                             _ptr(g._slot), _ptr(g._slot_t), _ptr(g._norm), _ptr(g._norm_t),
                             _ptr(g._sub) if nz else None, _ptr(g._sub_t) if nz else None)

    def _flush_guard(self) -> None:
        if self._pending:
            raise ValueError("tree has staged leaves with stale norms; call compute_norms() first")

    # -- reference-style accessors --------------------------------------------------------------
    def to_dense_tensor(self) -> torch.Tensor:
        self._flush_guard()
        out = torch.empty((self.m, self.n), dtype=torch.float32, device=self.device)
        if self.nleaf == 0:
            return out.zero_()
        v = self.view()
        _lib.check(_lib.lib().spamm_to_dense(C.byref(v), out.data_ptr(), out.stride(0), _stream()), "to_dense")
        return out

    def to_dense(self) -> DenseMatrix:
        return DenseMatrix(self.to_dense_tensor().cpu().numpy())

    def packed_leaves(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(keys, values, subnorms) on the host, ascending key order (`core.py:387-405`)."""
        self._flush_guard()
        n = self.nleaf
        if n == 0:
            return (np.empty(0, np.uint64), np.empty((0, 16, 16), np.float32), np.empty((0, 4, 4), np.float32))
        keys = self.keys[:n].cpu().numpy().astype(np.uint32).astype(np.uint64)
        rec = self.values[:n].cpu().numpy()
        vals = np.ascontiguousarray(rec[:, :256]).reshape(n, 16, 16)
        subs = np.ascontiguousarray(rec[:, 256:].reshape(n, 4, 4).transpose(0, 2, 1))   # tail is [q][p]
        if not getattr(self, "_keys_sorted", True):     # gathered from several ranks: rank order, unused slots
            keep = np.flatnonzero(keys != 0xFFFFFFFF)
            order = keep[np.argsort(keys[keep], kind="stable")]
            keys, vals, subs = keys[order], vals[order], subs[order]
        return keys, vals, subs

    def leaf_keys(self) -> np.ndarray:
        return self.packed_leaves()[0] if self.nleaf else np.empty(0, np.uint64)

    def level_norms(self, tier: int) -> np.ndarray:
        """Host copy of one tier's norm grid, -1 where no node is stored."""
        g = self.grids()
        s = 1 << tier
        off = _lib.level_offset(tier)
        return g.norm[off:off + s * s].cpu().numpy().reshape(s, s)

    def node(self, tier: int, index: int) -> TreeNode | None:
        if self.nleaf == 0 or not 0 <= tier <= self.depth:
            return None
        i, j = morton.decode(index)
        s = 1 << tier
        if i >= s or j >= s:
            return None
        v = float(self.level_norms(tier)[i, j])
        return TreeNode(tier, index, v) if v >= 0 else None

    # -- host-side accessors of the reference tree (`core.py:176-211`); each call copies from the device
    def leaf_items(self) -> list[tuple[int, TreeNode]]:
        """Stored leaves as (key, node) in ascending key order; node.norm is the leaf's Frobenius norm."""
        if self.nleaf == 0:
            return []
        keys = self.packed_leaves()[0]
        i, j = morton.decode_array(keys.astype(np.uint64))
        norms = self.level_norms(self.depth)[i, j]
        return [(int(k), TreeNode(self.depth, int(k), float(v))) for k, v in zip(keys.tolist(), norms)]

    @property
    def node_count(self) -> int:
        """Stored nodes of all tiers (`core.py:188-190`)."""
        if self.nleaf == 0:
            return 0
        return int(sum(int(np.count_nonzero(self.level_norms(t) >= 0)) for t in range(self.depth + 1)))

    def get_element(self, i: int, j: int) -> float:
        """Stored value at (i, j); 0.0 where no leaf is stored (`core.py:202-211`)."""
        i, j = int(i), int(j)
        if not (0 <= i < self.m and 0 <= j < self.n):
            raise IndexError(f"element ({i}, {j}) outside {self.m} x {self.n}")
        if self.nleaf == 0:
            return 0.0
        self._flush_guard()
        g = self.grids()
        slot = int(g.slot[(i // 16) * (1 << self.depth) + (j // 16)].item())
        return 0.0 if slot < 0 else float(self.values[slot, (i % 16) * 16 + (j % 16)].item())

    def set_element(self, i: int, j: int, value: float) -> None:
        """Not part of the multiply path (SURVEY.md section 8 marks `core.py:280-313` out of scope): edit the
        tree with put_leaf / compute_norms, or build it with from_dense / from_packed."""
        raise NotImplementedError("set_element is outside the B200 multiply path; use put_leaf + compute_norms")

    # -- staged mutation: put_leaf ... compute_norms (`core.py:315-345`) --------------------------
    def put_leaf(self, key: int, values: np.ndarray) -> None:
        self._require_16()
        values = np.asarray(values)
        if values.shape != (self.n_b, self.n_b):
            raise ValueError(f"leaf values must be {self.n_b} x {self.n_b}")
        if key < 0 or key >> (2 * self.depth):
            raise ValueError(f"leaf key {key} outside depth {self.depth}")
        self._pending[int(key)] = np.ascontiguousarray(values, dtype=np.float32)
        self._rev += 1

    def clear(self) -> None:
        self._pending.clear()
        self._set_empty()
        self._rev += 1

    def sparsify(self, eps: float) -> int:
        """Zero every 4x4 sub-block with 0 < sub-norm < eps, drop the leaves left empty and rebuild
        the interior norms (`core.py:347-383`).  Returns the number of sub-blocks dropped;
        ``eps = 0`` is an exact no-op.  The comparison is done in float32, as numpy does for a
        float32 array against a Python float."""
        self._require_16()
        if not eps >= 0:
            raise ValueError(f"eps must be nonnegative, got {eps}")
        self._flush_guard()
        if eps == 0 or self.nleaf == 0:
            return 0
        n = self.nleaf
        if not getattr(self, "_keys_sorted", True):
            raise ValueError("sparsify needs a tree with its leaves in key order")
        if self._values_t is None:
            self.view()                                         # builds the transposed copies
        values, values_t = self.values[:n].contiguous(), self.values_t[:n].contiguous()
        leaf_sq = self._packed_leaf_sq()[:n].clone()
        dropped = torch.zeros((1,), dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().spamm_sparsify_leaves(values.data_ptr(), values_t.data_ptr(), leaf_sq.data_ptr(), n,
                                                    float(np.float32(eps)), dropped.data_ptr(), _stream()), "sparsify")
        keep = torch.nonzero(leaf_sq > 0).flatten()
        if keep.numel() == 0:
            self._set_empty()
            self._rev += 1
        elif keep.numel() == n:
            self._adopt_packed(self.keys[:n].contiguous(), values, values_t, leaf_sq, n)
        else:
            self._adopt_packed(self.keys[:n][keep].contiguous(), values[keep].contiguous(), values_t[keep].contiguous(),
                               leaf_sq[keep].contiguous(), int(keep.numel()))
        return int(dropped.item())

    def compute_norms(self) -> None:
        """Rebuild all norms bottom-up from leaf values (`core.py:331-345`)."""
        self._require_16()
        leaves: dict[int, np.ndarray] = {}
        if self.nleaf:
            keys = self.keys[: self.nleaf].cpu().numpy()
            vals = self.values[: self.nleaf, :256].cpu().numpy().reshape(-1, 16, 16)
            leaves.update({int(k): v for k, v in zip(keys.tolist(), vals)})
        leaves.update(self._pending)
        self._pending.clear()
        ks = sorted(leaves)
        if not ks:
            self._set_empty()
            self._rev += 1
            return
        keys_t = torch.tensor(ks, dtype=torch.int32, device=self.device)
        rec = np.zeros((len(ks), _lib.REC), np.float32)
        rec[:, :256] = np.stack([leaves[k] for k in ks]).reshape(-1, 256)
        self._set_packed_values(keys_t, torch.from_numpy(rec).to(self.device))

    def _set_packed_values(self, keys: torch.Tensor, values: torch.Tensor) -> None:
        """Leaves given by keys (ascending) and (n, 272) value records; norms in compute_norms order."""
        n = int(keys.numel())
        values_t = self._alloc((n, _lib.REC), torch.float32)
        leaf_sq = self._alloc((n,), torch.float64)
        _lib.check(_lib.lib().spamm_leaf_norms_packed(values.data_ptr(), n, values_t.data_ptr(), leaf_sq.data_ptr(),
                                                     _stream()), "leaf_norms_packed")
        self._adopt_packed(keys, values, values_t, leaf_sq, n)

    def __repr__(self) -> str:
        return (f"QuadtreeMatrix({self.m}x{self.n}, n_b={self.n_b}, depth={self.depth}, "
                f"leaves={self.leaf_count}, device={self.device})")
