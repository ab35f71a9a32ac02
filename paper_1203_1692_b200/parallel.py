"""Row-block sharding of the SpAMM product across the GPUs of one box.

The reference is single process (`SPEC.md:542` lists distribution as a non-goal); this is the
split BASELINE.json's north_star asks for.  Every product leaf C(i,j) has exactly one owner and
accumulates over k locally, so no reduction crosses ranks and the ascending-k order -- hence the
bitwise result -- is the same for any number of ranks.

* Operands enter row-sharded: rank r holds the stored leaves of its block of leaf rows, as a
  ``PackedShard`` (keys, 272-float leaf records with their sub-norm tails, leaf square sums).
  Block boundaries are multiples of 4 leaf rows, so every aligned 4x4 block of leaves -- the unit
  the numeric kernel stages with one bulk copy -- has one owner and stays contiguous.
* One exchange step: an all-gather of the shards (NCCL over NVLink/NVSwitch; only stored leaves
  travel).  The transposed copies are rebuilt locally instead of being sent.
* Every rank then plans the product on the (replicated) norm pyramids, counts the surviving tasks
  per leaf row, cuts the rows of C into contiguous blocks of about equal task count, and runs the
  fused multiply restricted to its own block (``row_range``).

The collective and partition logic is plain ``torch.distributed`` on whatever device the tensors
live on, so it is covered on CPU with the gloo backend (tests/test_parallel.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

ROW_ALIGN = 4      # leaf rows; shard boundaries are multiples of this


@dataclass
class PackedShard:
    """Stored leaves of a block of leaf rows (any device)."""

    keys: torch.Tensor       # (n,) int32 Morton keys in GLOBAL leaf coordinates
    records: torch.Tensor    # (n, 272) float32: row-major leaf values + transposed sub-norm tail
    leaf_sq: torch.Tensor    # (n,) float64 leaf square sums

    @property
    def n(self) -> int:
        return int(self.keys.shape[0])


def even_row_split(nrows: int, world: int) -> list[tuple[int, int]]:
    """Contiguous blocks of leaf rows of (nearly) equal height, boundaries aligned to ROW_ALIGN."""
    units = -(-nrows // ROW_ALIGN)
    cuts = [min(nrows, ROW_ALIGN * ((units * r) // world)) for r in range(world + 1)]
    cuts[-1] = nrows
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def balanced_row_split(row_tasks: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous blocks of leaf rows with about equal numbers of surviving tasks.

    Cut r sits where the running task count first reaches r/world of the total, rounded to
    ROW_ALIGN rows; every rank evaluates this on the same counts and gets the same answer."""
    row_tasks = np.asarray(row_tasks, np.int64)
    nrows = int(row_tasks.shape[0])
    total = int(row_tasks.sum())
    if total == 0:
        return even_row_split(nrows, world)
    csum = np.concatenate([[0], np.cumsum(row_tasks)])
    cuts = [0]
    for r in range(1, world):
        x = int(np.searchsorted(csum, total * r / world, side="left"))
        x = min(nrows, max(cuts[-1], ROW_ALIGN * int(round(x / ROW_ALIGN))))
        cuts.append(x)
    cuts.append(nrows)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def _spread16(x: torch.Tensor) -> torch.Tensor:
    x = x & 0xFFFF
    x = (x | (x << 8)) & 0x00FF00FF
    x = (x | (x << 4)) & 0x0F0F0F0F
    x = (x | (x << 2)) & 0x33333333
    x = (x | (x << 1)) & 0x55555555
    return x


def _squeeze16(x: torch.Tensor) -> torch.Tensor:
    x = x & 0x55555555
    x = (x | (x >> 1)) & 0x33333333
    x = (x | (x >> 2)) & 0x0F0F0F0F
    x = (x | (x >> 4)) & 0x00FF00FF
    x = (x | (x >> 8)) & 0x0000FFFF
    return x


def shift_keys(keys: torch.Tensor, row_offset: int) -> torch.Tensor:
    """Morton keys of leaves (i, j) -> keys of (i + row_offset, j) (row bit above column bit)."""
    k = keys.to(torch.int64)
    i = _squeeze16(k >> 1) + int(row_offset)
    j = _squeeze16(k)
    return ((_spread16(i) << 1) | _spread16(j)).to(torch.int32)


def shard_from_dense_rows(dense_rows, row0_leaf: int, device=None) -> PackedShard:
    """Shard of the leaf rows starting at ``row0_leaf`` from the matching rows of the dense matrix
    (``QuadtreeMatrix.from_dense`` on the row block, keys moved to global coordinates)."""
    from .tree import QuadtreeMatrix
    if row0_leaf % ROW_ALIGN:
        raise ValueError(f"row blocks must start at a multiple of {ROW_ALIGN} leaf rows")
    local = QuadtreeMatrix.from_dense(dense_rows, device=device)
    n = local.nleaf
    if n == 0:
        dev = local.device
        return PackedShard(torch.empty((0,), dtype=torch.int32, device=dev),
                           torch.empty((0, 272), dtype=torch.float32, device=dev),
                           torch.empty((0,), dtype=torch.float64, device=dev))
    return PackedShard(shift_keys(local.keys[:n], row0_leaf), local.values[:n], local._packed_leaf_sq()[:n])


def shard_of_tree(tree, r0: int, r1: int) -> PackedShard:
    """The stored leaves of leaf rows [r0, r1) of a whole tree (benchmarks and tests)."""
    n = tree.nleaf
    keys = tree.keys[:n]
    rows = _squeeze16(keys.to(torch.int64) >> 1)
    sel = torch.nonzero((rows >= r0) & (rows < r1)).flatten()
    return PackedShard(keys[sel].contiguous(), tree.values[:n][sel].contiguous(),
                       tree._packed_leaf_sq()[:n][sel].contiguous())


HOLE = -1          # key of an unused slot in a gathered shard (0xFFFFFFFF on the device)


def allgather_shards(shard: PackedShard, group=None) -> PackedShard:
    """Every rank's shard in rank order, gathered straight into its final buffers.

    Shard sizes differ, so each rank's part occupies ``cap`` = the largest shard size slots of the
    result; the unused slots at the end of a part carry the key ``HOLE`` and are never indexed
    (`spamm_index_leaves` skips them).  One collective per array, no staging copy of the payload
    beyond padding the rank's own shard; with a single rank nothing is copied at all."""
    world = dist.get_world_size(group)
    if world == 1:
        return shard
    dev = shard.keys.device
    sizes = [torch.zeros((1,), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([shard.n], dtype=torch.int64, device=dev), group=group)
    cap = max(max(int(c.item()) for c in sizes), 1)

    def gather(x: torch.Tensor, fill) -> torch.Tensor:
        pad = torch.empty((cap,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        pad[: x.shape[0]] = x
        if fill is not None:
            pad[x.shape[0]:] = fill
        out = torch.empty((world * cap,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(out, pad, group=group)
        else:
            dist.all_gather(list(out.chunk(world)), pad, group=group)
        return out

    return PackedShard(gather(shard.keys, HOLE), gather(shard.records, None), gather(shard.leaf_sq, 0.0))


def needed_rows(a_shard: PackedShard, nrows_b: int, reach: torch.Tensor | None = None) -> torch.Tensor:
    """Leaf rows of B that a rank holding ``a_shard`` can reach: the leaf columns of its stored A
    leaves (only those marked in ``reach``, see ``reaching_leaves``, when given), widened to whole
    groups of ROW_ALIGN rows so 4x4 blocks of leaves travel complete."""
    groups = -(-nrows_b // ROW_ALIGN)
    hit = torch.zeros((groups,), dtype=torch.bool, device=a_shard.keys.device)
    if a_shard.n:
        cols = _squeeze16(a_shard.keys.to(torch.int64))
        if reach is not None:
            cols = cols[reach]
        hit[torch.div(cols, ROW_ALIGN, rounding_mode="floor").clamp_(max=groups - 1)] = True
    return hit.repeat_interleave(ROW_ALIGN)[:nrows_b]


def row_max_norms(b_shard: PackedShard, nrows_b: int, group=None) -> torch.Tensor:
    """Largest leaf norm in every leaf row of B (float32, 0 for an empty row), from all ranks' shards:
    one MAX all-reduce of nrows_b floats (set-up)."""
    out = torch.zeros((nrows_b,), dtype=torch.float32, device=b_shard.keys.device)
    if b_shard.n:
        rows = _squeeze16(b_shard.keys.to(torch.int64) >> 1)
        out.scatter_reduce_(0, rows, torch.sqrt(b_shard.leaf_sq).to(torch.float32), reduce="amax")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.MAX, group=group)
    return out


def reaching_leaves(a_shard: PackedShard, rowmax_b: torch.Tensor, tau: float) -> torch.Tensor:
    """Which stored leaves of A take part in at least one task: leaf (i,k) does iff
    double(|A_ik|) * double(max_j |B_kj|) >= tau -- the planner's own test (`symbolic.py:118-125`)
    against the largest norm in row k of B."""
    if a_shard.n == 0:
        return torch.zeros((0,), dtype=torch.bool, device=a_shard.keys.device)
    cols = _squeeze16(a_shard.keys.to(torch.int64))
    na = torch.sqrt(a_shard.leaf_sq).to(torch.float32).to(torch.float64)
    nb = rowmax_b[cols].to(torch.float64)
    return (nb > 0) & (na * nb >= float(tau))


def exchange_needed_rows(b_shard: PackedShard, need: torch.Tensor, splits: list[tuple[int, int]], group=None) -> PackedShard:
    """The band-limited alternative to ``allgather_shards``: every rank receives only the leaf rows
    of B it asked for (``need``, a bool per leaf row of B), from the ranks that own them
    (``splits[r]`` = rows of rank r).  One small all-gather of the requests and of the piece sizes,
    then point-to-point transfers straight into the result (pieces in rank order, own rows in
    place, no unused slots).  For a banded matrix split over N ranks a rank fetches its band, not
    (N-1)/N of the matrix."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = b_shard.keys.device
    nrows = int(need.shape[0])
    asked = [torch.zeros((nrows,), dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(asked, need.to(torch.uint8), group=group)
    r0, r1 = splits[rank]
    my_rows = _squeeze16(b_shard.keys.to(torch.int64) >> 1) if b_shard.n else torch.zeros((0,), dtype=torch.int64, device=dev)
    picks = []
    for p in range(world):
        want = asked[p].to(torch.bool)
        want[:r0] = False
        want[r1:] = False
        picks.append(torch.nonzero(want[my_rows]).flatten() if b_shard.n else my_rows)
    sizes = torch.tensor([int(x.numel()) for x in picks], dtype=torch.int64, device=dev)
    table = [torch.zeros((world,), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(table, sizes, group=group)
    incoming = [int(table[src][rank].item()) for src in range(world)]        # leaves rank src sends me
    offs = [0]
    for c in incoming:
        offs.append(offs[-1] + c)
    out = PackedShard(torch.empty((offs[-1],), dtype=b_shard.keys.dtype, device=dev),
                      torch.empty((offs[-1], 272), dtype=torch.float32, device=dev),
                      torch.empty((offs[-1],), dtype=torch.float64, device=dev))
    ops, keep = [], []
    for p in range(world):
        sel = picks[p]
        if p == rank:
            sl = slice(offs[p], offs[p + 1])
            out.keys[sl], out.records[sl], out.leaf_sq[sl] = b_shard.keys[sel], b_shard.records[sel], b_shard.leaf_sq[sel]
            continue
        if sel.numel():
            bufs = (b_shard.keys[sel].contiguous(), b_shard.records[sel].contiguous(), b_shard.leaf_sq[sel].contiguous())
            keep.append(bufs)
            ops += [dist.P2POp(dist.isend, t, p, group) for t in bufs]
        if incoming[p]:
            sl = slice(offs[p], offs[p + 1])
            ops += [dist.P2POp(dist.irecv, t[sl], p, group) for t in (out.keys, out.records, out.leaf_sq)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out


def drop_holes(shard: PackedShard) -> PackedShard:
    """The stored leaves of a gathered shard, unused slots removed (tests and host export)."""
    keep = torch.nonzero(shard.keys != HOLE).flatten()
    return PackedShard(shard.keys[keep], shard.records[keep], shard.leaf_sq[keep])


# ---------------------------------------------------------------------------------------------------
# Set-up objects: everything about an exchange that needs the host (sizes, offsets, who sends what)
# is found ONCE; the timed step then only moves payload -- no .item(), no allocation.

@dataclass
class GatherLayout:
    """What ``allgather_shards`` needs to run without a host round trip: the common stride ``cap`` (the
    largest shard) and the buffers the collective writes into."""

    world: int
    sizes: list            # stored leaves per rank
    cap: int
    pad: PackedShard | None     # staging of the own shard when it is shorter than cap
    out: PackedShard


def gather_layout(shard: PackedShard, group=None) -> GatherLayout:
    world = dist.get_world_size(group)
    dev = shard.keys.device
    sizes_t = [torch.zeros((1,), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes_t, torch.tensor([shard.n], dtype=torch.int64, device=dev), group=group)
    sizes = [int(c.item()) for c in sizes_t]
    cap = max(max(sizes), 1)

    def buf(n):
        return PackedShard(torch.empty((n,), dtype=torch.int32, device=dev),
                           torch.empty((n, 272), dtype=torch.float32, device=dev),
                           torch.empty((n,), dtype=torch.float64, device=dev))
    pad = None
    if shard.n < cap:
        pad = buf(cap)
        pad.keys[shard.n:] = HOLE
        pad.leaf_sq[shard.n:] = 0.0
    return GatherLayout(world, sizes, cap, pad, buf(world * cap))


def allgather_with_layout(shard: PackedShard, lay: GatherLayout, group=None, async_op: bool = False):
    """The all-gather of ``allgather_shards`` into the layout's buffers; with ``async_op`` returns the
    work handles to wait on (the collective then overlaps with whatever is enqueued meanwhile)."""
    if lay.world == 1:
        return (shard, []) if async_op else shard
    src = shard
    if lay.pad is not None:
        n = shard.n
        lay.pad.keys[:n].copy_(shard.keys)
        lay.pad.records[:n].copy_(shard.records)
        lay.pad.leaf_sq[:n].copy_(shard.leaf_sq)
        src = lay.pad
    works = []
    nccl = dist.get_backend(group) == "nccl"
    for o, x in ((lay.out.keys, src.keys), (lay.out.records, src.records), (lay.out.leaf_sq, src.leaf_sq)):
        if nccl:
            w = dist.all_gather_into_tensor(o, x, group=group, async_op=async_op)
        else:
            w = dist.all_gather(list(o.chunk(lay.world)), x, group=group, async_op=async_op)
        works.append(w)
    return (lay.out, works) if async_op else lay.out


@dataclass
class NeededLayout:
    """What ``exchange_needed_rows`` needs to run without a host round trip."""

    world: int
    rank: int
    picks: list            # per peer: indices into the own shard of the leaves it asked for
    offs: list             # start of every source rank's part in the result
    incoming: list
    out: PackedShard
    send: list             # per peer: staging buffers (keys, records, leaf_sq) or None


def needed_layout(b_shard: PackedShard, need: torch.Tensor, splits, group=None) -> NeededLayout:
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = b_shard.keys.device
    nrows = int(need.shape[0])
    asked = [torch.zeros((nrows,), dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(asked, need.to(torch.uint8), group=group)
    r0, r1 = splits[rank]
    my_rows = _squeeze16(b_shard.keys.to(torch.int64) >> 1) if b_shard.n else torch.zeros((0,), dtype=torch.int64, device=dev)
    picks = []
    for p in range(world):
        want = asked[p].to(torch.bool)
        want[:r0] = False
        want[r1:] = False
        picks.append(torch.nonzero(want[my_rows]).flatten() if b_shard.n else my_rows)
    sizes = torch.tensor([int(x.numel()) for x in picks], dtype=torch.int64, device=dev)
    table = [torch.zeros((world,), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(table, sizes, group=group)
    incoming = [int(table[src][rank].item()) for src in range(world)]
    offs = [0]
    for c in incoming:
        offs.append(offs[-1] + c)
    out = PackedShard(torch.empty((offs[-1],), dtype=b_shard.keys.dtype, device=dev),
                      torch.empty((offs[-1], 272), dtype=torch.float32, device=dev),
                      torch.empty((offs[-1],), dtype=torch.float64, device=dev))
    send = []
    for p in range(world):
        k = int(picks[p].numel())
        send.append(None if (p == rank or k == 0) else (torch.empty((k,), dtype=b_shard.keys.dtype, device=dev),
                                                         torch.empty((k, 272), dtype=torch.float32, device=dev),
                                                         torch.empty((k,), dtype=torch.float64, device=dev)))
    return NeededLayout(world, rank, picks, offs, incoming, out, send)


def exchange_with_layout(b_shard: PackedShard, lay: NeededLayout, group=None, async_op: bool = False):
    """The transfers of ``exchange_needed_rows`` with everything host-side prepared: gathers of the
    asked-for leaves into the staging buffers, then one batch of isend / irecv into the result."""
    ops = []
    for p in range(lay.world):
        sel = lay.picks[p]
        sl = slice(lay.offs[p], lay.offs[p + 1])
        if p == lay.rank:
            if sel.numel():
                torch.index_select(b_shard.keys, 0, sel, out=lay.out.keys[sl])
                torch.index_select(b_shard.records, 0, sel, out=lay.out.records[sl])
                torch.index_select(b_shard.leaf_sq, 0, sel, out=lay.out.leaf_sq[sl])
            continue
        if lay.send[p] is not None:
            for dst, src in zip(lay.send[p], (b_shard.keys, b_shard.records, b_shard.leaf_sq)):
                torch.index_select(src, 0, sel, out=dst)
            ops += [dist.P2POp(dist.isend, t, p, group) for t in lay.send[p]]
        if lay.incoming[p]:
            ops += [dist.P2POp(dist.irecv, t[sl], p, group) for t in (lay.out.keys, lay.out.records, lay.out.leaf_sq)]
    reqs = dist.batch_isend_irecv(ops) if ops else []
    if async_op:
        return lay.out, reqs
    for r in reqs:
        r.wait()
    return lay.out


def interior_rows(a_shard: PackedShard, own_rows: tuple[int, int], b_rows: tuple[int, int],
                  reach: torch.Tensor | None = None) -> tuple[int, int]:
    """The largest run [i0, i1) of this rank's leaf rows of A (``own_rows``), aligned to ROW_ALIGN, whose
    stored leaves (those marked in ``reach`` when given) all sit in leaf columns inside ``b_rows`` --
    the rows of B the rank holds itself.  Those rows of C need nothing from other ranks: their
    product can run while the exchange is in flight.  (Host side, set-up only.)"""
    r0, r1 = own_rows
    if a_shard.n == 0 or r1 <= r0:
        return (r0, r0)
    k = a_shard.keys.to(torch.int64)
    if reach is not None:
        k = k[reach]
    rows = (_squeeze16(k >> 1) - r0).cpu().numpy()
    cols = _squeeze16(k).cpu().numpy()
    local = np.ones(r1 - r0, bool)
    out = (cols < b_rows[0]) | (cols >= b_rows[1])
    local[np.unique(rows[out])] = False
    groups = local[: (len(local) // ROW_ALIGN) * ROW_ALIGN].reshape(-1, ROW_ALIGN).all(axis=1) if r0 % ROW_ALIGN == 0 else np.zeros(0, bool)
    best, cur_start, best_len = (0, 0), None, 0
    for i, ok in enumerate(list(groups) + [False]):
        if ok and cur_start is None:
            cur_start = i
        if not ok and cur_start is not None:
            if i - cur_start > best_len:
                best, best_len = (cur_start, i), i - cur_start
            cur_start = None
    return (r0 + ROW_ALIGN * best[0], r0 + ROW_ALIGN * best[1])


class ShardedMultiply:
    """C = A B for one rank of a row-block split, prepared once and run many times.

    Set-up (host round trips allowed): the exchange layout (sizes, offsets, who sends what), the choice
    between the all-gather and the band-limited exchange (``exchange="auto"``: the latter when the rank
    needs less than half of B), and the INTERIOR rows -- the rows of the rank's block of A whose stored
    leaves only reach rows of B the rank holds itself.  ``run()`` then (1) starts the exchange
    asynchronously, (2) multiplies the interior rows against the rank's own rows of B while the
    exchange is in flight, (3) waits for the exchange, indexes B and multiplies the remaining rows
    (above and below the interior run).  Every product leaf is still computed in one pass in ascending
    k, so the rows of C are bit-identical to the single-GPU product whatever the rank count; the result
    is a list of (row range, C tree, plan, counters) with disjoint row ranges.
    The reference has no counterpart (`SPEC.md:542`)."""

    def __init__(self, a_shard: PackedShard, b_shard: PackedShard | None, shape_a, shape_b, cfg, group=None,
                 splits=None, exchange: str = "auto", overlap: bool = True, device=None, a_tree=None):
        self.cfg, self.group, self.shape_a, self.shape_b, self.device = cfg, group, shape_a, shape_b, device
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.mine_b = a_shard if b_shard is None else b_shard
        nrows_b = -(-shape_b[0] // 16)
        # one split for the leaf rows of A (= of C) and of B: rank r holds rows splits[r] of both
        self.splits = splits if splits is not None else even_row_split(nrows_b, self.world)
        self.rows = self.splits[self.rank]
        self.a_tree = a_tree if a_tree is not None else tree_from_shard(shape_a[0], shape_a[1], a_shard, device)
        # only leaves that take part in a task reach out: |A_ik| * max_j |B_kj| >= tau
        self.rowmax_b = row_max_norms(self.mine_b, nrows_b, group)
        reach = reaching_leaves(a_shard, self.rowmax_b, cfg.tau)
        need = needed_rows(a_shard, nrows_b, reach)
        self.need_fraction = float(need.float().mean().item()) if need.numel() else 0.0
        if exchange == "auto":
            exchange = "needed" if (self.world > 1 and self.need_fraction < 0.5) else "all"
        if exchange not in ("all", "needed"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.exchange = exchange
        if self.world > 1:
            self.layout = needed_layout(self.mine_b, need, self.splits, group) if exchange == "needed" \
                else gather_layout(self.mine_b, group)
        else:
            self.layout = None
        self.interior = (self.rows[0], self.rows[0])
        self.b_own = None
        if overlap and self.world > 1:
            self.interior = interior_rows(a_shard, self.rows, self.splits[self.rank], reach)
            if self.interior[1] > self.interior[0]:
                self.b_own = tree_from_shard(shape_b[0], shape_b[1], self.mine_b, device, transposed=False)

    def run(self):
        from .numeric import multiply_async
        out = []
        r0, r1 = self.rows
        i0, i1 = self.interior
        if self.world == 1:
            b_full = tree_from_shard(self.shape_b[0], self.shape_b[1], self.mine_b, self.device, transposed=False)
            c, plan, k = multiply_async(self.a_tree, b_full, self.cfg, None, row_range=(r0, r1))
            return [((r0, r1), c, plan, k)]
        if self.exchange == "needed":
            got, works = exchange_with_layout(self.mine_b, self.layout, self.group, async_op=True)
        else:
            got, works = allgather_with_layout(self.mine_b, self.layout, self.group, async_op=True)
        if i1 > i0:          # needs nothing from the other ranks: runs while the exchange is in flight
            c, plan, k = multiply_async(self.a_tree, self.b_own, self.cfg, None, row_range=(i0, i1))
            out.append(((i0, i1), c, plan, k))
        for w in works:
            w.wait()
        b_full = tree_from_shard(self.shape_b[0], self.shape_b[1], got, self.device, transposed=False)
        for lo, hi in ((r0, i0), (i1, r1)) if i1 > i0 else ((r0, r1),):
            if hi > lo:
                c, plan, k = multiply_async(self.a_tree, b_full, self.cfg, None, row_range=(lo, hi))
                out.append(((lo, hi), c, plan, k))
        return sorted(out, key=lambda x: x[0])


def tree_from_shard(m: int, n: int, shard: PackedShard, device=None, transposed: bool = True):
    """Tree of an m x n matrix from packed leaves (global keys, possibly with HOLE slots): leaf
    grids and the norm pyramid are built on the device from the norms the owners computed.

    ``transposed=False`` skips the transposed leaf copies: enough for a right-hand operand, which the
    numeric kernel reads through ``values`` only (the left-hand operand is read through ``values_t``)."""
    from . import _lib
    from .tree import QuadtreeMatrix, _stream
    q = QuadtreeMatrix(m, n, device=device)
    cnt = shard.n
    if cnt == 0:
        return q
    keys = shard.keys.to(q.device).contiguous()
    values = shard.records.to(q.device).contiguous()
    leaf_sq = shard.leaf_sq.to(q.device).contiguous()
    values_t = None
    if transposed:
        values_t = torch.empty_like(values)
        _lib.check(_lib.lib().spamm_transpose_records(values.data_ptr(), cnt, values_t.data_ptr(), _stream()),
                   "transpose_records")
    q._adopt_packed(keys, values, values_t, leaf_sq, cnt)
    q._keys_sorted = False          # rank order with unused slots, not one ascending Morton sequence
    return q


def row_task_counts(plan, depth: int) -> torch.Tensor:
    """Surviving tasks per leaf row of the product (device int32 tensor of length 2^depth)."""
    import ctypes as C
    from . import _lib
    from .tree import _stream
    out = torch.empty((1 << depth,), dtype=torch.int32, device=plan.steps.device)
    bufs = plan.buffers()
    _lib.check(_lib.lib().spamm_plan_row_counts(C.byref(bufs), depth, out.data_ptr(), _stream()), "row_counts")
    return out


def multiply_sharded(a_shard: PackedShard, b_shard: PackedShard | None, shape_a: tuple[int, int],
                     shape_b: tuple[int, int], cfg, group=None, device=None, exchange: str = "all",
                     splits: list[tuple[int, int]] | None = None, a_tree=None):
    """C = A B with C's leaf rows split across the ranks of ``group`` like the rows of A.

    ``a_shard`` / ``b_shard`` are this rank's row blocks of the operands (``b_shard is None`` means
    B is A).  The one exchange step brings B's packed leaves to the rank: ``exchange="all"`` is the
    all-gather; ``exchange="needed"`` fetches only the leaf rows of B that the columns of the local A
    reach (``splits`` = the row block of every rank, needed to find the owners).  The left operand
    stays local: a tree holding only this rank's rows of A times B gives exactly this rank's rows of
    C, so the partition of A (see ``balanced_row_split``) is the partition of the work.
    ``a_tree``: the tree of the local rows when the caller already holds one (a resident operand, or
    the product of a previous sharded multiply), which saves rebuilding its transposed leaf copies.
    Returns ``(c, plan, counters)``; ``c`` has the global shape and holds this rank's rows."""
    from .numeric import multiply_async
    if cfg.beta != 0:
        raise ValueError("the sharded multiply computes C = alpha A B; merge an accumulator with multiply() (beta != 0)")
    a_local = a_tree if a_tree is not None else tree_from_shard(shape_a[0], shape_a[1], a_shard, device)
    mine_b = a_shard if b_shard is None else b_shard
    if exchange == "all":
        got = allgather_shards(mine_b, group)
    elif exchange == "needed":
        if splits is None:
            raise ValueError('exchange="needed" needs the row blocks of all ranks (splits)')
        got = exchange_needed_rows(mine_b, needed_rows(a_shard, -(-shape_b[0] // 16)), splits, group)
    else:
        raise ValueError(f"unknown exchange {exchange!r}")
    b_full = tree_from_shard(shape_b[0], shape_b[1], got, device, transposed=False)
    return multiply_async(a_local, b_full, cfg, None)
