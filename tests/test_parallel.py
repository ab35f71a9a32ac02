"""Host-side logic of the multi-GPU row-block split, on CPU with gloo (world size 2).

The collective path (all-gather of packed leaf shards) and the partition arithmetic are the
same code that runs over NCCL; the leaf products are done here by the CPU oracle, restricted to each
rank's row block, so the test checks what the split must guarantee: every product leaf has one
owner, the union of the per-rank task sets is the global task set, and the rows of C computed by
the ranks are bit-identical to the single-process product.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1203_1692_b200 import inputs, morton, parallel


def test_even_and_balanced_splits_cover_all_rows():
    rng = np.random.default_rng(0)
    for nrows in (1, 3, 4, 17, 64, 250, 2048):
        for world in (1, 2, 3, 4, 8):
            for split in (parallel.even_row_split(nrows, world),
                          parallel.balanced_row_split(rng.integers(0, 50, nrows), world),
                          parallel.balanced_row_split(np.zeros(nrows, np.int64), world)):
                assert len(split) == world
                assert split[0][0] == 0 and split[-1][1] == nrows
                for (a0, a1), (b0, b1) in zip(split, split[1:]):
                    assert a1 == b0 and a0 <= a1
                for r0, _ in split[1:]:
                    assert r0 % parallel.ROW_ALIGN == 0 or r0 == nrows


def test_balanced_split_balances_tasks():
    # config-5-like profile: uniform interior, lighter edges
    counts = np.full(2048, 4636, np.int64)
    counts[:64] = np.linspace(1800, 4636, 64).astype(np.int64)
    counts[-64:] = counts[:64][::-1]
    for world in (2, 4, 8):
        split = parallel.balanced_row_split(counts, world)
        loads = np.array([counts[r0:r1].sum() for r0, r1 in split])
        assert loads.max() <= 1.02 * loads.mean()


def test_shift_keys_matches_encode():
    rng = np.random.default_rng(1)
    i = rng.integers(0, 500, 1000)
    j = rng.integers(0, 2048, 1000)
    keys = torch.from_numpy(morton.encode_array(i, j).astype(np.int32))
    for off in (0, 4, 256, 1500):
        got = parallel.shift_keys(keys, off).numpy().astype(np.uint64)
        assert np.array_equal(got, morton.encode_array(i + off, j))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_of_oracle_tree(t: O.OracleTree, r0: int, r1: int) -> parallel.PackedShard:
    ii, jj = np.nonzero(t.slot >= 0)
    sel = (ii >= r0) & (ii < r1)
    ii, jj = ii[sel], jj[sel]
    order = np.argsort(morton.encode_array(ii, jj), kind="stable")     # a rank's store is in Morton order
    ii, jj = ii[order], jj[order]
    slots = t.slot[ii, jj]
    rec = np.zeros((slots.size, 272), np.float32)
    rec[:, :256] = t.values[slots].reshape(-1, 256)
    rec[:, 256:] = t.subnorms[slots].transpose(0, 2, 1).reshape(-1, 16)
    sq = t.sq_levels[O.level_offset(t.depth):].reshape(t.L, t.L)[ii, jj]
    return parallel.PackedShard(torch.from_numpy(morton.encode_array(ii, jj).astype(np.int32)),
                                torch.from_numpy(rec), torch.from_numpy(np.ascontiguousarray(sq)))


def _worker(rank: int, world: int, port: int, n: int, tau: float, out_dir: str):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = inputs.exponential_decay(n, 0.9, seed=3)
        full = O.tree_from_dense(a)
        nrows = -(-n // 16)
        r0, r1 = parallel.even_row_split(nrows, world)[rank]
        mine = _shard_of_oracle_tree(full, r0, r1)
        raw = parallel.allgather_shards(mine)                           # the one exchange step
        # every rank's part sits at a fixed stride; the unused slots behind a part carry the HOLE key
        assert raw.n % world == 0 and int((raw.keys != parallel.HOLE).sum()) == full.keys.size
        part = raw.keys.numpy().reshape(world, -1)
        for r in range(world):
            used = part[r] != parallel.HOLE
            assert not used[np.argmin(used):].any() or used.all()         # holes only at the end of a part
        gathered = parallel.drop_holes(raw)
        # the gathered leaves are exactly the stored leaves of the whole matrix, with their norms
        order = np.argsort(gathered.keys.numpy().astype(np.uint64), kind="stable")
        assert np.array_equal(gathered.keys.numpy().astype(np.uint64)[order], full.keys.astype(np.uint64))
        assert np.array_equal(gathered.records.numpy()[order][:, :256].reshape(-1, 16, 16), full.values)
        assert np.array_equal(gathered.records.numpy()[order][:, 256:].reshape(-1, 4, 4).transpose(0, 2, 1), full.subnorms)
        # every 4x4 block of leaves arrived contiguous and in Morton order (what the bulk copies need)
        k = gathered.keys.numpy().astype(np.int64)
        same_block = (k[1:] >> 4) == (k[:-1] >> 4)
        assert np.all(k[1:][same_block] > k[:-1][same_block])
        blocks = k >> 4
        starts = np.flatnonzero(np.r_[True, blocks[1:] != blocks[:-1]])
        assert np.unique(blocks[starts]).size == starts.size          # one run per block
        # band-limited exchange: ask only for the leaf rows of B that the local columns of A reach
        splits = parallel.even_row_split(nrows, world)
        need = parallel.needed_rows(mine, nrows)
        part = parallel.exchange_needed_rows(mine, need, splits)
        cols = np.unique(np.nonzero(full.slot[r0:r1] >= 0)[1])                  # leaf columns of my A rows
        want_rows = np.unique(np.concatenate([np.arange(4 * (c // 4), min(nrows, 4 * (c // 4) + 4)) for c in cols]))
        assert np.array_equal(np.flatnonzero(need.numpy()), want_rows)
        pi, pj = morton.decode_array(part.keys.numpy().astype(np.uint64))
        fi, fj = np.nonzero(full.slot >= 0)
        sel = np.isin(fi, want_rows)
        assert sorted(zip(pi.tolist(), pj.tolist())) == sorted(zip(fi[sel].tolist(), fj[sel].tolist()))
        assert np.array_equal(part.records.numpy()[:, :256].reshape(-1, 16, 16),
                              full.values[full.slot[pi.astype(np.int64), pj.astype(np.int64)]])
        sq_grid = full.sq_levels[O.level_offset(full.depth):].reshape(full.L, full.L)
        assert np.array_equal(part.leaf_sq.numpy(), sq_grid[pi.astype(np.int64), pj.astype(np.int64)])
        pk = part.keys.numpy().astype(np.int64)
        same_block = (pk[1:] >> 4) == (pk[:-1] >> 4)
        assert np.all(pk[1:][same_block] > pk[:-1][same_block])                 # blocks stay in Morton order
        # balance on the replicated norms, then compute this rank's row block with the oracle
        plan = O.build_plan(full, full, tau)
        counts = np.bincount(plan.ti, minlength=nrows)
        c0, c1 = parallel.balanced_row_split(counts, world)[rank]
        sel = (plan.ti >= c0) & (plan.ti < c1)
        sub = O.OraclePlan(plan.ti[sel], plan.tk[sel], plan.tj[sel], plan.norm_product[sel], tau)
        c, k4 = O.execute_plan(sub, full, full, None, tau)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), rows=np.array([c0, c1]), dense=c.to_dense(),
                 tasks=np.stack([sub.ti, sub.tk, sub.tj], axis=1), products4=k4.products4)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_split_reproduces_single_process_product(tmp_path):
    n, tau, world = 384, 1e-6, 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, tau, str(tmp_path)), nprocs=world, join=True)
    a = inputs.exponential_decay(n, 0.9, seed=3)
    full = O.tree_from_dense(a)
    c_ref, plan, k_ref = O.multiply(full, full, tau)
    dense_ref = c_ref.to_dense()
    got = np.zeros_like(dense_ref)
    tasks, p4, covered = [], 0, 0
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        c0, c1 = z["rows"]
        assert c0 == covered
        covered = c1
        got[c0 * 16:c1 * 16] = z["dense"][c0 * 16:c1 * 16]
        assert not z["dense"][:c0 * 16].any() and not z["dense"][c1 * 16:].any()   # nothing outside its rows
        tasks.append(z["tasks"])
        p4 += int(z["products4"])
    assert covered == -(-n // 16)
    assert np.array_equal(got, dense_ref)                                   # bitwise, any number of ranks
    allt = np.concatenate(tasks)
    ref = np.stack([plan.ti, plan.tk, plan.tj], axis=1)
    assert np.array_equal(allt[np.lexsort(allt.T[::-1])], ref[np.lexsort(ref.T[::-1])])
    assert p4 == k_ref.products4


def test_interior_rows_need_nothing_from_other_ranks():
    """ShardedMultiply's overlap: the tasks of the interior rows of a rank's block only touch rows of B
    the rank holds itself (checked against the oracle's task list), and the run is maximal."""
    n, tau = 1024, 1e-6
    a = inputs.exponential_decay(n, 0.8, seed=4)
    full = O.tree_from_dense(a)
    plan = O.build_plan(full, full, tau)
    nrows = n // 16
    whole = _shard_of_oracle_tree(full, 0, nrows)
    rowmax = parallel.row_max_norms(whole, nrows)
    assert np.array_equal(rowmax.numpy(), np.where(full.leaf_norm.max(axis=1) > 0, full.leaf_norm.max(axis=1), 0).astype(np.float32))
    for world in (2, 3):
        splits = parallel.even_row_split(nrows, world)
        for rank, (r0, r1) in enumerate(splits):
            mine = _shard_of_oracle_tree(full, r0, r1)
            reach = parallel.reaching_leaves(mine, rowmax, tau)
            # exactly the stored leaves of A that occur in a task
            mi, mk = morton.decode_array(mine.keys.numpy().astype(np.uint64))
            in_task = set(zip(plan.ti.tolist(), plan.tk.tolist()))
            assert [(int(i), int(k)) in in_task for i, k in zip(mi, mk)] == reach.tolist()
            i0, i1 = parallel.interior_rows(mine, (r0, r1), splits[rank], reach)
            assert r0 <= i0 <= i1 <= r1 and i0 % parallel.ROW_ALIGN == 0 and (i1 % parallel.ROW_ALIGN == 0 or i1 == r1)
            assert i1 > i0, "a banded matrix has interior rows"
            sel = (plan.ti >= i0) & (plan.ti < i1)
            assert plan.tk[sel].min() >= r0 and plan.tk[sel].max() < r1
            # maximal: the aligned groups just outside the run have a task that reaches a foreign row
            for g0 in (i0 - parallel.ROW_ALIGN, i1):
                if r0 <= g0 and g0 + parallel.ROW_ALIGN <= r1:
                    sel = (plan.ti >= g0) & (plan.ti < g0 + parallel.ROW_ALIGN)
                    assert plan.tk[sel].min() < r0 or plan.tk[sel].max() >= r1
            # the band-limited exchange asks for exactly the (aligned) rows of B the tasks touch
            need = parallel.needed_rows(mine, nrows, reach).numpy()
            sel = (plan.ti >= r0) & (plan.ti < r1)
            want = np.zeros(nrows, bool)
            want[np.unique(plan.tk[sel])] = True
            want = want.reshape(-1, parallel.ROW_ALIGN).any(axis=1).repeat(parallel.ROW_ALIGN)
            assert np.array_equal(need, want)


def _layout_worker(rank: int, world: int, port: int, n: int):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = inputs.exponential_decay(n, 0.9, seed=3)
        full = O.tree_from_dense(a)
        nrows = -(-n // 16)
        splits = parallel.even_row_split(nrows, world)
        r0, r1 = splits[rank]
        mine = _shard_of_oracle_tree(full, r0, r1)
        # the prepared (host-sync-free) forms move exactly what the one-shot forms move, and can be reused
        want = parallel.allgather_shards(mine)
        lay = parallel.gather_layout(mine)
        for _ in range(2):
            got = parallel.allgather_with_layout(mine, lay)
            assert torch.equal(got.keys, want.keys) and torch.equal(got.leaf_sq, want.leaf_sq)
            used = want.keys != parallel.HOLE
            assert torch.equal(got.records[used], want.records[used])
        got, works = parallel.allgather_with_layout(mine, lay, async_op=True)
        for w in works:
            w.wait()
        assert torch.equal(got.keys, want.keys)
        need = parallel.needed_rows(mine, nrows)
        want = parallel.exchange_needed_rows(mine, need, splits)
        nl = parallel.needed_layout(mine, need, splits)
        for _ in range(2):
            got = parallel.exchange_with_layout(mine, nl)
            assert torch.equal(got.keys, want.keys) and torch.equal(got.records, want.records)
            assert torch.equal(got.leaf_sq, want.leaf_sq)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_prepared_exchanges_match_the_one_shot_ones():
    mp.spawn(_layout_worker, args=(2, _free_port(), 384), nprocs=2, join=True)
