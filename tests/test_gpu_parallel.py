"""Row-block sharding on the device, emulated on one GPU by running the ranks one after another
(never concurrently): shards -> gathered tree -> per-rank row_range multiply.  The union of the
per-rank products must be bit-identical to the single-GPU product, for any number of ranks."""

import numpy as np
import pytest
import torch

from paper_1203_1692_b200 import inputs, parallel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_row_blocks_reproduce_single_gpu_product(world):
    import paper_1203_1692_b200 as P
    n, tau = 1024, 1e-6
    a = inputs.exponential_decay(n, 0.9, seed=0)
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau)
    c_ref, plan_ref, k_ref = P.multiply(qa, qa, cfg)
    dense_ref = c_ref.to_dense().data
    nrows = n // 16
    # what the ranks would hold, and what the all-gather would deliver (rank order)
    shards = [parallel.shard_from_dense_rows(a[r0 * 16:r1 * 16], r0) for r0, r1 in parallel.even_row_split(nrows, world)]
    gathered = parallel.PackedShard(torch.cat([s.keys for s in shards]), torch.cat([s.records for s in shards]),
                                    torch.cat([s.leaf_sq for s in shards]))
    full = parallel.tree_from_shard(n, n, gathered)
    # the gathered tree is the same matrix with the same norms
    assert np.array_equal(full.to_dense().data, a)
    for t in range(qa.depth + 1):
        assert np.array_equal(full.level_norms(t), qa.level_norms(t))
    plan = P.build_plan(full, full, tau)
    assert len(plan) == len(plan_ref)
    counts = parallel.row_task_counts(plan, plan.depth).cpu().numpy()
    assert counts.sum() == len(plan)
    assert np.array_equal(counts, np.bincount(plan.ikj()[:, 0], minlength=counts.size))
    split = parallel.balanced_row_split(counts[:nrows], world)
    got = np.zeros_like(dense_ref)
    total_tasks = total_p4 = 0
    for r0, r1 in split:
        c, p, k = P.numeric.multiply_async(full, full, cfg, None, row_range=(r0, r1))
        d = c.to_dense().data
        assert not d[:r0 * 16].any() and not d[r1 * 16:].any()
        got[r0 * 16:r1 * 16] = d[r0 * 16:r1 * 16]
        total_tasks += len(p)
        total_p4 += k.products4
        rows = p.ikj()[:, 0]
        assert rows.size == 0 or (rows.min() >= r0 and rows.max() < r1)
    assert total_tasks == len(plan_ref) and total_p4 == k_ref.products4
    assert np.array_equal(got, dense_ref)
    loads = np.array([counts[r0:r1].sum() for r0, r1 in split])
    assert loads.max() <= 1.35 * loads.mean()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_local_rows_of_a_times_gathered_b(world):
    """parallel.multiply_sharded's data flow without the collective: every rank multiplies a tree of
    its own rows of A by B rebuilt from the gathered buffer (fixed stride per rank, HOLE keys in
    the unused slots, no transposed copies) and gets exactly its rows of the single-GPU product."""
    import paper_1203_1692_b200 as P
    n, tau = 1000, 1e-6                       # ragged: 62.5 leaf rows
    a = inputs.exponential_decay(n, 0.9, seed=2)
    b = inputs.exponential_decay(n, 0.93, seed=5)
    qa, qb = P.QuadtreeMatrix.from_dense(a), P.QuadtreeMatrix.from_dense(b)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    c_ref, plan_ref, k_ref = P.multiply(qa, qb, cfg)
    dense_ref = c_ref.to_dense().data
    nrows = -(-n // 16)
    split = parallel.even_row_split(nrows, world)
    b_shards = [parallel.shard_of_tree(qb, r0, r1) for r0, r1 in split]
    cap = max(s.n for s in b_shards)
    dev = b_shards[0].keys.device
    keys = torch.full((world * cap,), parallel.HOLE, dtype=torch.int32, device=dev)
    recs = torch.full((world * cap, 272), float("nan"), dtype=torch.float32, device=dev)   # garbage must never be read
    sq = torch.zeros((world * cap,), dtype=torch.float64, device=dev)
    for r, s in enumerate(b_shards):
        keys[r * cap:r * cap + s.n] = s.keys
        recs[r * cap:r * cap + s.n] = s.records
        sq[r * cap:r * cap + s.n] = s.leaf_sq
    b_full = parallel.tree_from_shard(n, n, parallel.PackedShard(keys, recs, sq), transposed=False)
    assert np.array_equal(b_full.to_dense().data, b)
    bk, bv, bs = b_full.packed_leaves()
    rk, rv, rs = qb.packed_leaves()
    assert np.array_equal(bk, rk) and np.array_equal(bv, rv) and np.array_equal(bs, rs)
    got = np.zeros_like(dense_ref)
    tasks = p4 = 0
    for r0, r1 in split:
        a_local = parallel.tree_from_shard(n, n, parallel.shard_of_tree(qa, r0, r1))
        c, p, k = P.numeric.multiply_async(a_local, b_full, cfg, None)
        d = c.to_dense().data
        assert not d[:r0 * 16].any() and not d[r1 * 16:].any()
        got[r0 * 16:r1 * 16] = d[r0 * 16:r1 * 16]
        tasks += len(p)
        p4 += k.products4
    assert tasks == len(plan_ref) and p4 == k_ref.products4
    assert np.array_equal(got, dense_ref)
    # a right-hand-only tree still works on the left: the transposed copies are made on first use
    c2, _, _ = P.multiply(b_full, qa, P.MultiplyConfig(tau=tau, exact=True))
    c3, _, _ = P.multiply(qb, qa, P.MultiplyConfig(tau=tau, exact=True))
    assert np.array_equal(c2.to_dense().data, c3.to_dense().data)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_band_limited_exchange_gives_the_same_rows(world):
    """exchange="needed": a rank multiplies its rows of A by ONLY the leaf rows of B its columns
    reach (what parallel.exchange_needed_rows delivers, pieces in owner order).  Rows of C must be
    bit-identical to the single-GPU product, and for a banded matrix most of B is never fetched."""
    import paper_1203_1692_b200 as P
    n, tau = 2048, 1e-6
    a = inputs.exponential_decay(n, 0.5, seed=0)            # narrow band: entries underflow ~150 columns out
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    c_ref, plan_ref, k_ref = P.multiply(qa, qa, cfg)
    dense_ref = c_ref.to_dense().data
    nrows = n // 16
    split = parallel.even_row_split(nrows, world)
    shards = [parallel.shard_of_tree(qa, r0, r1) for r0, r1 in split]
    got = np.zeros_like(dense_ref)
    tasks = fetched = 0
    for rank, (r0, r1) in enumerate(split):
        need = parallel.needed_rows(shards[rank], nrows)
        rows_of = [parallel._squeeze16(s.keys.to(torch.int64) >> 1) for s in shards]
        pieces = [torch.nonzero(need[rows_of[src]]).flatten() for src in range(world)]
        part = parallel.PackedShard(torch.cat([shards[s].keys[pieces[s]] for s in range(world)]),
                                    torch.cat([shards[s].records[pieces[s]] for s in range(world)]),
                                    torch.cat([shards[s].leaf_sq[pieces[s]] for s in range(world)]))
        fetched += part.n - int(pieces[rank].numel())
        b_part = parallel.tree_from_shard(n, n, part, transposed=False)
        a_local = parallel.tree_from_shard(n, n, shards[rank])
        c, p, k = P.numeric.multiply_async(a_local, b_part, cfg, None)
        d = c.to_dense().data
        got[r0 * 16:r1 * 16] = d[r0 * 16:r1 * 16]
        assert not d[:r0 * 16].any() and not d[r1 * 16:].any()
        tasks += len(p)
    assert tasks == len(plan_ref)
    assert np.array_equal(got, dense_ref)
    if world == 8:
        assert fetched < 0.3 * (world - 1) * qa.nleaf          # an all-gather would move (world-1) * nleaf
