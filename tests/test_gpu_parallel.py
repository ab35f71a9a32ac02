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
