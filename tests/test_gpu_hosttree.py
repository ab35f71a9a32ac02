"""Operands that stay in host memory (paper_1203_1692_b200.hosttree): the device gets keys, norms and sub-block
norms, plans, and fetches only the leaves a surviving task reads.  The product must equal the one of fully
resident trees bit for bit (EXACT mode), for C = A A and C = A B, and the leaves fetched must be exactly the
leaves that occur in a task (counted from the oracle's plan).  The reference side is `core.py:387-405`
(packed_leaves) and `numeric.py:302-313` (multiply)."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _touched(oplan):
    return np.unique(oplan.a_keys).size, np.unique(oplan.b_keys).size


@pytest.mark.parametrize("n,lam,tau,gran", [(256, 0.8, 1e-5, "fine4"), (1000, 0.9, 1e-6, "fine4"), (2048, 0.95, 1e-8, "coarse16")])
def test_host_resident_square(n, lam, tau, gran):
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(n, lam, seed=7)
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau, granularity=gran, exact=True)
    want, wplan, wk = P.multiply(qa, qa, cfg)
    ha = P.HostTree.from_device(qa)
    assert ha.nleaf == qa.nleaf and ha.blocks.is_pinned()
    for _ in range(2):
        c, plan, k, fetched = P.multiply_host(ha, None, cfg)
        assert len(plan) == len(wplan) and k.products4 == wk.products4
        for x, y in zip(c.packed_leaves(), want.packed_leaves()):
            assert np.array_equal(x, y)
        for tier in range(want.depth + 1):
            assert np.array_equal(c.level_norms(tier), want.level_norms(tier))
    oa = O.tree_from_dense(a)
    oplan = O.build_plan(oa, oa, tau)
    both = np.unique(np.concatenate([oplan.a_keys, oplan.b_keys])).size
    assert int(fetched[0].item()) == both, "exactly the leaves that occur in a task are fetched"
    assert both <= ha.nleaf


def test_host_resident_two_operands():
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    n, tau = 1024, 1e-6
    a, b = inputs.algebraic_decay(n, seed=0), inputs.algebraic_decay(n, seed=1)
    qa, qb = P.QuadtreeMatrix.from_dense(a), P.QuadtreeMatrix.from_dense(b)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    want, wplan, wk = P.multiply(qa, qb, cfg)
    ha, hb = P.HostTree.from_device(qa), P.HostTree.from_device(qb)
    c, plan, k, fetched = P.multiply_host(ha, hb, cfg)
    assert len(plan) == len(wplan) and k.products4 == wk.products4
    for x, y in zip(c.packed_leaves(), want.packed_leaves()):
        assert np.array_equal(x, y)
    oa, ob = O.tree_from_dense(a), O.tree_from_dense(b)
    oplan = O.build_plan(oa, ob, tau)
    ta, tb = _touched(oplan)
    assert (int(fetched[0].item()), int(fetched[1].item())) == (ta, tb)
    with pytest.raises(ValueError):
        P.multiply_host(ha, hb, P.MultiplyConfig(tau=tau, beta=1.0))


@pytest.mark.parametrize("parts", [2, 3])
def test_host_resident_in_row_blocks(parts):
    """multiply_host_parts: the product in blocks of leaf rows, each enqueued behind the other; together they are the
    product of fully resident trees, bit for bit, on the first call (plan + execute) and on the fused repeat."""
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    n, tau = 2048, 1e-7
    a = inputs.exponential_decay(n, 0.93, seed=3)
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    want, wplan, wk = P.multiply(qa, qa, cfg)
    wd = want.to_dense().data
    ha = P.HostTree.from_device(qa)
    for rep in range(3):
        seen = []
        res = P.multiply_host_parts(ha, None, cfg, parts=parts, on_part=lambda p: seen.append(p[0]))
        assert [p[0] for p in res] == seen and len(res) == parts
        assert res[0][0][0] == 0 and res[-1][0][1] == 128 and all(x[0][1] == y[0][0] for x, y in zip(res[:-1], res[1:]))
        got = np.zeros_like(wd)
        for (r0, r1), c, plan, k, fetched in res:
            assert r0 % 4 == 0
            d = c.to_dense().data
            assert not d[: r0 * 16].any() and not d[r1 * 16:].any(), "a block holds its rows only"
            got[r0 * 16:r1 * 16] = d[r0 * 16:r1 * 16]
        assert np.array_equal(got, wd), f"repetition {rep}"
        assert sum(len(p[2]) for p in res) == len(wplan) and sum(p[3].products4 for p in res) == wk.products4
