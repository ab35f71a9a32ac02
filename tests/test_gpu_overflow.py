"""Plan buffers that turn out too small: the multiply flags it on the device (plan counts[2]), the host repeats
it with larger buffers when it first reads the counts, and the result is the product of an undisturbed run.
Capacities come from the last product of the same shape (`symbolic.plan_capacity`), so the case arises when an
operand changes its values but not its leaf count; here the remembered capacity is made too small by hand.
Both planners: count + emit kernels (n <= 4096) and the look-back kernel (n = 8192).  The reference has no
counterpart (its lists grow on the host, `symbolic.py:92-159`)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,lam,tau", [(1024, 0.9, 1e-6), (4096, 0.95, 1e-8), (8192, 0.95, 1e-6)])
@pytest.mark.parametrize("caps", [(64, 16), (1 << 20, 16), (64, 1 << 16)])
def test_too_small_capacity_is_repeated(n, lam, tau, caps):
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs, symbolic
    a = inputs.exponential_decay(n, lam, seed=1)
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau)
    c0, p0, k0 = P.multiply(qa, qa, cfg)
    want = [x.copy() for x in c0.packed_leaves()]
    n_tasks, p4 = len(p0), k0.products4
    key, _ = symbolic.plan_capacity(qa, qa, cfg.tau, p0.depth, 0, 1 << p0.depth)
    assert key in symbolic._capacity_hint
    symbolic._capacity_hint[key] = caps                 # (step records, product leaves): one or both far too small
    c1, p1, k1 = P.multiply(qa, qa, cfg)
    assert len(p1) == n_tasks and k1.products4 == p4
    for x, y in zip(c1.packed_leaves(), want):
        assert np.array_equal(x, y)
    for tier in range(c0.depth + 1):
        assert np.array_equal(c1.level_norms(tier), c0.level_norms(tier))
    # the repeat left a capacity that fits: the next product of this shape runs once
    steps_cap, leaf_cap = symbolic._capacity_hint[key]
    assert steps_cap >= p1.n_steps and leaf_cap >= p1.n_cleaves
    c2, p2, k2 = P.multiply(qa, qa, cfg)
    assert k2.products4 == p4 and np.array_equal(c2.packed_leaves()[1], want[1])
