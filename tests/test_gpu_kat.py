"""The reference's own known-answer tests for the path, replayed through the GPU `multiply`
("These small cases should be replayed through the GPU multiply as unit tests")."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _blocks(P, layout):
    a = np.zeros((32, 32), np.float32)
    for (bi, bj), v in layout.items():
        a[16 * bi:16 * bi + 16, 16 * bj:16 * bj + 16] = v
    return P.QuadtreeMatrix.from_dense(a)


def test_plan_dump_and_stats_on_constant_blocks():
    # tests/test_symbolic.py:73-91 of the reference
    import paper_1203_1692_b200 as P
    a = _blocks(P, {(0, 0): 0.25, (0, 1): 0.5, (1, 0): 1.0})
    b = _blocks(P, {(0, 0): 0.25, (1, 0): 0.125, (1, 1): 0.5})
    assert float(a.level_norms(1)[1, 0]) == 16.0
    assert P.plan_dump(P.build_plan(a, b, 0.0)) == (
        "2 0 2 6.400000000e+01\n0 0 0 1.600000000e+01\n1 3 1 6.400000000e+01\n1 2 0 1.600000000e+01\n")
    pruned = P.build_plan(a, b, 32.0)
    assert P.plan_dump(pruned) == "2 0 2 6.400000000e+01\n1 3 1 6.400000000e+01\n"
    st = pruned.stats
    assert (st.emitted, st.examined, st.pruned) == (2, 4, 2)


def test_tau_boundary_equality_survives():
    # tests/test_symbolic.py:109-113: a task whose norm product equals tau is kept
    import paper_1203_1692_b200 as P
    a = np.zeros((16, 16), np.float32)
    b = np.zeros((16, 16), np.float32)
    a[0, 0], b[0, 0] = 2.0, 3.0
    qa, qb = P.QuadtreeMatrix.from_dense(a), P.QuadtreeMatrix.from_dense(b)
    assert len(P.build_plan(qa, qb, 6.0)) == 1
    assert len(P.build_plan(qa, qb, 6.0 + 1e-12)) == 0
    c, plan, k = P.multiply(qa, qb, P.MultiplyConfig(tau=6.0))
    assert len(plan) == 1 and k.products4 == 1 and k.skipped4 == 63        # fine4 gate: equality survives too
    assert c.to_dense().data[0, 0] == 6.0
    c, plan, k = P.multiply(qa, qb, P.MultiplyConfig(tau=np.nextafter(6.0, 7.0)))
    assert len(plan) == 0 and c.leaf_count == 0


def test_exact_norms_and_depth_pins():
    # tests/test_core.py:21-26, :90-96
    import paper_1203_1692_b200 as P
    assert [P.tree_depth(*mn) for mn in ((16, 16), (17, 17), (7500, 7500), (1, 1000))] == [0, 1, 9, 6]
    d = np.zeros((16, 16), np.float32)
    d[0, 0], d[5, 9] = 3.0, 4.0
    q = P.QuadtreeMatrix.from_dense(d)
    keys, vals, subs = q.packed_leaves()
    assert float(q.level_norms(0)[0, 0]) == 5.0 and subs[0, 0, 0] == 3.0 and subs[0, 1, 2] == 4.0


def test_one_live_sub_block_runs_one_micro_product():
    # tests/test_numeric.py:89-100
    import paper_1203_1692_b200 as P
    av = np.zeros((16, 16), np.float32)
    bv = np.zeros((16, 16), np.float32)
    rng = np.random.default_rng(6)
    av[:4, :4] = rng.random((4, 4))
    bv[:4, :4] = rng.random((4, 4))
    c, plan, k = P.multiply(P.QuadtreeMatrix.from_dense(av), P.QuadtreeMatrix.from_dense(bv),
                            P.MultiplyConfig(tau=1e-30, exact=True))
    assert (k.products4, k.skipped4) == (1, 63)
    oc, _, _ = O.multiply(O.tree_from_dense(av), O.tree_from_dense(bv), 1e-30)
    assert np.array_equal(c.to_dense().data, oc.to_dense())
    ck, plan, kc = P.multiply(P.QuadtreeMatrix.from_dense(av), P.QuadtreeMatrix.from_dense(bv),
                              P.MultiplyConfig(tau=1e-30, granularity="coarse16"))
    assert (kc.products4, kc.skipped4) == (64, 0)


def test_tau_zero_equals_naive_single_precision_product():
    # tests/test_numeric.py:199-218: tau = 0 is bit-identical to the ascending-k fp32 product
    import paper_1203_1692_b200 as P
    rng = np.random.default_rng(5)
    a = (rng.random((80, 48)) * 2 - 1).astype(np.float32)
    b = (rng.random((48, 33)) * 2 - 1).astype(np.float32)
    c, plan, k = P.multiply(P.QuadtreeMatrix.from_dense(a), P.QuadtreeMatrix.from_dense(b), P.MultiplyConfig(exact=True))
    assert np.array_equal(c.to_dense().data, O.dense_multiply_single(a, b))
    assert k.products4 == 64 * len(plan) and k.skipped4 == 0
    # accumulator is mutated in place and returned (tests/test_numeric.py:281-289)
    dirty = P.QuadtreeMatrix.from_dense(np.ones((80, 33), np.float32))
    out, _, _ = P.multiply(P.QuadtreeMatrix.from_dense(a), P.QuadtreeMatrix.from_dense(b), P.MultiplyConfig(exact=True), dirty)
    assert out is dirty and np.array_equal(dirty.to_dense().data, O.dense_multiply_single(a, b))
