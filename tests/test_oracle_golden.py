"""Pins the CPU oracle (oracle/spamm_oracle.c) to the unmodified reference.

Every array the reference produced for the cases in tests/golden/cases.py is
compared bit for bit (in full for small cases, by SHA-256 for large ones):
packed leaves, sub-block / leaf / interior norms, plan order, norm products,
stats, plan dump, fine4 masks, recursive visit set, counters and the product.
"""

import hashlib

import numpy as np
import pytest

from helpers import CASES, build_inputs, check_oracle_tree, digest, golden, oracle_operands
from oracle import oracle as O


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(case):
    g = golden()
    name = case["name"]
    qa, qb, c0, (a_d, b_d, _) = oracle_operands(case)
    assert digest(a_d) == g.get(name, "in_a_sha"), "input generator drifted from the fixture"
    if b_d is not None:
        assert digest(b_d) == g.get(name, "in_b_sha")
    check_oracle_tree(g, name, "A_", qa)
    check_oracle_tree(g, name, "B_", qb)
    for run in case["runs"]:
        tag, tau = run["tag"], run["tau"]
        gran = run.get("granularity", "fine4")
        plan = O.build_plan(qa, qb, tau)
        assert len(plan) == g.get(name, f"{tag}/T")
        assert [plan.emitted, plan.examined, plan.pruned] == g.get(name, f"{tag}/stats").tolist()
        assert digest(plan.a_keys) == g.get(name, f"{tag}/akeys_sha"), "plan order (A keys)"
        assert digest(plan.b_keys) == g.get(name, f"{tag}/bkeys_sha"), "plan order (B keys)"
        assert digest(plan.norm_product) == g.get(name, f"{tag}/prods_sha")
        assert hashlib.sha256(plan.dump().encode()).hexdigest() == g.get(name, f"{tag}/dump_sha")
        masks = O.task_masks(qa, qb, plan, tau)
        assert digest(masks) == g.get(name, f"{tag}/masks_sha"), "fine4 masks"
        if run.get("recursive"):
            rec = O.recursive_tasks(qa, qb, tau)
            pairs = np.stack([O.encode(rec[:, 0], rec[:, 1]), O.encode(rec[:, 1], rec[:, 2])], axis=1)
            pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]
            assert digest(pairs.astype(np.uint64).reshape(-1, 2)) == g.get(name, f"{tag}/recursive_sha")
            # recursion == flat plan (test_reference.py:107-113)
            assert g.get(name, f"{tag}/recursive_sha") == g.get(name, f"{tag}/pairs_sorted_sha")
        c_in = c0 if run.get("use_c") else None
        c, counters = O.execute_plan(plan, qa, qb, c_in, tau, gran,
                                     run.get("alpha", 1.0), run.get("beta", 0.0))
        assert counters.products4 == g.get(name, f"{tag}/products4")
        assert counters.skipped4 == g.get(name, f"{tag}/skipped4")
        check_oracle_tree(g, name, f"{tag}/C_", c)
        assert digest(c.to_dense()) == g.get(name, f"{tag}/C_dense_sha"), "product values"


def test_known_answers_from_reference_tests():
    """KATs held by the reference's own tests for this path."""
    # tests/test_core.py:21-26
    assert [O.tree_depth(*mn) for mn in ((16, 16), (17, 17), (7500, 7500), (1, 1000))] == [0, 1, 9, 6]
    # tests/test_morton.py:25-30 (row bit high)
    assert int(O.encode(1, 0)) == 2 and int(O.encode(0, 1)) == 1 and int(O.encode(3, 5)) == 0b011011
    # tests/test_symbolic.py:73-91: pinned plan order and dump on constant blocks
    def blocks(layout):
        a = np.zeros((32, 32), np.float32)
        for (bi, bj), v in layout.items():
            a[16 * bi:16 * bi + 16, 16 * bj:16 * bj + 16] = v
        return O.tree_from_dense(a)
    a = blocks({(0, 0): 0.25, (0, 1): 0.5, (1, 0): 1.0})
    b = blocks({(0, 0): 0.25, (1, 0): 0.125, (1, 1): 0.5})
    assert a.leaf_norm[1, 0] == 16.0
    assert O.build_plan(a, b, 0.0).dump() == (
        "2 0 2 6.400000000e+01\n0 0 0 1.600000000e+01\n1 3 1 6.400000000e+01\n1 2 0 1.600000000e+01\n")
    pruned = O.build_plan(a, b, 32.0)
    assert pruned.dump() == "2 0 2 6.400000000e+01\n1 3 1 6.400000000e+01\n"
    assert (pruned.emitted, pruned.examined, pruned.pruned) == (2, 4, 2)
    # tests/test_core.py:90-96 style exact norms: a 3-4 pair gives 5
    d = np.zeros((16, 16), np.float32)
    d[0, 0], d[5, 9] = 3.0, 4.0
    t = O.tree_from_dense(d)
    assert t.norm == 5.0 and t.subnorms[0, 0, 0] == 3.0 and t.subnorms[0, 1, 2] == 4.0
    # tests/test_numeric.py:89-100: one live sub-block -> products4 = 1, skipped4 = 63
    av = np.zeros((16, 16), np.float32)
    bv = np.zeros((16, 16), np.float32)
    rng = np.random.default_rng(6)
    av[:4, :4] = rng.random((4, 4))
    bv[:4, :4] = rng.random((4, 4))
    _, _, k = O.multiply(O.tree_from_dense(av), O.tree_from_dense(bv), 1e-30)
    assert (k.products4, k.skipped4) == (1, 63)


def test_tau_boundary_and_validation():
    # tests/test_symbolic.py:109-113: p == tau survives
    a = np.zeros((16, 16), np.float32)
    b = np.zeros((16, 16), np.float32)
    a[0, 0], b[0, 0] = 2.0, 3.0
    ta, tb = O.tree_from_dense(a), O.tree_from_dense(b)
    assert len(O.build_plan(ta, tb, 6.0)) == 1
    assert len(O.build_plan(ta, tb, 6.0 + 1e-12)) == 0
    for bad in (-1.0, float("nan")):
        with pytest.raises(ValueError):
            O.build_plan(ta, tb, bad)
    with pytest.raises(ValueError):
        O.build_plan(ta, O.tree_from_dense(np.ones((32, 16), np.float32)), 0.0)


def test_tau_zero_equals_naive_single_product():
    # tests/test_numeric.py:199-207
    rng = np.random.default_rng(5)
    a = (rng.random((80, 48)) * 2 - 1).astype(np.float32)
    b = (rng.random((48, 33)) * 2 - 1).astype(np.float32)
    c, plan, k = O.multiply(O.tree_from_dense(a), O.tree_from_dense(b))
    assert np.array_equal(c.to_dense(), O.dense_multiply_single(a, b))
    assert k.products4 == 64 * len(plan) and k.skipped4 == 0
