"""Parity of the CUDA path (through the C ABI) with the reference and the oracle.

Every golden case of tests/golden/cases.py is replayed on the device:
  * trees: packed leaves, sub-norms, leaf and interior norms       -- bit exact vs the reference
  * plan: task set, fine4 masks, plan order, stats, dump           -- bit exact
  * product, EXACT rounding mode: leaves, values, norms, counters  -- bit exact
  * product, FMA mode: max |C - C_ref| / max |C_ref| <= 1e-5        -- north_star tolerance
"""

import hashlib

import numpy as np
import pytest

from helpers import (CASES, assert_trees_equal, build_inputs, check_device_tree, digest, golden,
                     oracle_operands)
from oracle import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5   # BASELINE.json north_star: C within 1e-5 relative max-norm of the reference output


def device_operands(case):
    import paper_1203_1692_b200 as P
    a_d, b_d, c_d = build_inputs(case)
    qa = P.QuadtreeMatrix.from_dense(a_d)
    qb = qa if b_d is None else P.QuadtreeMatrix.from_dense(b_d)
    if case.get("chain"):
        prod, _, _ = P.multiply(qa, qb, P.MultiplyConfig(tau=0.0, exact=True))
        qa = qb = prod
    return qa, qb, c_d


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_matches_reference(case):
    import paper_1203_1692_b200 as P
    g = golden()
    name = case["name"]
    qa, qb, c_d = device_operands(case)
    oa, ob, oc0, _ = oracle_operands(case)
    check_device_tree(g, name, "A_", qa)
    check_device_tree(g, name, "B_", qb)
    assert_trees_equal(qa, oa, "A")
    for run in case["runs"]:
        tag, tau = run["tag"], run["tau"]
        gran = run.get("granularity", "fine4")
        alpha, beta = run.get("alpha", 1.0), run.get("beta", 0.0)
        # ---- symbolic phase
        plan = P.build_plan(qa, qb, tau)
        assert len(plan) == g.get(name, f"{tag}/T")
        ka, kb = plan.pair_keys()
        pairs = np.stack([ka, kb], axis=1)
        order = np.lexsort((pairs[:, 1], pairs[:, 0]))
        assert digest(pairs[order].astype(np.uint64).reshape(-1, 2)) == g.get(name, f"{tag}/pairs_sorted_sha"), "task set"
        oplan = O.build_plan(oa, ob, tau)
        if gran == "fine4" and len(plan):
            omask = dict(zip(zip(oplan.a_keys.tolist(), oplan.b_keys.tolist()), O.task_masks(oa, ob, oplan, tau).tolist()))
            got = plan.masks()
            want = np.array([omask[(a, b)] for a, b in zip(ka.tolist(), kb.tolist())], np.uint64)
            assert np.array_equal(got, want), "fine4 masks"
            # the gate as the numeric kernel itself evaluated it (planner classification + per-lane
            # products in execute_kernel), not a host recomputation
            assert np.array_equal(plan.device_masks(), want), "fine4 masks evaluated by the device gate"
            full, dead = plan.classification()
            assert np.all(want[full] == np.uint64(0xFFFFFFFFFFFFFFFF)), "a task classified 'all pass' has a failing micro product"
            assert np.all(want[dead] == 0), "a task classified 'none passes' has a passing micro product"
            assert not np.any(full & dead)
        # ascending k inside every product leaf, leaves in ascending Morton order
        t = plan.ikj()
        if len(plan):
            ck = P.morton.encode_array(t[:, 0], t[:, 2]).astype(np.int64)
            assert np.all(np.diff(ck) >= 0)
            same = np.diff(ck) == 0
            assert np.all(np.diff(t[:, 1])[same] > 0)
        # reference plan order, stats and dump
        tasks = plan.tasks
        assert digest(np.array([x.a for x in tasks], np.uint64)) == g.get(name, f"{tag}/akeys_sha"), "plan order"
        assert digest(np.array([x.b for x in tasks], np.uint64)) == g.get(name, f"{tag}/bkeys_sha"), "plan order"
        assert digest(np.array([x.norm_product for x in tasks], np.float64)) == g.get(name, f"{tag}/prods_sha")
        st = plan.stats
        assert [st.emitted, st.examined, st.pruned] == g.get(name, f"{tag}/stats").tolist()
        assert hashlib.sha256(P.plan_dump(plan).encode()).hexdigest() == g.get(name, f"{tag}/dump_sha")
        # ---- numeric phase, exact rounding: bit for bit
        def c_in():
            return P.QuadtreeMatrix.from_dense(c_d) if (run.get("use_c") and c_d is not None) else None
        cfg = P.MultiplyConfig(tau=tau, granularity=gran, alpha=alpha, beta=beta, exact=True)
        c, counters = P.execute_plan(plan, qa, qb, c_in(), cfg)
        assert counters.products4 == g.get(name, f"{tag}/products4")
        assert counters.skipped4 == g.get(name, f"{tag}/skipped4")
        check_device_tree(g, name, f"{tag}/C_", c)
        cd = c.to_dense().data
        assert digest(cd) == g.get(name, f"{tag}/C_dense_sha"), "product values (exact mode)"
        # ---- numeric phase, FMA: tolerance
        cfg = P.MultiplyConfig(tau=tau, granularity=gran, alpha=alpha, beta=beta)
        c2, k2 = P.execute_plan(plan, qa, qb, c_in(), cfg)
        cd2 = c2.to_dense().data
        scale = float(np.abs(cd).max())
        if scale > 0:
            assert float(np.abs(cd2.astype(np.float64) - cd).max()) <= REL_TOL * scale
        assert k2.products4 == counters.products4
        assert np.array_equal(c2.leaf_keys(), c.leaf_keys())


def test_validation_errors_match_reference():
    import paper_1203_1692_b200 as P
    a = P.QuadtreeMatrix.from_dense(np.ones((32, 32), np.float32))
    with pytest.raises(ValueError):
        P.build_plan(a, P.QuadtreeMatrix(64, 32), 0.0)            # inner dimensions
    for bad in (-1.0, float("nan")):
        with pytest.raises(ValueError):
            P.build_plan(a, a, bad)
    plan = P.build_plan(a, a, 1e-8)
    with pytest.raises(ValueError, match="tau"):
        P.execute_plan(plan, a, a, None, P.MultiplyConfig(tau=1e-6))
    plan0 = P.build_plan(a, a, 0.0)
    with pytest.raises(ValueError, match="accumulator"):
        P.execute_plan(plan0, a, a, P.QuadtreeMatrix(16, 16), P.MultiplyConfig())
    b = P.QuadtreeMatrix.from_dense(np.ones((32, 32), np.float32))
    with pytest.raises(ValueError, match="stale"):
        P.execute_plan(plan0, b, b, None, P.MultiplyConfig())
    with pytest.raises(ValueError):
        P.QuadtreeMatrix.from_dense(np.ones((32, 32), np.float32), 8)   # the device path is n_b = 16 only
    with pytest.raises(ValueError):
        P.QuadtreeMatrix(32, 32, 12)


def test_empty_operands_and_beta_keep():
    import paper_1203_1692_b200 as P
    empty = P.QuadtreeMatrix(32, 32)
    rng = np.random.default_rng(27)
    c0_dense = (rng.random((32, 32)) * 2 - 1).astype(np.float32)
    c0 = P.QuadtreeMatrix.from_dense(c0_dense)
    plan = P.build_plan(empty, empty, 0.0)
    assert len(plan) == 0 and P.plan_dump(plan) == ""
    out, k = P.execute_plan(plan, empty, empty, c0, P.MultiplyConfig(beta=1.0))
    assert out is c0 and np.array_equal(out.to_dense().data, c0_dense)
    assert (k.products4, k.skipped4) == (0, 0)
    out2, _, _ = P.multiply(empty, empty)
    assert out2.leaf_count == 0 and out2.norm == 0.0


def test_put_leaf_compute_norms_equals_from_dense():
    # tests/test_core.py:215-226 of the reference, through the device kernels
    import paper_1203_1692_b200 as P
    rng = np.random.default_rng(3)
    d = (rng.random((80, 80)) * 2 - 1).astype(np.float32)
    d[16:48, 32:64] = 0
    q = P.QuadtreeMatrix.from_dense(d)
    keys, vals, _ = q.packed_leaves()
    r = P.QuadtreeMatrix(80, 80)
    for k, v in reversed(list(zip(keys.tolist(), vals))):
        r.put_leaf(k, v)
    r.compute_norms()
    assert np.array_equal(r.packed_leaves()[0], keys)
    assert np.array_equal(r.to_dense().data, d)
    want = O.tree_from_packed(80, 80, *[x.astype(np.int64) for x in P.morton.decode_array(keys)], vals)
    assert_trees_equal(r, want, "put_leaf tree")
