"""A plan made by a coarse16 multiply carries no fine4 classification of its tasks (the planner skips it when the
gating is known, csrc/plan.cu); executed with fine4 it must still give the reference's fine4 product -- every task
is then gated per micro product by the numeric kernel itself (`numeric.py:232-238`)."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,lam,tau", [(512, 0.8, 1e-5), (2048, 0.93, 1e-7)])
def test_plan_of_a_coarse_multiply_runs_fine4(n, lam, tau):
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(n, lam, seed=4)
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg16 = P.MultiplyConfig(tau=tau, granularity="coarse16")
    P.multiply(qa, qa, cfg16)                        # the first product of a shape sizes the buffers (plan + execute)
    c16, plan, k16 = P.multiply(qa, qa, cfg16)       # the fused multiply: its planner knows the gating
    full, dead = plan.classification()
    assert not full.any() and not dead.any(), "the fused coarse16 multiply does not classify its tasks"
    fine = P.MultiplyConfig(tau=tau, granularity="fine4", exact=True) if "exact" in P.MultiplyConfig.__dataclass_fields__ \
        else P.MultiplyConfig(tau=tau, granularity="fine4")
    c4, k4 = P.execute_plan(plan, qa, qa, None, fine)
    oa = O.tree_from_dense(a)
    oc, ok = O.execute_plan(O.build_plan(oa, oa, tau), oa, oa, None, tau, "fine4")
    assert k4.products4 == ok.products4
    got = c4.to_dense().data
    if getattr(fine, "exact", False):
        assert np.array_equal(got, oc.to_dense())
    else:
        assert np.allclose(got, oc.to_dense(), rtol=1e-5, atol=1e-5 * np.abs(oc.to_dense()).max())
    # and the fused multiply with fine4 agrees with it
    c4b, _, k4b = P.multiply(qa, qa, P.MultiplyConfig(tau=tau, granularity="fine4"))
    assert k4b.products4 == ok.products4
