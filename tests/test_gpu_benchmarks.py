"""The callers of multiply the reference ships in `spamm.bench` (run_scenario, sweep, calibrate_tau),
re-hosted on the GPU path: report fields against the oracle, CSV layout, calibration contract
(`pkg/tests/test_bench.py` of the reference checks the same properties on the CPU package)."""

import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1203_1692_b200 import inputs

pytestmark = pytest.mark.gpu


def test_flop_model_pins():
    from paper_1203_1692_b200 import benchmarks as B
    assert B.flop_model(16, 16, 16) == 8192 and B.flop_model(4, 4, 4) == 128      # tests/test_reference.py:58-65
    assert B.flop_model(3, 5, 7) == 3 * (5 * (1 + 2 * 7) - 7)
    with pytest.raises(ValueError):
        B.flop_model(0, 1, 1)


def test_run_scenario_reports_match_the_oracle():
    from paper_1203_1692_b200 import benchmarks as B
    n, tau = 512, 1e-6
    a = inputs.exponential_decay(n, 0.9, seed=0)
    oa = O.tree_from_dense(a)
    ref64 = a.astype(np.float64) @ a.astype(np.float64)
    for scen, gran in (("spamm4", "fine4"), ("spamm16", "coarse16")):
        r = B.run_scenario(scen, a, tau=tau, repeats=2)
        oc, oplan, ok = O.multiply(oa, oa, tau, gran)
        assert (r.scenario, r.n, r.tau, r.granularity) == (scen, n, tau, gran)
        assert r.products4 == ok.products4 and r.complexity == ok.products4      # numeric.py:58-61
        assert r.flops_model == 2 * n ** 3 and r.seconds > 0
        assert math.isclose(r.effective_rate, r.flops_model / r.seconds)
        want = np.abs(oc.to_dense().astype(np.float64) - ref64).max()
        assert abs(r.max_norm_error - want) <= 1e-5 * np.abs(ref64).max()
    d = B.run_scenario("dense-double", a, repeats=1)
    assert d.products4 == n ** 3 // 64 and d.max_norm_error < 1e-9
    s = B.run_scenario("dense-single", a, repeats=1)
    assert s.max_norm_error < 1e-3
    with pytest.raises(ValueError):
        B.run_scenario("spamm-dense-leaf", a)
    with pytest.raises(ValueError):
        B.run_scenario("dense-single", a, alpha=2.0)
    with pytest.raises(ValueError):
        B.run_scenario("spamm4", a[:100], tau=tau)
    text = B.reports_to_csv([r, d])
    lines = text.strip().split("\n")
    assert lines[0] == B.CSV_HEADER and len(lines) == 3 and lines[1].split(",")[0] == "spamm16"
    assert len(lines[1].split(",")) == len(B.CSV_HEADER.split(","))


def test_sweep_ratio_and_slope():
    from paper_1203_1692_b200 import benchmarks as B
    reps = B.sweep(lambda n: inputs.exponential_decay(n, 0.9, seed=0), [256, 512, 1024], [1e-6], repeats=1,
                   compute_error=False)
    assert [(r.n, r.scenario) for r in reps] == [(n, s) for n in (256, 512, 1024) for s in ("spamm4", "spamm16")]
    rows = B.ratio_table(reps)
    assert len(rows) == 3 and all(c >= 1.0 for _, _, c, _ in rows)        # coarse gating never does less work
    slope = B.fitted_slope([r for r in reps if r.scenario == "spamm4"])
    assert 0.8 < slope < 1.6                                              # banded input: work grows about linearly
    assert B.ratios_to_csv(rows).startswith(B.RATIO_HEADER)
    with pytest.raises(ValueError):
        B.fitted_slope(reps[:1])


def test_calibrate_tau_contract():
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import benchmarks as B
    a = inputs.exponential_decay(512, 0.9, seed=0)
    tree = P.QuadtreeMatrix.from_dense(a)
    oracle = B.dense_multiply_double(a)
    res = B.calibrate_tau(tree, oracle, target=1e-4, iters=6)
    assert res.converged and res.error <= 1e-4 and len(res.trace) == 7
    # the probe above the answer (if any) missed the target: bisection kept the bracketing half
    over = [t for t, e in res.trace if e > 1e-4]
    assert all(t > res.tau for t in over)
    # same probes as the reference's bisection: geometric midpoints of [1e-12, 1e-3]
    assert math.isclose(res.trace[1][0], math.sqrt(1e-12 * 1e-3))
    # oracle port agrees on the error at the calibrated tau
    oa = O.tree_from_dense(a)
    oc, _, _ = O.multiply(oa, oa, res.tau)
    want = np.abs(oc.to_dense().astype(np.float64) - oracle.cpu().numpy()).max()
    assert abs(want - res.error) <= 1e-5 * np.abs(oracle.cpu().numpy()).max()
    tight = B.calibrate_tau(tree, oracle, target=1e-30, iters=2)
    assert not tight.converged and tight.tau == 1e-12 and len(tight.trace) == 1
    with pytest.raises(ValueError):
        B.calibrate_tau(tree, oracle, target=0.0)
    with pytest.raises(ValueError):
        B.calibrate_tau(tree, oracle, target=1e-5, lo=1e-3, hi=1e-6)
