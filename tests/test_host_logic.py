"""Host-side logic that needs no GPU: Morton maps (pins from the reference's tests/test_morton.py),
configuration validation, capacity growth, work-unit arithmetic shared with the kernels, and the
seeded BASELINE.json input generators (drift would silently invalidate the golden fixtures)."""

import ctypes

import numpy as np
import pytest

from oracle import oracle as O


def test_morton_pins_and_round_trip():
    from paper_1203_1692_b200 import morton
    assert morton.encode(1, 0) == 2 and morton.encode(0, 1) == 1 and morton.encode(3, 5) == 0b011011   # test_morton.py:25-30
    rng = np.random.default_rng(0)
    i, j = rng.integers(0, 1 << 15, 5000), rng.integers(0, 1 << 15, 5000)
    keys = morton.encode_array(i, j)
    bi, bj = morton.decode_array(keys)
    assert np.array_equal(bi, i) and np.array_equal(bj, j)
    assert np.array_equal(keys, O.encode(i, j))
    for a, b in ((morton.encode(3, 7), morton.encode(7, 2)), (morton.encode(0, 0), morton.encode(0, 5))):
        # the k lanes stay interleaved, as in the reference (morton.py:77-95): column bits of A, row bits of B
        assert morton.k_of_a(a) == morton.encode(0, morton.decode(a)[1])
        assert morton.k_of_b(b) == morton.encode(morton.decode(b)[0], 0)
        assert morton.k_match(a, b) == (morton.decode(a)[1] == morton.decode(b)[0])
        if morton.k_match(a, b):
            assert morton.decode(morton.c_index(a, b)) == (morton.decode(a)[0], morton.decode(b)[1])
    # a key's four low bits are the leaf's position inside its 4x4 block (what the step records index)
    assert [morton.encode(di, dj) for di in range(2) for dj in range(2)] == [0, 1, 2, 3]


def test_multiply_config_validation():
    from paper_1203_1692_b200 import GRANULARITIES, MICRO_FLOPS, MultiplyConfig
    assert GRANULARITIES == ("fine4", "coarse16") and MICRO_FLOPS == 128       # numeric.py:26-29
    cfg = MultiplyConfig()
    assert (cfg.tau, cfg.granularity, cfg.alpha, cfg.beta, cfg.exact) == (0.0, "fine4", 1.0, 0.0, False)
    for kw in ({"granularity": "dense16"}, {"tau": -1e-9}, {"tau": float("nan")}, {"alpha": float("inf")},
               {"beta": float("nan")}):
        with pytest.raises(ValueError):
            MultiplyConfig(**kw)


def test_capacity_growth_terminates():
    from paper_1203_1692_b200.symbolic import grow_capacity
    depth = 6
    step, leaf = 64, 16
    cnt = [0] * 16
    for _ in range(64):
        cnt[0], cnt[3], cnt[4] = 4 * leaf, 3 * step, 3 * step          # the plan keeps reporting "more"
        try:
            step, leaf = grow_capacity(depth, step, leaf, cnt)
        except RuntimeError:
            break
    else:
        pytest.fail("capacities never reached the limit")
    assert leaf == 4 ** depth


def test_work_unit_arithmetic_matches_the_library():
    """unit_segments / unit_begin (csrc/plan_format.cuh) restated here: segments tile every
    super-tile's records exactly once, in order, for any segment length."""
    def segments(ns, seg_len):
        if seg_len <= 0:
            return 1
        n = -(-min(ns, 127) // seg_len)
        return max(1, min(63, n))
    for ns in list(range(1, 40)) + [127, 128, 500, 4000]:
        for seg_len in (0, 1, 2, 3, 5, 8, 64):
            nseg = segments(ns, seg_len)
            cuts = [(s * ns) // nseg for s in range(nseg + 1)]
            assert cuts[0] == 0 and cuts[-1] == ns and all(b > a for a, b in zip(cuts, cuts[1:]))
            assert nseg <= 63 and (seg_len == 0 or nseg == 63 or ns > 127 or max(b - a for a, b in zip(cuts, cuts[1:])) <= seg_len)


def test_arena_layout_scales_with_capacities():
    from paper_1203_1692_b200 import _lib
    lib = _lib.lib()
    small, big = _lib.ArenaLayout(), _lib.ArenaLayout()
    assert lib.spamm_multiply_arena_layout(8, 8, 4096, 1024, ctypes.byref(small)) == 0
    assert lib.spamm_multiply_arena_layout(8, 8, 8192, 2048, ctypes.byref(big)) == 0
    assert big.total > small.total and big.values - big.chain >= 4 * 2048
    assert big.values_t - big.values >= 2048 * _lib.REC * 4 and big.leaf_sq - big.values_t >= 2048 * _lib.REC * 4
    assert lib.spamm_multiply_arena_layout(16, 8, 4096, 1024, ctypes.byref(small)) == _lib.SPAMM_EINVAL
    assert lib.spamm_plan_workspace_bytes(8, 4096, 1024) > 0


def test_seeded_generators_are_frozen():
    from paper_1203_1692_b200 import inputs
    import hashlib
    def sig(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
    a = inputs.exponential_decay(96, 0.9, seed=0)
    assert a.dtype == np.float32 and np.array_equal(a, a.T)                       # symmetrised
    assert np.abs(a).max() <= 1.0 and np.abs(np.diag(a)).min() >= 0.5             # u in [0.5, 1], envelope 1 on the diagonal
    b = inputs.exponential_decay(96, 0.9, seed=0)
    assert sig(a) == sig(b) and sig(a) != sig(inputs.exponential_decay(96, 0.9, seed=1))
    # the draw order is chunk-independent: a prefix of rows of a larger draw differs (different n), same n repeats
    g = inputs.algebraic_decay(64, seed=3)
    assert np.array_equal(g, inputs.algebraic_decay(64, seed=3)) and np.array_equal(g, g.T)
    assert abs(abs(g[0, 63]) * (63 ** 3 + 1)) <= 1.0
    m = inputs.molecule_decay(4, seed=0)
    assert m.shape == (100, 100) and np.array_equal(m, m.T)
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        assert name in inputs.WORKLOADS and len(inputs.WORKLOADS[name].taus) >= 1
