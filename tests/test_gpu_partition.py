"""The planner's partition of the record stream for the numeric kernel (plan_order_kernel, csrc/plan.cu).

Every team of the numeric kernel (two per SM) runs a piece (b, mb, me, e) of the plan's step records: whole
super-tiles [mb, me), a head segment [me, e) of a tile the next piece finishes and a tail segment
[b, mb) of a tile the previous piece began.  Checked here on the device plan: the pieces tile the
record stream without gaps, segment boundaries sit where they must, every record carries the length
of its tile, and the piece weights are balanced.
The reference has no counterpart (its executor is sequential, `numeric.py:184-265`)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STEP_FIRST, STEP_LAST = 1 << 16, 1 << 17


def _units(plan):
    """(pieces of region A, [segments of layer 0, 1, 2 of region B], step records) of a device plan."""
    cnt = plan.counts.cpu().numpy()
    P, n, stride = int(cnt[12]), [int(x) for x in cnt[16:21]], int(cnt[21])
    raw4 = plan.tile_order[: 4 * (P + 5 * stride)].cpu().numpy().reshape(-1, 4).astype(np.int64)
    # a unit is (b, end of b's tile, start of the tile of e - 1, e); checked against the records below
    _units.raw4 = np.concatenate([raw4[:P]] + [raw4[P + x * stride: P + x * stride + n[x]] for x in range(5)])
    raw = raw4[:, [0, 3]]
    rng = [raw[P + x * stride: P + x * stride + n[x]] for x in range(5)]
    # ranges 0..2: first segments of the tiles with 3, 2, 1 segments; 3: second segments; 4: third segments
    return raw[:P], [np.concatenate(rng[:3]), rng[3], rng[4]], int(cnt[4])


def lens_of(rec, r):
    return int(rec[r, 15] & 0xFFFF)


@pytest.mark.parametrize("n,tau", [(256, 1e-6), (1024, 1e-6), (2048, 1e-8), (4096, 1e-8), (4096, 1e-4)])
def test_units_cover_the_plan(n, tau):
    import torch
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(n, 0.95, seed=0)
    qa = P.QuadtreeMatrix.from_dense(a)
    plan = P.build_plan(qa, qa, tau)
    pa, layers, R = _units(plan)
    assert R == plan.n_steps
    rec = plan.step_records()
    flags = rec[:, 1]
    units = np.concatenate([pa] + layers)
    b, e = units.T
    assert np.all(b <= e)
    # the units tile the record stream: region A's pieces in stream order, then region B's segments
    order = np.lexsort((e, b))
    nz = (e > b)[order]
    bs, es = b[order][nz], e[order][nz]
    assert bs[0] == 0 and es[-1] == R and np.array_equal(es[:-1], bs[1:]), "units must tile the record stream"
    npieces = len(pa)
    if npieces:
        assert pa[0, 0] == 0 and np.array_equal(pa[:-1, 1], pa[1:, 0]), "pieces of region A are contiguous"
    RA = int(pa[-1, 1]) if npieces else 0
    first = np.concatenate([(flags & STEP_FIRST) != 0, [True]])     # index R counts as a tile start
    assert first[RA], "region B begins on a tile boundary"
    # every record knows how many records its tile has and where in the tile it sits
    starts = np.flatnonzero(flags & STEP_FIRST)
    lens = np.diff(np.concatenate([starts, [R]]))
    assert np.array_equal(rec[:, 15] & 0xFFFF, np.repeat(lens, lens))
    assert np.array_equal(rec[:, 15] >> 16, np.concatenate([np.arange(x) for x in lens]))
    # the tile bounds stored with every unit: end of the tile of record b (b itself at a tile start), start of
    # the tile of record e - 1 (e itself at a tile end)
    tile_start = np.repeat(starts, lens)
    for ub, utb, uts, ue in _units.raw4:
        if ue > ub:
            assert utb == (ub if first[ub] else tile_start[ub] + lens_of(rec, ub)), (ub, utb)
            assert uts == (ue if first[ue] else tile_start[ue - 1]), (ue, uts)
    # region A: equal weights; weight = live tasks + rec_weight per record (default 32)
    w = np.zeros(R, np.int64)
    for kk in range(4):
        w += np.array([bin(int(x) & 0xFFFF).count("1") for x in rec[:, 8 + kk]], np.int64)
    w += 32
    cw = np.concatenate([[0], np.cumsum(w)])
    if npieces:
        pw = cw[pa[:, 1]] - cw[pa[:, 0]]
        assert npieces % (2 * torch.cuda.get_device_properties(0).multi_processor_count) == 0
        assert pw.max() <= cw[RA] / npieces + w.max() + 1, "a piece exceeds its share by more than one record"
    # region B: every tile is cut into a first segment (layer 0) and up to two short ones of 3 records
    # (layers 1, 2); a tile's segments sit in consecutive layers
    l0, l1, l2 = layers
    assert np.all(first[l0[:, 0]]), "layer 0 holds the first segments"
    assert len(l0) == int(np.count_nonzero(first[RA:R])), "one first segment per tile of region B"
    for later in (l1, l2):
        assert np.all(later[:, 1] - later[:, 0] == 3) and not np.any(first[later[:, 0]])
    ends0 = set(l0[:, 1].tolist())
    assert set(l1[:, 0].tolist()) <= ends0 and set(l2[:, 0].tolist()) <= set(l1[:, 1].tolist())
    for seg in units[npieces:]:
        assert not np.any(flags[seg[0] + 1:seg[1]] & STEP_FIRST), "a segment stays inside its tile"
    # region B exists only when a team's share of the records is a few records (under 3 per team)
    teams = 2 * torch.cuda.get_device_properties(0).multi_processor_count
    if R < 3 * teams:
        assert cw[R] - cw[RA] >= min(cw[R], cw[R] // 4) - w.max() * 16
    else:
        assert RA == R and not len(l0)
