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
    cnt = plan.counts.cpu().numpy()
    U, P = int(cnt[5]), int(cnt[12])
    return plan.tile_order[: 4 * U].cpu().numpy().reshape(U, 4).astype(np.int64), P, int(cnt[4])


@pytest.mark.parametrize("n,tau", [(256, 1e-6), (1024, 1e-6), (2048, 1e-8), (4096, 1e-8), (4096, 1e-4)])
def test_units_cover_the_plan(n, tau):
    import torch
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(n, 0.95, seed=0)
    qa = P.QuadtreeMatrix.from_dense(a)
    plan = P.build_plan(qa, qa, tau)
    units, npieces, R = _units(plan)
    assert R == plan.n_steps and len(units) >= 1
    rec = plan.step_records()
    flags = rec[:, 1]
    b, mb, me, e = units.T
    assert np.all(b <= mb) and np.all(mb <= me) and np.all(me <= e)
    # the units tile the record stream: region A's pieces in stream order, then region B's segments
    order = np.lexsort((e, b))
    nz = (e > b)[order]
    bs, es = b[order][nz], e[order][nz]
    assert bs[0] == 0 and es[-1] == R and np.array_equal(es[:-1], bs[1:]), "units must tile the record stream"
    pa = units[:npieces]
    if npieces:
        assert pa[0, 0] == 0 and np.array_equal(pa[:-1, 3], pa[1:, 0]), "pieces of region A are contiguous"
    RA = int(pa[-1, 3]) if npieces else 0
    first = np.concatenate([(flags & STEP_FIRST) != 0, [True]])     # index R counts as a tile start
    assert first[RA], "region B begins on a tile boundary"
    # whole-tile range: begins and ends on tile boundaries
    nzw = mb < me
    assert np.all(first[mb[nzw]]) and np.all(first[me[nzw]])
    # a head segment begins on a tile start and does not reach the tile's end
    hd = me < e
    assert np.all(first[me[hd]]) and not np.any(flags[e[hd] - 1] & STEP_LAST)
    # a tail segment begins inside a tile; it ends with the tile unless the whole unit lies inside one tile
    tl = b < mb
    assert not np.any(first[b[tl]])
    ends_tile = (flags[mb[tl] - 1] & STEP_LAST) != 0
    single = (mb[tl] == me[tl]) & (me[tl] == e[tl])
    assert np.all(ends_tile | single)
    # no record of a segment crosses a tile boundary
    for lo, hi in list(zip(me[hd], e[hd])) + list(zip(b[tl], mb[tl])):
        assert not np.any(flags[lo + 1:hi] & STEP_FIRST)
    # every record knows how many records its tile has
    starts = np.flatnonzero(flags & STEP_FIRST)
    lens = np.diff(np.concatenate([starts, [R]]))
    assert np.array_equal(rec[:, 15], np.repeat(lens, lens))
    # region A: equal weights; weight = live tasks that are not known dead + rec_weight per record (default 32)
    w = np.zeros(R, np.int64)
    dead = [rec[:, 13] & 0xFFFF, rec[:, 13] >> 16, rec[:, 14] & 0xFFFF, rec[:, 14] >> 16]
    for kk in range(4):
        w += np.array([bin(int(x) & 0xFFFF & ~int(d)).count("1") for x, d in zip(rec[:, 8 + kk], dead[kk])], np.int64)
    w += 32
    cw = np.concatenate([[0], np.cumsum(w)])
    if npieces:
        pw = cw[pa[:, 3]] - cw[pa[:, 0]]
        assert npieces % (2 * torch.cuda.get_device_properties(0).multi_processor_count) == 0
        assert pw.max() <= cw[RA] / npieces + w.max() + 1, "a piece exceeds its share by more than one record"
    # region B: layered segments of its tiles -- every later segment is the short kind (2 records),
    # and a tile's segments appear in the unit list in ascending order, a whole layer apart
    ub = units[npieces:]
    later = ub[ub[:, 0] < ub[:, 1]]
    assert np.all(later[:, 1] - later[:, 0] == 2)
    nB = int(np.count_nonzero(ub[:, 0] == ub[:, 1]))          # first segments = tiles of region B
    firsts = ub[:nB]
    assert np.all(firsts[:, 0] == firsts[:, 1]), "layer 0 holds exactly the first segments"
    pos = {int(x[0]): i for i, x in enumerate(ub)}              # unit that starts at a record
    for i, u in enumerate(ub):
        if u[3] < R and not first[u[3]]:                         # the tile continues: its next segment comes later
            assert pos[int(u[3])] > i
    assert cw[R] - cw[RA] >= min(cw[R], cw[R] // 4) - w.max() * 16
