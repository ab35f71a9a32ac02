"""The planner's partition of the record stream for the numeric kernel (plan_order_kernel, csrc/plan.cu).

The CTAs resident on one SM share a piece (b, mb, me, e) of the plan's step records: whole
super-tiles [mb, me), a head segment [me, e) of a tile the next piece finishes and a tail segment
[b, mb) of a tile the previous piece began.  Checked here on the device plan: the pieces tile the
record stream without gaps, segment boundaries sit where they must, every record carries the length
of its tile (the cursor hands out whole tiles), and the piece weights are balanced.
The reference has no counterpart (its executor is sequential, `numeric.py:184-265`)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STEP_FIRST, STEP_LAST = 1 << 16, 1 << 17


def _pieces(plan):
    cnt = plan.counts.cpu().numpy()
    P = int(cnt[5])
    return plan.tile_order[: 4 * P].cpu().numpy().reshape(P, 4).astype(np.int64), int(cnt[12]), int(cnt[4])


@pytest.mark.parametrize("n,tau", [(256, 1e-6), (1024, 1e-6), (2048, 1e-8), (4096, 1e-8), (4096, 1e-4)])
def test_pieces_cover_the_plan_and_are_balanced(n, tau):
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(n, 0.95, seed=0)
    qa = P.QuadtreeMatrix.from_dense(a)
    plan = P.build_plan(qa, qa, tau)
    pieces, rounds, R = _pieces(plan)
    assert R == plan.n_steps and len(pieces) >= 1 and rounds >= 1
    rec = plan.step_records()
    flags = rec[:, 1]
    b, mb, me, e = pieces.T
    assert b[0] == 0 and e[-1] == R
    assert np.array_equal(e[:-1], b[1:]), "pieces must tile the record stream"
    assert np.all(b <= mb) and np.all(mb <= me) and np.all(me <= e)
    first = np.concatenate([(flags & STEP_FIRST) != 0, [True]])     # index R counts as a tile start
    # whole-tile range: begins and ends on tile boundaries
    nz = mb < me
    assert np.all(first[mb[nz]]) and np.all(first[me[nz]])
    # a head segment begins on a tile start and does not reach the tile's end
    hd = me < e
    assert np.all(first[me[hd]]) and not np.any(flags[e[hd] - 1] & STEP_LAST)
    # a tail segment begins inside a tile; it ends with the tile unless the whole piece lies inside one tile
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
    # balance: weight = live tasks that are not known dead + rec_weight per record (default 6)
    w = np.zeros(R, np.int64)
    dead = [rec[:, 13] & 0xFFFF, rec[:, 13] >> 16, rec[:, 14] & 0xFFFF, rec[:, 14] >> 16]
    for kk in range(4):
        w += np.array([bin(int(x) & 0xFFFF & ~int(d)).count("1") for x, d in zip(rec[:, 8 + kk], dead[kk])], np.int64)
    w += 6
    cw = np.concatenate([[0], np.cumsum(w)])
    pw = cw[e] - cw[b]
    assert pw.sum() == cw[-1]
    import torch
    assert len(pieces) == rounds * torch.cuda.get_device_properties(0).multi_processor_count
    assert pw.max() <= cw[-1] / len(pieces) + w.max() + 1, "a piece exceeds its share by more than one record"
