"""Operands given as trees of the REFERENCE package (duck-typed) go through multiply / build_plan /
execute_plan unchanged: `numeric.py:302-313`, `symbolic.py:151-159`, `numeric.py:138-151` take the
reference's own `QuadtreeMatrix`; so does this package (tree.as_device_tree), copying the tree to the
device once per revision.  The reference itself is not on the GPU box, so a stand-in with the same
surface (`m, n, n_b, depth, _rev, packed_leaves(), leaf_items(), clear(), put_leaf(), compute_norms()`,
`core.py:146-405`) is filled from the oracle, which is pinned to the reference by tests/golden."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


class RefLikeTree:
    """The surface of spamm.QuadtreeMatrix that the multiply path touches, backed by numpy arrays."""

    def __init__(self, m, n, n_b=16):
        self.m, self.n, self.n_b = m, n, n_b
        self.depth = O.tree_depth(m, n) if hasattr(O, "tree_depth") else max(0, int(np.ceil(np.log2(max(1, -(-max(m, n) // 16))))))
        self._rev = 0
        self._leaves = {}           # key -> (values, subnorms, norm)

    @classmethod
    def from_oracle(cls, t):
        q = cls(t.m, t.n)
        q.depth = t.depth
        i, j = O.decode(t.keys) if hasattr(O, "decode") else (None, None)
        ln = t.leaf_norm
        for x, k in enumerate(t.keys.tolist()):
            ii, jj = (int(i[x]), int(j[x])) if i is not None else _decode(k)
            q._leaves[int(k)] = (t.values[x].reshape(16, 16).copy(), t.subnorms[x].reshape(4, 4).copy(), float(ln[ii, jj]))
        return q

    def packed_leaves(self):
        ks = sorted(self._leaves)
        if not ks:
            return np.empty(0, np.uint64), np.empty((0, 16, 16), np.float32), np.empty((0, 4, 4), np.float32)
        return (np.array(ks, np.uint64), np.stack([self._leaves[k][0] for k in ks]),
                np.stack([self._leaves[k][1] for k in ks]))

    def leaf_items(self):
        return [(k, SimpleNamespace(norm=self._leaves[k][2])) for k in sorted(self._leaves)]

    def clear(self):
        self._leaves.clear()
        self._rev += 1

    def put_leaf(self, key, values):
        self._leaves[int(key)] = (np.ascontiguousarray(values, np.float32), np.zeros((4, 4), np.float32), 0.0)
        self._rev += 1

    def compute_norms(self):
        self._rev += 1

    def to_dense(self):
        out = np.zeros((16 << self.depth, 16 << self.depth), np.float32)
        for k, (v, _, _) in self._leaves.items():
            i, j = _decode(k)
            out[16 * i:16 * i + 16, 16 * j:16 * j + 16] = v
        return out[: self.m, : self.n]


def _decode(key):
    i = j = 0
    for b in range(16):
        j |= ((key >> (2 * b)) & 1) << b
        i |= ((key >> (2 * b + 1)) & 1) << b
    return i, j


def test_reference_trees_as_operands_and_accumulator():
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(300, 0.8, seed=5)
    b = inputs.exponential_decay(300, 0.85, seed=6)
    oa, ob = O.tree_from_dense(a), O.tree_from_dense(b)
    ra, rb = RefLikeTree.from_oracle(oa), RefLikeTree.from_oracle(ob)
    tau = 1e-4
    oc, oplan, ok = O.multiply(oa, ob, tau)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    # one call
    c, plan, k = P.multiply(ra, rb, cfg)
    assert isinstance(c, P.QuadtreeMatrix) and len(plan) == len(oplan) and k.products4 == ok.products4
    assert np.array_equal(c.to_dense().data, oc.to_dense())
    ka, kb = plan.pair_keys()
    assert set(zip(ka.tolist(), kb.tolist())) == oplan.pair_set()
    # two-phase form on the same (cached) device copies
    plan2 = P.build_plan(ra, rb, tau)
    c2, k2 = P.execute_plan(plan2, ra, rb, None, cfg)
    assert np.array_equal(c2.to_dense().data, oc.to_dense()) and k2.products4 == ok.products4
    # an accumulator of the reference's type is mutated in place and returned (numeric.py:165-181)
    acc = RefLikeTree(300, 300)
    acc.depth = oa.depth
    acc.put_leaf(0, np.ones((16, 16), np.float32))
    out, _, _ = P.multiply(ra, rb, cfg, acc)
    assert out is acc
    assert np.array_equal(acc.to_dense(), oc.to_dense())
    # a mutated operand is copied again (cache keyed by the tree's revision, core.py:391-404)
    ra2 = RefLikeTree.from_oracle(oa)
    c3, _, _ = P.multiply(ra2, ra2, cfg)
    ra2._leaves = dict(RefLikeTree.from_oracle(ob)._leaves)
    ra2._rev += 1
    c4, _, _ = P.multiply(ra2, ra2, cfg)
    obb, _, _ = O.multiply(ob, ob, tau)
    assert np.array_equal(c4.to_dense().data, obb.to_dense())
    with pytest.raises(ValueError):
        bad = RefLikeTree(300, 300, n_b=8)
        P.multiply(bad, bad, cfg)
