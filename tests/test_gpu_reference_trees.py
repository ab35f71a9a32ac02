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


@pytest.mark.parametrize("n,lam", [(256, 0.8), (1000, 0.9)])
def test_from_packed_equals_from_dense(n, lam):
    """QuadtreeMatrix.from_packed (the key and value arrays of `core.py:387-405` from host memory) builds the
    tree from_dense builds: same records in both layouts, same norms at every tier, same product."""
    import torch
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(n, lam, seed=5)
    q0 = P.QuadtreeMatrix.from_dense(a)
    keys, vals, subs = q0.packed_leaves()
    for blocks in (vals, torch.from_numpy(vals.reshape(-1, 256).copy()).pin_memory()):
        q1 = P.QuadtreeMatrix.from_packed(n, n, keys.astype(np.int64), blocks)
        assert q1.nleaf == q0.nleaf and q1.depth == q0.depth
        k1, v1, s1 = q1.packed_leaves()
        assert np.array_equal(k1, keys) and np.array_equal(v1, vals) and np.array_equal(s1, subs)
        assert torch.equal(q1.values_t[: q1.nleaf], q0.values_t[: q0.nleaf])
        for tier in range(q0.depth + 1):
            assert np.array_equal(q1.level_norms(tier), q0.level_norms(tier))
        c0, _, _ = P.multiply(q0, q0, P.MultiplyConfig(tau=1e-6))
        c1, _, _ = P.multiply(q1, q1, P.MultiplyConfig(tau=1e-6))
        for x, y in zip(c0.packed_leaves(), c1.packed_leaves()):
            assert np.array_equal(x, y)
    # the oracle's tree of the same matrix holds the same leaves
    t = O.tree_from_dense(a)
    assert np.array_equal(np.asarray(t.keys, np.int64), keys.astype(np.int64))
    assert np.array_equal(np.asarray(t.values, np.float32).reshape(-1, 16, 16), vals)
    empty = P.QuadtreeMatrix.from_packed(n, n, np.zeros(0, np.int64), np.zeros((0, 16, 16), np.float32))
    assert empty.nleaf == 0
    with pytest.raises(ValueError):
        P.QuadtreeMatrix.from_packed(n, n, keys, vals.astype(np.float64))


def test_host_accessors_match_the_oracle_tree():
    """leaf_items / node_count / get_element (`core.py:176-211`) on the device tree against the oracle's tree."""
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(200, 0.7, seed=2)
    a[a < 1e-30] = 0.0
    q = P.QuadtreeMatrix.from_dense(a)
    t = O.tree_from_dense(a)
    items = q.leaf_items()
    assert [k for k, _ in items] == [int(k) for k in t.keys.tolist()]
    i, j = _decode_all(t.keys)
    assert np.array_equal(np.array([nd.norm for _, nd in items], np.float32), t.leaf_norm[i, j].astype(np.float32))
    assert q.node_count == sum(int(np.count_nonzero(q.level_norms(tier) >= 0)) for tier in range(q.depth + 1))
    for (r, c) in [(0, 0), (17, 3), (199, 199), (5, 190)]:
        assert q.get_element(r, c) == float(a[r, c])
    with pytest.raises(IndexError):
        q.get_element(200, 0)
    with pytest.raises(NotImplementedError):
        q.set_element(0, 0, 1.0)


def _decode_all(keys):
    ij = np.array([_decode(int(k)) for k in keys.tolist()], np.int64).reshape(-1, 2)
    return ij[:, 0], ij[:, 1]
