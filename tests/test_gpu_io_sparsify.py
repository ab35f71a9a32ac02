"""The rows either side of the multiply path: SPAMMQT1 tree files to and from
the packed device store, sparsify, and products fed back as operands -- against files and results
produced by the real reference (tests/golden/make_golden_io.py) and against the oracle."""

import os
import struct

import numpy as np
import pytest

from oracle import oracle as O
from helpers import CASES, assert_trees_equal, build_inputs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
BY_NAME = {c["name"]: c for c in CASES}


def test_reads_and_rewrites_the_reference_file_bit_for_bit(tmp_path):
    import paper_1203_1692_b200 as P
    src = os.path.join(HERE, "golden", "tree_rect.qt")              # written by spamm.io.save_quadtree
    a = build_inputs(BY_NAME["rect"])[0]
    q = P.load_quadtree(src)
    assert (q.m, q.n) == a.shape and np.array_equal(q.to_dense().data, a)
    assert_trees_equal(q, _refreshed(O.tree_from_dense(a)), "loaded tree")
    out = tmp_path / "again.qt"
    P.save_quadtree(out, q)
    assert out.read_bytes() == open(src, "rb").read()
    # a tree built on the device writes the same file
    P.save_quadtree(out, P.QuadtreeMatrix.from_dense(a))
    assert out.read_bytes() == open(src, "rb").read()


def _refreshed(t: O.OracleTree) -> O.OracleTree:
    """Norms in compute_norms order, which is what load_quadtree produces (io.py:147-148)."""
    from paper_1203_1692_b200 import morton
    i, j = morton.decode_array(t.keys.astype(np.uint64))
    return O.tree_from_packed(t.m, t.n, i.astype(np.int64), j.astype(np.int64), t.values)


def test_layout_pinned_and_empty_tree(tmp_path):
    # tests/test_io.py:136-160 of the reference
    import paper_1203_1692_b200 as P
    rng = np.random.default_rng(4)
    a = np.zeros((20, 20), np.float32)
    a[:16, :16] = rng.standard_normal((16, 16)).astype(np.float32)
    a[16:, 16:] = 1.0
    p = tmp_path / "t.qt"
    P.save_quadtree(p, P.QuadtreeMatrix.from_dense(a))
    raw = p.read_bytes()
    assert raw[:8] == P.QUADTREE_MAGIC == b"SPAMMQT1"
    assert struct.unpack_from("<5Q", raw, 8) == (20, 20, 16, 1, 2)
    record = 8 + 1024
    assert len(raw) == 48 + 2 * record
    assert struct.unpack_from("<Q", raw, 48)[0] == 0 and struct.unpack_from("<Q", raw, 48 + record)[0] == 3
    assert np.array_equal(np.frombuffer(raw, "<f4", 256, 56).reshape(16, 16), a[:16, :16])
    back = P.load_quadtree(p)
    assert np.array_equal(back.to_dense().data, a)
    e = tmp_path / "e.qt"
    P.save_quadtree(e, P.QuadtreeMatrix(33, 12))
    empty = P.load_quadtree(e)
    assert (empty.m, empty.n, empty.leaf_count) == (33, 12, 0) and not empty.to_dense().data.any()


@pytest.mark.parametrize("name,eps", [("exp96", 1e-3), ("exp96", 0.05), ("blocksparse128", 0.5), ("rand64", 10.0)])
def test_sparsify_matches_the_reference(name, eps):
    import paper_1203_1692_b200 as P
    z = np.load(os.path.join(HERE, "golden", "sparsify.npz"))
    tag = f"{name}:{eps}"
    a = build_inputs(BY_NAME[name])[0]
    q = P.QuadtreeMatrix.from_dense(a)
    assert q.sparsify(0.0) == 0
    dropped = q.sparsify(eps)
    assert dropped == int(z[f"{tag}:dropped"])
    keys, vals, subs = q.packed_leaves()
    assert np.array_equal(keys, z[f"{tag}:keys"])
    if keys.size:
        assert np.array_equal(vals, z[f"{tag}:values"]) and np.array_equal(subs, z[f"{tag}:subnorms"])
        for t in range(q.depth + 1):
            assert np.array_equal(q.level_norms(t), z[f"{tag}:norm{t}"]), f"tier {t} norms after sparsify"
        c, plan, k = P.multiply(q, q, P.MultiplyConfig(tau=1e-6, exact=True))
        assert len(plan) == int(z[f"{tag}:tasks"]) and k.products4 == int(z[f"{tag}:products4"])
        assert np.array_equal(c.to_dense().data, z[f"{tag}:c"])
    else:
        assert q.leaf_count == 0 and not q.to_dense().data.any()
    with pytest.raises(ValueError):
        q.sparsify(-1.0)


def test_products_fed_back_as_operands():
    """Purification-style squaring: C1 = A A, C2 = C1 C1, C3 = C2 A, every product
    consumed straight from the device store, bit-identical to the oracle doing the same chain."""
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(320, 0.8, seed=7)
    tau = 1e-7
    q = P.QuadtreeMatrix.from_dense(a)
    t = O.tree_from_dense(a)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    c1, p1, _ = P.multiply(q, q, cfg)
    o1, op1, _ = O.multiply(t, t, tau)
    assert len(p1) == len(op1)
    assert_trees_equal(c1, o1, "C1")
    c2, p2, k2 = P.multiply(c1, c1, cfg)
    o2, op2, ok2 = O.multiply(o1, o1, tau)
    assert len(p2) == len(op2) and k2.products4 == ok2.products4
    assert_trees_equal(c2, o2, "C2")
    c3, p3, _ = P.multiply(c2, q, cfg)
    o3, op3, _ = O.multiply(o2, t, tau)
    assert len(p3) == len(op3)
    assert_trees_equal(c3, o3, "C3")
    # thinning between the steps, as the paper does to keep the operands sparse
    eps = P.drop_tolerance(tau, float(c1.level_norms(0)[0, 0]), float(c1.level_norms(0)[0, 0]))
    assert c1.sparsify(eps) >= 0
    c4, _, _ = P.multiply(c1, c1, cfg)
    assert np.isfinite(c4.to_dense().data).all()
