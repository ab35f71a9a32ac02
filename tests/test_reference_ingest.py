"""Host side of the reference-tree ingestion (tree.pack_reference_leaves) against the REAL reference
package, when it is present (this container); the GPU half is tests/test_gpu_reference_trees.py.
Boundary: `pkg/src/spamm/core.py:387-405` (packed_leaves), `:138-143` (TreeNode.norm)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="the reference package only exists in the build container")
def test_pack_reference_leaves_matches_the_reference_tree():
    sys.path.insert(0, REF)
    try:
        import spamm
    finally:
        sys.path.remove(REF)
    from paper_1203_1692_b200.tree import pack_reference_leaves
    from paper_1203_1692_b200 import inputs
    a = inputs.exponential_decay(200, 0.7, seed=3)      # ragged size: padded leaves, some all-zero blocks
    t = spamm.QuadtreeMatrix.from_dense(spamm.DenseMatrix(a), 16)
    keys, rec, leaf_sq = pack_reference_leaves(t)
    rk, rv, rs = t.packed_leaves()
    assert np.array_equal(keys.astype(np.uint64), rk) and np.all(np.diff(keys) > 0)
    assert np.array_equal(rec[:, :256].reshape(-1, 16, 16), rv)
    assert np.array_equal(rec[:, 256:].reshape(-1, 4, 4).transpose(0, 2, 1), rs)
    want = np.array([nd.norm for _, nd in t.leaf_items()], np.float32)
    assert np.array_equal(np.sqrt(leaf_sq).astype(np.float32), want)
    with pytest.raises(ValueError):
        pack_reference_leaves(spamm.QuadtreeMatrix.from_dense(spamm.DenseMatrix(a), 8))
