"""Golden fixtures for the rows either side of the multiply path, made with the REAL reference
(`/root/reference/pkg/src`, importable in the build container only):

  tree_rect.qt         SPAMMQT1 file written by spamm.io.save_quadtree for the 'rect' golden case
  sparsify.npz         QuadtreeMatrix.sparsify(eps) results (dropped count, packed leaves, all norms)
                       and the product of the thinned tree, for two golden cases

Run:  python tests/golden/make_golden_io.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import spamm  # noqa: E402
from spamm.io import save_quadtree  # noqa: E402
from cases import CASES, build_inputs  # noqa: E402


def tree_blob(q):
    keys, vals, subs = q.packed_leaves()[:3]
    out = {"keys": np.asarray(keys, np.uint64), "values": np.asarray(vals, np.float32), "subnorms": np.asarray(subs, np.float32)}
    for t in range(q.depth + 1):
        grid = np.full((1 << t, 1 << t), -1.0, np.float32)
        for idx in range(4 ** t):
            node = q.node(t, idx)
            if node is not None:
                i, j = spamm.decode(idx)
                grid[i, j] = node.norm
        out[f"norm{t}"] = grid
    return out


def main():
    by_name = {c["name"]: c for c in CASES}
    a = build_inputs(by_name["rect"])[0]
    save_quadtree(os.path.join(HERE, "tree_rect.qt"), spamm.QuadtreeMatrix.from_dense(a))
    blob = {}
    for name, eps in (("exp96", 1e-3), ("exp96", 0.05), ("blocksparse128", 0.5), ("rand64", 10.0)):
        a = build_inputs(by_name[name])[0]
        q = spamm.QuadtreeMatrix.from_dense(a)
        dropped = q.sparsify(eps)
        tag = f"{name}:{eps}"
        blob[f"{tag}:dropped"] = np.int64(dropped)
        for k, v in tree_blob(q).items():
            blob[f"{tag}:{k}"] = v
        if q.leaf_count:
            c, plan, counters = spamm.multiply(q, q, spamm.MultiplyConfig(tau=1e-6))
            blob[f"{tag}:c"] = c.to_dense().data
            blob[f"{tag}:tasks"] = np.int64(len(plan.tasks))
            blob[f"{tag}:products4"] = np.int64(counters.products4)
    np.savez_compressed(os.path.join(HERE, "sparsify.npz"), **blob)
    print("wrote", len(blob), "arrays")


if __name__ == "__main__":
    main()
