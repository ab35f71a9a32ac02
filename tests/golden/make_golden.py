"""Generate tests/golden/golden.npz from the UNMODIFIED reference package.

Run in the build container only (the reference does not travel to the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``spamm`` from /root/reference/pkg/src, feeds it the seeded inputs of
``paper_1203_1692_b200.inputs`` (plus a few hand-built edge cases) and records,
per case: packed leaves, all norms, the plan in plan order, the fine4 masks
(recomputed from ``packed_leaves()`` sub-norms with the rule at
numeric.py:233-238), the recursive visit set, counters and the product.
Small cases are stored in full, large ones as SHA-256 digests of the same
arrays, so the fixture stays small.  ``cases.py`` (next to this file) defines the
cases and is shared with the tests, which rebuild the inputs from the seeds.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import spamm  # noqa: E402  (the reference)
from spamm.core import QuadtreeMatrix  # noqa: E402
from spamm.morton import decode_array  # noqa: E402
from spamm.numeric import MultiplyConfig, execute_plan  # noqa: E402
from spamm.reference import recursive_spamm  # noqa: E402
from spamm.symbolic import build_plan, plan_dump  # noqa: E402

from cases import CASES, FULL_LIMIT, build_inputs, digest  # noqa: E402


def tree_record(q: QuadtreeMatrix, full: bool) -> dict:
    keys, vals, subs = q.packed_leaves()
    rec = {"keys": keys.copy(), "m": q.m, "n": q.n, "depth": q.depth}
    leaf_norm = np.array([q.node(q.depth, int(k)).norm for k in keys], np.float32)
    tiers = []
    for t in range(q.depth + 1):
        items = sorted((key, nd.norm) for (tt, key), nd in q._nodes.items() if tt == t)
        tk = np.array([k for k, _ in items], np.uint64)
        tn = np.array([v for _, v in items], np.float32)
        tiers.append(np.concatenate([tk.view(np.uint8), tn.view(np.uint8)]))
    tier_blob = np.concatenate(tiers) if tiers else np.zeros(0, np.uint8)
    if full:
        rec.update(values=vals.copy(), subnorms=subs.copy(), leaf_norm=leaf_norm, tiers=tier_blob)
    rec.update(values_sha=digest(vals), subnorms_sha=digest(subs), leaf_norm_sha=digest(leaf_norm),
               tiers_sha=digest(tier_blob))
    return rec


def masks_from_packed(a: QuadtreeMatrix, b: QuadtreeMatrix, akeys, bkeys, tau) -> np.ndarray:
    """Bit r*16 + p*4 + q  <=>  float64(subA[p,r]) * float64(subB[r,q]) >= tau."""
    ka, _, sa = a.packed_leaves()
    kb, _, sb = b.packed_leaves()
    out = np.zeros(len(akeys), np.uint64)
    if len(akeys) == 0:
        return out
    an = sa[np.searchsorted(ka, akeys)].astype(np.float64)   # [t, p, r]
    bn = sb[np.searchsorted(kb, bkeys)].astype(np.float64)   # [t, r, q]
    for r in range(4):
        pn = an[:, :, r][:, :, None] * bn[:, r, :][:, None, :]
        live = pn >= tau
        for p in range(4):
            for q in range(4):
                out |= live[:, p, q].astype(np.uint64) << np.uint64(r * 16 + p * 4 + q)
    return out


def main() -> None:
    out: dict[str, np.ndarray] = {}
    meta = {"reference_version": spamm.__version__ if hasattr(spamm, "__version__") else "0.1.0",
            "numpy": np.__version__, "cases": {}}
    for case in CASES:
        name = case["name"]
        a_d, b_d, c_d = build_inputs(case)
        full = max(a_d.shape + (b_d.shape if b_d is not None else ())) <= FULL_LIMIT
        qa = QuadtreeMatrix.from_dense(a_d)
        qb = qa if b_d is None else QuadtreeMatrix.from_dense(b_d)
        if case.get("chain"):
            # operand with a stored all-zero leaf: the product of the two inputs is
            # itself used as both operands (zero-norm leaves stay stored, numeric.py:179)
            prod, _, _ = spamm.multiply(qa, qb, MultiplyConfig(tau=0.0))
            qa = qb = prod
        rec: dict = {"in_a_sha": digest(a_d), "in_b_sha": digest(b_d) if b_d is not None else ""}
        for side, q in (("A", qa), ("B", qb)):
            for k, v in tree_record(q, full).items():
                rec[f"{side}_{k}"] = v
        for run in case["runs"]:
            tau, gran = run["tau"], run.get("granularity", "fine4")
            alpha, beta = run.get("alpha", 1.0), run.get("beta", 0.0)
            tag = run["tag"]
            plan = build_plan(qa, qb, tau)
            akeys = np.array([t.a for t in plan.tasks], np.uint64)
            bkeys = np.array([t.b for t in plan.tasks], np.uint64)
            prods = np.array([t.norm_product for t in plan.tasks], np.float64)
            masks = masks_from_packed(qa, qb, akeys, bkeys, tau)
            cfg = MultiplyConfig(tau=tau, granularity=gran, alpha=alpha, beta=beta)
            c0 = QuadtreeMatrix.from_dense(c_d) if (c_d is not None and run.get("use_c")) else None
            c, counters = execute_plan(plan, qa, qb, c0, cfg)
            r = {
                "T": len(plan.tasks),
                "stats": np.array([plan.stats.emitted, plan.stats.examined, plan.stats.pruned], np.int64),
                "akeys_sha": digest(akeys), "bkeys_sha": digest(bkeys), "prods_sha": digest(prods),
                "masks_sha": digest(masks),
                "pairs_sorted_sha": digest(np.array(sorted(zip(akeys.tolist(), bkeys.tolist())), np.uint64).reshape(-1, 2)),
                "products4": counters.products4, "skipped4": counters.skipped4,
                "dump_sha": hashlib.sha256(plan_dump(plan).encode()).hexdigest(),
            }
            if run.get("recursive"):
                _, visits = recursive_spamm(qa, qb, tau)
                r["recursive_sha"] = digest(np.array(sorted(visits), np.uint64).reshape(-1, 2))
            for k, v in tree_record(c, full).items():
                r[f"C_{k}"] = v
            cd = c.to_dense().data
            r["C_dense_sha"] = digest(cd)
            if full:
                r.update(akeys=akeys, bkeys=bkeys, prods=prods, masks=masks, C_dense=cd)
            for k, v in r.items():
                rec[f"{tag}/{k}"] = v
        scal = {}
        for k, v in rec.items():
            if isinstance(v, np.ndarray):
                out[f"{name}/{k}"] = v
            else:
                scal[k] = v
        meta["cases"][name] = scal
        print(name, "done", flush=True)
    out["__meta__"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
