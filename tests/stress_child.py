"""Child process of test_gpu_stress.py: one product under the tuning knobs given in the environment
(they are read once per process), compared bit for bit with the oracle; prints OK or raises."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import paper_1203_1692_b200 as P  # noqa: E402
from paper_1203_1692_b200 import inputs  # noqa: E402

n, tau, reps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
a = inputs.exponential_decay(n, 0.95, seed=0)
oa = O.tree_from_dense(a)
qa = P.QuadtreeMatrix.from_dense(a)
for gran in ("fine4", "coarse16"):
    oc, oplan, ok = O.multiply(oa, oa, tau, gran)
    want = oc.to_dense()
    for it in range(reps):
        c, plan, k = P.multiply(qa, qa, P.MultiplyConfig(tau=tau, granularity=gran, exact=True))
        assert len(plan) == len(oplan) and k.products4 == ok.products4, (gran, it)
        assert np.array_equal(c.to_dense().data, want), (gran, it, "values")
        for t in range(oc.depth + 1):
            assert np.array_equal(c.level_norms(t), oc.level_norm(t)), (gran, it, "norms", t)
    cnt = plan.counts.cpu().numpy()
    npieces = int(cnt[12])
    u = plan.tile_order[: 4 * npieces].cpu().numpy().reshape(npieces, 4)[:, [0, 3]]
    flags = plan.step_records()[:, 1]
    chained = int(np.count_nonzero((flags[u[u[:, 1] > u[:, 0], 0]] & (1 << 16)) == 0))     # pieces that begin inside a super-tile
    print(f"{gran}: pieces={npieces} ranges={cnt[16:21].tolist()} chained={chained + int(cnt[19]) + int(cnt[20])} ")
print("OK")
