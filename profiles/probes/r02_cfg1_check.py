"""cfg1: the leaf-multiply kernel alone, timed as bench.py's measure_case does it (3 repetitions) and with more repetitions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs
import bench
a, _ = inputs.make_operands("cfg1")
qa = P.QuadtreeMatrix.from_dense(a)
flush = torch.empty((256 << 20,), dtype=torch.uint8, device="cuda")
for gran in ("fine4", "coarse16"):
    cfg = P.MultiplyConfig(tau=1e-6, granularity=gran)
    ts, (c, plan, k) = bench.timed_multiply(P, torch, qa, qa, cfg, 10, 3, flush)
    print(gran, "multiply median %.1f us" % (np.median(ts) * 1e3), "counts", plan.counts[:22].tolist())
    for reps in (3, 3, 10, 30):
        print("   kernel alone, %2d reps: %.1f us" % (reps, bench.kernel_time_execute(P, torch, plan, qa, qa, cfg, reps, flush) * 1e3))
    c2, plan2, k2 = P.multiply(qa, qa, cfg)
    print("   plan of a fresh multiply: %.1f us" % (bench.kernel_time_execute(P, torch, plan2, qa, qa, cfg, 10, flush) * 1e3))
