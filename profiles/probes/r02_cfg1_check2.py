"""cfg1: why k3_probe.py (one multiply, then the kernel alone) and bench.py (several multiplies first) time the same kernel differently."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs
import bench
a, _ = inputs.make_operands("cfg1")
qa = P.QuadtreeMatrix.from_dense(a)
cfg = P.MultiplyConfig(tau=1e-6, granularity="fine4")
keep = []
for it in range(6):
    c, plan, k = P.multiply(qa, qa, cfg)
    keep.append((c, plan))
    if it == 0:
        flush = torch.empty((256 << 20,), dtype=torch.uint8, device="cuda")
    t = bench.kernel_time_execute(P, torch, plan, qa, qa, cfg, 10, flush) * 1e3
    print("multiply #%d: kernel alone %.1f us; steps cap %d leaf cap %d; counts %s" % (
        it, t, plan._steps.shape[0] if hasattr(plan, "_steps") else -1, plan._c_keys.shape[0] if hasattr(plan, "_c_keys") else -1,
        plan.counts[:22].tolist()))
