import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs, symbolic
n, lam, tau, caps = 8192, 0.95, 1e-6, (64, 16)
a = inputs.exponential_decay(n, lam, seed=1)
qa = P.QuadtreeMatrix.from_dense(a)
cfg = P.MultiplyConfig(tau=tau)
c0, p0, k0 = P.multiply(qa, qa, cfg)
print("first: steps", p0.n_steps, "cleaves", p0.n_cleaves, "tasks", len(p0), flush=True)
key, _ = symbolic.plan_capacity(qa, qa, cfg.tau, p0.depth, 0, 1 << p0.depth)
print("hint after first:", symbolic._capacity_hint[key], flush=True)
symbolic._capacity_hint[key] = caps
c1, p1, k1 = P.multiply(qa, qa, cfg)
print("second resolved: tasks", len(p1), "hint:", symbolic._capacity_hint[key], flush=True)
torch.cuda.synchronize()
c2, p2, k2 = P.multiply(qa, qa, cfg)
torch.cuda.synchronize()
print("third ok", k2.products4 == k0.products4, flush=True)
