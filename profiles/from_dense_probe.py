"""Times QuadtreeMatrix.from_dense on a resident dense matrix (tuning aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
a, _ = inputs.make_operands(name)
d = torch.from_numpy(a).cuda()
ts = []
for it in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    q = P.QuadtreeMatrix.from_dense(d)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{name}: from_dense median {ts[len(ts) // 2] * 1e3:.1f} us, leaves {q.nleaf}, {a.nbytes / ts[len(ts) // 2] / 1e6:.0f} GB/s of dense input")
