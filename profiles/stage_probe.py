"""In-stream cost of each stage of one multiply (tuning aid): run with SPAMM_PIPE_STOP=1..4.
Capacity hints come from a first full multiply in a child process-free way: the hint table is
filled by a synchronous build_plan before timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
a, b = inputs.make_operands(name)
qa = P.QuadtreeMatrix.from_dense(a)
qb = qa if b is None else P.QuadtreeMatrix.from_dense(b)
cfg = P.MultiplyConfig(tau=tau)
P.build_plan(qa, qb, tau)            # records the capacity hint without running the pipeline
flush = torch.empty((256 << 20,), dtype=torch.uint8, device="cuda")
modes = (("back to back", False),) if os.environ.get("PROBE_ONLY_WARM") else (("back to back", False), ("L2 flushed", True))
for label, fl in modes:
    ts = []
    for it in range(30):
        if fl:
            flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = P.multiply(qa, qb, cfg)
        e1.record()
        torch.cuda.synchronize()
        if it >= 10:
            ts.append(e0.elapsed_time(e1))
        del out
    ts.sort()
    print(f"stop={os.environ.get('SPAMM_PIPE_STOP', '0')} {label:13s} median {ts[len(ts) // 2] * 1e3:.1f} us  min {ts[0] * 1e3:.1f} us")
