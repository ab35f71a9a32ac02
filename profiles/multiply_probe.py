"""Times whole multiplies back to back (tuning aid): async path, with and without resolving counts."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
gran = sys.argv[3] if len(sys.argv) > 3 else "fine4"
a, b = inputs.make_operands(name)
qa = P.QuadtreeMatrix.from_dense(a)
qb = qa if b is None else P.QuadtreeMatrix.from_dense(b)
cfg = P.MultiplyConfig(tau=tau, granularity=gran)

def run(n, resolve):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        c, plan, k = P.multiply(qa, qb, cfg)
        if resolve:
            len(plan)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return e0.elapsed_time(e1) / n, (t1 - t0) / n * 1e3, (t2 - t0) / n * 1e3

for label, resolve in (("first calls (guessed capacities), unresolved", False), ("resolved every call", True),
                       ("after hints, unresolved", False), ("after hints, unresolved again", False)):
    gpu_ms, cpu_ms, wall_ms = run(20, resolve)
    print(f"{label:50s} gpu {gpu_ms:.3f} ms  cpu-enqueue {cpu_ms:.3f} ms  wall {wall_ms:.3f} ms per multiply")

if os.environ.get("SPAMM_CPROFILE"):
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        c, plan, k = P.multiply(qa, qb, cfg)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
