"""Times the leaf-multiply kernel alone on one workload (tuning aid; knobs via SPAMM_EX_* env)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs
import bench

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
gran = sys.argv[3] if len(sys.argv) > 3 else "fine4"
n_over = int(sys.argv[4]) if len(sys.argv) > 4 else None
a, b = inputs.make_operands(name, n_over)
qa = P.QuadtreeMatrix.from_dense(a)
qb = qa if b is None else P.QuadtreeMatrix.from_dense(b)
cfg = P.MultiplyConfig(tau=tau, granularity=gran)
c, plan, k = P.multiply(qa, qb, cfg)
flush = torch.empty((1 if os.environ.get("PROBE_WARM_L2") else 256 << 20,), dtype=torch.uint8, device="cuda")
ms = bench.kernel_time_execute(P, torch, plan, qa, qb, cfg, 10, flush)
fl = 128 * k.products4 if gran == "fine4" else 8192 * len(plan)
print(json.dumps({"env": {k_: v for k_, v in os.environ.items() if k_.startswith("SPAMM_")}, "workload": name, "n": int(a.shape[0]), "tau": tau,
                  "gran": gran, "steps": plan.n_steps, "tasks": len(plan), "kernel_ms": round(ms, 4),
                  "tflops": round(fl / ms / 1e9, 2), "frac": round(fl / ms / 1e9 / 74.45, 3)}))
if os.environ.get("SPAMM_EX_TRACE"):
    # for the weight model of the planner's partition: the pieces (region A units) and per-record work of this plan
    npieces = int(plan.counts[12].item())
    pieces = plan.tile_order[: 4 * npieces].cpu().numpy().reshape(npieces, 4)
    rec = plan.step_records()
    np.savez(os.environ["SPAMM_EX_TRACE"] + ".plan.npz", pieces=pieces, rec=rec)
