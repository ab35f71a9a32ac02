"""Times the UNMODIFIED Python reference (/root/reference/pkg/src/spamm) on the BASELINE configs it can
finish, the way its own bench does (tree prebuilt; build_plan + execute_plan, `pkg/src/spamm/bench.py:133-145`).
Runs only in the build container (the reference is not on the GPU box); writes
profiles/python_reference_times.json, which bench.py quotes beside the C port's time."""
import json, os, platform, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
import spamm
from paper_1203_1692_b200 import inputs

out = {"where": "build container (no GPU), %s, %d cores visible, 1 used (the reference is single-threaded Python/numpy)"
                % (platform.processor() or platform.machine(), os.cpu_count()),
       "when": time.strftime("%Y-%m-%d"), "python": platform.python_version(), "numpy": np.__version__, "runs": {}}
for name, tau, gran in (("cfg1", 1e-6, "fine4"), ("cfg2", 1e-8, "fine4"), ("cfg2", 1e-8, "coarse16")):
    a, b = inputs.make_operands(name)
    t0 = time.perf_counter()
    qa = spamm.QuadtreeMatrix.from_dense(spamm.DenseMatrix(a), 16)
    qb = qa if b is None else spamm.QuadtreeMatrix.from_dense(spamm.DenseMatrix(b), 16)
    t_tree = time.perf_counter() - t0
    cfg = spamm.MultiplyConfig(tau=tau, granularity=gran)
    t0 = time.perf_counter()
    plan = spamm.build_plan(qa, qb, tau)
    t_plan = time.perf_counter() - t0
    t0 = time.perf_counter()
    c, k = spamm.execute_plan(plan, qa, qb, None, cfg)
    t_exec = time.perf_counter() - t0
    out["runs"][f"{name}:{tau:g}:{gran}"] = {"n": int(a.shape[0]), "tasks": len(plan.tasks), "products4": int(k.products4),
                                              "from_dense_s": t_tree, "build_plan_s": t_plan, "execute_plan_s": t_exec,
                                              "multiply_s": t_plan + t_exec}
    print(name, tau, gran, out["runs"][f"{name}:{tau:g}:{gran}"], flush=True)
with open(os.path.join(ROOT, "profiles", "python_reference_times.json"), "w") as f:
    json.dump(out, f, indent=1)
