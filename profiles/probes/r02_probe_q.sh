set -x
cd /root/repo
mkdir -p gpurun_out/r02q
timeout 600 python -m pytest tests/test_gpu_parallel.py -x -q 2>&1 | tail -5
SPAMM_EX_TRACE=gpurun_out/r02q/trace_c16.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace_summary.py gpurun_out/r02q/trace_c16.txt
SPAMM_TAIL_RECORDS=0 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_TAIL_PERCENT=10 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_TAIL_PERCENT=60 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_PLAN_TRACE=gpurun_out/r02q/plan_trace.txt python profiles/k3_probe.py cfg2 1e-8 coarse16 > /dev/null
python profiles/plan_trace_summary.py gpurun_out/r02q/plan_trace.txt
python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs
a,_ = inputs.make_operands('cfg2')
qa = P.QuadtreeMatrix.from_dense(a)
plan = P.build_plan(qa, qa, 1e-8)
cnt = plan.counts.cpu().numpy()
print("counts", cnt[:24].tolist())
Pn, stride = int(cnt[12]), int(cnt[21])
u = plan.tile_order[:2*Pn].cpu().numpy().reshape(-1,2)
print("pieces", Pn, "records per piece min/mean/max", (u[:,1]-u[:,0]).min(), (u[:,1]-u[:,0]).mean(), (u[:,1]-u[:,0]).max(), "RA", u[-1,1], "R", cnt[4])
PY
