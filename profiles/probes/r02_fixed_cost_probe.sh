#!/bin/bash
# Where the fixed cost of execute_kernel sits: cold vs warm L2, per-team fit of duration against records/tasks.
set -x
cd /root/repo
mkdir -p gpurun_out/r02w
for g in coarse16 fine4; do
  SPAMM_EX_TRACE=gpurun_out/r02w/trace_$g.txt python profiles/k3_probe.py cfg2 1e-8 $g
  python profiles/fit_weights.py gpurun_out/r02w/trace_$g.txt
  PROBE_WARM_L2=1 python profiles/k3_probe.py cfg2 1e-8 $g
  python profiles/k3_probe.py cfg2 1e-8 $g
done
PROBE_WARM_L2=1 python profiles/k3_probe.py cfg2 1e-8 coarse16 2048
python profiles/k3_probe.py cfg2 1e-8 coarse16 2048
python profiles/k3_probe.py cfg2 1e-8 coarse16 8192
PROBE_WARM_L2=1 python profiles/k3_probe.py cfg2 1e-8 coarse16 8192
python - <<'PY'
import torch
x=torch.zeros(1,device='cuda')
ts=[]
for i in range(20):
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(); x.fill_(1); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
print("tiny kernel between events: us", sorted(ts)[len(ts)//2])
PY
