#!/bin/bash
# What the fine4 path of execute_kernel costs beyond its arithmetic (debug instantiation, results are garbage for 4/8/12):
# 16 = no-op (baseline of the debug build), 4 = undecided tasks run whole, 8 = planner's dead tasks run, 12 = both
set -x
cd /root/repo
for d in 16 4 8 12; do
  SPAMM_EX_DEBUG=$d python profiles/k3_probe.py cfg2 1e-8 fine4
done
SPAMM_EX_DEBUG=16 python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/k3_probe.py cfg2 1e-8 fine4
python profiles/k3_probe.py cfg2 1e-8 coarse16
