#!/bin/bash
# Weight of a record (in tasks) in the planner's partition, fine4 and coarse16, after the zero-page gating.
set -x
cd /root/repo
mkdir -p gpurun_out/r02ac
for w in 32 64 128 256; do
  SPAMM_REC_WEIGHT=$w python profiles/k3_probe.py cfg2 1e-8 fine4
  SPAMM_REC_WEIGHT=$w python profiles/k3_probe.py cfg2 1e-8 coarse16
  SPAMM_REC_WEIGHT=$w python profiles/k3_probe.py cfg5 1e-8 fine4
done
for g in coarse16 fine4; do
  SPAMM_EX_TRACE=gpurun_out/r02ac/trace_$g.txt python profiles/k3_probe.py cfg2 1e-8 $g
  python profiles/fit_weights.py gpurun_out/r02ac/trace_$g.txt
done
