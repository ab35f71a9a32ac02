#!/bin/bash
# Small dense products: plan_count + plan_emit (2 kernels) against plan_tiles + plan_order (SPAMM_PLAN_SMALL=0).
set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
for rep in 1 2; do
  for f in 0 1; do
    SPAMM_PLAN_SMALL=$f python profiles/stage_probe.py cfg2
    SPAMM_PLAN_SMALL=$f python profiles/stage_probe.py cfg1 1e-6
    SPAMM_PLAN_SMALL=$f SPAMM_PIPE_STOP=2 python profiles/stage_probe.py cfg2
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02ak_launches.csv python profiles/stage_probe.py cfg2 > /dev/null 2>&1
