#!/bin/bash
# What plan_emit_kernel's band blocks spend their 10 us on: planner only (SPAMM_PIPE_STOP=2), per-block time stamps,
# with the cut placement and / or the task classification switched off.
set -x
cd /root/repo
for d in 0 1 2 3; do
  SPAMM_PLAN_DEBUG=$d SPAMM_PIPE_STOP=2 SPAMM_PLAN_TRACE=gpurun_out/r02aq_plan_$d.txt python profiles/stage_probe.py cfg2 > /dev/null 2>&1
  python profiles/plan_small_trace_summary.py gpurun_out/r02aq_plan_$d.txt
done
