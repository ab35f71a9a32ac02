#!/bin/bash
# Time line of one multiply on config 2: planner kernels per block, then the numeric kernel's teams.
set -x
cd /root/repo
SPAMM_PLAN_TRACE=gpurun_out/r02ao_plan.txt SPAMM_EX_TRACE=gpurun_out/r02ao_ex.txt python profiles/stage_probe.py cfg2 > /dev/null 2>&1
python profiles/plan_small_trace_summary.py gpurun_out/r02ao_plan.txt gpurun_out/r02ao_ex.txt
