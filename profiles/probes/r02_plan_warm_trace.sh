#!/bin/bash
# Planner time line with warm caches (no L2 flush between multiplies) against the flushed one: how much of
# plan_emit_kernel's tail is first-touch (instruction and data fetches from DRAM)?
set -x
cd /root/repo
PROBE_ONLY_WARM=1 SPAMM_PIPE_STOP=2 SPAMM_PLAN_TRACE=gpurun_out/r02be_warm.txt python profiles/stage_probe.py cfg2
python profiles/plan_small_trace_summary.py gpurun_out/r02be_warm.txt
SPAMM_PIPE_STOP=2 SPAMM_PLAN_TRACE=gpurun_out/r02be_cold.txt python profiles/stage_probe.py cfg2
python profiles/plan_small_trace_summary.py gpurun_out/r02be_cold.txt
