#!/bin/bash
# plan_emit_kernel walks only the block indices K that gave a record in plan_count_kernel (a 64-bit mask per super-tile).
set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2 3; do
  for v in variants/lib_head.so ""; do
    export SPAMM_B200_LIB=$v
    [ -z "$v" ] && unset SPAMM_B200_LIB
    python profiles/stage_probe.py cfg2 | grep flushed
    python profiles/stage_probe.py cfg1 1e-6 | grep flushed
  done
done
unset SPAMM_B200_LIB
SPAMM_PIPE_STOP=2 SPAMM_PLAN_TRACE=gpurun_out/r02bd_plan.txt python profiles/stage_probe.py cfg2 > /dev/null 2>&1
python profiles/plan_small_trace_summary.py gpurun_out/r02bd_plan.txt
