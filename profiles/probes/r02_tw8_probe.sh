#!/bin/bash
# plan_tiles with 8 nodes per block (small dense start): band blocks spread over the SMs.  A/B against the previous build.
set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  for v in variants/lib_head.so ""; do
    export SPAMM_B200_LIB=$v
    [ -z "$v" ] && unset SPAMM_B200_LIB
    python profiles/stage_probe.py cfg2
    python profiles/stage_probe.py cfg1 1e-6
    SPAMM_PIPE_STOP=2 python profiles/stage_probe.py cfg2
  done
done
unset SPAMM_B200_LIB
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02aj_launches.csv python profiles/stage_probe.py cfg2 > /dev/null 2>&1
SPAMM_PLAN_TRACE=gpurun_out/r02aj_plan_trace.txt python profiles/stage_probe.py cfg2 > /dev/null 2>&1
python profiles/plan_trace_summary.py gpurun_out/r02aj_plan_trace.txt
