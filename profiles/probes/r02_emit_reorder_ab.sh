#!/bin/bash
# plan_emit_kernel: slot loads issued before the sub-norm range loads (one round trip per pass).  A/B + time line.
set -x
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
for rep in 1 2 3; do
  for v in variants/lib_head.so ""; do
    export SPAMM_B200_LIB=$v
    [ -z "$v" ] && unset SPAMM_B200_LIB
    python profiles/stage_probe.py cfg2
    python profiles/stage_probe.py cfg1 1e-6
  done
done
unset SPAMM_B200_LIB
bash profiles/probes/r02_plan_timeline.sh
