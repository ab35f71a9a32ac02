#!/bin/bash
# A/B: plan_count prefetching plan_emit's operands into L2.
set -x
cd /root/repo
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -q -x 2>&1 | tail -3
for rep in 1 2 3; do
  for v in variants/lib_head.so ""; do
    export SPAMM_B200_LIB=$v
    [ -z "$v" ] && unset SPAMM_B200_LIB
    python profiles/stage_probe.py cfg2
    SPAMM_PIPE_STOP=2 python profiles/stage_probe.py cfg2
    python profiles/stage_probe.py cfg1 1e-6
  done
done
