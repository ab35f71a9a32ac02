#!/bin/bash
# plan_emit_kernel asks L2 for every record's operand blocks (cp.async.bulk.prefetch.L2); interior fold with both child loads in flight.
set -x
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for rep in 1 2 3; do
  for v in variants/lib_head.so "" "off"; do
    unset SPAMM_B200_LIB SPAMM_PLAN_PREFETCH
    [ "$v" = "off" ] && export SPAMM_PLAN_PREFETCH=0
    [ -n "$v" ] && [ "$v" != "off" ] && export SPAMM_B200_LIB=$v
    python profiles/stage_probe.py cfg2 | grep flushed
    python profiles/stage_probe.py cfg1 1e-6 | grep flushed
  done
done
