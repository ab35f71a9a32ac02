#!/bin/bash
# n = 8192 (2048 blocks of 8 super-tiles) through plan_count + plan_emit with sums per group of 4 blocks. A/B against the look-back kernel.
set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  for v in variants/lib_head.so ""; do
    export SPAMM_B200_LIB=$v
    [ -z "$v" ] && unset SPAMM_B200_LIB
    python profiles/stage_probe.py cfg3 | grep flushed
    SPAMM_PIPE_STOP=2 python profiles/stage_probe.py cfg3 | grep flushed
    python profiles/stage_probe.py cfg2 | grep flushed
    python profiles/k3_probe.py cfg2 1e-8 coarse16 8192 | cut -c1-200
  done
done
