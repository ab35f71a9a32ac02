#!/bin/bash
# execute_kernel: the unit a team most likely draws first is requested together with the counts and the ticket.
set -x
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_stress.py -q -x 2>&1 | tail -2
for rep in 1 2 3; do
  for v in variants/lib_head.so ""; do
    export SPAMM_B200_LIB=$v
    [ -z "$v" ] && unset SPAMM_B200_LIB
    python profiles/k3_probe.py cfg2 1e-8 fine4 | cut -c1-40,140-260
    python profiles/k3_probe.py cfg2 1e-8 coarse16 | cut -c1-40,140-260
    python profiles/stage_probe.py cfg2 | grep flushed
  done
done
