#!/bin/bash
# A/B on one box: 2-word units (previous commit) against 4-word units, alternating.
set -x
cd /root/repo
for rep in 1 2 3; do
  for v in variants/lib_unit2.so ""; do
    export SPAMM_B200_LIB=$v
    [ -z "$v" ] && unset SPAMM_B200_LIB
    python profiles/k3_probe.py cfg2 1e-8 coarse16
    python profiles/k3_probe.py cfg2 1e-8 fine4
  done
done
