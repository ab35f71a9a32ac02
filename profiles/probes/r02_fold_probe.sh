#!/bin/bash
# Interior levels of C folded in the numeric kernel (tile level in the epilogue, the rest by the last team; SPAMM_FOLD=0:
# all in the interior kernel).
set -x
cd /root/repo
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for rep in 1 2; do
  for f in 0 1; do
    SPAMM_FOLD=$f python profiles/stage_probe.py cfg2
    SPAMM_FOLD=$f python profiles/stage_probe.py cfg1 1e-6
    SPAMM_FOLD=$f python profiles/k3_probe.py cfg2 1e-8 fine4
  done
done
