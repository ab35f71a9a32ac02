#!/bin/bash
# Per-leaf staging (SPAMM_EX_LEAFCOPY = threshold in 128ths of a record's leaves; 0 = whole blocks always).
set -x
cd /root/repo
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for t in 0 64 96 128 1000; do
  export SPAMM_EX_LEAFCOPY=$t
  python profiles/k3_probe.py cfg2 1e-8 fine4
  python profiles/k3_probe.py cfg2 1e-8 coarse16
  python profiles/k3_probe.py cfg3 1e-8 fine4
  python profiles/k3_probe.py cfg5 1e-8 fine4
  python profiles/k3_probe.py cfg5 1e-8 coarse16
  python profiles/k3_probe.py cfg1 1e-6 fine4
done
