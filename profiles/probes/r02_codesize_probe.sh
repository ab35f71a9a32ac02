#!/bin/bash
# Code size of the consumer loop against the instruction cache: k loop unrolled 4 / 2 / 1, fine4 with and without the rolled path.
set -x
cd /root/repo
for v in "" variants/lib_KK2.so variants/lib_KK1.so variants/lib_NOROLL.so variants/lib_KK1NOROLL.so; do
  export SPAMM_B200_LIB=$v
  [ -z "$v" ] && unset SPAMM_B200_LIB
  python profiles/k3_probe.py cfg2 1e-8 fine4
  python profiles/k3_probe.py cfg2 1e-8 coarse16
  python profiles/k3_probe.py cfg3 1e-8 fine4
  python profiles/k3_probe.py cfg5 1e-8 fine4
  python profiles/k3_probe.py cfg5 1e-8 coarse16
done
unset SPAMM_B200_LIB
bash profiles/probes/r02_recweight_probe.sh
