#!/bin/bash
# 4-word work units (no record look-ups when a unit is claimed) + counts requested before the ticket.
set -x
cd /root/repo
timeout 1200 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
python profiles/k3_probe.py cfg2 1e-8 fine4
python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/k3_probe.py cfg3 1e-8 fine4
python profiles/k3_probe.py cfg5 1e-8 fine4
python profiles/k3_probe.py cfg5 1e-8 coarse16
python profiles/k3_probe.py cfg1 1e-6 fine4
python profiles/k3_probe.py cfg2 1e-8 coarse16 2048
python profiles/k3_probe.py cfg2 1e-8 coarse16 1024
mkdir -p gpurun_out/r02ae
SPAMM_EX_TRACE=gpurun_out/r02ae/trace_coarse16.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/stage_probe.py cfg2
python profiles/stage_probe.py cfg1 1e-6
