#!/bin/bash
# Region B no longer capped by a tenth of the unit slots (cfg1: 296 near-empty pieces in front of the layered segments).
set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python profiles/probes/r02_cfg1_check2.py
SPAMM_PLAN_SMALL=0 python profiles/probes/r02_cfg1_check2.py
python profiles/stage_probe.py cfg1 1e-6
python profiles/stage_probe.py cfg2
python profiles/k3_probe.py cfg2 1e-8 coarse16 1024
python profiles/k3_probe.py cfg2 1e-8 fine4 512
