#!/bin/bash
# fine4 with gated-off micro products reading zeros (no divergent slow path): parity first, then timing.
set -x
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
python profiles/k3_probe.py cfg2 1e-8 fine4
python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/k3_probe.py cfg3 1e-8 fine4
python profiles/k3_probe.py cfg5 1e-8 fine4
python profiles/k3_probe.py cfg4 1e-8 fine4
python profiles/k3_probe.py cfg1 1e-6 fine4
python profiles/k3_probe.py cfg2 1e-6 fine4
python profiles/k3_probe.py cfg2 1e-10 fine4
