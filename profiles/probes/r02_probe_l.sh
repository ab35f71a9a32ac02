set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for w in cfg2 cfg5 cfg3 cfg4; do for g in coarse16 fine4; do python profiles/k3_probe.py $w 1e-8 $g; done; done
python profiles/k3_probe.py cfg1 1e-6 fine4
python profiles/k3_probe.py cfg1 1e-6 coarse16
SPAMM_EX_STAGES=2 python profiles/k3_probe.py cfg2 1e-8 coarse16
python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-configs
