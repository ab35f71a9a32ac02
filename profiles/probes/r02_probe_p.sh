set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for w in cfg2 cfg5 cfg3 cfg4; do for g in coarse16 fine4; do python profiles/k3_probe.py $w 1e-8 $g; done; done
python profiles/k3_probe.py cfg1 1e-6 fine4
SPAMM_TAIL_PERCENT=40 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_TAIL_RECORDS=2 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_REC_WEIGHT=48 python profiles/k3_probe.py cfg2 1e-8 coarse16
python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-configs > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err
cut -c1-600 gpurun_out/r02p_bench.json
