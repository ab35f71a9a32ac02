set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for w in cfg2 cfg5 cfg3 cfg4; do for g in coarse16 fine4; do python profiles/k3_probe.py $w 1e-8 $g; done; done
python profiles/k3_probe.py cfg1 1e-6 fine4
python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-configs > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
cut -c1-1500 gpurun_out/r02o_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02o_launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-configs > /dev/null 2>&1
tail -40 gpurun_out/r02o_launches.csv | cut -d, -f5,12- | cut -c1-120
