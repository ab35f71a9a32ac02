set -x
cd /root/repo
python bench.py --steps 20 --warmup 5 > gpurun_out/r02u_bench.json 2> gpurun_out/r02u_bench.err
tail -c 600 gpurun_out/r02u_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02u_bench_ref.json 2>> gpurun_out/r02u_bench.err
cut -c1-900 gpurun_out/r02u_bench_ref.json
SPAMM_BENCH_SHARDED=1 python bench.py --steps 5 --warmup 3 --workload cfg5 > gpurun_out/r02u_bench_sh.json 2> gpurun_out/r02u_bench_sh.err
cut -c1-1500 gpurun_out/r02u_bench_sh.json; tail -c 800 gpurun_out/r02u_bench_sh.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02u_launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-configs > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()"
