set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python profiles/k3_probe.py cfg2 1e-8 fine4 && ncu --set full --clock-control none --import-source on -k regex:execute_kernel -c 1 -o gpurun_out/r02s_k3_cfg2_fine4 -f python profiles/k3_probe.py cfg2 1e-8 fine4 > gpurun_out/r02s_ncu_fine4.log 2>&1
python profiles/k3_probe.py cfg2 1e-8 coarse16 && ncu --set full --clock-control none --import-source on -k regex:execute_kernel -c 1 -o gpurun_out/r02s_k3_cfg2_coarse16 -f python profiles/k3_probe.py cfg2 1e-8 coarse16 > gpurun_out/r02s_ncu_c16.log 2>&1
python profiles/k3_probe.py cfg1 1e-6 fine4
python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-configs | cut -c1-2500
