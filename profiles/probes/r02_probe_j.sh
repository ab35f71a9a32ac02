set -x
cd /root/repo
mkdir -p gpurun_out/r02j
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_stress.py tests/test_gpu_kat.py -x -q 2>&1 | tail -15
for g in coarse16 fine4; do
  python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_TAIL_RECORDS=3 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_TAIL_RECORDS=1 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_TAIL_RECORDS=0 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_REC_WEIGHT=48 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_REC_WEIGHT=16 python profiles/k3_probe.py cfg2 1e-8 $g
done
SPAMM_EX_TRACE=gpurun_out/r02j/trace_c16.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace_summary.py gpurun_out/r02j/trace_c16.txt
python profiles/k3_probe.py cfg5 1e-8 coarse16
python profiles/k3_probe.py cfg5 1e-8 fine4
python profiles/k3_probe.py cfg3 1e-8 coarse16
python profiles/k3_probe.py cfg1 1e-6 fine4
python profiles/k3_probe.py cfg4 1e-8 coarse16
