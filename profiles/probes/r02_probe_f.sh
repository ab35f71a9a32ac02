set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for g in coarse16 fine4; do
  python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_EX_STAGES=2 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_REC_WEIGHT=24 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_REC_WEIGHT=12 python profiles/k3_probe.py cfg2 1e-8 $g
done
mkdir -p gpurun_out/r02f
SPAMM_EX_TRACE=gpurun_out/r02f/trace_fine4.txt python profiles/k3_probe.py cfg2 1e-8 fine4
python profiles/trace_summary.py gpurun_out/r02f/trace_fine4.txt
SPAMM_EX_TRACE=gpurun_out/r02f/trace_c16.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace_summary.py gpurun_out/r02f/trace_c16.txt
python profiles/k3_probe.py cfg5 1e-8 coarse16
SPAMM_PIECE_RECORDS=64 python profiles/k3_probe.py cfg5 1e-8 coarse16
SPAMM_PIECE_RECORDS=1000000 python profiles/k3_probe.py cfg5 1e-8 coarse16
python profiles/k3_probe.py cfg5 1e-8 fine4
python profiles/k3_probe.py cfg3 1e-8 coarse16
python profiles/k3_probe.py cfg3 1e-8 fine4
python profiles/k3_probe.py cfg1 1e-6 fine4
python profiles/k3_probe.py cfg4 1e-8 coarse16
python profiles/k3_probe.py cfg4 1e-8 fine4
python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-configs
