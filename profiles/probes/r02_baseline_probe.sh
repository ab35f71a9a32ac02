set -x
mkdir -p gpurun_out/r02a
cd /root/repo
for g in fine4 coarse16; do
  python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_EX_DEBUG=1 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_EX_DEBUG=2 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_EX_STAGES=2 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_EX_STAGES=2 SPAMM_EX_CTAS=3 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_EX_CTAS=1 SPAMM_EX_STAGES=6 python profiles/k3_probe.py cfg2 1e-8 $g
  SPAMM_UNIT_TARGET=0 python profiles/k3_probe.py cfg2 1e-8 $g
done
SPAMM_EX_TRACE=gpurun_out/r02a/trace_fine4.txt python profiles/k3_probe.py cfg2 1e-8 fine4
python profiles/trace_summary.py gpurun_out/r02a/trace_fine4.txt
python profiles/k3_probe.py cfg5 1e-8 coarse16
SPAMM_EX_DEBUG=1 python profiles/k3_probe.py cfg5 1e-8 coarse16
python profiles/k3_probe.py cfg2 1e-8 coarse16 16384
SPAMM_EX_DEBUG=1 python profiles/k3_probe.py cfg2 1e-8 coarse16 16384
