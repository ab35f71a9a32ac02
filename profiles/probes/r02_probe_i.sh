set -x
cd /root/repo
mkdir -p gpurun_out/r02i
export SPAMM_REC_WEIGHT=28
for sk in 0 160 320 480 640; do
  SPAMM_EX_SKEW=$sk python profiles/k3_probe.py cfg2 1e-8 coarse16
done
for sk in 0 320; do
  SPAMM_EX_SKEW=$sk python profiles/k3_probe.py cfg2 1e-8 fine4
  SPAMM_EX_SKEW=$sk python profiles/k3_probe.py cfg5 1e-8 coarse16
done
SPAMM_EX_SKEW=320 SPAMM_EX_TRACE2=gpurun_out/r02i/t2_skew.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace2_summary.py gpurun_out/r02i/t2_skew.txt 2>/dev/null | head -24
SPAMM_EX_SKEW=320 SPAMM_EX_TRACE=gpurun_out/r02i/trace_c16.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace_summary.py gpurun_out/r02i/trace_c16.txt
python profiles/fit_weights.py gpurun_out/r02i/trace_c16.txt
