set -x
cd /root/repo
mkdir -p gpurun_out/r02h
SPAMM_EX_TRACE2=gpurun_out/r02h/t2_c16.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace2_summary.py gpurun_out/r02h/t2_c16.txt
SPAMM_EX_TRACE2=gpurun_out/r02h/t2_c16_nocopy.txt SPAMM_EX_DEBUG=1 python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace2_summary.py gpurun_out/r02h/t2_c16_nocopy.txt | tail -3
for h in 0 1000; do
  SPAMM_B200_LIB=/root/repo/variants/lib_hint$h.so python profiles/k3_probe.py cfg2 1e-8 coarse16
  SPAMM_B200_LIB=/root/repo/variants/lib_hint$h.so SPAMM_REC_WEIGHT=28 python profiles/k3_probe.py cfg2 1e-8 coarse16
done
SPAMM_REC_WEIGHT=28 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_REC_WEIGHT=28 SPAMM_EX_DEBUG=1 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_REC_WEIGHT=28 SPAMM_EX_DEBUG=2 python profiles/k3_probe.py cfg2 1e-8 coarse16
SPAMM_REC_WEIGHT=28 SPAMM_EX_DEBUG=3 python profiles/k3_probe.py cfg2 1e-8 coarse16
