set -x
cd /root/repo
for t in -1 0 2 3; do
  SPAMM_TAIL_RECORDS=$t python profiles/k3_probe.py cfg2 1e-8 coarse16 1024
  SPAMM_TAIL_RECORDS=$t python profiles/k3_probe.py cfg1 1e-6 fine4
  SPAMM_TAIL_RECORDS=$t python profiles/k3_probe.py cfg2 1e-8 coarse16 2048
done
SPAMM_TAIL_RECORDS=3 SPAMM_TAIL_PERCENT=100 python profiles/k3_probe.py cfg2 1e-8 coarse16 1024
SPAMM_TAIL_RECORDS=3 SPAMM_TAIL_PERCENT=100 python profiles/k3_probe.py cfg1 1e-6 fine4
python profiles/stage_probe.py cfg2
python profiles/stage_probe.py cfg1 1e-6
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02v_launches.csv python profiles/stage_probe.py cfg2 > /dev/null 2>&1
