set -x
cd /root/repo
for nap in 0 64 256 1000; do
  SPAMM_EX_NAP=$nap python profiles/k3_probe.py cfg2 1e-8 coarse16
  SPAMM_EX_NAP=$nap python profiles/k3_probe.py cfg2 1e-8 fine4
done
for nap in 0 256 1000; do
  SPAMM_EX_NAP=$nap python profiles/k3_probe.py cfg3 1e-8 coarse16
  SPAMM_EX_NAP=$nap python profiles/k3_probe.py cfg5 1e-8 coarse16
done
python profiles/k3_probe.py cfg4 1e-8 coarse16
python profiles/k3_probe.py cfg1 1e-6 fine4
