set -x
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/order profiles/microbench/ffma2_order.cu && /tmp/order
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/inner profiles/microbench/inner_loop.cu && /tmp/inner
for w in cfg2 cfg5; do for g in coarse16 fine4; do
  python profiles/k3_probe.py $w 1e-8 $g
  SPAMM_B200_LIB=/root/repo/variants/lib_mb3.so SPAMM_EX_STAGES=2 SPAMM_EX_CTAS=3 python profiles/k3_probe.py $w 1e-8 $g
  SPAMM_B200_LIB=/root/repo/variants/lib_mb3.so SPAMM_EX_STAGES=3 SPAMM_EX_CTAS=2 python profiles/k3_probe.py $w 1e-8 $g
done; done
