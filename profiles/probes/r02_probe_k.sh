set -x
cd /root/repo
mkdir -p gpurun_out/r02k
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/inner_order profiles/microbench/inner_order.cu && /tmp/inner_order
for lib in "" /root/repo/variants/lib_teams1.so; do
  export SPAMM_B200_LIB=$lib
  [ -z "$lib" ] && unset SPAMM_B200_LIB
  for g in coarse16 fine4; do
    python profiles/k3_probe.py cfg2 1e-8 $g
    SPAMM_TAIL_PERCENT=45 python profiles/k3_probe.py cfg2 1e-8 $g
    SPAMM_TAIL_PERCENT=70 python profiles/k3_probe.py cfg2 1e-8 $g
    SPAMM_TAIL_PERCENT=100 python profiles/k3_probe.py cfg2 1e-8 $g
  done
  python profiles/k3_probe.py cfg5 1e-8 coarse16
  python profiles/k3_probe.py cfg3 1e-8 coarse16
  python profiles/k3_probe.py cfg1 1e-6 fine4
done
export SPAMM_B200_LIB=/root/repo/variants/lib_teams1.so
SPAMM_TAIL_PERCENT=45 SPAMM_EX_TRACE=gpurun_out/r02k/trace_c16_t1.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace_summary.py gpurun_out/r02k/trace_c16_t1.txt
