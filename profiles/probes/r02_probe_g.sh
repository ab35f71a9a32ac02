set -x
cd /root/repo
mkdir -p gpurun_out/r02g
for g in coarse16 fine4; do
  SPAMM_EX_TRACE=gpurun_out/r02g/trace_$g.txt python profiles/k3_probe.py cfg2 1e-8 $g
  python profiles/trace_summary.py gpurun_out/r02g/trace_$g.txt
  python profiles/fit_weights.py gpurun_out/r02g/trace_$g.txt
  for w in 24 32 48; do SPAMM_REC_WEIGHT=$w python profiles/k3_probe.py cfg2 1e-8 $g; done
done
timeout 600 python -m pytest tests/test_gpu_reference_trees.py tests/test_gpu_partition.py tests/test_gpu_stress.py -x -q 2>&1 | tail -5
