#!/bin/bash
# Per-warp time stamps of the first records of one team: where a record's time goes on cfg3 (sparse records) and cfg2.
set -x
cd /root/repo
mkdir -p gpurun_out/r02y
timeout 600 python -m pytest tests/test_gpu_reference_trees.py -x -q 2>&1 | tail -3
for w in "cfg3 1e-8 fine4" "cfg3 1e-8 coarse16" "cfg2 1e-8 coarse16"; do
  tag=$(echo $w | tr ' ' '_')
  SPAMM_EX_TRACE2=gpurun_out/r02y/t2_$tag.txt python profiles/k3_probe.py $w
  python profiles/trace2_summary.py gpurun_out/r02y/t2_$tag.txt > gpurun_out/r02y/t2_$tag.summary
done
for d in 1 2 3; do SPAMM_EX_DEBUG=$d python profiles/k3_probe.py cfg3 1e-8 fine4; done
python bench.py --steps 20 --warmup 3 > gpurun_out/r02y/bench.json 2> gpurun_out/r02y/bench.err
