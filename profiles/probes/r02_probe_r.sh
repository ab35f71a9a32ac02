set -x
cd /root/repo
mkdir -p gpurun_out/r02r
export SPAMM_TAIL_RECORDS=0
for w in cfg2 cfg5 cfg3 cfg4; do for g in coarse16 fine4; do python profiles/k3_probe.py $w 1e-8 $g; done; done
python profiles/k3_probe.py cfg1 1e-6 fine4
for rw in 16 24 48; do SPAMM_REC_WEIGHT=$rw python profiles/k3_probe.py cfg2 1e-8 coarse16; SPAMM_REC_WEIGHT=$rw python profiles/k3_probe.py cfg2 1e-8 fine4; done
for pr in 48 96 384; do SPAMM_PIECE_RECORDS=$pr python profiles/k3_probe.py cfg5 1e-8 coarse16; done
SPAMM_PIECE_RECORDS=96 python profiles/k3_probe.py cfg4 1e-8 coarse16
SPAMM_EX_TRACE=gpurun_out/r02r/trace_c16.txt python profiles/k3_probe.py cfg2 1e-8 coarse16
python profiles/trace_summary.py gpurun_out/r02r/trace_c16.txt
python profiles/fit_weights.py gpurun_out/r02r/trace_c16.txt
SPAMM_EX_TRACE=gpurun_out/r02r/trace_fine4.txt python profiles/k3_probe.py cfg2 1e-8 fine4
python profiles/trace_summary.py gpurun_out/r02r/trace_fine4.txt
python profiles/fit_weights.py gpurun_out/r02r/trace_fine4.txt
unset SPAMM_TAIL_RECORDS
python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu --no-configs | cut -c1-700
