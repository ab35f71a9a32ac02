#!/bin/bash
# Round-2 evidence run (one GPU): plain bench first, then the ncu launch list of the same command, then one
# `ncu --set full` capture per kernel, each only after its command exited 0 without ncu.  Outputs: gpurun_out/r02_final/.
set -x
cd /root/repo
O=gpurun_out/r02_final
mkdir -p $O
python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-configs > $O/bench_short.json 2> $O/bench_short.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/r02_launches_bench_steps3.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-configs > /dev/null 2>&1
cap() {   # name, kernel regex, command...
  local name=$1 k=$2; shift 2
  "$@" > $O/$name.plain.log 2>&1 || return 1
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/$name -f "$@" > $O/$name.ncu.log 2>&1
  python profiles/ncu_summary.py $O/$name.ncu-rep 30 > $O/$name.txt 2>&1
}
cap r02_ncu_k3_cfg2_fine4 execute_kernel python profiles/k3_probe.py cfg2 1e-8 fine4
cap r02_ncu_k3_cfg2_coarse16 execute_kernel python profiles/k3_probe.py cfg2 1e-8 coarse16
cap r02_ncu_k3_cfg3_fine4 execute_kernel python profiles/k3_probe.py cfg3 1e-8 fine4
cap r02_ncu_k3_cfg5_fine4 execute_kernel python profiles/k3_probe.py cfg5 1e-8 fine4
cap r02_ncu_k3_cfg5_coarse16 execute_kernel python profiles/k3_probe.py cfg5 1e-8 coarse16
cap r02_ncu_plan_count plan_count_kernel python profiles/stage_probe.py cfg2
cap r02_ncu_plan_emit plan_emit_kernel python profiles/stage_probe.py cfg2
rm -f $O/r02_ncu_k3_cfg5_*.ncu-rep      # large; the summaries stay
ls -la $O
