#!/bin/bash
# plan_emit_kernel variants: sub-norm ranges requested early (same pass / one pass ahead), cut positions in double arithmetic.
set -x
cd /root/repo
for v in "" variants/lib_SUBS1.so variants/lib_SUBS2.so variants/lib_CUTD.so variants/lib_SUBS1CUTD.so; do
  export SPAMM_B200_LIB=$v
  [ -z "$v" ] && unset SPAMM_B200_LIB
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -q -x 2>&1 | tail -1
  SPAMM_PIPE_STOP=2 SPAMM_PLAN_TRACE=gpurun_out/r02ar_plan.txt python profiles/stage_probe.py cfg2 > /dev/null 2>&1
  python profiles/plan_small_trace_summary.py gpurun_out/r02ar_plan.txt | grep "emit: end"
  python profiles/stage_probe.py cfg2 | grep flushed
  python profiles/stage_probe.py cfg2 | grep flushed
  python profiles/stage_probe.py cfg1 1e-6 | grep flushed
done
