#!/bin/bash
# dense starts up to n = 8192 through plan_count + plan_emit; warm-cache kernel durations (ncu without its own flush)
set -x
cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for f in 0 1; do
  SPAMM_PLAN_SMALL=$f python profiles/stage_probe.py cfg3
  SPAMM_PLAN_SMALL=$f SPAMM_PIPE_STOP=2 python profiles/stage_probe.py cfg3
  SPAMM_PLAN_SMALL=$f python profiles/stage_probe.py cfg2
done
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file gpurun_out/r02am_launches_nocc.csv python profiles/stage_probe.py cfg2 > /dev/null 2>&1
