#!/bin/bash
# What the driver does at round end, on one fresh box: GPU tests, smoke(), both bench arms; plus the sharded arm with one rank.
set -x
cd /root/repo
O=gpurun_out/r02_driver
mkdir -p $O
timeout 1800 python -m pytest tests/ -x -q -m gpu > $O/tests.log 2>&1; tail -2 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.err
SPAMM_BENCH_SHARDED=1 python bench.py --steps 5 --warmup 3 --workload cfg5 > $O/bench_sh.json 2> $O/bench_sh.err; tail -c 300 $O/bench_sh.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err; tail -c 300 $O/bench_torchrun1.err
