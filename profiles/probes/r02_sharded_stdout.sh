#!/bin/bash
# The sharded arm must print exactly one line (the JSON) on stdout, whatever NCCL logs.
set -x
cd /root/repo
SPAMM_BENCH_SHARDED=1 python bench.py --steps 3 --warmup 3 --workload cfg5 > gpurun_out/r02aw_sh.json 2> gpurun_out/r02aw_sh.err
wc -l gpurun_out/r02aw_sh.json; head -c 200 gpurun_out/r02aw_sh.json; echo; grep -c "NCCL version" gpurun_out/r02aw_sh.err
NCCL_DEBUG=INFO SPAMM_BENCH_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 3 --warmup 3 --workload cfg5 > gpurun_out/r02aw_sh2.json 2> gpurun_out/r02aw_sh2.err
wc -l gpurun_out/r02aw_sh2.json; head -c 200 gpurun_out/r02aw_sh2.json; echo; python -c "
import json; d=json.loads(open('gpurun_out/r02aw_sh2.json').read()); print(d['ms_per_step'], d['config']['without_exchange']['ms_per_step'])"
timeout 600 python -m pytest tests/test_gpu_bench_contract.py tests/test_gpu_parallel.py -q 2>&1 | tail -2
