"""One rank of a multi-GPU check (run under torchrun by tests/test_gpu_parallel.py, needs >= 2 GPUs):
ShardedMultiply with every exchange mode, with and without overlap, against the single-GPU product of
the same operands, bit for bit (EXACT arithmetic) -- and bench.py's own sharded arm afterwards."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs, parallel
from paper_1203_1692_b200.symbolic import build_plan

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
try:
    for n, lam, tau in ((1024, 0.9, 1e-6), (4096, 0.95, 1e-8)):
        a = inputs.exponential_decay(n, lam, seed=0)
        qa = P.QuadtreeMatrix.from_dense(a)
        cfg = P.MultiplyConfig(tau=tau, exact=True)
        want = P.multiply(qa, qa, cfg)[0].to_dense().data
        nrows = -(-n // 16)
        counts = parallel.row_task_counts(build_plan(qa, qa, tau), qa.depth).cpu().numpy()
        splits = parallel.balanced_row_split(counts[:nrows], world)
        r0, r1 = splits[rank]
        mine = parallel.shard_of_tree(qa, r0, r1)
        for exchange in ("all", "needed", "auto"):
            for overlap in (False, True):
                sm = parallel.ShardedMultiply(mine, None, (n, n), (n, n), cfg, splits=splits, exchange=exchange, overlap=overlap)
                for _ in range(2):
                    parts = sm.run()
                    got = np.zeros_like(want)
                    for (lo, hi), c, plan, k in parts:
                        got[lo * 16:hi * 16] = c.to_dense().data[lo * 16:hi * 16]
                    assert np.array_equal(got[r0 * 16:r1 * 16], want[r0 * 16:r1 * 16]), (n, exchange, overlap, rank)
                    covered = sorted(p[0] for p in parts)
                    assert covered[0][0] == r0 and covered[-1][1] == r1
        c, plan, k = parallel.multiply_sharded(mine, None, (n, n), (n, n), cfg, exchange="needed", splits=splits)
        assert np.array_equal(c.to_dense().data[r0 * 16:r1 * 16], want[r0 * 16:r1 * 16])
    dist.barrier()
    if rank == 0:
        print("SHARDED OK", world)
finally:
    dist.destroy_process_group()
