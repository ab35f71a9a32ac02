"""Where the time of one sharded multiply goes (world size 1, NCCL): tuning aid for parallel.py."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs, parallel
from paper_1203_1692_b200.numeric import multiply_async
from paper_1203_1692_b200.symbolic import build_plan

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
a, _ = inputs.make_operands(name)
m = a.shape[0]
q = P.QuadtreeMatrix.from_dense(a)
mine = parallel.shard_of_tree(q, 0, 1 << 30)
del q, a
cfg = P.MultiplyConfig(tau=1e-8)

def timed(label, fn, reps=5):
    out = None
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{label:40s} {min(ts):8.3f} ms")
    return out

g = timed("allgather_shards", lambda: parallel.allgather_shards(mine))
timed("tree_from_shard (B: no transposed copy)", lambda: parallel.tree_from_shard(m, m, g, transposed=False))
full = timed("tree_from_shard (A: with transposed copy)", lambda: parallel.tree_from_shard(m, m, g))
plan = timed("build_plan (sync)", lambda: build_plan(full, full, cfg.tau))
cnt = timed("row_task_counts + cpu", lambda: parallel.row_task_counts(plan, plan.depth).cpu().numpy())
timed("multiply_async(row_range) + sync", lambda: multiply_async(full, full, cfg, None, row_range=(0, -(-m // 16))))
timed("multiply_sharded total", lambda: parallel.multiply_sharded(mine, None, (m, m), (m, m), cfg))
dist.destroy_process_group()
