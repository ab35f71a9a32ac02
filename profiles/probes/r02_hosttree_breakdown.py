"""Where the end-to-end time of multiply_host goes (config 2): phases separated by synchronisations (so their
sum exceeds the un-synchronised step)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, ctypes as C
import paper_1203_1692_b200 as P
from paper_1203_1692_b200 import inputs, _lib
from paper_1203_1692_b200.tree import _stream
a, _ = inputs.make_operands("cfg2")
qa = P.QuadtreeMatrix.from_dense(a)
cfg = P.MultiplyConfig(tau=1e-8)
h = P.HostTree.from_device(qa)
lib = _lib.lib()
host_vals = torch.empty((20000, _lib.REC), dtype=torch.float32).pin_memory()
def sync():
    torch.cuda.synchronize(); return time.perf_counter()
acc = {}
for it in range(8):
    t0 = sync()
    q = h.skeleton(); t1 = sync()
    plan = P.build_plan(q, q, cfg.tau); t2 = sync()
    fa = torch.zeros((h.nleaf,), dtype=torch.uint8, device="cuda")
    copied = torch.zeros((2,), dtype=torch.int64, device="cuda")
    bufs = plan.buffers()
    lib.spamm_mark_touched(C.byref(bufs), fa.data_ptr(), fa.data_ptr(), _stream()); t3 = sync()
    lib.spamm_gather_blocks(h.blocks.data_ptr(), fa.data_ptr(), h.nleaf, 3, q.values.data_ptr(), q.values_t.data_ptr(), copied.data_ptr(), _stream()); t4 = sync()
    c, k = P.execute_plan(plan, q, q, None, cfg); t5 = sync()
    nc = c.nleaf
    host_vals[:nc].copy_(c.values[:nc], non_blocking=True); t6 = sync()
    if it >= 3:
        for name, d in (("skeleton", t1 - t0), ("build_plan", t2 - t1), ("mark", t3 - t2), ("gather", t4 - t3), ("execute_plan", t5 - t4), ("d2h", t6 - t5), ("total", t6 - t0)):
            acc.setdefault(name, []).append(d * 1e3)
for k_, v in acc.items():
    print(f"{k_:14s} {np.median(v):7.3f} ms")
print("leaves fetched", int(copied[0].item()), "GB/s of the gather", int(copied[0].item()) * 1024 / (np.median(acc["gather"]) * 1e-3) / 1e9)
