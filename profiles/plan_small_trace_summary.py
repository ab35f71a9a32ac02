"""Summary of a SPAMM_PLAN_TRACE dump of the count / emit planner (n <= 4096): per block of 8 super-tiles,
plan_count_kernel start / end, plan_emit_kernel entry / released by its predecessor / prefix known / end (ns)."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
t0 = d[:, 1].min()
names = ["count: start", "count: end", "emit: entered", "emit: released", "emit: prefix known", "emit: end"]
for k, nm in enumerate(names):
    x = (d[:, 1 + k] - t0) / 1e3
    print(f"{nm:20s} min {x.min():6.2f}  median {np.median(x):6.2f}  max {x.max():6.2f} us")
if len(sys.argv) > 2:          # SPAMM_EX_TRACE dump of the numeric kernel that followed
    tr = np.loadtxt(sys.argv[2], dtype=np.int64)
    for k, nm in ((1, "execute: start"), (2, "execute: first data"), (3, "execute: end")):
        x = (tr[:, k] - t0) / 1e3
        print(f"{nm:20s} min {x.min():6.2f}  median {np.median(x):6.2f}  max {x.max():6.2f} us")
