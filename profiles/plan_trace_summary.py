"""Summary of a SPAMM_PLAN_TRACE dump: per block start / tile claimed / candidates listed / counted / look-back done / end (ns)."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
d = d[d[:, 2] > 0]                      # blocks that got a tile
t0 = d[:, 1].min()
names = ["start", "tile claimed", "candidates", "counted (phase 1)", "look-back done", "end"]
for k, nm in enumerate(names):
    x = d[:, 1 + k] - t0
    print(f"{nm:20s} median {np.median(x) / 1e3:6.2f} us   max {x.max() / 1e3:6.2f} us")
