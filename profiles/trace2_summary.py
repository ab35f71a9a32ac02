"""Summary of a SPAMM_EX_TRACE2 dump: per record of team 0 / CTA 0, SM-clock time stamps of its 8 consumer
warps (wait begin, data ready, math done) and of its producer (stage wanted, stage free, copies issued)."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
n = d[:, 0].max() + 1
t = d[:, 2:5].reshape(n, 9, 3).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
cons, prod = t[:, :8, :], t[:, 8, :]
wait = cons[:, :, 1] - cons[:, :, 0]
work = cons[:, :, 2] - cons[:, :, 1]
gap = cons[1:, :, 0] - cons[:-1, :, 2]
print("per record, cycles (mean over warps): wait for data, work, gap to next wait")
for r in range(min(n, 40)):
    print(f"rec {r:3d}: ready-at {np.nanmin(cons[r,:,1]):9.0f}  wait {np.nanmean(wait[r]):7.0f} (max {np.nanmax(wait[r]):6.0f})  "
          f"work {np.nanmean(work[r]):7.0f} (min {np.nanmin(work[r]):6.0f} max {np.nanmax(work[r]):6.0f})  "
          f"prod: want {prod[r,0]:9.0f} free +{prod[r,1]-prod[r,0]:6.0f} issued +{prod[r,2]-prod[r,1]:5.0f}  "
          f"data latency {np.nanmin(cons[r,:,1]) - prod[r,2]:7.0f}")
print("totals over %d records: wait %.0f  work %.0f  (cycles per record, mean over warps); record period %.0f" % (
    n, np.nanmean(wait), np.nanmean(work), (np.nanmax(cons[-1, :, 2]) - np.nanmin(cons[0, :, 0])) / n))
