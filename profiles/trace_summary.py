"""Summary of a SPAMM_EX_TRACE dump (per CTA: start, first data, end in ns, units): ramp and tail."""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], dtype=np.int64)
t0 = d[:, 1].min()
start, first, end, units = d[:, 1] - t0, d[:, 2] - t0, d[:, 3] - t0, d[:, 4] & 0xFFFFFFFF
print(f"CTAs {len(d)}  units/CTA min {units.min()} mean {units.mean():.2f} max {units.max()}")
print(f"start   : max {start.max() / 1e3:.1f} us")
print(f"1st data: mean {first.mean() / 1e3:.1f} us  max {first.max() / 1e3:.1f} us")
print(f"end     : min {end.min() / 1e3:.1f}  p10 {np.percentile(end, 10) / 1e3:.1f}  median {np.median(end) / 1e3:.1f}  "
      f"p90 {np.percentile(end, 90) / 1e3:.1f}  max {end.max() / 1e3:.1f} us")
busy = (end - first).sum() / (len(d) * (end.max()))
print(f"CTA busy fraction of the kernel span: {busy:.3f}")
