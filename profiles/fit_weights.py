"""Least-squares fit of the time a team of execute_kernel needs for its piece against the piece's
records and live tasks (SPAMM_EX_TRACE dump + the plan saved by k3_probe.py): how much a record
weighs, in tasks, in the planner's partition (SPAMM_REC_WEIGHT).
    python profiles/fit_weights.py <trace.txt>"""
import sys
import numpy as np
tr = np.loadtxt(sys.argv[1], dtype=np.int64)
z = np.load(sys.argv[1] + ".plan.npz")
pieces, rec = z["pieces"].astype(np.int64), z["rec"]
t0 = tr[:, 1].min()
first, end, units, piece0 = (tr[:, 2] - t0) / 1e3, (tr[:, 3] - t0) / 1e3, tr[:, 4] & 0xFFFFFFFF, tr[:, 4] >> 32
R = rec.shape[0]
tasks = np.zeros(R, np.int64)
passes = np.zeros(R, np.int64)
dead = [rec[:, 13] & 0xFFFF, rec[:, 13] >> 16, rec[:, 14] & 0xFFFF, rec[:, 14] >> 16]
fine = "fine4" in sys.argv[1]
for kk in range(4):
    live = rec[:, 8 + kk] & 0xFFFF
    if fine:
        live = live & ~dead[kk]
    tasks += np.array([bin(int(x)).count("1") for x in live])
    for w in range(8):
        passes += ((live >> (2 * w)) & 3) != 0
cr, ct, cp = (np.concatenate([[0], np.cumsum(x)]) for x in (np.ones(R, np.int64), tasks, passes))
b, e = pieces[:, 0], pieces[:, -1]
if len(pieces) != len(tr):
    print("pieces", len(pieces), "teams", len(tr), ": fit needs one round (one piece per team)")
    sys.exit(0)
# the trace records the first piece every team drew
b, e = b[piece0], e[piece0]
dur = end - first
X = np.stack([cr[e] - cr[b], ct[e] - ct[b], np.ones(len(b))], 1).astype(float)
coef, res, *_ = np.linalg.lstsq(X, dur, rcond=None)
print("dur = %.3f us/record + %.4f us/task + %.2f us ; a record weighs %.1f tasks" % (coef[0], coef[1], coef[2], coef[0] / max(coef[1], 1e-9)))
Xp = np.stack([cr[e] - cr[b], cp[e] - cp[b], np.ones(len(b))], 1).astype(float)
cf2, *_ = np.linalg.lstsq(Xp, dur, rcond=None)
print("dur = %.3f us/record + %.4f us/warp-pass + %.2f us" % tuple(cf2))
print("duration min %.1f median %.1f max %.1f; records/piece min %d max %d; tasks/piece min %d max %d" % (
    dur.min(), np.median(dur), dur.max(), X[:, 0].min(), X[:, 0].max(), X[:, 1].min(), X[:, 1].max()))
print("residual rms %.2f us (tasks model), %.2f us (passes model)" % (np.sqrt(np.mean((X @ coef - dur) ** 2)), np.sqrt(np.mean((Xp @ cf2 - dur) ** 2))))
