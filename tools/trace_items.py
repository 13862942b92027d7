"""Per-item timeline of one slab solve (task 1, CTA 0) from an HS_SWEEP_TRACE dump:
issue (producer), data ready (consumer after the mbarrier), consumed; all in ns
from the CTA's task start, plus the phase end stamps."""
import sys
import numpy as np
rows = [l.split() for l in open(sys.argv[1]) if not l.startswith('#')]
A = np.array([[int(v) for v in r] for r in rows])
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
a = A[cta]
t0 = a[0]
print("phase ends:", [int(v - t0) for v in a[1:12] if v > 0], " tips", a[40] - t0, " R", a[41] - t0,
      " corr", a[42] - t0, " out", a[43] - t0)
it = a[256:1024].reshape(-1, 3)
print("  r   issue  ready   done   (ready-issue)")
for r in range(it.shape[0]):
    if it[r, 0] < 0 and it[r, 1] < 0:
        break
    i, rd, d = (int(v - t0) if v >= 0 else -1 for v in it[r])
    print(f"{r:3d} {i:7d} {rd:7d} {d:7d}   {rd - i:6d}")
