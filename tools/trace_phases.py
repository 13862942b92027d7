"""Per-phase stamps of one slab step from an HS_SWEEP_TRACE file (ns from the
step start, per CTA of the first cluster): rhs, forward levels + dense top,
group A done, tips in, R GEMV, level-2 post / seen / (P, Q) / corrected,
spike correction, outputs, end."""
import re
import sys

import numpy as np

path = sys.argv[1]
hdr = open(path).readline().strip()
rows = [l.split() for l in open(path) if not l.startswith('#')]
A = np.array([[int(v) for v in r[:128]] for r in rows])
L = int(re.search(r'L=(\d+)', hdr).group(1))
print(hdr)
names = [("rhs", 1)] + [(f"p{p}", 2 + p) for p in range(L + 1)] + [
    ("A done", 48), ("tips in", 40), ("R gemv", 44), ("post", 45), ("seen", 46), ("PQ", 47),
    ("B done", 41), ("spikes", 42), ("outputs", 43), ("end", 63)]
print("cta " + " ".join(f"{n:>8s}" for n, _ in names))
for b in range(A.shape[0]):
    a = A[b]
    if a[63] <= 0:
        continue
    print(f"{b:3d} " + " ".join(f"{(a[k] - a[0]) / 1e3 if a[k] > 0 else float('nan'):8.2f}" for _, k in names))
