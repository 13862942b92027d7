import sys, numpy as np
rows = [l.split() for l in open(sys.argv[1]) if not l.startswith('#')]
A = np.array([[int(v) for v in r] for r in rows])
hdr = open(sys.argv[1]).readline()
import re
L = int(re.search(r'L=(\d+)', hdr).group(1))
NP = 2 * L + (1 if 'q=' in hdr else 0)
a = A[0]
print(hdr.strip())
print("rhs", a[1]-a[0], " local phases:", [int(a[2+p]-(a[1+p] if p else a[1])) for p in range(NP)])
print("tips barrier", a[40]-a[1+NP], " R gemv", a[41]-a[40], " correction+out+barrier", a[63]-a[41], " total", a[63]-a[0])
print("rank0 warp0 item j=0 per phase [start->seq, seq->mbar, mbar->done] and phase start offset:")
for p in range(NP):
    st = a[1+p] if p else a[1]
    it = a[64+5*p:64+5*p+5]
    if p < 12 and it[0] > 0:
        print(f"  p{p}: start+{it[0]-st}  seq {it[1]-it[0]}  mbar {it[2]-it[1]}  compute {it[3]-it[2]}  release {it[4]-it[3]}  phase end +{a[2+p]-it[4]}")
if A.shape[1] >= 256:
    pr = a[128:256].reshape(64, 2)
    print("producer (task 1, first 64 items): [spin->issued duration, gap to previous issue]")
    prev = None
    out = []
    for k in range(64):
        if pr[k, 0] < 0: break
        out.append(f"{k}:{pr[k,1]-pr[k,0]}/{(pr[k,0]-prev) if prev is not None else 0}")
        prev = pr[k, 1]
    print(" ".join(out))
