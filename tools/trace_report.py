import sys, numpy as np
rows = [l.split() for l in open(sys.argv[1]) if not l.startswith('#')]
A = np.array([[int(v) for v in r] for r in rows])
L = int(open(sys.argv[1]).readline().split('L=')[1])
NP = 2 * L
print("CTA0 task: rhs", A[0,1]-A[0,0], "end", A[0,63]-A[0,0])
ends = [A[0,1]] + [A[0,2+p] for p in range(NP)]
for p in range(NP):
    st = ends[p]; en = ends[p+1]
    items = [(b, A[b,64+8*p:64+8*p+5]) for b in range(A.shape[0]) if A[b,64+8*p] >= 0]
    desc = " ".join(f"c{b}:[{it[1]-it[0]},{it[2]-it[1]},{it[3]-it[2]},{it[4]-it[3]}]@{it[0]-st}" for b, it in items[:6])
    last = max([it[4] for b, it in items], default=st)
    print(f"p{p:2d} dur {en-st:5d}  last item done +{last-st:5d}  items(seq,mbar,comp,refill)@start: {desc}")
