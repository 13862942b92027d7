"""DGKS gate statistics of a BASELINE config's solve: per Arnoldi step the
ratio ||w'||^2 / ||w||^2 after the first Gram-Schmidt pass for w = A M v_k
(what the solver does) and what it would be for the shifted vector
w - v_k = (A M - I) v_k (same Krylov space, same remainder w')."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import paper_1412_0464_b200 as hb
from paper_1412_0464_b200 import krylov
from paper_1412_0464_b200.configs import config

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = config(idx)
cycle, _ = hb.build_two_grid(p.mesh, p.model, smoother=hb.SmootherConfig(p.omega_jac, p.nu),
                             coarse="sweep",
                             sweep=hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                             keep_slab_ops=False)
rows = []
orig = krylov._givens_column


def spy(hess, cs, sn, g, k):
    rows.append((k, complex(hess[k, k]), float(abs(hess[k + 1, k]) ** 2),
                 float(np.sum(np.abs(hess[:k + 1, k]) ** 2))))
    return orig(hess, cs, sn, g, k)


krylov._givens_column = spy
f = torch.from_numpy(p.f[0].ravel()).cuda()
u, rep = hb.gmres(cycle.fine_csr, cycle.as_preconditioner(), f,
                  hb.GmresConfig(p.tol, p.max_iter, p.restart), pipelined=False)
print(f"config {idx}: {rep.iterations} iterations")
open_now = open_shift = 0
for k, hkk, rem2, proj2 in rows:
    w2 = proj2 + rem2                         # ||w||^2 = ||V^H w||^2 + ||w'||^2
    ws2 = w2 - 2.0 * hkk.real + 1.0           # ||w - v_k||^2
    r_now, r_shift = rem2 / w2, rem2 / ws2
    open_now += r_now < 0.5
    open_shift += r_shift < 0.5
print(f"gate open (second pass runs): now {open_now}/{len(rows)}, shifted {open_shift}/{len(rows)}")
rs = np.array([rem2 / (proj2 + rem2 - 2.0 * hkk.real + 1.0) for k, hkk, rem2, proj2 in rows])
rn = np.array([rem2 / (proj2 + rem2) for k, hkk, rem2, proj2 in rows])
print("ratio now    : min %.3g median %.3g max %.3g" % (rn.min(), np.median(rn), rn.max()))
print("ratio shifted: min %.3g median %.3g max %.3g" % (rs.min(), np.median(rs), rs.max()))
