"""hs_sweep_apply_many check + timing on a BASELINE config's coarse level:
nrhs right-hand sides through one chain of slab solves vs one application
per right-hand side (bitwise comparison, ms per application).

    python tools/time_many.py CONFIG [SCALE] [NRHS ...]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import empty, ptr, to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1
counts = [int(v) for v in sys.argv[3:]] or [1, 2, 4, 8]
p = config(idx, scale)
hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                        hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                        keep_slab_ops=False)
sw = hh.partition.device()
n = sw.n
rng = np.random.default_rng(0)
nmax = max(counts)
Z = rng.standard_normal((nmax, n)) + 1j * rng.standard_normal((nmax, n))
F, _ = to_device(Z, nmax * n)
F = F.reshape(nmax, n)
print(f"config {idx}/{scale}: J={p.subdomains} M={hh.coarse_op.shape[1]} segments={sw.segments} "
      f"chunks={sw.chunks} rhs_width={sw.rhs_width()}")
only_many = os.environ.get("HS_MANY_ONLY") is not None   # (profiling: no single applications)
for vname, vid in (("x", 1), ("ud", 0)):
    single = torch.empty_like(F)
    for r in range(0 if only_many else nmax):
        sw.ctx.call("hs_sweep_apply", sw.h, vid, ptr(F[r]), ptr(single[r]))
    torch.cuda.synchronize()

    def timed(fn, N=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(N):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / N

    u1 = empty(n)
    t1 = float("nan") if only_many else timed(
        lambda: sw.ctx.call("hs_sweep_apply", sw.h, vid, ptr(F[0]), ptr(u1)))
    for k in counts:
        U = torch.full((k, n), float("nan"), dtype=torch.complex128, device=F.device)
        tk = timed(lambda: sw.ctx.call("hs_sweep_apply_many", sw.h, vid, k, ptr(F), ptr(U), n))
        same = bool(torch.equal(U.view(torch.float64), single[:k].view(torch.float64)))
        err = float((U - single[:k]).norm() / single[:k].norm())
        print(f"  {vname}: nrhs={k}: {tk:.3f} ms ({tk / k:.3f} per rhs; single {t1:.3f}) "
              f"bitwise={same} relerr={err:.2e}")
