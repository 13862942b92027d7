"""Kernel-class times of one lockstep batch solve (solve_many(batch=True),
one group) of a multi-right-hand-side config vs its wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import paper_1412_0464_b200 as hb
from paper_1412_0464_b200._lib import context
from paper_1412_0464_b200.configs import config

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = config(idx, scale)
cycle, _ = hb.build_two_grid(p.mesh, p.model, smoother=hb.SmootherConfig(p.omega_jac, p.nu),
                             coarse="sweep",
                             sweep=hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                             keep_slab_ops=False)
ctx = context()
fs = [torch.from_numpy(p.f[r].ravel()).cuda() for r in range(p.f.shape[0])]
cfg = hb.GmresConfig(p.tol, p.max_iter, p.restart)
for _ in range(2):
    out = hb.solve_many(cycle, fs, cfg, batch=True, lanes=1)
torch.cuda.synchronize()
t0 = time.perf_counter()
out = hb.solve_many(cycle, fs, cfg, batch=True, lanes=1)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
ctx.profile_reset()
ctx.profile(True)
out = hb.solve_many(cycle, fs, cfg, batch=True, lanes=1)
prof = ctx.profile_read()
ctx.profile(False)
tot = sum(v["ms"] for v in prof.values())
print(f"wall {wall * 1e3:.1f} ms, kernel sum {tot:.1f} ms, its {[r.iterations for _, r in out]}")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"  {k:16s} {v['ms']:9.1f} ms {v['launches']:6d} launches  {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f} GB/s")
