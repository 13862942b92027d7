"""Fine-level kernel classes of the V-cycle on a BASELINE config (event
profiler: us per launch, algorithmic GB/s)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import paper_1412_0464_b200 as hb
from paper_1412_0464_b200._lib import context
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = config(idx)
cycle, _ = hb.build_two_grid(p.mesh, p.model, smoother=hb.SmootherConfig(p.omega_jac, p.nu),
                             coarse="sweep",
                             sweep=hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                             keep_slab_ops=False)
dev = cycle.device()
ctx = context()
z = np.random.default_rng(0).standard_normal(dev.n) + 1j
f, _ = to_device(z, dev.n)
for _ in range(3):
    dev.vcycle_dev(f)
torch.cuda.synchronize()
ctx.profile_reset()
ctx.profile(True)
for _ in range(10):
    dev.vcycle_dev(f)
prof = ctx.profile_read()
ctx.profile(False)
for k in ("pre_fused", "post_fused", "restrict", "stencil", "residual"):
    if k in prof:
        v = prof[k]
        print(f"config {idx} {k:11s} {1e3 * v['ms'] / v['launches']:8.1f} us  "
              f"{v['bytes'] / v['ms'] / 1e6:7.1f} GB/s")
