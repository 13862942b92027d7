"""Apply the C5 3-D X sweep to a seeded vector and save the result (A/B of two libraries)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import to_device, empty, ptr
p = config(4)
hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                        hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains), keep_slab_ops=False)
sw = hh.partition.device()
rng = np.random.default_rng(0)
z = rng.standard_normal(sw.n) + 1j * rng.standard_normal(sw.n)
f, _ = to_device(z, sw.n)
u = empty(sw.n)
sw.ctx.call("hs_sweep_apply", sw.h, 1, ptr(f), ptr(u))
torch.cuda.synchronize()
np.save(sys.argv[1], u.cpu().numpy())
