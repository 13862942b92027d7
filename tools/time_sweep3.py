"""Time the 3-D sweep (C5 coarse level): ms per X sweep and per slab solve."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import to_device, empty, ptr
p = config(4)
t0 = time.time()
hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                        hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains), keep_slab_ops=False)
sw = hh.partition.device()
print(f"setup {time.time() - t0:.1f} s, factors {sw.factor_bytes / 1e9:.1f} GB" if hasattr(sw, "factor_bytes") else f"setup {time.time()-t0:.1f} s")
z = np.random.default_rng(0).standard_normal(sw.n) + 0j
f, _ = to_device(z, sw.n)
u = empty(sw.n)
sw.ctx.call("hs_sweep_apply", sw.h, 1, ptr(f), ptr(u))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 3
e0.record()
for _ in range(N):
    sw.ctx.call("hs_sweep_apply", sw.h, 1, ptr(f), ptr(u))
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / N
J = p.subdomains
print(f"C5 3-D X sweep {ms:.2f} ms -> {ms / (J + 2) * 1e3:.0f} us per slab step ({ms / (2 * J) * 1e3:.0f} us per slab solve)")
