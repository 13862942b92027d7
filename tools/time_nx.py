"""Time the X and NX sweeps (n cells) on a BASELINE config's coarse level."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import to_device, empty, ptr
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = config(idx)
hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                        hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                        keep_slab_ops=False)
sw = hh.partition.device()
f, _ = to_device(np.random.default_rng(0).standard_normal(sw.n) + 0j, sw.n)
u = empty(sw.n)
for label, v in [("X", sw.variant_id("x"))] + [
        (f"NX({n})", sw.variant_id("nx", hb.make_nx_cells(p.subdomains, n))) for n in (1, 2, 4, 8)]:
    for _ in range(3):
        sw.ctx.call("hs_sweep_apply", sw.h, v, ptr(f), ptr(u))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sw.ctx.call("hs_sweep_apply", sw.h, v, ptr(f), ptr(u))
    e1.record(); torch.cuda.synchronize()
    print(f"config {idx} {label:6s} {e0.elapsed_time(e1) / 10:.3f} ms per sweep")
