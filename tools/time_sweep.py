"""Time hs_sweep_apply on a BASELINE config's coarse level (ms per X sweep)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import to_device, empty, ptr
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
assembly = sys.argv[2] if len(sys.argv) > 2 else "device"
p = config(idx)
hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                        hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains), keep_slab_ops=False,
                        assembly=assembly)
sw = hh.partition.device()
z = np.random.default_rng(0).standard_normal(sw.n) + 0j
f, _ = to_device(z, sw.n)
u = empty(sw.n)
for _ in range(3):
    sw.ctx.call("hs_sweep_apply", sw.h, 1, ptr(f), ptr(u))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 10
e0.record()
for _ in range(N):
    sw.ctx.call("hs_sweep_apply", sw.h, 1, ptr(f), ptr(u))
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / N
print(f"[{assembly} assembly] config {idx}: J={p.subdomains} M={hh.coarse_op.shape[1]} "
      f"segments={sw.segments} chunks={sw.chunks} factor_bytes={sw.factor_bytes / 1e9:.2f} GB "
      f"sweep {ms:.3f} ms  -> {1e3*ms/(p.subdomains+2):.1f} us per slab step")
