"""Setup time of build_two_grid (host vs device assembly) on a BASELINE config,
with a cProfile of the device-assembly build."""
import cProfile, pstats, sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = config(idx)
def build(assembly):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cyc, _ = hb.build_two_grid(p.mesh, p.model, smoother=hb.SmootherConfig(p.omega_jac, p.nu),
                               coarse="sweep", sweep=hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                               keep_slab_ops=False, assembly=assembly)
    cyc.device(); torch.cuda.synchronize()
    return time.perf_counter() - t0
build("device")
for a in ("host", "device", "host", "device"):
    print(a, round(build(a), 3))
pr = cProfile.Profile(); pr.enable(); build("device"); pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
