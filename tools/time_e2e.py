"""Where the e2e (host-buffer) solve spends its extra time over the device-resident one."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import to_device, from_device
p = config(1)
cycle, _ = hb.build_two_grid(p.mesh, p.model, smoother=hb.SmootherConfig(p.omega_jac, p.nu), coarse="sweep",
                             sweep=hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains), keep_slab_ops=False)
cfg = hb.GmresConfig(p.tol, p.max_iter, p.restart)
prec = cycle.as_preconditioner()
fh = torch.from_numpy(p.f[0].ravel()).pin_memory().numpy()
fd = torch.from_numpy(p.f[0].ravel()).cuda()
for _ in range(2):
    hb.gmres(cycle.fine_csr, prec, fd, cfg); hb.gmres(cycle.fine_csr, prec, fh, cfg)
def t(fn, n=3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("solve dev   %.2f ms" % t(lambda: hb.gmres(cycle.fine_csr, prec, fd, cfg)))
print("solve host  %.2f ms" % t(lambda: hb.gmres(cycle.fine_csr, prec, fh, cfg)))
print("to_device   %.2f ms" % t(lambda: to_device(fh), 10))
u = fd.clone()
print("from_device %.2f ms" % t(lambda: from_device(u, True), 10))
