"""Time the fine-level stencil kernels on a BASELINE config (GB/s vs algorithmic bytes)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import to_device, empty, ptr
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = config(idx)
from paper_1412_0464_b200.configs import fe_fine_operator
fine = fe_fine_operator(p.mesh, p.model) if p.fine != "fd5" else None
cycle, _ = hb.build_two_grid(p.mesh, p.model, fine_op=fine, smoother=hb.SmootherConfig(p.omega_jac, p.nu), coarse="sweep",
                             sweep=hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains), keep_slab_ops=False)
dev = cycle.device()
op = dev.fine
n = op.n
z = np.random.default_rng(0).standard_normal(n) + 1j
x, _ = to_device(z, n); f, _ = to_device(z[::-1].copy(), n); y = empty(n)
S = len(op.offsets)
ctx = op.ctx
def t(fn, nb, name, N=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N): fn()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / N * 1e3
    print(f"{name:10s} {us:8.2f} us  {nb * n / us / 1e3:7.1f} GB/s")
t(lambda: ctx.call("hs_stencil_apply", op.h, ptr(x), ptr(y), 1), (S + 2) * 16, "apply")
t(lambda: ctx.call("hs_stencil_residual", op.h, ptr(f), ptr(x), ptr(y), 1), (S + 3) * 16, "residual")
t(lambda: ctx.call("hs_jacobi", op.h, ptr(y), ptr(f), 0.8, 2, 0, 1), 2 * (S + 3) * 16, "jacobi x2")
t(lambda: ctx.call("hs_jacobi", op.h, ptr(y), ptr(f), 0.8, 2, 1, 1), (S + 2) * 16, "jacobi2z")
