"""Two-level face partition check: the coarse X sweep of a BASELINE config
built with G = 1 and with G segments per front (HS_SWEEP_SEGMENTS /
HS_SWEEP_CPC), outputs compared and timed.

    python tools/check_segments.py CONFIG [SCALE] [G,C G,C ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import empty, ptr, to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1
variants = [tuple(int(v) for v in a.split(",")) for a in sys.argv[3:]] or [(1, 16), (2, 16), (4, 16)]
p = config(idx, scale)
z = None
ref = None
for G, C in variants:
    os.environ["HS_SWEEP_SEGMENTS"] = str(G)
    os.environ["HS_SWEEP_CPC"] = str(C)
    t0 = time.perf_counter()
    hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                            hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                            keep_slab_ops=False)
    sw = hh.partition.device()
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    if z is None:
        z = np.random.default_rng(0).standard_normal(sw.n) + 1j * np.random.default_rng(1).standard_normal(sw.n)
    f, _ = to_device(z, sw.n)
    u = empty(sw.n)
    for variant, vid in (("x", 1), ("ud", 0)):
        for _ in range(3):
            sw.ctx.call("hs_sweep_apply", sw.h, vid, ptr(f), ptr(u))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        N = 10
        e0.record()
        for _ in range(N):
            sw.ctx.call("hs_sweep_apply", sw.h, vid, ptr(f), ptr(u))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / N
        out = u.cpu().numpy()
        key = variant
        if ref is None:
            ref = {}
        if key not in ref:
            ref[key] = out
            err = 0.0
        else:
            err = float(np.linalg.norm(out - ref[key]) / np.linalg.norm(ref[key]))
        # bitwise run-to-run
        sw.ctx.call("hs_sweep_apply", sw.h, vid, ptr(f), ptr(u))
        torch.cuda.synchronize()
        same = bool(np.array_equal(u.cpu().numpy(), out))
        print(f"config {idx}/{scale} G={G} C={C} (built G={sw.segments} C={sw.chunks}) "
              f"{variant}: {ms:.3f} ms/apply ({1e3 * ms / (p.subdomains + 2):.1f} us/step), "
              f"rel diff vs first {err:.2e}, repeat-bitwise {same}, setup {setup:.1f} s, "
              f"factors {sw.factor_bytes / 1e9:.2f} GB", flush=True)
    del sw, hh
