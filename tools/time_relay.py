"""Relay vs replication of the coarse sweep, one B200:
the X sweep as one plan (replicated coarse level: every GPU runs it whole)
against the same sweep cut into one launch per sweep-axis shard step
(hs_sweep_plan_relay: the critical path of a relay in which each of G GPUs
owns its region's slabs; the P2P trace hop itself is not included).

    python tools/time_relay.py [config=2] [shards...]
"""
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import numpy as np
import torch
import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import config
from paper_1412_0464_b200.device import empty, ptr, to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
shards = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
p = config(idx)
hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                        hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                        keep_slab_ops=False)
sw = hh.partition.device()
z = np.random.default_rng(0).standard_normal(sw.n) + 1j * np.random.default_rng(1).standard_normal(sw.n)
f, _ = to_device(z, sw.n)


def timed(variant, n=10):
    u = empty(sw.n)
    for _ in range(3):
        sw.ctx.call("hs_sweep_apply", sw.h, variant, ptr(f), ptr(u))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        sw.ctx.call("hs_sweep_apply", sw.h, variant, ptr(f), ptr(u))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, u


ms_x, ux = timed(sw.variant_id("x"))
out = {"config": p.name, "J": p.subdomains, "segments": sw.segments, "x_plan_ms": ms_x,
       "relay": {}}
for g in shards:
    v = sw.relay_variant(g)
    ms, u = timed(v)
    # (bitwise equal with one face segment; with the two-level partition a
    # front's first task after a cut reads its trace from global memory
    # instead of the level-2 edge values: equal to rounding)
    out["relay"][g] = {"ms": ms, "launches": sw.ctx.lib.hs_sweep_plan_launches(sw.h, v),
                       "rel_diff_vs_x": float(torch.linalg.norm(u - ux) / torch.linalg.norm(ux))}
print(json.dumps(out))
