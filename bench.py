#!/usr/bin/env python
"""Benchmark: TGSP-GMRES solve on BASELINE configs[2] (C3) on B200.

A "step" = one full right-preconditioned GMRES(20) solve to 1e-6 with the
two-grid sweeping preconditioner (the north_star hot path), inputs resident
in HBM.  The default workload is C3 (4095^2 smooth random medium, 17.2 M
fine DOF), the largest BASELINE config on one GPU.  ``value`` = fine DOF/s
(n_fine * distinct solves / time, time = max over ranks of CUDA-event
time).  ``e2e`` = the same metric through the public API with the
right-hand side in host memory and the solution copied back (H2D + D2H
inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2] [--scale 1]

``--impl reference`` times the CPU oracle port of the reference algorithm
(oracle/, numpy + scipy SuperLU exactly like the reference, 2 host threads: the X sweep's two fronts concurrently) on the
same config: each step is a bounded sample of whole GMRES iterations,
projected to a full solve with the reference's own iteration count
(tests/golden/large_anchors.json, made by running the reference).
N>1 (torchrun, one process per GPU): a single-right-hand-side config is
solved ONCE, sharded along the sweep axis (strong scaling, shards.py); a
multi-right-hand-side config (C4) spreads its right-hand sides over the
ranks (each solve counted once).  See DESIGN.md section 7.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0   # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
L2_BYTES = 126 * 2**20
CPU_CORES = 2               # host threads the CPU oracle uses (the two X-sweep fronts)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=2, help="BASELINE configs index (0-based)")
    p.add_argument("--scale", type=int, default=1, help="divide the grid size (debug)")
    p.add_argument("--cpu-iters", type=int, default=1,
                   help="GMRES iterations in each bounded CPU-oracle sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--orth", default="cgs2")
    p.add_argument("--shard", action="store_true",
                   help="one solve sharded along the sweep axis over the ranks (strong "
                        "scaling; halos P2P, dots all-reduced, coarse level replicated)")
    p.add_argument("--local-shards", type=int, default=0,
                   help="with --shard on one process: G logical shards on one GPU")
    p.add_argument("--lanes", type=int, default=4,
                   help="multi-RHS configs (C4): right-hand sides in flight at once per GPU")
    p.add_argument("--no-batch", dest="batch", action="store_false",
                   help="multi-RHS configs: independent solves on concurrent lanes instead of "
                        "the default lockstep batches (gmres_many: the solves advance together "
                        "and their coarse sweeps share one chain of slab solves per group)")
    p.add_argument("--batch-groups", type=int, default=4,
                   help="with --batch: lockstep groups running side by side (one lane each)")
    p.add_argument("--segments", type=int, default=-1,
                   help="face segments per sweep front (-1: 1 when several right-hand sides "
                        "run as lanes, else automatic)")
    p.add_argument("--clock-sampler", choices=["smi", "nvml", "none"], default="smi")
    p.add_argument("--no-pipeline", action="store_true",
                   help="synchronous Arnoldi loop (A/B against the pipelined default)")
    return p.parse_args()


# ---------------------------------------------------------------------------
def dist_info():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def assign_rhs(nrhs: int, world: int, rank: int) -> list[int]:
    """Right-hand sides solved by ``rank``: round-robin over ranks.  A rank
    left without one gets none (no replicas: every solve counted is a
    distinct right-hand side; single-RHS configs shard instead, --shard)."""
    return [r for r in range(nrhs) if r % world == rank]


def reduce_over_ranks(x: float, world: int, op: str = "max", device=None) -> float:
    """max / sum of a per-rank scalar over the process group (identity for
    world == 1); ``device``: "cuda" under NCCL, "cpu" under gloo."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def job_value(n_fine: int, solves_all_ranks: float, ms_max: float) -> float:
    """Whole-job throughput: fine DOF of every solve on every rank / slowest rank's time."""
    return n_fine * solves_all_ranks / (ms_max / 1e3)


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            d = json.loads(f.read_text())
            return float(d["hbm_gbs"]), "measured"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region by a
    separate ``nvidia-smi -lms 200`` process (the profiling recipe's clocks
    line).  In-process NVML polling was measured to stall the launching
    thread (driver lock) and is only the fallback; ``mode="none"`` skips."""

    FIELDS = os.environ.get("HS_SMI_FIELDS", "clocks.sm,clocks.max.sm,clocks_event_reasons.active")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, device_index, mode="smi"):
        self.idx, self.mode = device_index, mode
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.proc = None
        self.nv = None
        self._stop = threading.Event()

    def __enter__(self):
        import shutil
        import subprocess
        import tempfile
        if self.mode == "smi" and shutil.which("nvidia-smi"):
            self.out = tempfile.TemporaryFile(mode="w+")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("HS_SMI_LMS", "200")],
                stdout=self.out, stderr=subprocess.DEVNULL)
            # nvidia-smi's start-up and its first periodic query were measured
            # to stall this process's launches (20-55 ms, once): start timing
            # only after its second sample is written
            t_end = time.perf_counter() + 5.0
            while time.perf_counter() < t_end:
                self.out.seek(0)
                if self.out.read().count("\n") >= 2:
                    break
                time.sleep(0.02)
            self.out.seek(0, 2)
        elif self.mode in ("smi", "nvml"):
            try:
                import pynvml
                pynvml.nvmlInit()
                self.nv = pynvml
                self.h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
                self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                self.t = threading.Thread(target=self._run, daemon=True)
                self.t.start()
            except Exception:
                self.nv = None
        return self

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.out.seek(0)
            for line in self.out.read().splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) < 3:
                    continue
                try:
                    self.samples.append(float(f[0]))
                    self.max_mhz = float(f[1])
                except ValueError:
                    continue
                if len(f) == 3:   # clocks_event_reasons.active: the NVML bit mask
                    try:
                        mask = int(f[2], 16) if f[2].lower().startswith("0x") else int(f[2])
                    except ValueError:
                        mask = 0
                    for bit, name in self.REASONS.items():
                        if mask & bit:
                            self.reasons.add(name)
                else:
                    for name, v in zip(self.NAMES, f[2:6]):
                        if v.lower() == "active":
                            self.reasons.add(name)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": ["unavailable" if self.mode != "none" else "not sampled"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "sampler": "nvidia-smi -lms 200" if self.proc is not None else "nvml"}


def fine_operator(p):
    """The config's fine operator: None = the 5-point FD default (SURVEY F2
    (ii)); "fe9" / "fe27" = the literal compact FE-opt operator (C5's
    27-point stencil, BASELINE configs[4])."""
    if p.fine == "fd5":
        return None
    from paper_1412_0464_b200.configs import fe_fine_operator
    return fe_fine_operator(p.mesh, p.model)


def reference_iterations(p, args):
    """GMRES iterations of the REFERENCE solver on this config (committed
    anchors, tests/golden/large_anchors.json), or None."""
    if args.scale != 1:
        return None
    f = ROOT / "tests" / "golden" / "large_anchors.json"
    try:
        d = json.loads(f.read_text())
    except Exception:
        return None
    if args.config == 3:   # C4: mean over its eight right-hand sides
        its = [d[k]["iterations"] for k in (f"C4_rhs{r}" for r in range(8)) if k in d]
        return int(round(float(np.mean(its)))) if its else None
    key = {0: "C1_x", 1: "C2", 2: "C3", 4: "C5"}.get(args.config)
    a = d.get(key)
    return None if a is None else int(a["iterations"])


def bench_config(p, args, world):
    """The ``config`` object of both arms (identical keys and values)."""
    nrhs = int(p.f.shape[0])
    if world > 1:
        par = f"rhs across {world} ranks" if nrhs > 1 else f"sweep-axis shards x{world}"
    else:
        par = "single GPU" + (f", {nrhs} rhs" if nrhs > 1 else "")
    return {"workload": workload_name(p), "fine_dof": p.n_fine, "rhs": nrhs,
            "subdomains": int(p.subdomains), "parallelism": par,
            "l2": "working set > L2 (slab factors + GMRES basis + operators stream every "
                  "step); no flush"}


def workload_name(p):
    op = {"fd5": "5-point fine op (SURVEY F2 ii)", "fe9": "9-point compact fine op",
          "fe27": "27-point compact fine op"}[p.fine]
    return (f"{p.name}: {p.mesh.dim}-D {'x'.join(map(str, p.mesh.unknowns))} fine DOF incl. PML, "
            f"{op}, TGSP X-sweep J={p.subdomains}, nu={p.nu}, GMRES({p.restart}) to {p.tol:g}")


# ---------------------------------------------------------------------------
def cpu_oracle(hh):
    """The CPU oracle (numpy/scipy restatement of the reference, SuperLU slab
    factorisations) built from the host hierarchy; setup is not timed."""
    from oracle import tgsp_oracle as orc
    t0 = time.perf_counter()
    tg = orc.from_hierarchy(hh)
    tg.fine.csr, tg.part.op.csr        # assemble the CSR matrices outside the sample
    if hasattr(tg.part, "parallel"):   # the X sweep's two fronts on two host threads
        tg.part.parallel = True         # (the reference's prec_x(parallel=True))
    return tg, time.perf_counter() - t0


def cpu_sample(problem, tg, its_target, iters):
    """Bounded sample of the CPU oracle (reference algorithm, the two X-sweep fronts on two threads):
    ``iters`` whole GMRES(restart) iterations on the config's right-hand
    side (each = one A M v + orthogonalisation) plus the solve's closing
    M dv and residual, timed, then projected per iteration to a solve of
    ``its_target`` iterations (the reference's own count)."""
    from oracle import tgsp_oracle as orc
    f = problem.f[0].ravel()
    t0 = time.perf_counter()
    _, its, _, _, _ = orc.gmres(lambda v: tg.fine.csr @ v, tg.as_preconditioner(), f,
                                tol=1e-300, max_iter=iters, restart=problem.restart)
    dt = time.perf_counter() - t0
    per_it = dt / (its + 1)           # its x (A M v + orth) + final (M dv, f - A u)
    projected = per_it * (its_target + 1)
    return {"value": problem.n_fine / projected, "projected_solve_s": projected,
            "per_iteration_s": per_it, "sample_s": dt, "sample_iterations": its}


def _sample_text(r, its_target, source, setup_s):
    return (f"{r['sample_iterations']} GMRES iteration(s) + the closing M dv / residual of the "
            f"numpy/scipy oracle port (SuperLU slab solves like the reference) timed in "
            f"{r['sample_s']:.1f} s, projected per iteration to a {its_target}-iteration solve "
            f"({source}); oracle setup {setup_s:.0f} s untimed; 2 threads (the X sweep's two "
            f"fronts run concurrently, the reference's prec_x(parallel=True); the rest is "
            f"single-threaded like the reference), host has {os.cpu_count()} cores")


def run_reference(args):
    world, rank, _ = dist_info()
    if rank != 0:
        return
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.configs import config
    p = config(args.config, args.scale)
    hh = hb.build_hierarchy(p.mesh, p.model, fine_operator(p), hb.SmootherConfig(p.omega_jac, p.nu),
                            hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                            device=False)
    its_ref = reference_iterations(p, args)
    its_target = its_ref if its_ref is not None else 50
    source = ("reference iteration count from tests/golden/large_anchors.json"
              if its_ref is not None else "no reference anchor: 50 iterations assumed")
    tg, setup_s = cpu_oracle(hh)
    vals = []
    for s_ in range(args.warmup + args.steps):
        r = cpu_sample(p, tg, its_target, args.cpu_iters)
        if s_ >= args.warmup:
            vals.append(r)
    value = float(np.median([r["value"] for r in vals]))
    ms = float(np.median([r["projected_solve_s"] for r in vals])) * 1e3
    med = sorted(vals, key=lambda r: r["value"])[len(vals) // 2]
    line = {
        "impl": "reference", "metric": "TGSP-GMRES fine DOF/s (solve to 1e-6 rel-res)",
        "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 and p.f.shape[0] == 1 else "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": bench_config(p, args, world),
        "projection": True,
        "reference_iterations": its_target,
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": CPU_CORES, "kind": "port",
                         "sample": _sample_text(med, its_target, source, setup_s)},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    world, rank, local = dist_info()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200._lib import context
    from paper_1412_0464_b200.configs import config

    p = config(args.config, args.scale)
    nrhs_total = p.f.shape[0]
    mine = assign_rhs(nrhs_total, world, rank)
    # several right-hand sides in flight as lanes: one cluster per sweep front
    # (the lanes' sweeps run side by side); one at a time: the widest layout
    # lockstep batches side by side (one lane each): small clusters with
    # several segments pack concurrent batches best (cluster CTAs x segments
    # per front, measured at C4: profiles/r2/c4_layouts.log).  Candidates in
    # order of speed; the first whose clusters all co-reside on this device
    # (hs_sweep_max_fronts) is used, the last one always fits
    groups = max(1, min(args.batch_groups, len(mine) // 2)) if args.batch else 1
    if args.batch:
        args.lanes = groups
    layouts = {4: [(4, 4), (3, 5)], 3: [(6, 3)], 2: [(6, 5)]}.get(groups, []) if args.batch else []
    if groups > 1:
        layouts = layouts + [(0, max(1, 7 // groups))]   # default 9-CTA clusters: 14 co-reside
    cluster = 0
    if args.segments >= 0:
        segments, layouts = args.segments, []
    elif args.batch:
        cluster, segments = layouts.pop(0) if layouts else (0, 0)
    else:
        segments = 1 if len(mine) > 1 and args.lanes > 1 else 0
    t0 = time.perf_counter()
    keep = (rank == 0 and world == 1 and not args.no_cpu_baseline)
    def build(segments, cluster):
        return hb.build_two_grid(p.mesh, p.model, fine_op=fine_operator(p),
                                 smoother=hb.SmootherConfig(p.omega_jac, p.nu),
                                 coarse="sweep",
                                 sweep=hb.SweepOptions(p.w_dd, p.s_dd, "x",
                                                       subdomains=p.subdomains,
                                                       segments=segments, cluster=cluster),
                                 keep_slab_ops=keep)[0]

    cycle = build(segments, cluster)
    if groups > 1:
        from paper_1412_0464_b200.twogrid import _lane_capable
        while layouts and not _lane_capable(cycle, groups):   # does not co-reside here: next
            cycle = None
            cluster, segments = layouts.pop(0)
            cycle = build(segments, cluster)
    dev = cycle.device()
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    ctx = context()
    f_dev = [torch.from_numpy(p.f[r].ravel()).cuda() for r in mine]
    cfg = hb.GmresConfig(p.tol, p.max_iter, p.restart)
    prec = cycle.as_preconditioner()

    def solve(fd):
        return hb.gmres(cycle.fine_csr, prec, fd, cfg, orth=args.orth,
                        pipelined=not args.no_pipeline)

    # warm-up, holding each step's solutions like the timed loop does: the
    # caching allocator then already owns the second solution buffer (a
    # fresh cudaMalloc inside the 2nd timed step was measured to stall it)
    reports = []
    held = None
    for _ in range(args.warmup):
        held = [solve(fd) for fd in f_dev]
    held = None
    # ---- timed region: K steps (each step solves this rank's right-hand sides)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    def all_launches():   # this context plus the lanes' (lanes / batch groups launch on their own)
        return ctx.launches + sum(ln.ctx.launches for ln in getattr(cycle, "_lanes", []))

    launches0 = None      # taken after the (lane-creating) warm-up below
    multi = len(f_dev) > 1 and (args.lanes > 1 or args.batch)

    def step(fs):
        if multi:
            return hb.solve_many(cycle, fs, cfg, lanes=args.lanes, orth=args.orth,
                                 batch=args.batch)
        return [solve(fd) for fd in fs]

    if multi:   # (lanes) same holding pattern as the timed loop
        for _ in range(args.warmup):
            held = step(f_dev)
        held = None
    launches0 = all_launches()
    with ClockSampler(local, args.clock_sampler) as clk:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        # ncu --profile-from-start off captures exactly the timed region
        # (cudaProfilerStart/Stop are no-ops without a profiler attached)
        torch.cuda.cudart().cudaProfilerStart()
        ev0.record(stream)
        evs[0].record(stream)
        for s in range(args.steps):
            for u, rep in step(f_dev):
                reports.append(rep)
            evs[s + 1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    launches = all_launches() - launches0
    if world > 1:
        torch.distributed.barrier()
    ms_local = ev0.elapsed_time(ev1)
    ms_steps = [evs[s].elapsed_time(evs[s + 1]) for s in range(args.steps)]
    # kernel-class attribution: the same K steps again with the library's
    # event profiler on (events bracket every launch, so this pass is not
    # the timed one; its per-kernel durations feed roofline/kernel_shares)
    ctx.profile_reset()
    ctx.profile(True)
    for _ in range(args.steps):
        if multi and args.batch:   # the batch's kernels (one group: the main context sees them all)
            hb.solve_many(cycle, f_dev, cfg, lanes=1, batch=True)
        else:
            for fd in f_dev:
                solve(fd)
    prof = ctx.profile_read() or {"none": {"ms": 0.0, "bytes": 0.0, "launches": 0}}
    ctx.profile(False)
    ms = reduce_over_ranks(ms_local, world, "max")
    solves = reduce_over_ranks(args.steps * len(f_dev), world, "sum")
    value = job_value(p.n_fine, solves, ms)
    its = [r.iterations for r in reports] or [0]
    # true residual of the last solve
    true_res = None
    if f_dev:
        u_h = u.cpu().numpy()
        f0 = p.f[mine[-1]].ravel()
        true_res = float(np.linalg.norm(f0 - cycle.fine_csr @ u_h) / np.linalg.norm(f0))

    # ---- e2e: public API with host buffers (H2D + D2H inside the timed region)
    f_host = [torch.from_numpy(p.f[r].ravel()).pin_memory().numpy() for r in mine]
    # two untimed passes of the host-buffer path: the pinned output buffers
    # of two consecutive solves come from torch's host cache afterwards
    # (a fresh 18-MB cudaHostAlloc costs ~14 ms)
    for _ in range(2):
        if multi:
            outs = step(f_host)
        else:
            outs = [hb.gmres(cycle.fine_csr, prec, fh, cfg, orth=args.orth,
                             pipelined=not args.no_pipeline) for fh in f_host]
    outs = None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eevs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    eevs[0].record(stream)
    for s_ in range(args.steps):
        if multi:
            step(f_host)
        else:
            for fh in f_host:
                u_out, _ = hb.gmres(cycle.fine_csr, prec, fh, cfg, orth=args.orth,
                                    pipelined=not args.no_pipeline)
        eevs[s_ + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = reduce_over_ranks(e0.elapsed_time(e1), world, "max")
    e2e_steps = [eevs[i].elapsed_time(eevs[i + 1]) for i in range(args.steps)]
    e2e_value = job_value(p.n_fine, solves, e2e_ms)

    # ---- roofline of the dominant kernel class (profiler events over the timed region)
    peak, peak_kind = peaks()
    total_ms = sum(v["ms"] for v in prof.values()) or 1.0
    dom = max(prof, key=lambda k: prof[k]["ms"])
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            tj = json.loads(tf.read_text())
            # ncu traffic was captured on one config (C2): not another config's
            traffic = tj.get(dom) if tj.get("config", 1) == args.config and args.scale == 1 else None
        except Exception:
            traffic = None

    def roof(names):
        ms_ = sum(prof[k]["ms"] for k in names if k in prof)
        by = sum(prof[k]["bytes"] for k in names if k in prof)
        n = sum(prof[k]["launches"] for k in names if k in prof)
        if not n or ms_ <= 0:
            return None
        ach = (by / n) / ((ms_ / n) / 1e3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "peak_kind": peak_kind,
                "bytes_per_launch": by / n, "ms_per_launch": ms_ / n, "launches": n}

    roofline = roof([dom])
    if roofline is not None:
        roofline["kernel"] = dom
        roofline["traffic"] = traffic
    stencil_roof = roof(["stencil", "residual", "jacobi", "jacobi2z"])
    fused_roof = roof(["pre_fused", "post_fused"])
    shares = {k: {"share": v["ms"] / total_ms, "ms": v["ms"], "launches": v["launches"],
                  "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None}
              for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        its_ref = reference_iterations(p, args)
        its_t = its_ref if its_ref is not None else int(np.median(its))
        src = ("reference iteration count from tests/golden/large_anchors.json"
               if its_ref is not None else "this solve's iteration count")
        tg, osetup = cpu_oracle(cycle.hierarchy)
        r = cpu_sample(p, tg, its_t, args.cpu_iters)
        tg = None
        cpu = {"value": r["value"], "unit": "DOF/s", "cores": CPU_CORES, "kind": "port",
               "sample": _sample_text(r, its_t, src, osetup),
               "projected_solve_s": r["projected_solve_s"]}

    if rank == 0:
        fac = dev.sweep.factor_bytes
        if roofline and roofline.get("kernel") == "sweep_front":
            # bytes_per_launch above = SURVEY 8(d)'s banded-LU floor of the
            # launch's slab solves; the own factor format streams factor_bytes
            # per pass (each slab solved twice per X application)
            roofline["bytes_basis"] = (
                "SURVEY 8(d) banded no-pivot LU floor of the slabs solved"
                + (" x the right-hand sides a launch carries (each is one solve of every slab; "
                   "the factor blocks themselves are read once per launch)"
                   if multi and args.batch else ""))
            roofline["own_format_bytes_per_application"] = 2 * fac
            roofline["launches_per_application"] = dev.sweep.launches_per_apply()
        line = {
            "metric": "TGSP-GMRES fine DOF/s (solve to 1e-6 rel-res)",
            "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "ms_steps_rank0": ms_steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic",
            "config": bench_config(p, args, world),
            "coarse_dof": int(np.prod(cycle.coarse_op.shape)),
            "slab_factor_bytes": fac,
            "sweep_segments": dev.sweep.segments if p.mesh.dim == 2 else None,
            "rhs_per_rank": len(f_dev),
            "rhs_in_flight": (len(f_dev) if args.batch else min(args.lanes, len(f_dev))) if multi else 1,
            "rhs_per_chain": (min(dev.sweep.rhs_width(), max(1, len(f_dev) // groups))
                              if multi and args.batch else 1),
            "rhs_mode": (f"{groups} lockstep batch(es) (several right-hand sides per chain of "
                         "slab solves)" if args.batch else "lanes") if multi else "single",
            "reference_iterations": reference_iterations(p, args),
            "solve_s": ms / 1e3 / max(1, args.steps * len(f_dev)),
            "setup_s": setup_s,
            "iterations": int(np.median(its)),
            "true_residual": true_res,
            "e2e": {"value": e2e_value, "unit": "DOF/s",
                    "h2d_bytes_per_step": 16 * p.n_fine * len(f_dev),
                    "d2h_bytes_per_step": 16 * p.n_fine * len(f_dev),
                    "ms_steps_rank0": e2e_steps},
            "gpu_launches": launches,
            "roofline": roofline,
            "roofline_stencil": stencil_roof,
            "roofline_vcycle_fused": fused_roof,
            "kernel_shares": shares,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded(args):
    """--shard: the single right-hand side solve decomposed along the sweep
    axis (paper_1412_0464_b200/shards.py).  Each rank owns a slab of fine
    rows; value = fine DOF / max-over-ranks solve time (strong scaling)."""
    import torch
    world, rank, local = dist_info()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.configs import config
    from paper_1412_0464_b200.shards import (CudaShardBackend, DistComm, LocalComm,
                                             ShardedTGSP, plan_shards, scatter_rows)
    p = config(args.config, args.scale)
    t0 = time.perf_counter()
    hh = hb.build_hierarchy(p.mesh, p.model, fine_operator(p), hb.SmootherConfig(p.omega_jac, p.nu),
                            hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                            keep_slab_ops=False)
    G = world if world > 1 else max(1, args.local_shards)
    plans = plan_shards(hh.fine_op.shape, hh.cmap, G)
    comm = DistComm(plans, rank) if world > 1 else LocalComm(plans)
    be = CudaShardBackend(hh, plans, comm.local)
    st = ShardedTGSP(plans, be, comm)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    fh = p.f[0]
    f = {g: be.upload(g, scatter_rows(plans[g], fh)) for g in comm.local}
    cfg = hb.GmresConfig(p.tol, p.max_iter, p.restart)
    for _ in range(args.warmup):
        st.gmres(f, cfg)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = be.ctx.launches
    reps = []
    with ClockSampler(local, args.clock_sampler) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            u, rep = st.gmres(f, cfg)
            reps.append(rep)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = be.ctx.launches - launches0
    ms = reduce_over_ranks(ev0.elapsed_time(ev1), world, "max")
    # true residual of the sharded solution (owned rows gathered on rank 0)
    resid = {g: be.zeros(g) for g in comm.local}
    comm.exchange(u)
    for g in comm.local:
        be.residual(g, f[g], u[g], resid[g])
    true_res = st.norm(resid) / st.norm(f)
    if rank == 0:
        line = {
            "metric": "TGSP-GMRES fine DOF/s (solve to 1e-6 rel-res)",
            "value": p.n_fine * args.steps / (ms / 1e3), "unit": "DOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic",
            "config": bench_config(p, args, world),
            "shards": G, "logical_shards_on_one_gpu": world == 1,
            "iterations": int(np.median([r.iterations for r in reps])),
            "true_residual": true_res, "setup_s": setup_s, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    world = dist_info()[0]
    if not args.shard and world > 1 and args.impl == "ours":
        from paper_1412_0464_b200.configs import config
        # one right-hand side: no replicas -- the solve itself is sharded
        args.shard = config(args.config, args.scale).f.shape[0] == 1
    if args.impl == "reference":
        run_reference(args)
    elif args.shard:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
