"""Two-grid sweeping preconditioner (TGSP): drop-in for reference ``twogrid.py``.

* ``SmootherConfig``, ``jacobi_smooth``                 :27-50
* ``prolongation_matrix``, ``prolongate``, ``restrict`` :53-93
* ``TwoGridCycle`` (vcycle, as_preconditioner)          :119-164
* ``tgsp_apply``, ``vcycle``                            :167-176
* ``SweepOptions``, ``build_two_grid``                  :179-229

``build_two_grid`` assembles the hierarchy on the host (setup), uploads it and
factorises the coarse slabs on the device.  Every cycle application is a
chain of CUDA kernels (``hs_vcycle``): fused two-step pre-smoothing from zero,
residual, h^d-scaled restriction, the X/UD sweep, prolongation-correction,
post-smoothing.  Inputs may be numpy arrays (copied in/out) or torch CUDA
complex128 tensors (zero-copy).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .discretize import (StencilOperator, WaveModel, coarsen_wavenumber,
                         wavenumber_cell_midpoints)
from .mesh import CoarseningMap, Mesh, coarsen_mesh
from .sweepdd import (HelmholtzLevel, Partition, SweepingPreconditioner, build_partition,
                      coarse_level, fine_level)


@dataclass(frozen=True)
class SmootherConfig:
    omega_jac: float = 0.8
    nu: int = 3

    def __post_init__(self):
        if not 0.0 < self.omega_jac <= 1.0:
            raise ValueError(f"relaxation weight must be in (0, 1], got {self.omega_jac}")
        if self.nu < 0:
            raise ValueError(f"smoothing step count must be >= 0, got {self.nu}")


@dataclass(frozen=True)
class SweepOptions:
    w_dd: int = 4
    s_dd: float = 20.0
    variant: str = "ud"
    n_cell: int | None = None
    subdomains: int | None = None
    parallel: bool = False
    # device layout of the 2-D slab solves (not in the reference): face
    # segments per sweep front, 0 = automatic (fastest single sweep); 1 keeps
    # one cluster per front so that several right-hand sides' sweeps (solve_many
    # lanes) run side by side
    segments: int = 0
    # CTAs (face chunks) per segment's cluster, 0 = automatic (9)
    cluster: int = 0


def default_dd_strength(w_dd: int) -> float:
    return 5.0 * w_dd


def jacobi_smooth(op: StencilOperator, u, f, omega: float, steps: int):
    """u <- u + omega D^-1 (f - A u), ``steps`` times, on the GPU."""
    from .device import from_device, to_device
    diag = op.diagonal()
    zero = np.argwhere(diag == 0)
    if zero.size:
        raise ZeroDivisionError(f"zero operator diagonal at node {tuple(zero[0])}")
    dev = op.device()
    ut, was_np = to_device(u, op.n, dev.ctx)
    ut = ut.clone()
    ft, _ = to_device(f, op.n, dev.ctx)
    dev.jacobi(ut, ft, omega, steps)
    return from_device(ut, was_np, op.shape if was_np else None)


# ---------------------------------------------------------------------------
# transfers

def _prolong_1d(fp, refined) -> sp.csr_matrix:
    """1-D tent prolongation (host matrix; inspection / drop-in helper)."""
    fp = np.asarray(fp)
    n_f, n_c = int(fp[-1]) - 1, len(fp) - 2
    rows = list(fp[1:n_c + 1] - 1)
    cols = list(range(n_c))
    vals = [1.0] * n_c
    for cell in np.flatnonzero(np.asarray(refined)):
        for cp in (cell, cell + 1):
            if 1 <= cp <= n_c:
                rows.append(fp[cell])
                cols.append(cp - 1)
                vals.append(0.5)
    return sp.csr_matrix((vals, (rows, cols)), shape=(n_f, n_c))


def empty_like_dev(t):
    import torch
    return torch.empty_like(t)


def prolongation_matrix(cmap: CoarseningMap) -> sp.csr_matrix:
    p = _prolong_1d(cmap.fine_point_of_coarse[0], cmap.refined_cell[0])
    for a in range(1, cmap.dim):
        p = sp.kron(p, _prolong_1d(cmap.fine_point_of_coarse[a], cmap.refined_cell[a]),
                    format="csr")
    return p


def prolongate(cmap: CoarseningMap, u_coarse):
    """Coarse-to-fine tent interpolation on the GPU (field in, field out)."""
    from .device import DeviceTransfer
    t = DeviceTransfer(cmap)
    was_np = not hasattr(u_coarse, "data_ptr")
    out = t.prolong(np.asarray(u_coarse, dtype=complex) if was_np else u_coarse)
    return out.reshape(t.fine_shape)


def restrict(cmap: CoarseningMap, r_fine):
    """Fine-to-coarse transfer P^T on the GPU."""
    from .device import DeviceTransfer
    t = DeviceTransfer(cmap)
    was_np = not hasattr(r_fine, "data_ptr")
    out = t.restrict(np.asarray(r_fine, dtype=complex) if was_np else r_fine)
    return out.reshape(t.coarse_shape)


# ---------------------------------------------------------------------------
# coarse solvers

class ExactCoarseSolver:
    """Exact coarse solve (twogrid.py:99-105): device block-LU factors of the
    coarse operator (:class:`.sparselin.Factorization`)."""

    def __init__(self, factor, shape):
        self.factor = factor
        self.shape = tuple(shape)

    def solve(self, rc):
        out = self.factor.solve(rc.reshape(-1) if hasattr(rc, "reshape") else rc)
        return out.reshape(self.shape)

    def device_plan(self):
        """(device solver handle, C-ABI variant id) for hs_cycle_create."""
        dev = self.factor.device
        return dev, dev.variant_id()


class SweepCoarseSolver:
    """One sweep application, never iterated."""

    def __init__(self, prec: SweepingPreconditioner):
        self.prec = prec
        self.shape = prec.part.shape

    def solve(self, rc):
        return self.prec(rc.reshape(self.shape) if hasattr(rc, "reshape") else rc)

    def device_plan(self):
        sw = self.prec.part.device()
        return sw, sw.variant_id(self.prec.variant, self.prec.cells)


class FineOperator:
    """Device fine operator usable as ``apply_a`` (``fine_csr @ v``)."""

    def __init__(self, op: StencilOperator):
        self.op = op
        self.shape = (op.n, op.n)

    def __matmul__(self, v):
        return self.op.device().apply(v)

    def __call__(self, v):
        return self @ v


@dataclass
class TwoGridCycle:
    """Fixed linear V-cycle (pre-smoothing from zero), executed on the GPU."""

    fine_op: StencilOperator
    coarse_op: StencilOperator
    cmap: CoarseningMap
    smoother: SmootherConfig
    coarse_solver: object
    restrict_scale: float = 1.0
    variant: str = "x"
    fine_csr: object = None
    _dev: object = field(default=None, repr=False)

    def __post_init__(self):
        if self.fine_csr is None:
            self.fine_csr = FineOperator(self.fine_op)

    @property
    def generic(self) -> bool:
        """built from an explicit prolongation matrix (the reference's
        ``TwoGridCycle(fine, coarse, p_matrix, ...)``) instead of a CoarseningMap"""
        return sp.issparse(self.cmap)

    @property
    def p_matrix(self):
        return sp.csr_matrix(self.cmap) if self.generic else prolongation_matrix(self.cmap)

    @property
    def r_matrix(self):
        return self.p_matrix.T

    def device(self):
        if self.generic:
            raise ValueError("an explicit-matrix cycle has no fused device plan")
        if self._dev is None:
            from .device import DeviceCycle, DeviceTransfer
            fine = self.fine_op.device()
            solver, vid = self.coarse_solver.device_plan()
            self._dev = DeviceCycle(fine, DeviceTransfer(self.cmap, fine.ctx),
                                    self.coarse_op.device(), solver, self.smoother.omega_jac,
                                    self.smoother.nu, self.restrict_scale, vid, fine.ctx)
        return self._dev

    def _vcycle_matrix(self, f):
        """V-cycle with an explicit prolongation matrix P (twogrid.py:150-159):
        device Jacobi / residual kernels, P^T and P as device CSR products
        (hs_csr_apply), the coarse solver's own device solve."""
        from .device import DeviceCSR, from_device, to_device
        mats = self.__dict__.get("_pmats")
        fine = self.fine_op.device()
        if mats is None:
            p = sp.csr_matrix(self.cmap, dtype=complex)
            mats = (DeviceCSR(p, fine.ctx), DeviceCSR(p.T.tocsr(), fine.ctx))
            self.__dict__["_pmats"] = mats
        pd, rd = mats
        ft, was_np = to_device(f, fine.n, fine.ctx)
        nu, w = self.smoother.nu, self.smoother.omega_jac
        if nu:
            diag = self.fine_op.diagonal()
            zero = np.argwhere(diag == 0)
            if zero.size:
                raise ZeroDivisionError(f"zero operator diagonal at node {tuple(zero[0])}")
        u = empty_like_dev(ft)
        u.zero_()
        if nu:
            fine.jacobi(u, ft, w, nu, u_is_zero=True)
        r = fine.residual(ft, u)
        rc = rd.apply(r, alpha=self.restrict_scale)
        uc = self.coarse_solver.solve(rc)
        pd.apply(uc.reshape(-1), out=u, accumulate=True)
        if nu:
            fine.jacobi(u, ft, w, nu)
        if was_np:
            return from_device(u, True, self.fine_op.shape)
        return u.reshape(f.shape)

    def vcycle(self, f):
        from .device import from_device, to_device
        if self.generic:
            return self._vcycle_matrix(f)
        dev = self.device()
        ft, was_np = to_device(f, dev.n, dev.ctx)
        u = dev.vcycle_dev(ft)
        if was_np:
            return from_device(u, True, self.fine_op.shape)
        return u.reshape(f.shape)

    def vcycle_many(self, F):
        """One cycle per row of the stack F (nrhs, ...): the coarse sweeps of
        all rows through one chain of slab solves (hs_vcycle_many); row r is
        bitwise ``vcycle(F[r])``."""
        from .device import from_device, to_device
        if self.generic:
            return np.stack([self._vcycle_matrix(F[r]) for r in range(F.shape[0])])
        dev = self.device()
        nrhs = int(F.shape[0])
        was_np = not hasattr(F, "is_cuda")
        if was_np:
            F = np.ascontiguousarray(np.asarray(F, dtype=complex))
        ft, _ = to_device(F, nrhs * dev.n, dev.ctx)
        u = dev.vcycle_many_dev(ft.reshape(nrhs, dev.n))
        if was_np:
            return from_device(u, True, tuple(F.shape))
        return u.reshape(F.shape)

    def as_preconditioner(self, lane=None):
        """The flat-vector preconditioner callable (twogrid.py:161-164);
        ``lane``: run on a :class:`Lane` (its own context and stream)."""
        dev_cycle = self
        the_lane = lane

        class _Prec:
            cycle = dev_cycle
            lane = the_lane

            def __call__(self, v):
                out = dev_cycle.vcycle(v)
                return out.reshape(-1)

        return _Prec()

    def lanes(self, n: int):
        """``n`` lanes of this cycle for right-hand sides in flight at once on
        one GPU (2-D levels): each has its own library context, CUDA stream
        and cycle/sweep scratch and shares the operators and slab factors."""
        return [Lane(self) for _ in range(n)]


class Lane:
    """One right-hand side in flight: a private libhsweep context bound to its
    own CUDA stream and a lane of the cycle's device handle."""

    def __init__(self, cycle: TwoGridCycle):
        import torch
        from ._lib import Context
        base = cycle.device()
        self.cycle = cycle
        self.stream = torch.cuda.Stream(device=base.ctx.device)
        self.ctx = Context(base.ctx.device)
        with torch.cuda.stream(self.stream):
            self.ctx.bind_stream()
            self.dev = base.lane(self.ctx)

    def preconditioner(self):
        return self.cycle.as_preconditioner(lane=self)


def solve_many(cycle: TwoGridCycle, rhs, config=None, lanes: int = 4, orth: str = "cgs2",
               batch: bool = False):
    """Independent GMRES solves of several right-hand sides (C4's sources).
    ``batch=True``: the solves advance in lockstep and every Arnoldi step's
    coarse sweeps go through one chain of slab solves (``gmres_many``:
    several right-hand sides per pass over the slab factors).  Otherwise
    ``lanes`` of them are in flight at once on one GPU (one host thread and
    one CUDA stream per lane; the sweeps of different lanes run on disjoint
    clusters).  Stream-ordered with the caller: the lanes start after the
    caller's current stream and the caller's stream waits for all of them.
    Either way each solve is bitwise the sequential ``gmres``.
    Returns [(u, SolveReport)] in input order."""
    import concurrent.futures as cf
    import threading
    import torch
    from .krylov import gmres, gmres_many
    rhs = list(rhs)
    if not rhs:
        return []
    if batch and orth == "cgs2":
        groups = max(1, min(lanes, len(rhs) // 2))
        if groups <= 1 or not _lane_capable(cycle, groups):
            return gmres_many(cycle.fine_csr, cycle.as_preconditioner(), rhs, config)
        # `groups` lockstep batches side by side, one lane (thread, stream,
        # work set) each: one batch's fine-level kernels overlap the other's
        # sweep, and the sweeps' clusters share the device
        pool = getattr(cycle, "_lanes", [])
        if len(pool) < groups:
            pool = pool + cycle.lanes(groups - len(pool))
            cycle._lanes = pool
        pool = pool[:groups]
        main = torch.cuda.current_stream(pool[0].ctx.device)
        start = torch.cuda.Event()
        start.record(main)
        per = -(-len(rhs) // groups)
        parts = [rhs[i * per:(i + 1) * per] for i in range(groups)]

        def run(i):
            ln = pool[i]
            with torch.cuda.stream(ln.stream):
                ln.stream.wait_event(start)
                return gmres_many(cycle.fine_csr, ln.preconditioner(), parts[i], config)

        with cf.ThreadPoolExecutor(max_workers=groups) as ex:
            outs = list(ex.map(run, range(groups)))
        for ln in pool:
            main.wait_stream(ln.stream)
        return [o for part in outs for o in part]
    if lanes <= 1 or not _lane_capable(cycle, min(lanes, len(rhs))):
        # 3-D levels and the exact coarse solve run one cooperative all-SM
        # chain per slab solve: no concurrent lanes, solves in order
        prec = cycle.as_preconditioner()
        return [gmres(cycle.fine_csr, prec, f, config, orth=orth) for f in rhs]
    pool = getattr(cycle, "_lanes", [])
    want = max(1, min(lanes, len(rhs)))
    if len(pool) < want:
        pool = pool + cycle.lanes(want - len(pool))
        cycle._lanes = pool
    pool = pool[:want]
    main = torch.cuda.current_stream(pool[0].ctx.device)
    start = torch.cuda.Event()
    start.record(main)
    free = list(pool)
    lock = threading.Lock()

    def one(f):
        with lock:
            ln = free.pop()
        try:
            with torch.cuda.stream(ln.stream):
                ln.stream.wait_event(start)
                return gmres(cycle.fine_csr, ln.preconditioner(), f, config, orth=orth)
        finally:
            with lock:
                free.append(ln)

    with cf.ThreadPoolExecutor(max_workers=len(pool)) as ex:
        out = list(ex.map(one, rhs))
    for ln in pool:
        main.wait_stream(ln.stream)
    return out


def _lane_capable(cycle: TwoGridCycle, lanes: int = 2) -> bool:
    """Lanes need a 2-D sweep coarse solver (private sweep scratch per lane).
    The G clusters of a two-level-partition front wait on each other, so
    with G > 1 every lane's two fronts must be co-resident at once:
    2 * lanes <= the fronts the device holds (hs_sweep_max_fronts); with one
    cluster per front nothing waits across clusters and any lane count runs."""
    if not (isinstance(cycle.coarse_solver, SweepCoarseSolver) and cycle.coarse_op.dim == 2):
        return False
    sw = cycle.hierarchy.partition.device()
    return sw.segments == 1 or 2 * lanes <= sw.max_fronts


def vcycle(cycle: TwoGridCycle, f):
    return cycle.vcycle(f)


def tgsp_apply(cycle: TwoGridCycle, f):
    if not isinstance(cycle.coarse_solver, SweepCoarseSolver):
        raise ValueError("tgsp_apply needs a cycle with a sweeping coarse solver")
    return cycle.vcycle(f)


@dataclass
class HostHierarchy:
    """Everything build_two_grid assembles on the host (the device's inputs)."""

    mesh: Mesh
    fine_op: StencilOperator
    coarse_op: StencilOperator
    cmap: CoarseningMap
    clevel: HelmholtzLevel
    partition: Partition
    smoother: SmootherConfig
    sweep: SweepOptions
    restrict_scale: float

    @property
    def beta(self):
        return self.partition.beta

    @property
    def beta_tilde(self):
        return self.partition.beta_tilde

    @property
    def slabs(self):
        return [(sd.pt_lo, sd.pt_hi, sd.op) for sd in self.partition.subs]


def build_hierarchy(mesh: Mesh, model: WaveModel, fine_op=None, smoother=None, sweep=None,
                    table=None, device=True, keep_slab_ops=True,
                    assembly: str | None = None, coarse: str = "sweep") -> HostHierarchy:
    """Assembly of the TGSP hierarchy (reference twogrid.py:196-229).

    ``assembly="device"`` (the default when ``device``): the fine FD operator,
    the PML coarse FE operator and every slab operator are formed on the GPU
    (:mod:`.assembly`); ``"host"``: numpy assembly (the oracle's inputs).  The
    wavenumber transfers and the per-axis profiles stay on the host."""
    if assembly is None:
        assembly = "device" if device else "host"
    if assembly not in ("device", "host"):
        raise ValueError(f"assembly must be 'device' or 'host', got {assembly!r}")
    on_gpu = assembly == "device"
    if on_gpu and fine_op is None:
        from .assembly import assemble_fine_device
        fine_op = assemble_fine_device(mesh, model)
    flevel = fine_level(mesh, model, fine_op)
    mesh_c, cmap = coarsen_mesh(mesh)
    model_c = WaveModel(model.omega, coarsen_wavenumber(model.k, cmap))
    k_cells = wavenumber_cell_midpoints(model.k, cmap)
    has_pml = any(s.kind == "pml" for pair in mesh_c.layers for s in pair)
    coarse_op, fields = None, None
    if on_gpu and has_pml:
        from .assembly import CoarseFields, assemble_fe_pml_coarse_device
        from ._lib import context
        fields = CoarseFields(model_c, k_cells, context())
        coarse_op = assemble_fe_pml_coarse_device(mesh_c, cmap, model_c, k_cells, table,
                                                  fields=fields)
    clevel = coarse_level(mesh_c, cmap, model_c, op=coarse_op, k_cells=k_cells, table=table)
    clevel.fields = fields
    if smoother is None:
        smoother = SmootherConfig(omega_jac=0.8 if mesh.dim == 2 else 0.6, nu=3)
    sweep = sweep or SweepOptions()
    part = None
    if coarse == "sweep":
        from ._lib import context
        ctx = context() if device else None
        if ctx is not None:
            ctx.lib.hs_ctx_set_sweep_segments(ctx.h, int(sweep.segments))
            ctx.lib.hs_ctx_set_sweep_cluster(ctx.h, int(sweep.cluster))
        try:
            part = build_partition(clevel, sweep.w_dd, sweep.s_dd, J=sweep.subdomains,
                                   device=device, keep_slab_ops=keep_slab_ops)
        finally:
            if ctx is not None:
                ctx.lib.hs_ctx_set_sweep_segments(ctx.h, 0)
                ctx.lib.hs_ctx_set_sweep_cluster(ctx.h, 0)
    h = float(mesh.spacing[0][0])
    return HostHierarchy(mesh, flevel.op, clevel.op, cmap, clevel, part, smoother, sweep,
                         h ** mesh.dim)


def build_two_grid(mesh: Mesh, model: WaveModel, fine_op: StencilOperator | None = None,
                   smoother: SmootherConfig | None = None, coarse: str = "exact",
                   sweep: SweepOptions | None = None, table=None, keep_slab_ops=True,
                   assembly: str = "device"):
    """Assemble the two-grid hierarchy; returns (cycle, coarse level)
    (twogrid.py:196-229).

    ``coarse="sweep"``: the TGSP path (one sweep application per cycle).
    ``coarse="exact"``: the coarse operator factorised on the device (block
    LU, :mod:`.sparselin`) and solved exactly in every cycle.
    """
    if coarse not in ("exact", "sweep"):
        raise ValueError(f"coarse solver must be 'exact' or 'sweep', got {coarse!r}")
    sweep = sweep or SweepOptions()
    if sweep.variant not in ("ud", "x", "nx"):
        raise ValueError(f"unknown sweep variant {sweep.variant!r}")
    hh = build_hierarchy(mesh, model, fine_op, smoother, sweep, table,
                         keep_slab_ops=keep_slab_ops, assembly=assembly, coarse=coarse)
    if coarse == "exact":
        from .sparselin import factorize
        solver = ExactCoarseSolver(factorize(hh.coarse_op), hh.coarse_op.shape)
        variant = "exact"
    else:
        prec = SweepingPreconditioner(hh.partition, sweep.variant, cells=sweep.n_cell,
                                      parallel=sweep.parallel)
        solver = SweepCoarseSolver(prec)
        variant = sweep.variant
    cycle = TwoGridCycle(hh.fine_op, hh.coarse_op, hh.cmap, hh.smoother, solver,
                         restrict_scale=hh.restrict_scale, variant=variant)
    cycle.hierarchy = hh
    return cycle, hh.clevel
