"""Sweeping domain-decomposition preconditioner: partition (host setup) and
its device application.

Drop-in names of reference ``sweepdd.py``:

* ``HelmholtzLevel``, ``fine_level``, ``coarse_level``   :33-87
* ``TransmissionMatrix``, ``extract_transmission``      :98-141, :221-230
* ``spaced_interfaces``, ``default_subdomain_count``    :179-189
* ``build_partition``                                    :192-218
* ``prec_ud``, ``prec_x``, ``SweepingPreconditioner``    :312-359, :437-467
* ``NxCells``, ``make_nx_cells``, ``prec_nx``           :362-434
* ``subdom_solve``, ``forward_sweep``, ``backward_sweep``,
  ``midsolve_in``, ``midsolve_out``                      :236-306

Setup (geometry, slab operator assembly) runs on the host; the slabs are
factorised on the device at ``build_partition`` time and every application
runs the CUDA slab-solve chains (``csrc/hs_sweep.cu``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .discretize import (StencilOperator, WaveModel, assemble_fe_pml_coarse, assemble_fine,
                         assemble_opt_fd_coarse, assemble_sponge, default_table,
                         interior_spacing, robin1d_operator, subdomain_fd_operator,
                         subdomain_fe_operator, subdomain_robin1d_operator, _nodes_to_cells)
from .mesh import PML, SPONGE, CoarseningMap, Mesh


@dataclass
class HelmholtzLevel:
    op: StencilOperator
    kind: str
    mesh: Mesh | None = None
    model: WaveModel | None = None
    cmap: CoarseningMap | None = None
    k_cells: np.ndarray | None = None
    table: object = None
    k1d: float = 0.0
    h1d: float = 0.0

    fields: object = None   # device wavenumbers (assembly.CoarseFields): slabs assembled on the GPU

    def subdomain_operator(self, core_lo, core_hi, w_dd, s_dd, open_left, open_right):
        if self.kind == "fe" and self.fields is not None and self.k_cells is not None:
            from .assembly import subdomain_fe_operator_device
            return subdomain_fe_operator_device(self.mesh, self.model, self.k_cells, self.table,
                                                core_lo, core_hi, w_dd, s_dd, open_left,
                                                open_right, self.fields)
        if self.kind == "fd":
            return subdomain_fd_operator(self.mesh, self.model, core_lo, core_hi, w_dd, s_dd,
                                         open_left, open_right)
        if self.kind == "fe":
            return subdomain_fe_operator(self.mesh, self.model, self.k_cells, self.table,
                                         core_lo, core_hi, w_dd, s_dd, open_left, open_right)
        if self.kind == "robin1d":
            return subdomain_robin1d_operator(self.k1d, self.h1d, core_lo, core_hi, open_left,
                                              open_right)
        raise ValueError(f"unknown level kind {self.kind!r}")


def fine_level(mesh: Mesh, model: WaveModel, op: StencilOperator | None = None):
    if op is None:
        sponge = any(s.kind == SPONGE for pair in mesh.layers for s in pair)
        op = assemble_sponge(mesh, model) if sponge else assemble_fine(mesh, model)
    return HelmholtzLevel(op, "fd", mesh=mesh, model=model)


def robin_level_1d(k: float, h: float, n_cells: int) -> HelmholtzLevel:
    """The 1-D line of ``n_cells`` cells (n_cells - 1 unknowns) with exact
    radiating end closures (reference sweepdd.py:90-92): the sweep's
    known-answer level, solved on the device like the 2-D/3-D levels."""
    return HelmholtzLevel(robin1d_operator(k, h, n_cells - 1), "robin1d", k1d=k, h1d=h)


def _lift_line(op):
    """A 1-D line operator as the (n, 1, 1) 3-D stencil the device sweep
    takes (same memory layout; the slab solve is the 3-D block chain with
    one T x T block per slab)."""
    if op.dim != 1:
        return op
    return StencilOperator((op.shape[0], 1, 1),
                           {(o[0], 0, 0): c.reshape(-1, 1, 1) for o, c in op.coeffs.items()})


def coarse_level(mesh_c: Mesh, cmap: CoarseningMap, model_c: WaveModel, op=None,
                 k_cells=None, table=None):
    """FE rows on PML-coarsened meshes, else h^d-scaled optimized FD."""
    has_pml = any(s.kind == PML for pair in mesh_c.layers for s in pair)
    table = table or default_table(mesh_c.dim)
    if has_pml:
        if k_cells is None:
            k_cells = _nodes_to_cells(model_c.k)
        if op is None:
            op = assemble_fe_pml_coarse(mesh_c, cmap, model_c, k_cells, table)
    else:
        k_cells = None
        if op is None:
            op = assemble_opt_fd_coarse(mesh_c, model_c, table).scaled(
                interior_spacing(mesh_c) ** mesh_c.dim, fe_scaled=True)
    return HelmholtzLevel(op, "fe", mesh=mesh_c, model=model_c, cmap=cmap, k_cells=k_cells,
                          table=table)


# ---------------------------------------------------------------------------
# transmission (the sweep kernels read the global operator rows directly;
# this object is the drop-in view, reference sweepdd.py:98-141)

@dataclass
class TransmissionMatrix:
    """Two-layer interface map of the global operator at layers (b, b+1)
    (reference ``sweepdd.py:98-118``): ``apply(buf)`` returns
    ``[sign * A[b, b+1] buf[1], -sign * A[b+1, b] buf[0]]`` -- the face
    blocks applied as (d-1)-dimensional compact stencils on the GPU."""

    point: int
    block01: dict
    block10: dict
    sign: int

    def _face_ops(self, face):
        """device stencils of the two blocks, the sign folded into the
        coefficients (exact: a negation)"""
        ops = self.__dict__.get("_dev")
        if ops is None or ops[0] != face:
            from .device import DeviceStencil
            shape = face if face else (1,)
            dev = []
            for blk, sg in ((self.block01, self.sign), (self.block10, -self.sign)):
                offs = sorted(blk) or [(0,) * len(face)]
                co = [np.broadcast_to(np.asarray(blk[o], dtype=complex), face).reshape(-1) * sg
                      if o in blk else np.zeros(int(np.prod(shape)), complex) for o in offs]
                offs = [o if face else (0,) for o in offs]
                dev.append(DeviceStencil(shape, offs, np.stack(co)))
            ops = (face, dev[0], dev[1])
            self.__dict__["_dev"] = ops
        return ops[1], ops[2]

    def apply(self, buf):
        """out[0] = sign * A[b,:;b+1,:] buf[1], out[1] = -sign * A[b+1,:;b,:] buf[0]
        (two face-stencil applications on the device).  numpy in -> numpy out;
        a torch CUDA tensor in -> tensor out."""
        import torch
        is_t = isinstance(buf, torch.Tensor)
        shp = tuple(buf.shape) if is_t else np.shape(np.asarray(buf))
        if len(shp) < 1 or shp[0] != 2:
            raise ValueError(f"transmission buffer must have 2 layers, got shape {shp}")
        face = tuple(int(v) for v in shp[1:])
        d01, d10 = self._face_ops(face)
        b = buf if is_t else np.asarray(buf, dtype=complex)
        o0 = d01.apply(b[1].reshape(-1) if is_t else np.ascontiguousarray(b[1]).ravel())
        o1 = d10.apply(b[0].reshape(-1) if is_t else np.ascontiguousarray(b[0]).ravel())
        if is_t:
            return torch.stack([o0, o1]).reshape(shp)
        return np.stack([np.asarray(o0), np.asarray(o1)]).reshape(shp)

    def dense(self):
        """Full 2m x 2m matrix (small sizes only; inspection helper)."""
        blk = self.block01 or self.block10
        shape = next(iter(blk.values())).shape if blk else ()
        m = int(np.prod(shape)) if shape else 1
        t = np.zeros((2 * m, 2 * m), dtype=complex)
        for j in range(m):
            e = np.zeros(m)
            e[j] = 1.0
            e = e.reshape(shape)
            t[:m, m + j] = self.sign * _face_apply(self.block01, e).ravel()
            t[m:, j] = -self.sign * _face_apply(self.block10, e).ravel()
        return t


def _face_apply(block, v):
    out = np.zeros(np.shape(v), dtype=complex)
    for off, c in block.items():
        if len(off) == 0:
            out = out + c * v
            continue
        dst = tuple(slice(max(0, -o), n - max(0, o)) for o, n in zip(off, np.shape(v)))
        src = tuple(slice(max(0, o), n - max(0, -o)) for o, n in zip(off, np.shape(v)))
        out[dst] += c[dst] * v[src]
    return out


def _extract(op: StencilOperator, b: int, sign: int) -> TransmissionMatrix:
    x0 = b - 1
    b01 = {off[1:]: c[x0] for off, c in op.coeffs.items() if off[0] == 1}
    b10 = {off[1:]: c[x0 + 1] for off, c in op.coeffs.items() if off[0] == -1}
    return TransmissionMatrix(b, b01, b10, sign)


# ---------------------------------------------------------------------------
# partition

def default_subdomain_count(n_unknowns: int, w_dd: int) -> int:
    return n_unknowns // (2 * w_dd + 1)


def spaced_interfaces(n_unknowns: int, J: int) -> np.ndarray:
    """Interfaces as even as possible; the remainder goes to the leading slabs."""
    w, r = divmod(n_unknowns, J)
    widths = np.full(J, w, dtype=int)
    widths[:r] += 1
    return np.concatenate([[0], np.cumsum(widths)]).astype(int)


@dataclass
class Subdomain:
    j: int
    pt_lo: int
    pt_hi: int
    core_lo: int
    core_hi: int
    op: StencilOperator | None

    @property
    def factor(self):
        """The slab's own LU (reference ``Subdomain.factor``): a device
        factorisation of the slab operator, made on first use (the sweep
        itself solves from the partition's packed device factors)."""
        f = self.__dict__.get("_factor")
        if f is None:
            if self.op is None:
                raise ValueError("slab operator not kept (build_partition(keep_slab_ops=False))")
            from .sparselin import factorize
            op = self.op
            if hasattr(op, "to_host"):
                op = op.to_host()
            f = factorize(op)
            self.__dict__["_factor"] = f
        return f


@dataclass
class Partition:
    level: HelmholtzLevel
    J: int
    beta: np.ndarray
    beta_tilde: np.ndarray
    w_dd: int
    s_dd: float
    subs: list
    _device: object = field(default=None, repr=False)

    @property
    def shape(self):
        return self.level.op.shape

    @property
    def t_fwd(self):
        return {j: _extract(self.level.op, int(self.beta[j - 1]), +1) for j in range(2, self.J + 1)}

    @property
    def t_bwd(self):
        return {j: _extract(self.level.op, int(self.beta_tilde[j]), -1) for j in range(1, self.J)}

    def device(self):
        """Factorise every slab on the device (once) and return the handle."""
        if self._device is None:
            from .device import DeviceStencil, DeviceSweep
            from .assembly import DeviceOperator
            if self.level.op.dim == 1:     # the line: lifted to (n, 1, 1)
                coarse = _lift_line(self.level.op).device()
            else:
                coarse = self.level.op.device()
            slab_ops = [sd.op.device() if isinstance(sd.op, DeviceOperator)
                        else DeviceStencil.from_host(_lift_line(sd.op), coarse.ctx)
                        for sd in self.subs]
            self._device = DeviceSweep(coarse, self.J, self.beta, self.beta_tilde,
                                       [sd.pt_lo for sd in self.subs],
                                       [sd.pt_hi for sd in self.subs], slab_ops, coarse.ctx)
            del slab_ops
        return self._device

    def apply_global(self, u):
        return self.level.op.apply(u)

    @property
    def csr(self):
        """The level operator as ``apply_a`` (reference ``part.csr @ v``,
        cli.py:248): a device matvec object, not a host CSR matrix."""
        from .twogrid import FineOperator
        return FineOperator(self.level.op)


def partition_geometry(n1: int, J: int, tilde_right: bool = False):
    if J < 2:
        raise ValueError(f"{J} subdomains: the sweep needs at least 2")
    beta = spaced_interfaces(n1, J)
    if np.any(np.diff(beta) < 2):
        raise ValueError("subdomain thinner than 2 cells")
    bt = beta.copy()
    bt[1:J] = beta[1:J] + (1 if tilde_right else -1)
    return beta, bt


def build_partition(level: HelmholtzLevel, w_dd: int = 4, s_dd: float = 20.0,
                    J: int | None = None, tilde_right: bool = False,
                    device: bool = True, keep_slab_ops: bool = True) -> Partition:
    """Staggered interfaces, slab operators (host) and device factorisations."""
    n1 = level.op.shape[0]
    if J is None:
        J = default_subdomain_count(n1, w_dd)
    beta, bt = partition_geometry(n1, J, tilde_right)
    subs = []
    for j in range(1, J + 1):
        core_lo = min(beta[j - 1], bt[j - 1]) + 1
        core_hi = max(beta[j], bt[j])
        op_j, lo, hi = level.subdomain_operator(int(core_lo), int(core_hi), w_dd, s_dd,
                                                j > 1, j < J)
        subs.append(Subdomain(j, int(lo), int(hi), int(core_lo), int(core_hi), op_j))
    part = Partition(level, J, beta, bt, w_dd, s_dd, subs)
    if device:
        part.device()
        if not keep_slab_ops:      # the factors live on the device now
            for sd in subs:
                sd.op = None
    return part


def extract_transmission(part: Partition, j: int, direction: str) -> TransmissionMatrix:
    if direction == "forward":
        if not 1 < j <= part.J:
            raise ValueError(f"forward transmission needs 1 < j <= J, got {j}")
        return _extract(part.level.op, int(part.beta[j - 1]), +1)
    if direction == "backward":
        if not 1 <= j < part.J:
            raise ValueError(f"backward transmission needs 1 <= j < J, got {j}")
        return _extract(part.level.op, int(part.beta_tilde[j]), -1)
    raise ValueError(f"direction must be forward or backward, got {direction!r}")


# ---------------------------------------------------------------------------
# applications (device)

def subdom_solve(part: Partition, u, f, j, a, b, ta, tb, tau1=False, B1=None, tau2=False,
                 tau3=False, B3=None, tau4=False):
    """One slab solve (sweepdd.py:236-268) on the device (hs_sweep_solve_one):
    right-hand side rows a..b-1 of f plus the transmission sources of the
    incoming traces, u[ta:tb] += the solution rows (u updated in place: a
    numpy array or a torch CUDA tensor), returns the outgoing traces (out2,
    out4) that were asked for (2 x face arrays) or None."""
    import ctypes as C
    import torch
    from .device import ptr, to_device
    J = part.J
    if tau1 and j > 1 and B1 is None:
        raise RuntimeError(f"forward transmission buffer for slab {j} not populated")
    if tau3 and j < J and B3 is None:
        raise RuntimeError(f"backward transmission buffer for slab {j} not populated")
    sw = part.device()
    ctx = sw.ctx
    shape = part.shape
    face = int(np.prod(shape[1:]))
    ft, _ = to_device(f, sw.n, ctx)
    is_np = not isinstance(u, torch.Tensor)
    ut, _ = to_device(u, sw.n, ctx)
    if not is_np and ut.data_ptr() != u.data_ptr():
        raise ValueError("u must be a contiguous complex128 CUDA tensor (updated in place)")
    ut = ut.clone() if is_np else ut

    def trace_in(B, used):
        if not used or B is None:
            return None
        return to_device(np.asarray(B) if not isinstance(B, torch.Tensor) else B, 2 * face,
                         ctx)[0]
    b1 = trace_in(B1, tau1 and j > 1)
    b3 = trace_in(B3, tau3 and j < J)
    o2 = torch.empty(2 * face, dtype=torch.complex128, device=ut.device) \
        if tau2 and j < J else None
    o4 = torch.empty(2 * face, dtype=torch.complex128, device=ut.device) \
        if tau4 and j > 1 else None
    nul = C.c_void_p(None)
    ctx.call("hs_sweep_solve_one", sw.h, int(j), int(a), int(b), int(ta), int(tb),
             ptr(b1) if b1 is not None else nul, ptr(b3) if b3 is not None else nul,
             ptr(o2) if o2 is not None else nul, ptr(o4) if o4 is not None else nul,
             ptr(ft), ptr(ut))
    if is_np:
        u[...] = ut.cpu().numpy().reshape(np.shape(u))
    tshape = (2,) + tuple(shape[1:])

    def out(t):
        if t is None:
            return None
        return t.cpu().numpy().reshape(tshape) if is_np else t.reshape(tshape)
    return out(o2), out(o4)


def forward_sweep(part, u, f, j0, j1, B=None):
    """Slab solves j0..j1 ascending with forward transmission; out-of-range
    slab numbers are skipped (sweepdd.py:271-282)."""
    for j in range(j0, j1 + 1):
        if j < 1 or j > part.J:
            continue
        out, _ = subdom_solve(part, u, f, j, part.beta[j - 1], part.beta[j],
                              part.beta[j - 1], part.beta[j],
                              tau1=j > 1, B1=B, tau2=j < part.J)
        if out is not None:
            B = out
    return B


def backward_sweep(part, u, f, j0, j1, B=None):
    """Slab solves j0..j1 descending with backward transmission (sweepdd.py:285-294)."""
    for j in range(j0, j1 - 1, -1):
        if j < 1 or j > part.J:
            continue
        _, out = subdom_solve(part, u, f, j, part.beta_tilde[j - 1], part.beta_tilde[j],
                              part.beta_tilde[j - 1], part.beta_tilde[j],
                              tau3=j < part.J, B3=B, tau4=j > 1)
        if out is not None:
            B = out
    return B


def midsolve_in(part, u, f, j, B1, B3):
    """sweepdd.py:297-300."""
    subdom_solve(part, u, f, j, part.beta[j - 1], part.beta_tilde[j],
                 part.beta[j - 1], part.beta_tilde[j], tau1=True, B1=B1, tau3=True, B3=B3)


def midsolve_out(part, u, f, j):
    """sweepdd.py:303-306: returns (out2, out4)."""
    return subdom_solve(part, u, f, j, part.beta_tilde[j - 1], part.beta[j],
                        part.beta_tilde[j - 1], part.beta[j], tau2=True, tau4=True)


def _apply(part: Partition, f, variant: str, cells=None):
    from .device import from_device
    shape = part.shape
    u, was_np = part.device().apply(f, variant, cells)
    if was_np:
        return from_device(u, True, shape)
    return u.reshape(f.shape) if hasattr(f, "shape") else u


def prec_many(part: Partition, F, variant: str = "x", cells=None):
    """The sweep applied to a stack of right-hand sides F[r] (shape
    (nrhs,) + level shape, or (nrhs, n)): groups of up to
    ``part.device().rhs_width()`` right-hand sides go through one chain of
    slab solves, every factor block streamed once per group
    (hs_sweep_apply_many; the reference solves multi-column right-hand sides
    in one SuperLU call, sparselin.py:58-62).  Row r is bitwise
    ``prec_x(part, F[r])`` / ``prec_ud`` / ``prec_nx``."""
    from .device import from_device
    if variant == "x" and part.J % 2 != 0:
        raise ValueError(f"X-sweep needs an even subdomain count, got {part.J}")
    nrhs = int(F.shape[0])
    n = int(np.prod(part.shape))
    flat = F.reshape(nrhs, n)
    u, was_np = part.device().apply_many(flat, variant, cells)
    if was_np:
        return from_device(u, True, tuple(F.shape))
    return u.reshape(F.shape)


def prec_ud(part: Partition, f):
    return _apply(part, f, "ud")


def prec_x(part: Partition, f, parallel: bool = False):
    """X sweep; the two half-sweep fronts always run concurrently on the device
    (``parallel`` is accepted for drop-in compatibility; results are identical)."""
    if part.J % 2 != 0:
        raise ValueError(f"X-sweep needs an even subdomain count, got {part.J}")
    return _apply(part, f, "x")


@dataclass(frozen=True)
class NxCells:
    """Grouping for partial intersecting sweeps (reference sweepdd.py:362-390):
    cell boundaries with -1 and J+1 sentinels and each cell's meeting slab."""

    j_cell: tuple
    j_mid: tuple

    @property
    def n_cell(self):
        return len(self.j_cell) - 1

    def _span(self, m, J):
        """Slabs of cell m (1-based), clipped to 1..J."""
        return max(1, self.j_cell[m - 1] + 1), min(J, self.j_cell[m] - 1)

    def validate(self, J):
        b = np.asarray(self.j_cell)
        if b[0] != -1 or b[-1] != J + 1:
            raise ValueError("cell boundaries must start at -1 and end at J+1")
        if len(self.j_mid) != len(b) - 1:
            raise ValueError("one meeting slab per cell required")
        if np.any(np.diff(b) <= 0):
            raise ValueError("cell boundaries must be strictly increasing")
        for m, mid in enumerate(self.j_mid, start=1):
            lo, hi = self._span(m, J)
            if mid < lo or mid > hi:
                raise ValueError(f"cell {m}: meeting slab {mid} outside [{lo},{hi}]")


def make_nx_cells(J: int, n_cell: int) -> NxCells:
    """n_cell cells of ~J/n_cell slabs (boundaries round(m J / n_cell)), each
    meeting at the upper middle of its slab span (sweepdd.py:392-401)."""
    if n_cell < 1 or 2 * n_cell > J:
        raise ValueError(f"need 1 <= n_cell <= J/2, got {n_cell} for J={J}")
    inner = tuple(round(m * J / n_cell) for m in range(1, n_cell))
    bounds = (-1,) + inner + (J + 1,)
    probe = NxCells(bounds, ())
    mids = tuple(sum(probe._span(m, J)) // 2 + (sum(probe._span(m, J)) % 2)
                 for m in range(1, n_cell + 1))
    cells = NxCells(bounds, mids)
    cells.validate(J)
    return cells


def prec_nx(part: Partition, f, cells: NxCells):
    """NX sweep: partial intersecting X sweeps over slab groups (sweepdd.py:
    403-434).  Every cell's fronts run concurrently on the device (one
    cluster per front); the group-boundary input solve runs after both
    neighbouring cells, as in the reference."""
    cells.validate(part.J)
    return _apply(part, f, "nx", cells)


@dataclass
class SweepingPreconditioner:
    part: Partition
    variant: str = "ud"
    cells: object = None
    parallel: bool = False

    def __post_init__(self):
        if self.variant not in ("ud", "x", "nx"):
            raise ValueError(f"unknown sweep variant {self.variant!r}")
        if self.variant == "x" and self.part.J % 2 != 0:
            raise ValueError(f"X-sweep needs an even subdomain count, got {self.part.J}")
        if self.variant == "nx":
            if isinstance(self.cells, (int, np.integer)):
                self.cells = make_nx_cells(self.part.J, int(self.cells))
            if self.cells is None:
                raise ValueError("NX-sweep needs its cell grouping")
            self.cells.validate(self.part.J)

    def __call__(self, f):
        flat = np.ndim(f) == 1 if not hasattr(f, "dim") else f.dim() == 1
        if self.variant == "x":
            u = prec_x(self.part, f)
        elif self.variant == "ud":
            u = prec_ud(self.part, f)
        else:
            u = prec_nx(self.part, f, self.cells)
        return u.reshape(-1) if flat else u
