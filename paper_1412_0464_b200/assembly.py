"""Operator assembly on the device.

Drop-in device versions of the reference's assembly routines
(``/root/reference/pkg/src/helmsweep/discretize.py``):

* ``assemble_fine_device``            -- ``assemble_fine`` / ``assemble_sponge`` :191-253
* ``assemble_fe_pml_coarse_device``   -- ``assemble_fe_pml_coarse`` :514-537 (FE engine :428-506)
* ``subdomain_fe_operator_device``    -- ``subdomain_fe_operator`` :685-723

The host evaluates only the per-axis 1-D arrays with the same numpy
expressions as :mod:`.discretize` (stretching factors, widths, damping
profiles); ``hs_assemble_fd`` / ``hs_assemble_fe`` form every per-node
coefficient on the device in the reference's operation order and keep it
there.  The result is a :class:`DeviceOperator`: a ``StencilOperator`` whose
device copy is authoritative and whose host ``coeffs`` are downloaded only
if something asks for them (tests, the shard planner).
"""

from __future__ import annotations

import ctypes as C
import itertools

import numpy as np

from .discretize import (StencilOperator, _check_model, _extend_rows, _slab_sigma, _stretch,
                         _TWO_PI, axis_gamma_fn, axis_sigma_fn, default_table,
                         interior_spacing, _nodes_to_cells)
from .mesh import PML, SPONGE, CoarseningMap, Mesh


def _dp(a):
    return np.ascontiguousarray(a).view(np.float64).ctypes.data_as(C.POINTER(C.c_double))


class DeviceOperator(StencilOperator):
    """A stencil operator assembled on (and owned by) the device."""

    def __init__(self, dev, fe_scaled=False):
        self.shape = dev.shape
        self.fe_scaled = fe_scaled
        self._device = dev
        self._coeffs = None

    @property
    def coeffs(self):
        if self._coeffs is None:
            arr = self._device.download()
            self._coeffs = {o: arr[s].reshape(self.shape)
                            for s, o in enumerate(self._device.offsets)}
        return self._coeffs

    def device(self, ctx=None):
        return self._device

    def scaled(self, factor, fe_scaled=None):
        return StencilOperator(self.shape, {o: c * factor for o, c in self.coeffs.items()},
                               fe_scaled=self.fe_scaled if fe_scaled is None else fe_scaled)


class DeviceField:
    """A float64 field uploaded once (wavenumbers of a level)."""

    def __init__(self, arr, ctx):
        import torch
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.float64))
        self.shape = a.shape
        self.t = torch.from_numpy(a).to(f"cuda:{ctx.device}")

    @property
    def ptr(self):
        return C.c_void_p(self.t.data_ptr())


def _ctx(ctx):
    from ._lib import context
    return ctx or context()


def assemble_fine_device(mesh: Mesh, model, ctx=None, k_field: DeviceField | None = None):
    """Fine-level 5/7-point FD operator (PML stretching, or sponge damping)."""
    from .device import DeviceStencil
    ctx = _ctx(ctx)
    _check_model(mesh, model)
    if not mesh.is_uniform():
        raise ValueError("fine assembly expects uniform spacing")
    kinds = {s.kind for pair in mesh.layers for s in pair}
    if PML in kinds and SPONGE in kinds:
        raise ValueError("mesh mixes PML and sponge layers")
    sponge = SPONGE in kinds
    h = float(mesh.spacing[0][0])
    dim = mesh.dim
    a_half, a_node, gam = [], [], []
    for a in range(dim):
        p = mesh.points(a)
        if sponge:
            a_half.append(np.ones(mesh.cells[a], dtype=complex))
            a_node.append(np.ones(mesh.cells[a] - 1, dtype=complex))
            g = axis_gamma_fn(mesh, a)
            gam.append(np.zeros(mesh.cells[a] - 1) if g is None else np.asarray(g(p[1:-1]), float))
        else:
            sig = axis_sigma_fn(mesh, a)
            a_half.append(_stretch(sig, 0.5 * (p[:-1] + p[1:]), model.omega))
            a_node.append(_stretch(sig, p[1:-1], model.omega))
    k = k_field or DeviceField(model.k, ctx)
    shape = np.asarray(mesh.unknowns, dtype=np.int64)
    h_ = C.c_void_p()
    gcat = np.concatenate(gam) if sponge else None
    ctx.call("hs_assemble_fd", dim, shape.ctypes.data_as(C.POINTER(C.c_int64)), h,
             _dp(np.concatenate(a_half)), _dp(np.concatenate(a_node)),
             _dp(gcat) if sponge else None, k.ptr, C.byref(h_))
    offs = sorted([tuple(-1 if m == a else 0 for m in range(dim)) for a in range(dim)]
                  + [tuple(1 if m == a else 0 for m in range(dim)) for a in range(dim)]
                  + [(0,) * dim])
    dev = DeviceStencil.adopt(h_, mesh.unknowns, offs, ctx)
    dev._k = k
    return DeviceOperator(dev)


def _fe_device(widths, origins, sigma_fns, gamma_fns, omega, kn: DeviceField,
               kc: DeviceField, rowmap, table, h_ref, ctx):
    """The FE engine (discretize._fe_operator, k per cell) on the device."""
    from .device import DeviceStencil
    dim = len(widths)
    widths = [np.asarray(w, dtype=float) for w in widths]
    shape = tuple(w.size - 1 for w in widths)
    woa, aow, cw, gc = [], [], [], []
    for a in range(dim):
        p = np.zeros(widths[a].size + 1)
        np.cumsum(widths[a], out=p[1:])
        p = origins[a] + p
        mids = 0.5 * (p[:-1] + p[1:])
        alpha = _stretch(sigma_fns[a], mids, omega)
        woa.append(widths[a].astype(complex) / alpha)
        aow.append(alpha / widths[a])
        cw.append(widths[a] * (1.0 / alpha))
        gc.append(np.zeros(widths[a].size) if gamma_fns[a] is None
                  else np.asarray(gamma_fns[a](mids), float))
    any_g = any(g is not None for g in gamma_fns)
    shp = np.asarray(shape, dtype=np.int64)
    rm = np.asarray(rowmap, dtype=np.int32)
    tx = np.ascontiguousarray(table.inv_g, dtype=np.float64)
    tc = np.ascontiguousarray(table.coeffs, dtype=np.float64)
    gcat = np.concatenate(gc) if any_g else None
    h_ = C.c_void_p()
    ctx.call("hs_assemble_fe", dim, shp.ctypes.data_as(C.POINTER(C.c_int64)),
             _dp(np.concatenate(woa)), _dp(np.concatenate(aow)), _dp(np.concatenate(cw)),
             _dp(gcat) if any_g else None, kn.ptr, int(np.prod(kn.shape[1:])), kc.ptr,
             int(np.prod(kc.shape[1:])), rm.ctypes.data_as(C.POINTER(C.c_int32)),
             float(h_ref), len(tx), tc.shape[1], _dp(tx), _dp(tc), C.byref(h_))
    offs = list(itertools.product((-1, 0, 1), repeat=dim))
    dev = DeviceStencil.adopt(h_, shape, offs, ctx)
    dev._fields = (kn, kc)
    return DeviceOperator(dev, fe_scaled=True)


class CoarseFields:
    """The coarse level's wavenumbers on the device (nodes and cells)."""

    def __init__(self, model_c, k_cells, ctx):
        self.kn = DeviceField(model_c.k, ctx)
        self.kc = DeviceField(k_cells, ctx)


def assemble_fe_pml_coarse_device(mesh_c: Mesh, cmap: CoarseningMap, model_c, k_cells=None,
                                  table=None, ctx=None, fields: CoarseFields | None = None):
    """FE coarse operator on a PML-coarsened mesh (rows carry h^d), on the device."""
    ctx = _ctx(ctx)
    _check_model(mesh_c, model_c)
    if cmap.dim != mesh_c.dim or any(len(cmap.coarse_widths[a]) != mesh_c.cells[a]
                                     for a in range(mesh_c.dim)):
        raise ValueError("coarsening map does not match the coarse mesh")
    dim = mesh_c.dim
    table = table or default_table(dim)
    if k_cells is None:
        k_cells = _nodes_to_cells(model_c.k)
    if k_cells.shape != mesh_c.cells:
        raise ValueError(f"k_cells shape {k_cells.shape} != cells {mesh_c.cells}")
    fields = fields or CoarseFields(model_c, k_cells, ctx)
    n0 = mesh_c.unknowns[0]
    rowmap = (0, 0, n0 - 1, 0, 0, n0)
    return _fe_device(mesh_c.spacing, [0.0] * dim,
                      [axis_sigma_fn(mesh_c, a) for a in range(dim)],
                      [axis_gamma_fn(mesh_c, a) for a in range(dim)],
                      model_c.omega, fields.kn, fields.kc, rowmap, table,
                      interior_spacing(mesh_c), ctx)


def subdomain_fe_operator_device(mesh_c: Mesh, model_c, k_cells, table, core_lo, core_hi,
                                 w_dd, s_dd, open_left, open_right, fields: CoarseFields,
                                 ctx=None):
    """Coarse-level FE slab with added PML (discretize.subdomain_fe_operator) on
    the device; the slab's replicated edge rows of k are a row map into the
    level's device fields, not copies."""
    ctx = _ctx(ctx)
    dim = mesh_c.dim
    wl = w_dd if open_left else 0
    wr = w_dd if open_right else 0
    lo, hi = core_lo - wl, core_hi + wr
    wx = np.asarray(mesh_c.spacing[0], dtype=float)
    core_cells = wx[core_lo - 1:core_hi + 1]
    edge_l, edge_r = float(core_cells[0]), float(core_cells[-1])
    wx_loc = np.concatenate([np.full(wl, edge_l), core_cells, np.full(wr, edge_r)])
    xg = mesh_c.points(0)
    sig0 = _slab_sigma(axis_sigma_fn(mesh_c, 0), model_c.omega, model_c.k, core_lo, core_hi,
                       0.5 * (xg[core_lo - 1] + xg[core_lo]),
                       0.5 * (xg[core_hi] + xg[core_hi + 1]),
                       w_dd * edge_l, w_dd * edge_r, s_dd, open_left, open_right)
    if k_cells is None:
        raise ValueError("the device slab assembly needs per-cell wavenumbers (PML levels)")
    rowmap = (core_lo - 1 - wl, core_lo - 1, core_hi - 1, core_lo - 1 - wl, core_lo - 1, core_hi)
    op = _fe_device([wx_loc] + [mesh_c.spacing[a] for a in range(1, dim)],
                    [float(xg[core_lo - 1]) - wl * edge_l] + [0.0] * (dim - 1),
                    [sig0] + [axis_sigma_fn(mesh_c, a) for a in range(1, dim)],
                    [axis_gamma_fn(mesh_c, a) for a in range(dim)],
                    model_c.omega, fields.kn, fields.kc, rowmap, table or default_table(dim),
                    interior_spacing(mesh_c), ctx)
    return op, lo, hi
