"""Device-side handles over libhsweep: operators, transfers, sweep, cycle.

Vectors: numpy arrays are copied to the device (and results copied back as
numpy); torch CUDA complex128 tensors are used zero-copy and results are
returned as torch tensors.  Everything is stream-ordered on torch's current
stream.  Device memory of handles is released when the handle is collected.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import context, i64


def _torch():
    import torch
    return torch


def to_device(x, n: int | None = None, ctx=None):
    """(tensor on device, was_numpy).  complex128, contiguous, flat view."""
    torch = _torch()
    ctx = ctx or context()
    if isinstance(x, torch.Tensor):
        t = x
        if (t.device.type != "cuda" or t.device.index != ctx.device
                or t.dtype != torch.complex128 or not t.is_contiguous()):
            t = t.to(device=f"cuda:{ctx.device}", dtype=torch.complex128).contiguous()
        t = t.reshape(-1)
        was_np = False
    else:
        a = np.ascontiguousarray(np.asarray(x, dtype=complex)).reshape(-1)
        t = torch.from_numpy(a).to(f"cuda:{ctx.device}", non_blocking=False)
        was_np = True
    if n is not None and t.numel() != n:
        raise ValueError(f"vector has {t.numel()} entries, expected {n}")
    return t, was_np


def from_device(t, was_numpy: bool, shape=None):
    if was_numpy:
        # DMA into pinned host memory (the numpy result keeps the buffer
        # alive): a pageable .cpu() would stage through a bounce buffer
        torch = _torch()
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t.detach(), non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        a = h.numpy()
        return a.reshape(shape) if shape is not None else a
    return t.reshape(shape) if shape is not None else t


def ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def empty(n: int, ctx=None):
    torch = _torch()
    ctx = ctx or context()
    return torch.empty(n, dtype=torch.complex128, device=f"cuda:{ctx.device}")


class _Handle:
    _destroy = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and self._destroy:
            try:
                getattr(self.ctx.lib, self._destroy)(self.ctx.h, h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None


class DeviceStencil(_Handle):
    """Uploaded compact-stencil operator (reference StencilOperator)."""

    _destroy = "hs_stencil_destroy"

    def __init__(self, shape, offsets, coeffs, ctx=None):
        self.ctx = ctx or context()
        self.shape = tuple(int(s) for s in shape)
        self.n = int(np.prod(self.shape))
        offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int8).reshape(-1, len(shape)))
        co = np.ascontiguousarray(np.asarray(coeffs, dtype=complex).reshape(len(offs), self.n))
        self.offsets = [tuple(int(v) for v in o) for o in offs]
        shp, pshp = i64(self.shape)
        h = C.c_void_p()
        self.ctx.call("hs_stencil_create", len(self.shape), pshp, len(offs),
                      offs.ctypes.data_as(C.POINTER(C.c_int8)),
                      co.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), C.byref(h))
        self.h = h

    @classmethod
    def adopt(cls, h, shape, offsets, ctx):
        """Wrap a handle created on the device (hs_assemble_*)."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.shape = tuple(int(s) for s in shape)
        self.n = int(np.prod(self.shape))
        self.offsets = [tuple(int(v) for v in o) for o in offsets]
        self.h = h
        return self

    def download(self) -> np.ndarray:
        """[S][n] complex128 coefficients back on the host (synchronises)."""
        out = np.empty((len(self.offsets), self.n), dtype=complex)
        self.ctx.call("hs_stencil_download", self.h,
                      out.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)))
        return out

    @classmethod
    def from_host(cls, op, ctx=None):
        offs = sorted(op.coeffs)
        return cls(op.shape, offs, np.stack([op.coeffs[o].reshape(-1) for o in offs]), ctx)

    def apply(self, x, shape=None, nrhs: int = 1):
        xt, was_np = to_device(x, self.n * nrhs, self.ctx)
        y = empty(self.n * nrhs, self.ctx)
        self.ctx.call("hs_stencil_apply", self.h, ptr(xt), ptr(y), nrhs)
        if shape is None and was_np and np.ndim(x) > 1:
            shape = np.shape(x)
        return from_device(y, was_np, shape)

    __call__ = apply

    def __matmul__(self, x):
        return self.apply(x)

    def residual(self, f, u, out=None):
        ft, _ = to_device(f, self.n, self.ctx)
        ut, _ = to_device(u, self.n, self.ctx)
        r = out if out is not None else empty(self.n, self.ctx)
        self.ctx.call("hs_stencil_residual", self.h, ptr(ft), ptr(ut), ptr(r), 1)
        return r

    def jacobi(self, u, f, omega, steps, u_is_zero=False):
        """In-place on a device tensor u (flat)."""
        self.ctx.call("hs_jacobi", self.h, ptr(u), ptr(f), float(omega), int(steps),
                      int(bool(u_is_zero)), 1)
        return u


class DeviceTransfer(_Handle):
    """Tent prolongation / restriction tables from a CoarseningMap."""

    _destroy = "hs_transfer_destroy"

    def __init__(self, cmap, ctx=None, window=None):
        """``window``: (fw_lo, fw_hi, cr_lo, cr_hi, fr_lo, fr_hi) on axis 0 for
        one shard of a sweep-axis decomposition (hs_transfer_create_window)."""
        self.ctx = ctx or context()
        fps = [np.asarray(f, dtype=np.int64) for f in cmap.fine_point_of_coarse]
        refs = [np.asarray(r, dtype=np.uint8) for r in cmap.refined_cell]
        self.fine_shape = tuple(int(f[-1]) - 1 for f in fps)
        self.coarse_shape = tuple(len(f) - 2 for f in fps)
        self.nf = int(np.prod(self.fine_shape))
        self.nc = int(np.prod(self.coarse_shape))
        lens, plen = i64([len(f) for f in fps])
        cat, pcat = i64(np.concatenate(fps))
        rc = np.ascontiguousarray(np.concatenate(refs), dtype=np.uint8)
        h = C.c_void_p()
        if window is None:
            self.ctx.call("hs_transfer_create", len(fps), plen, pcat,
                          rc.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(h))
        else:
            win, pwin = i64(window)
            self.ctx.call("hs_transfer_create_window", len(fps), plen, pcat,
                          rc.ctypes.data_as(C.POINTER(C.c_uint8)), pwin, C.byref(h))
        self.h = h

    def restrict(self, r, scale=1.0):
        rt, was_np = to_device(r, self.nf, self.ctx)
        out = empty(self.nc, self.ctx)
        self.ctx.call("hs_restrict", self.h, ptr(rt), ptr(out), float(scale), 1)
        return from_device(out, was_np, self.coarse_shape if was_np else None)

    def prolong(self, uc, u=None):
        ut, was_np = to_device(uc, self.nc, self.ctx)
        out = empty(self.nf, self.ctx) if u is None else u
        self.ctx.call("hs_prolong_add", self.h, ptr(ut), ptr(out), int(u is not None), 1)
        return from_device(out, was_np, self.fine_shape if was_np else None)


class DeviceSweep(_Handle):
    """Factorised slabs + UD/X schedules of one partition (device)."""

    _destroy = "hs_sweep_destroy"

    def __init__(self, coarse: DeviceStencil, J, beta, beta_tilde, slab_lo, slab_hi,
                 slab_ops, ctx=None):
        self.ctx = ctx or context()
        self.coarse = coarse
        self.slab_ops = list(slab_ops)   # keep alive during factorisation
        self.shape = coarse.shape
        self.n = coarse.n
        self.J = int(J)
        b, pb = i64(beta)
        bt, pbt = i64(beta_tilde)
        lo, plo = i64(slab_lo)
        hi, phi = i64(slab_hi)
        arr = (C.c_void_p * self.J)(*[op.h for op in self.slab_ops])
        h = C.c_void_p()
        self.ctx.call("hs_sweep_create", coarse.h, self.J, pb, pbt, plo, phi, arr, C.byref(h))
        self.h = h
        # the factors are self-contained on the device: slab coefficient copies can go
        self.slab_ops = None

    @property
    def factor_bytes(self) -> int:
        return int(self.ctx.lib.hs_sweep_factor_bytes(self.h))

    @property
    def segments(self) -> int:
        """face segments per front (two-level partition; 1 = one cluster)"""
        return int(self.ctx.lib.hs_sweep_segments(self.h))

    @property
    def chunks(self) -> int:
        return int(self.ctx.lib.hs_sweep_chunks(self.h))

    @property
    def max_fronts(self) -> int:
        """sweep fronts whose clusters co-reside on the device (hs_sweep_max_fronts)"""
        return int(self.ctx.lib.hs_sweep_max_fronts(self.h))

    def launches_per_apply(self, variant="x") -> int:
        """slab-solve launches of one application of the variant's plan"""
        return int(self.ctx.lib.hs_sweep_plan_launches(self.h, self.variant_id(variant)))

    def variant_id(self, variant="x", cells=None) -> int:
        """C-ABI variant id: HS_VARIANT_X / HS_VARIANT_UD, or the plan of an
        NX cell grouping (registered once per grouping, hs_sweep_plan_nx)."""
        if variant == "x":
            return _lib.HS_VARIANT_X
        if variant == "ud":
            return _lib.HS_VARIANT_UD
        if variant != "nx" or cells is None:
            raise ValueError(f"unknown sweep variant {variant!r}")
        key = (tuple(int(v) for v in cells.j_cell), tuple(int(v) for v in cells.j_mid))
        plans = self.__dict__.setdefault("_nx_plans", {})
        if key not in plans:
            jc, pjc = i64(key[0])
            jm, pjm = i64(key[1])
            v = C.c_int()
            self.ctx.call("hs_sweep_plan_nx", self.h, len(key[1]), pjc, pjm, C.byref(v))
            plans[key] = int(v.value)
        return plans[key]

    def relay_variant(self, shards: int) -> int:
        """Variant id of the X plan cut at `shards` sweep-axis shard
        boundaries (hs_sweep_plan_relay: the relay's critical path on one
        device); registered once per shard count."""
        plans = self.__dict__.setdefault("_relay_plans", {})
        if shards not in plans:
            v = C.c_int()
            self.ctx.call("hs_sweep_plan_relay", self.h, int(shards), C.byref(v))
            plans[shards] = int(v.value)
        return plans[shards]

    def apply(self, f, variant="x", cells=None):
        v = variant if isinstance(variant, int) else self.variant_id(variant, cells)
        ft, was_np = to_device(f, self.n, self.ctx)
        u = empty(self.n, self.ctx)
        self.ctx.call("hs_sweep_apply", self.h, v, ptr(ft), ptr(u))
        return u, was_np

    def rhs_width(self) -> int:
        """right-hand sides one chain of slab solves carries (hs_sweep_rhs_width)"""
        return int(self.ctx.lib.hs_sweep_rhs_width(self.h))

    def apply_many(self, F, variant="x", cells=None):
        """Rows of F (nrhs x n) through hs_sweep_apply_many: groups of up to
        rhs_width() right-hand sides share one pass over the slab factors."""
        v = variant if isinstance(variant, int) else self.variant_id(variant, cells)
        torch = _torch()
        was_np = not isinstance(F, torch.Tensor)
        if was_np:
            F = np.ascontiguousarray(np.asarray(F, dtype=complex))
        nrhs = int(F.shape[0])
        ft, _ = to_device(F, nrhs * self.n, self.ctx)
        u = empty(nrhs * self.n, self.ctx)
        self.ctx.call("hs_sweep_apply_many", self.h, v, nrhs, ptr(ft), ptr(u), self.n)
        return u.reshape(nrhs, self.n), was_np


class DeviceCSR(_Handle):
    """A general sparse matrix on the device for y = alpha A x (+ y)
    (hs_csr_*): explicit prolongation / restriction matrices."""

    _destroy = "hs_csr_destroy"

    def __init__(self, mat, ctx=None):
        import scipy.sparse as sp
        self.ctx = ctx or context()
        a = sp.csr_matrix(mat, dtype=complex)
        a.sum_duplicates()
        self.rows, self.cols = (int(v) for v in a.shape)
        ip, pip = i64(a.indptr)
        ix, pix = i64(a.indices)
        vals = np.ascontiguousarray(a.data, dtype=complex)
        h = C.c_void_p()
        self.ctx.call("hs_csr_create", self.rows, self.cols, int(a.nnz), pip, pix,
                      vals.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), C.byref(h))
        self.h = h

    def apply(self, x, out=None, alpha=1.0, accumulate=False):
        """device tensor in, device tensor out"""
        xt, _ = to_device(x, self.cols, self.ctx)
        y = out if out is not None else empty(self.rows, self.ctx)
        a = complex(alpha)
        self.ctx.call("hs_csr_apply", self.h, ptr(xt), ptr(y), a.real, a.imag,
                      int(bool(accumulate) and out is not None))
        return y


class DeviceExactCSR(_Handle):
    """Exact solver of a general sparse matrix (hs_exact_create_csr): its CSR
    rows cut into block rows of ``block`` >= bandwidth unknowns, factorised as
    a block-tridiagonal chain on the device."""

    _destroy = "hs_sweep_destroy"

    def __init__(self, csr, ctx=None):
        self.ctx = ctx or context()
        a = csr.tocsr().astype(complex)
        a.sum_duplicates()
        self.n = int(a.shape[0])
        coo = a.tocoo()
        bw = int(np.abs(coo.row.astype(np.int64) - coo.col.astype(np.int64)).max()) if a.nnz else 0
        # pivoting happens inside the blocks: small matrices are one dense
        # block (partial pivoting over every row, like SuperLU's), larger ones
        # get blocks of at least 64 rows
        self.block = self.n if self.n <= 1024 else max(bw, 64)
        self.n_pad = -(-self.n // self.block) * self.block
        ip, pip = i64(a.indptr)
        ix, pix = i64(a.indices)
        vals = np.ascontiguousarray(a.data, dtype=complex)
        h = C.c_void_p()
        self.ctx.call("hs_exact_create_csr", self.n, int(a.nnz), pip, pix,
                      vals.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
                      self.block, C.byref(h))
        self.h = h

    def variant_id(self, variant="ud", cells=None) -> int:
        if self.n_pad != self.n:
            raise ValueError("a padded general-matrix factorisation cannot be a cycle's "
                             "coarse solver")
        return _lib.HS_VARIANT_UD

    def apply(self, f):
        """x = A^{-1} f (flat, n entries); returns (tensor, was_numpy)."""
        torch = _torch()
        ft, was_np = to_device(f, self.n, self.ctx)
        if self.n_pad != self.n:
            fp = torch.zeros(self.n_pad, dtype=torch.complex128, device=ft.device)
            fp[:self.n] = ft
            ft = fp
        u = empty(self.n_pad, self.ctx)
        self.ctx.call("hs_sweep_apply", self.h, _lib.HS_VARIANT_UD, ptr(ft), ptr(u))
        return (u[:self.n] if self.n_pad != self.n else u), was_np

    def apply_many(self, F):
        """Rows of the device tensor F (k x n) solved through
        hs_sweep_apply_many (groups of right-hand sides per block chain);
        returns a (k x n) device tensor."""
        torch = _torch()
        k = int(F.shape[0])
        fp = torch.zeros((k, self.n_pad), dtype=torch.complex128, device=F.device)
        fp[:, :self.n] = F
        u = torch.empty_like(fp)
        self.ctx.call("hs_sweep_apply_many", self.h, _lib.HS_VARIANT_UD, k, ptr(fp), ptr(u),
                      self.n_pad)
        return u[:, :self.n]


class DeviceExact(_Handle):
    """Exact solver of a whole stencil operator (hs_exact_create): one block-LU
    slab behind the sweep interface (variant HS_VARIANT_UD)."""

    _destroy = "hs_sweep_destroy"

    def __init__(self, op: DeviceStencil):
        self.ctx = op.ctx
        self.op = op              # the factors copy the coefficients; kept for shape
        self.n = op.n
        self.shape = op.shape
        h = C.c_void_p()
        self.ctx.call("hs_exact_create", op.h, C.byref(h))
        self.h = h

    @property
    def factor_bytes(self) -> int:
        return int(self.ctx.lib.hs_sweep_factor_bytes(self.h))

    def variant_id(self, variant="ud", cells=None) -> int:
        return _lib.HS_VARIANT_UD

    def apply(self, f, variant="ud", cells=None):
        ft, was_np = to_device(f, self.n, self.ctx)
        u = empty(self.n, self.ctx)
        self.ctx.call("hs_sweep_apply", self.h, _lib.HS_VARIANT_UD, ptr(ft), ptr(u))
        return u, was_np

    def apply_many(self, F):
        """Rows of the contiguous device tensor F (k x n) through
        hs_sweep_apply_many; returns a (k x n) device tensor."""
        torch = _torch()
        k = int(F.shape[0])
        F = F.contiguous()
        u = torch.empty_like(F)
        self.ctx.call("hs_sweep_apply_many", self.h, _lib.HS_VARIANT_UD, k, ptr(F), ptr(u), self.n)
        return u

    def rhs_width(self) -> int:
        return int(self.ctx.lib.hs_sweep_rhs_width(self.h))


class DeviceCycle(_Handle):
    """The TGSP two-grid cycle (fine smoother + transfers + coarse sweep)."""

    _destroy = "hs_cycle_destroy"

    def __init__(self, fine: DeviceStencil, transfer: DeviceTransfer, coarse: DeviceStencil,
                 sweep, omega_jac, nu, restrict_scale, variant, ctx=None, cells=None):
        """``sweep``: a DeviceSweep or DeviceExact; ``variant``: a C-ABI
        variant id, or "x" / "ud" / "nx" (with ``cells``)."""
        self.ctx = ctx or context()
        self.fine, self.transfer, self.coarse, self.sweep = fine, transfer, coarse, sweep
        self.n = fine.n
        v = variant if isinstance(variant, int) else sweep.variant_id(variant, cells)
        h = C.c_void_p()
        self.ctx.call("hs_cycle_create", fine.h, transfer.h, coarse.h, sweep.h,
                      float(omega_jac), int(nu), float(restrict_scale), v, C.byref(h))
        self.h = h

    def lane(self, ctx):
        """A lane of this cycle on another context (hs_cycle_create_lane):
        shared operators and factors, private scratch."""
        ln = DeviceCycle.__new__(DeviceCycle)
        ln.ctx = ctx
        ln.fine, ln.transfer, ln.coarse, ln.sweep = self.fine, self.transfer, self.coarse, \
            self.sweep
        ln.base = self            # keeps the shared handles alive
        ln.n = self.n
        h = C.c_void_p()
        ctx.call("hs_cycle_create_lane", self.h, C.byref(h))
        ln.h = h
        return ln

    def vcycle_dev(self, f_dev, out=None):
        u = out if out is not None else empty(self.n, self.ctx)
        self.ctx.call("hs_vcycle", self.h, ptr(f_dev), ptr(u))
        return u

    def vcycle_many_dev(self, F_dev, out=None):
        """Rows of F_dev (nrhs x n, contiguous device tensor) through
        hs_vcycle_many: one chain of slab solves for all of them."""
        nrhs = int(F_dev.shape[0])
        u = out if out is not None else empty(nrhs * self.n, self.ctx).reshape(nrhs, self.n)
        self.ctx.call("hs_vcycle_many", self.h, nrhs, ptr(F_dev), ptr(u), self.n)
        return u

    def apply_a_begin(self, f_dev):
        """First half of w = A M f (pre-smoothing, residual, restriction)."""
        self.ctx.call("hs_vcycle_apply_a_begin", self.h, ptr(f_dev))

    def apply_a_part(self, f_dev, w, part):
        """hs_vcycle_apply_a_part: 0 begin, 1 the sweep's first launch, 2 the rest (-> w)."""
        self.ctx.call("hs_vcycle_apply_a_part", self.h, ptr(f_dev), ptr(w) if w is not None
                      else None, int(part))
        return w

    def apply_az_part(self, f_dev, z, w, part):
        """hs_vcycle_apply_az_part: z = M f kept, w = A z (parts 0/1/2, 3 = whole)."""
        self.ctx.call("hs_vcycle_apply_az_part", self.h, ptr(f_dev), ptr(z),
                      ptr(w) if w is not None else None, int(part))
        return w

    def apply_a_end(self, f_dev, w):
        """Second half (sweep, prolongation, post-smoothing, fine matvec) into w."""
        self.ctx.call("hs_vcycle_apply_a_end", self.h, ptr(f_dev), ptr(w))
        return w

    def apply_a_dev(self, f_dev, out=None):
        w = out if out is not None else empty(self.n, self.ctx)
        self.ctx.call("hs_vcycle_apply_a", self.h, ptr(f_dev), ptr(w))
        return w
