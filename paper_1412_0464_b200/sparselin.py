"""Direct solves on the device: drop-in for reference ``sparselin.py``.

* ``to_csr``                          :21-37  (host CSR, setup / checking only)
* ``Factorization``, ``factorize``    :40-68
* ``solve_factored``                  :71-76

A compact stencil operator is factorised on the GPU (``hs_exact_create``):
block LU along its second axis with dense planes of the first (and third)
axis, cuSOLVER/cuBLAS at setup, and the solve is the same cooperative
block-tridiagonal chain kernel as a 3-D sweep slab (``csrc/hs_sweep3.cu``).
It replaces SuperLU on the reference's exact coarse solve and ``factorize``
calls.  General scipy matrices are not factorised here (no host fallback).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .discretize import StencilOperator


def to_csr(op) -> sp.csr_matrix:
    """CSR matrix of a stencil operator (row-major unknown ordering), host:
    for every offset, the (row, row + offset) pairs whose neighbour lies in
    the box carry that offset's coefficient at the row."""
    shape = tuple(op.shape)
    idx = np.arange(int(np.prod(shape))).reshape(shape)
    rows, cols, vals = [], [], []
    for off, coef in op.coeffs.items():
        keep = np.ones(shape, dtype=bool)
        for ax, o in enumerate(off):
            n = shape[ax]
            sl = [slice(None)] * len(shape)
            if o > 0:
                sl[ax] = slice(n - o, n)
            elif o < 0:
                sl[ax] = slice(0, -o)
            else:
                continue
            keep[tuple(sl)] = False
        r = idx[keep]
        strides = [int(np.prod(shape[ax + 1:])) for ax in range(len(shape))]
        c = r + sum(o * st for o, st in zip(off, strides))
        rows.append(r)
        cols.append(c)
        vals.append(np.asarray(coef, dtype=complex)[keep])
    n = idx.size
    a = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n), dtype=complex)
    a.sort_indices()
    return a


class Factorization:
    """Device LU factors of a stencil operator; reusable for many right-hand
    sides.  Raises ZeroDivisionError("zero pivot at row i ...") on a singular
    pivot block (sparselin.py:53-56)."""

    _hs_device = True   # solve() takes torch CUDA vectors (krylov._device_callable)

    def __init__(self, op):
        from .device import DeviceExact, DeviceExactCSR
        if sp.issparse(op) or isinstance(op, np.ndarray):
            a = sp.csr_matrix(op, dtype=complex)
            if a.shape[0] != a.shape[1]:
                raise ValueError("matrix must be square")
            self.shape = (int(a.shape[0]),)
            self.n = self.shape[0]
            self.device = DeviceExactCSR(a)
            return
        if not hasattr(op, "device") or not hasattr(op, "shape"):
            raise TypeError("factorize takes a StencilOperator or a scipy sparse matrix, "
                            f"got {type(op).__name__}")
        if len(op.shape) == 1:   # a line: its rows as a general band (pivoting across rows)
            self.shape = tuple(op.shape)
            self.n = int(op.shape[0])
            self.device = DeviceExactCSR(to_csr(op))
            return
        self.shape = tuple(op.shape)
        self.n = int(np.prod(self.shape))
        self.device = DeviceExact(op.device())

    def solve(self, rhs):
        """x = A^{-1} rhs for rhs of shape (n,) or (n, k); numpy in, numpy out
        (torch CUDA tensors: zero-copy in, tensor out)."""
        if hasattr(rhs, "is_cuda"):
            if rhs.shape[0] != self.n:
                raise ValueError(f"rhs has {rhs.shape[0]} rows, expected {self.n}")
            if rhs.dim() == 1:
                return self.device.apply(rhs)[0]
            return self._solve_columns(rhs)
        rhs = np.asarray(rhs, dtype=complex)
        if rhs.shape[0] != self.n:
            raise ValueError(f"rhs has {rhs.shape[0]} rows, expected {self.n}")
        if rhs.ndim == 1:
            return self._solve1(rhs)
        import torch
        from .device import from_device
        dev = f"cuda:{self.device.ctx.device}"
        x = self._solve_columns(torch.from_numpy(np.ascontiguousarray(rhs)).to(dev))
        return from_device(x.contiguous(), True, tuple(rhs.shape))

    def _solve_columns(self, rhs):
        """(n, k) device tensor: the k columns as one multi-right-hand-side
        solve (hs_sweep_apply_many: groups of columns per block chain, every
        factor plane streamed once per group -- the reference's multi-column
        SuperLU solve, sparselin.py:58-62); column j is bitwise solve(rhs[:, j])."""
        import torch
        x = self.device.apply_many(rhs.t().to(torch.complex128).contiguous())
        return x.t().contiguous()

    def _solve1(self, b):
        from .device import from_device
        u, was_np = self.device.apply(np.ascontiguousarray(b))
        return from_device(u, True, (self.n,))


def factorize(matrix) -> Factorization:
    """Factorization of a stencil operator or a scipy sparse matrix
    (sparselin.py:65-68); both are factorised on the device."""
    return Factorization(matrix)


def solve_factored(factor: Factorization, rhs):
    """Solve for one vector or a block of right-hand sides (sparselin.py:71-76)."""
    return factor.solve(rhs)


_DENSE_CAP = 10_000


def dense_solve(op, rhs):
    """Dense LU solve of a small operator, the reference's ground-truth
    checker (sparselin.py:79-87): the operator densified from its CSR rows
    and solved on the device (torch.linalg.solve); capped at 10 000
    unknowns so that it stays a checker, not a solver."""
    import torch
    n = int(np.prod(op.shape)) if hasattr(op, "coeffs") else int(op.shape[0])
    if n > _DENSE_CAP:
        raise ValueError(f"dense oracle capped at {_DENSE_CAP} unknowns, got {n}")
    a = (to_csr(op) if hasattr(op, "coeffs") else sp.csr_matrix(op)).toarray()
    b = np.asarray(rhs, dtype=complex).reshape(n, -1)
    from ._lib import context
    dev = f"cuda:{context().device}"
    x = torch.linalg.solve(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)).cpu().numpy()
    return x[:, 0] if b.shape[1] == 1 else x


def write_matrix_market(path, matrix):
    """Matrix Market coordinate dump, complex general, 1-based
    (sparselin.py:90-94; host file I/O of the assembled matrix)."""
    import scipy.io
    if hasattr(matrix, "coeffs"):
        matrix = to_csr(matrix)
    scipy.io.mmwrite(path, matrix, field="complex")
