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

    def __init__(self, op):
        from .device import DeviceExact
        if not hasattr(op, "device") or not hasattr(op, "shape"):
            raise TypeError("factorize on the device takes a StencilOperator "
                            f"(compact stencil), got {type(op).__name__}")
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
            return _stack([self.device.apply(rhs[:, j].contiguous())[0]
                           for j in range(rhs.shape[1])])
        rhs = np.asarray(rhs, dtype=complex)
        if rhs.shape[0] != self.n:
            raise ValueError(f"rhs has {rhs.shape[0]} rows, expected {self.n}")
        if rhs.ndim == 1:
            return self._solve1(rhs)
        return np.column_stack([self._solve1(rhs[:, j]) for j in range(rhs.shape[1])])

    def _solve1(self, b):
        from .device import from_device
        u, was_np = self.device.apply(np.ascontiguousarray(b))
        return from_device(u, True, (self.n,))


def _stack(cols):
    import torch
    return torch.stack(cols, dim=1)


def factorize(matrix) -> Factorization:
    """Factorization of a stencil operator (sparselin.py:65-68)."""
    return Factorization(matrix)


def solve_factored(factor: Factorization, rhs):
    """Solve for one vector or a block of right-hand sides (sparselin.py:71-76)."""
    return factor.solve(rhs)
