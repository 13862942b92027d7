"""Harness I/O with the reference's file formats: the
results-CSV row, velocity-model ingestion and complex field dumps, so GPU
runs emit reference-identical reports and files.

* ``ResultRow``, ``write_rows``, ``read_rows``   cli.py:83-108, 287-318
* ``load_model``                                  cli.py:114-125
* ``save_field``, ``load_field``                  cli.py:128-143

Formats: velocities are raw little-endian float32, x-fastest (axis 0
fastest), on the interior unknown lattice; fields are interleaved (re, im)
little-endian float64 in the same order.  ``save_field`` takes a numpy array
or a torch CUDA tensor (the x-fastest reordering then runs on the device
and one pinned D2H copy moves the bytes).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, fields
from pathlib import Path

import numpy as np


@dataclass
class ResultRow:
    key: str
    model: str
    dim: int
    size: int
    freq: float
    layer: str
    solver: str
    variant: str
    w_dd: int
    subdomains: int
    seed: object
    iterations: int
    converged: bool
    final_residual: float
    setup_time: float
    solve_time: float
    residual_file: str = ""

    @staticmethod
    def columns():
        return [f.name for f in fields(ResultRow)]

    def values(self):
        return [getattr(self, name) for name in self.columns()]


def _cell(v):
    return repr(v) if isinstance(v, float) else v


def write_rows(path, rows, append=False):
    """CSV with a header row; floats written with repr (round-trip exact)."""
    mode = "a" if append and Path(path).exists() else "w"
    with open(path, mode, newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        if mode == "w":
            w.writerow(ResultRow.columns())
        for row in rows:
            w.writerow([_cell(v) for v in row.values()])


_INT = ("dim", "size", "w_dd", "subdomains", "iterations")
_FLOAT = ("freq", "final_residual", "setup_time", "solve_time")


def read_rows(path):
    out = []
    with open(path, newline="", encoding="utf-8") as fh:
        for rec in csv.DictReader(fh):
            for k in _INT:
                rec[k] = int(rec[k])
            for k in _FLOAT:
                rec[k] = float(rec[k])
            rec["converged"] = rec["converged"] == "True"
            out.append(rec)
    return out


def load_model(path, dims, dtype="<f4") -> np.ndarray:
    """Velocities on the lattice ``dims`` (x-fastest raw file) as float64."""
    dims = tuple(int(d) for d in dims)
    raw = np.fromfile(path, dtype=dtype)
    expected = int(np.prod(dims))
    if raw.size != expected:
        raise ValueError(f"{path}: {raw.size} samples, expected {expected} "
                         f"({expected * 4} bytes) for dims {dims}")
    bad = np.flatnonzero(raw <= 0.0)
    if bad.size:
        raise ValueError(f"{path}: nonpositive velocity at flat index {bad[0]}")
    return raw.reshape(dims[::-1]).T.astype(float)


def save_field(path, u):
    """Complex field as interleaved (re, im) float64, x-fastest."""
    if hasattr(u, "is_cuda") and u.is_cuda:
        import torch
        t = u.to(torch.complex128)
        t = t.permute(*reversed(range(t.dim()))).contiguous()   # x-fastest, on the device
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        inter = torch.view_as_real(h).numpy().reshape(-1)
    else:
        flat = np.ascontiguousarray(np.asarray(u, dtype=complex).T)
        inter = np.empty(flat.size * 2)
        inter[0::2] = flat.real.ravel()
        inter[1::2] = flat.imag.ravel()
    np.asarray(inter, dtype="<f8").tofile(path)


def load_field(path, dims) -> np.ndarray:
    dims = tuple(int(d) for d in dims)
    raw = np.fromfile(path, dtype="<f8")
    if raw.size != 2 * int(np.prod(dims)):
        raise ValueError(f"{path}: wrong size for dims {dims}")
    u = raw[0::2] + 1j * raw[1::2]
    return u.reshape(dims[::-1]).T
