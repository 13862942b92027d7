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
    """One results-CSV row; the field order is the CSV column order."""

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
        return [self.__dict__[name] for name in self.columns()]


_TYPES = {"dim": int, "size": int, "w_dd": int, "subdomains": int, "iterations": int,
          "freq": float, "final_residual": float, "setup_time": float, "solve_time": float,
          "converged": lambda v: v == "True"}


def write_rows(path, rows, append=False):
    """Rows to CSV (header first when the file is new); floats as repr, so a
    read-back is exact."""
    path = Path(path)
    fresh = not (append and path.exists())
    with path.open("w" if fresh else "a", newline="", encoding="utf-8") as fh:
        out = csv.writer(fh)
        if fresh:
            out.writerow(ResultRow.columns())
        out.writerows([[repr(v) if isinstance(v, float) else v for v in r.values()]
                       for r in rows])


def read_rows(path):
    """CSV rows as dicts with the numeric / boolean columns converted."""
    with open(path, newline="", encoding="utf-8") as fh:
        return [{k: _TYPES[k](v) if k in _TYPES else v for k, v in rec.items()}
                for rec in csv.DictReader(fh)]


def _xfast(dims):
    """Reshape order of an x-fastest file: the raw samples are the C-order
    array of the reversed shape, transposed back."""
    return tuple(int(n) for n in dims)[::-1]


def load_model(path, dims, dtype="<f4") -> np.ndarray:
    """Velocities on the lattice ``dims`` (x-fastest raw file) as float64."""
    dims = tuple(int(n) for n in dims)
    raw = np.fromfile(path, dtype=dtype)
    need = int(np.prod(dims))
    if raw.size != need:
        raise ValueError(f"{path}: {raw.size} samples, expected {need} "
                         f"({need * 4} bytes) for dims {dims}")
    nonpos = np.nonzero(raw <= 0.0)[0]
    if len(nonpos):
        raise ValueError(f"{path}: nonpositive velocity at flat index {nonpos[0]}")
    return np.transpose(raw.reshape(_xfast(dims))).astype(np.float64)


def save_field(path, u):
    """Complex field as interleaved (re, im) float64, x-fastest."""
    if hasattr(u, "is_cuda") and u.is_cuda:
        import torch
        t = u.to(torch.complex128)
        t = t.permute(*reversed(range(t.dim()))).contiguous()   # x-fastest, on the device
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        flat = h.numpy().reshape(-1)
    else:
        flat = np.transpose(np.asarray(u, dtype=np.complex128)).reshape(-1)
    # complex128 in memory is exactly (re, im) float64 pairs
    np.ascontiguousarray(flat).view(np.float64).astype("<f8").tofile(path)


def load_field(path, dims) -> np.ndarray:
    dims = tuple(int(n) for n in dims)
    raw = np.fromfile(path, dtype="<f8")
    if raw.size != 2 * int(np.prod(dims)):
        raise ValueError(f"{path}: wrong size for dims {dims}")
    z = raw.astype(np.float64).view(np.complex128)
    return np.transpose(z.reshape(_xfast(dims)))
