"""BASELINE.json configurations restated as problem builders (host setup).

Each builder returns ``Problem(mesh, model, f, smoother, sweep, gmres)``
following SURVEY.md section 8(d):

* ``build_mesh(dim, size, 1/size, AbsorbingLayerSpec("pml", w, 20, max c))``;
  S_pml = 20 is the reference CLI default (reference ``cli.py:177-179``).
* c sampled at interior unknowns x_i = i h and edge-padded into the PML
  (reference ``cli.py:193-194``); omega from min(c) and the points/wavelength.
* point sources delta * h^-d at unknown index ``w + round(p * size) - 1``.
* TGSP: nu = 2, omega_jac 0.8 (2-D) / 0.6 (3-D), X sweep with
  J = (n_coarse_0 // lines) // 2 * 2, w_dd = 5 / s_dd = 25 (2-D) and
  w_dd = 3 / s_dd = 15 (3-D); GMRES(tol 1e-6, restart 20, max_iter 400).

Media are seeded synthetic stand-ins (no dataset is read): C2's three-layer
wedge from BASELINE's formula, C3/C4 smooth random media (seed 0 / 1),
C5 a Gaussian low-velocity lens.  C2-C4 use the 5-point fine operator
(SURVEY F2 decision (ii): the literal 9-point FE-opt fine operator stalls in
the reference); ``fine="fe9"`` builds the literal 9-point operator instead.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import PML, AbsorbingLayerSpec, build_mesh
from .discretize import (WaveModel, _fe_operator, axis_gamma_fn, axis_sigma_fn,
                         default_table)


@dataclass
class Problem:
    name: str
    mesh: object
    model: object
    f: np.ndarray                 # (nrhs,) + unknowns, complex128
    omega_jac: float
    nu: int
    w_dd: int
    s_dd: float
    subdomains: int
    lines: int
    fine: str = "fd5"
    tol: float = 1e-6
    restart: int = 20
    max_iter: int = 400
    notes: dict = field(default_factory=dict)

    @property
    def n_fine(self):
        return int(np.prod(self.mesh.unknowns))


def _interior_coords(size, dim):
    x = np.arange(1, size) / size
    return np.meshgrid(*([x] * dim), indexing="ij")


def _point_sources(mesh, size, width, points):
    h = 1.0 / size
    f = np.zeros((len(points),) + mesh.unknowns, dtype=complex)
    for r, p in enumerate(points):
        idx = tuple(width + int(round(pa * size)) - 1 for pa in p)
        f[(r,) + idx] += h ** (-mesh.dim)
    return f


def _subdomains(mesh, lines):
    from .mesh import coarsen_mesh
    mesh_c, _ = coarsen_mesh(mesh)
    return (mesh_c.unknowns[0] // lines) // 2 * 2


def _make(name, dim, size, width, c_int, ppw, sources, omega_jac, w_dd, s_dd, lines,
          sum_sources=True, fine="fd5", **notes):
    mesh = build_mesh(dim, size, 1.0 / size,
                      AbsorbingLayerSpec(PML, width, 20.0, float(np.max(c_int))))
    pad = [(width, width)] * dim
    c_full = np.pad(c_int, pad, mode="edge")
    freq = float(np.min(c_int)) * size / ppw
    model = WaveModel.from_velocity(mesh, 2.0 * np.pi * freq, c_full)
    f = _point_sources(mesh, size, width, sources)
    if sum_sources:
        f = f.sum(axis=0, keepdims=True)
    return Problem(name, mesh, model, f, omega_jac, 2, w_dd, s_dd,
                   _subdomains(mesh, lines), lines, fine=fine, notes=notes)


def smooth_random_velocity(size, seed, sigma_cells=20.0):
    from scipy.ndimage import gaussian_filter
    g = gaussian_filter(np.random.default_rng(seed).standard_normal((size - 1, size - 1)),
                        sigma=sigma_cells)
    g = (g - g.mean()) / g.std()
    return 1.0 + 0.3 * np.tanh(g)


def config(idx: int, scale: int = 1, fine: str = "fd5") -> Problem:
    """BASELINE configs[idx] (0-based); ``scale`` > 1 divides the grid size."""
    if idx == 0:
        size = 256 // scale
        return _make("C1", 2, size, 16, np.ones((size - 1,) * 2), 10.0, [(0.5, 0.5)],
                     0.8, 5, 25.0, 4, fine="fd5")
    if idx == 1:
        size = 1024 // scale
        x, y = _interior_coords(size, 2)
        c = np.where(y < 0.4 + 0.2 * x, 1.0, np.where(y < 0.75 - 0.15 * x, 1.5, 2.0))
        return _make("C2", 2, size, 16, c, 8.0, [(0.25, 0.1), (0.75, 0.1)],
                     0.8, 5, 25.0, 4, fine=fine)
    if idx == 2:
        size = 4096 // scale
        c = smooth_random_velocity(size, 0)
        return _make("C3", 2, size, 24, c, 8.0, [(0.5, 0.5)], 0.8, 5, 25.0, 4, fine=fine)
    if idx == 3:
        size = 2048 // scale
        c = smooth_random_velocity(size, 1)
        src = [(m / 9.0, 0.05) for m in range(1, 9)]
        return _make("C4", 2, size, 16, c, 8.0, src, 0.8, 5, 25.0, 4,
                     sum_sources=False, fine=fine)
    if idx == 4:
        size = 128 // scale
        x, y, z = _interior_coords(size, 3)
        r2 = (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2
        c = 1.0 - 0.4 * np.exp(-r2 / (2 * 0.15**2))
        return _make("C5", 3, size, 12, c, 8.0, [(0.5, 0.5, 0.1)], 0.6, 3, 15.0, 3,
                     fine="fe27")
    raise ValueError(f"no BASELINE config {idx}")


def fe_fine_operator(mesh, model):
    """The literal 9-point (2-D) / 27-point (3-D) compact fine operator: the FE
    engine on the fine mesh with node-sampled k, rescaled by h^-d."""
    dim = mesh.dim
    h = float(mesh.spacing[0][0])
    op = _fe_operator(mesh.spacing, [0.0] * dim, [axis_sigma_fn(mesh, a) for a in range(dim)],
                      [axis_gamma_fn(mesh, a) for a in range(dim)], model.omega, model.k,
                      None, default_table(dim), h)
    return op.scaled(h ** (-dim), fe_scaled=False)
