"""Iteration-count / solution anchors of BASELINE configs at (near) full
size, computed by running the REFERENCE solver (build container only, ~15
min of one core):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_large_anchors.py

The problem inputs (velocity sampling, omega, sources, J) come from this
package's host-side recipe (``paper_1412_0464_b200.configs``, no GPU
needed); the mesh, model, hierarchy and GMRES are the reference's own.
Writes ``tests/golden/large_anchors.json`` (``--out=PATH`` for a partial
file that is merged afterwards, so several cases can run in parallel);
``tests/test_gpu_parity.py`` solves the same problems on the GPU and checks
iterations (+-1), the residual history and the solution norm.

``apply_*`` cases store the reference's ``tgsp_apply(cycle, z)`` for a seeded
complex standard-normal z (``default_rng(APPLY_SEED + config)``) at full
config size: its 2-norm, 256 sampled entries and the sums over 1024
contiguous blocks of the flat output -- enough to bound the relative L2
error of a GPU apply at the north_star's 1e-10 without committing the
vector (C3: 275 MB).  Consecutive cases of the same problem reuse one
reference hierarchy (C4's eight right-hand sides).
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = os.environ.get("HELMSWEEP_REF", "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, REF)
sys.path.insert(1, str(ROOT))

import helmsweep as hs  # noqa: E402  (the reference)
from helmsweep.discretize import _assemble_fe, axis_gamma_fn, axis_sigma_fn  # noqa: E402
from helmsweep.mesh import PML, AbsorbingLayerSpec  # noqa: E402
from helmsweep.twogrid import SmootherConfig, SweepOptions  # noqa: E402
from paper_1412_0464_b200.configs import config  # noqa: E402  (inputs only)

OUT = Path(__file__).resolve().parent / "large_anchors.json"
CASES = [("C2", 1, 1, 0), ("C4_rhs0", 3, 1, 0), ("C3_half", 2, 2, 0), ("C5_half", 4, 2, 0),
         ("C1_exact", 0, 1, 0), ("C1_nx4", 0, 1, 0), ("C1_x", 0, 1, 0),
         ("C3", 2, 1, 0), ("apply_C3", 2, 1, None),
         ("apply_C4", 3, 1, None)] + [(f"C4_rhs{r}", 3, 1, r) for r in range(1, 8)] + [
         ("apply_C2", 1, 1, None), ("apply_C1", 0, 1, None),
         ("C5", 4, 1, 0), ("apply_C5", 4, 1, None)]
APPLY_SEED = 100
N_BLOCKS = 1024


def apply_vector(config_idx, n):
    """the seeded preconditioner-apply input of ``apply_*`` anchors"""
    rng = np.random.default_rng(APPLY_SEED + config_idx)
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def block_sums(y, nb=N_BLOCKS):
    """sums of y over nb contiguous blocks (np.array_split bounds)"""
    return np.array([b.sum() for b in np.array_split(np.asarray(y).ravel(), nb)])


def fe_fine(mesh, model):
    """The literal 27-point (3-D) / 9-point (2-D) compact fine operator: the
    reference FE engine on the fine mesh, rescaled by h^-d."""
    dim = mesh.dim
    h = float(mesh.spacing[0][0])
    op = _assemble_fe(mesh.spacing, [0.0] * dim, [axis_sigma_fn(mesh, a) for a in range(dim)],
                      [axis_gamma_fn(mesh, a) for a in range(dim)], model.omega, model.k,
                      None, hs.discretize.default_table(dim), h)
    return op.scaled(h ** (-dim), fe_scaled=False)


def _coarse(name):
    """coarse solver and sweep variant of a case: C1_exact -> the reference's
    default exact coarse solve; C1_nx4 -> NX sweep with 4 cells."""
    if name.endswith("_exact"):
        return "exact", "x", None
    if name.endswith("_nx4"):
        return "sweep", "nx", 4
    return "sweep", "x", None


_CACHE = {}


def _problem(name, idx, scale):
    """(p, cycle, setup seconds), reusing the last hierarchy of the same problem"""
    coarse, variant, n_cell = _coarse(name)
    key = (idx, scale, coarse, variant, n_cell)
    if key in _CACHE:
        return _CACHE[key]
    _CACHE.clear()
    p = config(idx, scale)
    m = p.mesh
    size = m.interior_cells(0)
    lay = m.layers[0][0]
    spec = AbsorbingLayerSpec(PML, lay.width, lay.strength, lay.ref_speed)
    mesh = hs.build_mesh(m.dim, size, 1.0 / size, spec)
    assert tuple(mesh.unknowns) == tuple(m.unknowns)
    model = hs.WaveModel(p.model.omega, np.asarray(p.model.k))
    t0 = time.perf_counter()
    fine_op = fe_fine(mesh, model) if p.fine != "fd5" else None
    cycle, _ = hs.build_two_grid(mesh, model, fine_op=fine_op,
                                 smoother=SmootherConfig(p.omega_jac, p.nu),
                                 coarse=coarse,
                                 sweep=SweepOptions(p.w_dd, p.s_dd, variant, n_cell=n_cell,
                                                    subdomains=p.subdomains))
    setup = time.perf_counter() - t0
    _CACHE[key] = (p, cycle, setup)
    return _CACHE[key]


def run_apply(name, idx, scale):
    p, cycle, setup = _problem(name, idx, scale)
    m = p.mesh
    z = apply_vector(idx, p.n_fine).reshape(m.unknowns)
    t0 = time.perf_counter()
    y = hs.tgsp_apply(cycle, z).ravel()
    t_apply = time.perf_counter() - t0
    sel = np.unique(np.linspace(0, y.size - 1, 256).astype(np.int64))
    bs = block_sums(y)
    print(f"{name}: |tgsp_apply(z)| = {np.linalg.norm(y):.12e}, {t_apply:.1f} s", flush=True)
    return {"config": idx, "scale": scale, "seed": APPLY_SEED + idx,
            "subdomains": int(p.subdomains), "fine_operator": p.fine,
            "fine_unknowns": list(m.unknowns), "y_norm": float(np.linalg.norm(y)),
            "y_sample_idx": sel.tolist(), "y_sample_re": y[sel].real.tolist(),
            "y_sample_im": y[sel].imag.tolist(), "n_blocks": N_BLOCKS,
            "block_sums_re": bs.real.tolist(), "block_sums_im": bs.imag.tolist(),
            "reference_setup_s": setup, "reference_apply_s": t_apply}


def run(name, idx, scale, rhs):
    if rhs is None:
        return run_apply(name, idx, scale)
    p, cycle, setup = _problem(name, idx, scale)
    m = p.mesh
    coarse, variant, n_cell = _coarse(name)
    f = p.f[rhs].ravel()
    t0 = time.perf_counter()
    u, rep = hs.gmres(lambda v: cycle.fine_csr @ v, cycle.as_preconditioner(), f,
                      hs.GmresConfig(tol=p.tol, max_iter=p.max_iter, restart=p.restart))
    solve = time.perf_counter() - t0
    true_res = float(np.linalg.norm(f - cycle.fine_csr @ u) / np.linalg.norm(f))
    sel = np.arange(0, u.size, max(1, u.size // 64))
    out = {"config": idx, "scale": scale, "rhs": rhs, "subdomains": int(p.subdomains),
           "fine_operator": p.fine, "coarse": coarse, "variant": variant, "n_cell": n_cell,
           "fine_unknowns": list(m.unknowns), "iterations": int(rep.iterations),
           "history": [float(v) for v in rep.residual_history], "true_residual": true_res,
           "u_norm": float(np.linalg.norm(u)), "u_sample_idx": sel.tolist(),
           "u_sample_re": u[sel].real.tolist(), "u_sample_im": u[sel].imag.tolist(),
           "reference_setup_s": setup, "reference_solve_s": solve}
    print(f"{name}: {rep.iterations} its, true residual {true_res:.3e}, setup {setup:.1f} s, "
          f"solve {solve:.1f} s", flush=True)
    return out


def main():
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    out = Path(outs[0]) if outs else OUT
    res = json.loads(out.read_text()) if out.exists() else {}
    only = [a for a in sys.argv[1:] if not a.startswith("--")]
    for name, idx, scale, rhs in CASES:
        if only and name not in only:
            continue
        res[name] = run(name, idx, scale, rhs)
        out.write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
