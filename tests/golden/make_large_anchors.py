"""Iteration-count / solution anchors of BASELINE configs at (near) full
size, computed by running the REFERENCE solver (build container only, ~15
min of one core):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_large_anchors.py

The problem inputs (velocity sampling, omega, sources, J) come from this
package's host-side recipe (``paper_1412_0464_b200.configs``, no GPU
needed); the mesh, model, hierarchy and GMRES are the reference's own.
Writes ``tests/golden/large_anchors.json``; ``tests/test_gpu_parity.py``
solves the same problems on the GPU and checks iterations (+-1), the
residual history and the solution norm.
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
         ("C1_exact", 0, 1, 0), ("C1_nx4", 0, 1, 0)]


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


def run(name, idx, scale, rhs):
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
    coarse, variant, n_cell = _coarse(name)
    cycle, _ = hs.build_two_grid(mesh, model, fine_op=fine_op,
                                 smoother=SmootherConfig(p.omega_jac, p.nu),
                                 coarse=coarse,
                                 sweep=SweepOptions(p.w_dd, p.s_dd, variant, n_cell=n_cell,
                                                    subdomains=p.subdomains))
    setup = time.perf_counter() - t0
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
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    only = sys.argv[1:]
    for name, idx, scale, rhs in CASES:
        if only and name not in only:
            continue
        res[name] = run(name, idx, scale, rhs)
        OUT.write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
