"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/*.npz`` / ``*.json``: operator coefficients, partition
geometry, transfer/smoother/sweep/TGSP outputs and GMRES histories computed by
``helmsweep`` itself on small seeded cases, plus the config-1 (BASELINE
configs[0]) anchors.  These pin both the numpy oracle (``oracle/``) and the
package's host-side assembly; the GPU tests then compare against the oracle.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("HELMSWEEP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import helmsweep as hs  # noqa: E402  (the reference)
from helmsweep.discretize import _assemble_fe, axis_gamma_fn, axis_sigma_fn  # noqa: E402
from helmsweep.twogrid import SmootherConfig, SweepOptions  # noqa: E402
from helmsweep.mesh import PML, SPONGE, AbsorbingLayerSpec  # noqa: E402

OUT = Path(__file__).resolve().parent


def crand(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def pack_op(prefix, op, out):
    offs = sorted(op.coeffs)
    out[prefix + "offsets"] = np.array(offs, dtype=np.int8).reshape(len(offs), op.dim)
    out[prefix + "coeffs"] = np.stack([op.coeffs[o] for o in offs])
    out[prefix + "fe_scaled"] = np.array(op.fe_scaled)


def constant_case(dim, interior, layer, ppw):
    h = 1.0 / interior
    mesh = hs.build_mesh(dim, interior, h, layer)
    model = hs.WaveModel.constant(mesh, 2 * np.pi * interior / ppw)
    return mesh, model


def hetero_case(interior, width, ppw, seed):
    h = 1.0 / interior
    mesh = hs.build_mesh(2, interior, h, AbsorbingLayerSpec(PML, width, 20.0, 2.0))
    rng = np.random.default_rng(seed)
    x = np.arange(1, interior) * h
    xx, yy = np.meshgrid(x, x, indexing="ij")
    c = np.where(yy < 0.4 + 0.2 * xx, 1.0, np.where(yy < 0.75 - 0.15 * xx, 1.5, 2.0))
    c = c * (1.0 + 0.05 * rng.random(c.shape))
    c_full = np.pad(c, width, mode="edge")
    model = hs.WaveModel.from_velocity(mesh, 2 * np.pi * c.min() * interior / ppw, c_full)
    return mesh, model


def fe9_fine(mesh, model):
    dim = mesh.dim
    h = float(mesh.spacing[0][0])
    op = _assemble_fe(mesh.spacing, [0.0] * dim, [axis_sigma_fn(mesh, a) for a in range(dim)],
                      [axis_gamma_fn(mesh, a) for a in range(dim)], model.omega, model.k,
                      None, hs.discretize.default_table(dim), h)
    return op.scaled(h ** (-dim), fe_scaled=False)


def point_rhs(mesh):
    f = np.zeros(mesh.unknowns, complex)
    idx = tuple(mesh.layers[a][0].width + mesh.interior_cells(a) // 2 for a in range(mesh.dim))
    f[idx] = (1.0 / mesh.spacing[0][0]) ** mesh.dim
    return f


def case_fixture(name, mesh, model, smoother, sweep, fine_op=None, solve=True, seed=7):
    rng = np.random.default_rng(seed)
    out = {}
    cycle, clevel = hs.build_two_grid(mesh, model, fine_op=fine_op, smoother=smoother,
                                      coarse="sweep", sweep=sweep)
    part = cycle.coarse_solver.prec.part
    out["fine_shape"] = np.array(cycle.fine_op.shape)
    out["coarse_shape"] = np.array(clevel.op.shape)
    out["omega"] = np.array(model.omega)
    out["k"] = model.k
    pack_op("fine_", cycle.fine_op, out)
    pack_op("coarse_", clevel.op, out)
    out["coarse_k"] = clevel.model.k
    out["coarse_k_cells"] = clevel.k_cells if clevel.k_cells is not None else np.zeros(0)
    out["beta"] = part.beta
    out["beta_tilde"] = part.beta_tilde
    out["slab_lo"] = np.array([s.pt_lo for s in part.subs])
    out["slab_hi"] = np.array([s.pt_hi for s in part.subs])
    out["slab_core"] = np.array([[s.core_lo, s.core_hi] for s in part.subs])
    for s in part.subs:
        pack_op(f"slab{s.j}_", s.op, out)
    _, cmap = hs.coarsen_mesh(mesh)
    for a in range(mesh.dim):
        out[f"fp{a}"] = cmap.fine_point_of_coarse[a]
        out[f"refined{a}"] = cmap.refined_cell[a]
    out["restrict_scale"] = np.array(cycle.restrict_scale)
    out["omega_jac"] = np.array(cycle.smoother.omega_jac)
    out["nu"] = np.array(cycle.smoother.nu)
    out["variant"] = np.array(sweep.variant)

    # kernel-level probes
    x = crand(rng, cycle.fine_op.shape)
    fvec = crand(rng, cycle.fine_op.shape)
    xc = crand(rng, clevel.op.shape)
    out["probe_x"], out["probe_f"], out["probe_xc"] = x, fvec, xc
    out["apply_fine"] = cycle.fine_op.apply(x)
    out["apply_coarse"] = clevel.op.apply(xc)
    out["jacobi2"] = hs.jacobi_smooth(cycle.fine_op, x, fvec, cycle.smoother.omega_jac, 2)
    out["restrict"] = (cycle.restrict_scale * (cycle.p_matrix.T @ fvec.ravel())).reshape(
        clevel.op.shape)
    out["prolong"] = (cycle.p_matrix @ xc.ravel()).reshape(cycle.fine_op.shape)
    out["sweep_x"] = hs.prec_x(part, xc)
    out["sweep_ud"] = hs.prec_ud(part, xc)
    z = crand(np.random.default_rng(0), cycle.fine_op.shape)
    out["tgsp_z"] = z
    out["tgsp_out"] = hs.tgsp_apply(cycle, z)
    if solve:
        f = point_rhs(mesh)
        out["rhs"] = f
        u, rep = hs.gmres(lambda v: cycle.fine_csr @ v, cycle.as_preconditioner(), f.ravel(),
                          hs.GmresConfig(tol=1e-6, max_iter=200, restart=20))
        out["gmres_u"] = u.reshape(mesh.unknowns)
        out["gmres_history"] = rep.residual_history
        out["gmres_iterations"] = np.array(rep.iterations)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: fine {cycle.fine_op.shape} coarse {clevel.op.shape} J={part.J}"
          + (f" its={out['gmres_iterations']}" if solve else ""))


def c1_anchors():
    """BASELINE configs[0] per SURVEY 8(d): anchors only (norms, samples, counts)."""
    size, width = 256, 16
    mesh = hs.build_mesh(2, size, 1.0 / size, AbsorbingLayerSpec(PML, width, 20.0, 1.0))
    model = hs.WaveModel.constant(mesh, 2 * np.pi * size / 10.0)
    mesh_c, _ = hs.coarsen_mesh(mesh)
    J = (mesh_c.unknowns[0] // 4) // 2 * 2
    f = np.zeros(mesh.unknowns, complex)
    c = width + 128 - 1
    f[c, c] = size**2.0
    res = {"J": J, "fine_shape": list(mesh.unknowns), "coarse_shape": list(mesh_c.unknowns)}
    for variant in ("x", "ud"):
        cycle, _ = hs.build_two_grid(mesh, model, smoother=SmootherConfig(0.8, 2),
                                     coarse="sweep",
                                     sweep=SweepOptions(5, 25.0, variant, subdomains=J))
        z = crand(np.random.default_rng(0), mesh.unknowns)
        t = hs.tgsp_apply(cycle, z)
        u, rep = hs.gmres(lambda v: cycle.fine_csr @ v, cycle.as_preconditioner(), f.ravel(),
                          hs.GmresConfig(tol=1e-6, max_iter=400, restart=20))
        true_res = np.linalg.norm(f.ravel() - cycle.fine_csr @ u) / np.linalg.norm(f)
        sel = np.arange(0, t.size, 997)
        res[variant] = {
            "tgsp_norm": float(np.linalg.norm(t)),
            "tgsp_sample_idx": sel.tolist(),
            "tgsp_sample_re": t.ravel()[sel].real.tolist(),
            "tgsp_sample_im": t.ravel()[sel].imag.tolist(),
            "iterations": int(rep.iterations),
            "history": [float(v) for v in rep.residual_history],
            "true_residual": float(true_res),
            "u_norm": float(np.linalg.norm(u)),
        }
        print(f"C1 {variant}: |tgsp(z)| = {res[variant]['tgsp_norm']:.12e} its={rep.iterations}")
    (OUT / "c1_anchors.json").write_text(json.dumps(res, indent=1))


def known_answers():
    """Known-answer vectors from the reference's own tests (small, exact)."""
    out = {}
    # tridiagonal hand solve (test_sparselin.py:44-47)
    diag = np.full(3, 2.0, complex)
    off = np.full(3, -1.0, complex)
    op = hs.StencilOperator((3,), {(0,): diag, (-1,): off, (1,): off})
    out["tridiag_solve"] = hs.factorize(op).solve(np.ones(3, complex))
    # prolongation midpoint (test_twogrid.py:68-73)
    cmap = hs.CoarseningMap((np.array([0, 2, 4]),), (np.array([True, True]),),
                            (np.array([0.5, 0.5]),))
    out["prolong_mid"] = hs.prolongate(cmap, np.array([1.0]))
    # fine_point_of_coarse by hand (test_mesh.py:64-68)
    mesh = hs.build_mesh(1, 6, 1.0 / 6, AbsorbingLayerSpec(PML, 1, 20.0))
    _, cm = hs.coarsen_mesh(mesh)
    out["fp_hand"] = cm.fine_point_of_coarse[0]
    # jacobi mode damping (test_twogrid.py:36-47)
    n, h, w = 64, 1.0 / 64, 0.8
    d = np.full(n - 1, 2 / h**2, complex)
    o = np.full(n - 1, -1 / h**2, complex)
    lap = hs.StencilOperator((n - 1,), {(0,): d, (-1,): o, (1,): o})
    v = np.sin(np.pi * 17 * np.arange(1, n) * h).astype(complex)
    out["jacobi_mode_in"] = v
    out["jacobi_mode_out"] = hs.jacobi_smooth(lap, v, np.zeros(n - 1, complex), w, 1)
    np.savez_compressed(OUT / "known_answers.npz", **out)


NX_CUSTOM = ((-1, 3, 6, 9), (1, 5, 7))   # J = 8: empty forward / backward chains in both passes


def nx_fixture():
    """NX sweep (prec_nx, sweepdd.py:403-434) on a J = 8 wedge case: the TGSP
    cycle with NX(2) coarse sweeps plus raw prec_nx outputs for n_cell 1..4
    and a hand grouping whose cells have empty chains."""
    mesh, model = hetero_case(64, 8, 8.0, seed=5)
    case_fixture("nx2d", mesh, model, SmootherConfig(0.8, 2),
                 SweepOptions(5, 25.0, "nx", n_cell=2, subdomains=8))
    path = OUT / "nx2d.npz"
    d = dict(np.load(path))
    cycle, clevel = hs.build_two_grid(mesh, model, smoother=SmootherConfig(0.8, 2),
                                      coarse="sweep",
                                      sweep=SweepOptions(5, 25.0, "nx", n_cell=2, subdomains=8))
    part = cycle.coarse_solver.prec.part
    xc = d["probe_xc"]
    for nc in (1, 2, 3, 4):
        cells = hs.sweepdd.make_nx_cells(part.J, nc)
        d[f"nx{nc}_cells"] = np.array(cells.j_cell)
        d[f"nx{nc}_mid"] = np.array(cells.j_mid)
        d[f"sweep_nx{nc}"] = hs.sweepdd.prec_nx(part, xc, cells)
    cells = hs.sweepdd.NxCells(*NX_CUSTOM)
    d["nxc_cells"] = np.array(cells.j_cell)
    d["nxc_mid"] = np.array(cells.j_mid)
    d["sweep_nxc"] = hs.sweepdd.prec_nx(part, xc, cells)
    np.savez_compressed(path, **d)
    print("nx2d: n_cell 1..4 + custom grouping")


def exact_fixture():
    """Exact coarse solve (ExactCoarseSolver, factorize / SuperLU): a 2-D
    two-grid cycle with coarse="exact" (vcycle + GMRES) and factorize().solve
    on the 2-D and 3-D coarse operators and a 1-D operator."""
    out = {}
    rng = np.random.default_rng(11)
    mesh, model = constant_case(2, 32, AbsorbingLayerSpec(PML, 4, 20.0), 10.0)
    cycle, clevel = hs.build_two_grid(mesh, model, smoother=SmootherConfig(0.8, 2),
                                      coarse="exact")
    pack_op("fine_", cycle.fine_op, out)
    pack_op("coarse_", clevel.op, out)
    out["fine_shape"] = np.array(cycle.fine_op.shape)
    out["coarse_shape"] = np.array(clevel.op.shape)
    _, cmap = hs.coarsen_mesh(mesh)
    for a in range(mesh.dim):
        out[f"fp{a}"] = cmap.fine_point_of_coarse[a]
        out[f"refined{a}"] = cmap.refined_cell[a]
    out["restrict_scale"] = np.array(cycle.restrict_scale)
    out["omega_jac"] = np.array(cycle.smoother.omega_jac)
    out["nu"] = np.array(cycle.smoother.nu)
    z = crand(np.random.default_rng(0), cycle.fine_op.shape)
    out["vcycle_z"] = z
    out["vcycle_out"] = cycle.vcycle(z)
    b = crand(rng, clevel.op.n)
    out["coarse_b"] = b
    out["coarse_x"] = hs.factorize(clevel.op).solve(b)
    f = point_rhs(mesh)
    out["rhs"] = f
    u, rep = hs.gmres(lambda v: cycle.fine_csr @ v, cycle.as_preconditioner(), f.ravel(),
                      hs.GmresConfig(tol=1e-6, max_iter=200, restart=20))
    out["gmres_u"] = u.reshape(mesh.unknowns)
    out["gmres_history"] = rep.residual_history
    out["gmres_iterations"] = np.array(rep.iterations)
    # 3-D coarse operator (pml3d recipe) and a 1-D PML operator
    mesh3, model3 = constant_case(3, 8, AbsorbingLayerSpec(PML, 3, 15.0), 6.0)
    _, cl3 = hs.build_two_grid(mesh3, model3, smoother=SmootherConfig(0.6, 2), coarse="exact")
    pack_op("c3_", cl3.op, out)
    out["c3_shape"] = np.array(cl3.op.shape)
    b3 = crand(rng, cl3.op.n)
    out["c3_b"] = b3
    out["c3_x"] = hs.factorize(cl3.op).solve(b3)
    mesh1 = hs.build_mesh(1, 64, 1.0 / 64, AbsorbingLayerSpec(PML, 8, 20.0))
    op1 = hs.assemble_fine(mesh1, hs.WaveModel.constant(mesh1, 2 * np.pi * 64 / 10.0))
    pack_op("l1_", op1, out)
    out["l1_shape"] = np.array(op1.shape)
    b1 = crand(rng, op1.n)
    out["l1_b"] = b1
    out["l1_x"] = hs.factorize(op1).solve(b1)
    np.savez_compressed(OUT / "exact2d.npz", **out)
    print(f"exact2d: coarse {clevel.op.shape} its={rep.iterations}; 3-D coarse {cl3.op.shape}; "
          f"1-D {op1.shape}")


def harness_fixture():
    """Reference file formats (cli.py:83-143): bytes of save_field, a velocity
    file read by load_model, and a results CSV written by write_rows."""
    import tempfile
    from helmsweep import cli
    out = {}
    rng = np.random.default_rng(21)
    u = crand(rng, (5, 4, 3))
    out["field_u"] = u
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "u.bin"
        cli.save_field(p, u)
        out["field_bytes"] = np.frombuffer(p.read_bytes(), dtype=np.uint8)
        vel = (1.0 + rng.random(6 * 7)).astype("<f4")
        vp = Path(td) / "v.bin"
        vel.tofile(vp)
        out["model_raw"] = np.frombuffer(vp.read_bytes(), dtype=np.uint8)
        out["model_loaded"] = cli.load_model(vp, (6, 7))
        rows = [cli.ResultRow("k1", "constant", 2, 64, 6.4, "pml", "tg-sweep", "x", 5, 6, "",
                              12, True, 7.5e-7, 0.1234567890123, 1.0 / 3.0, "k1.csv"),
                cli.ResultRow("k2", "wedge", 3, 32, 3.2, "sponge", "sweep-only", "nx", 3, 4, 7,
                              40, False, 2.5e-3, 10.0, 2.0 ** -40, "k2.csv")]
        cp = Path(td) / "r.csv"
        cli.write_rows(cp, rows)
        out["csv_bytes"] = np.frombuffer(cp.read_bytes(), dtype=np.uint8)
    np.savez_compressed(OUT / "harness.npz", **out)
    print("harness: field / model / csv bytes")


def main():
    if sys.argv[1:] == ["harness"]:
        harness_fixture()
        return
    if sys.argv[1:] == ["nx"]:
        nx_fixture()
        return
    if sys.argv[1:] == ["exact"]:
        exact_fixture()
        return
    sm2 = SmootherConfig(0.8, 2)
    mesh, model = constant_case(2, 32, AbsorbingLayerSpec(PML, 4, 20.0), 10.0)
    case_fixture("pml2d", mesh, model, sm2, SweepOptions(3, 15.0, "x", subdomains=4))
    mesh, model = hetero_case(48, 8, 8.0, seed=3)
    case_fixture("wedge2d", mesh, model, sm2, SweepOptions(5, 25.0, "x", subdomains=6))
    mesh, model = constant_case(2, 40, AbsorbingLayerSpec(SPONGE, 8, 1.0), 10.0)
    case_fixture("sponge2d", mesh, model, SmootherConfig(0.8, 3),
                 SweepOptions(4, 20.0, "ud", subdomains=4))
    mesh, model = hetero_case(48, 8, 8.0, seed=4)
    case_fixture("fe9_2d", mesh, model, sm2, SweepOptions(5, 25.0, "x", subdomains=6),
                 fine_op=fe9_fine(mesh, model), solve=False)
    mesh, model = constant_case(3, 8, AbsorbingLayerSpec(PML, 3, 15.0), 6.0)
    case_fixture("pml3d", mesh, model, SmootherConfig(0.6, 2),
                 SweepOptions(3, 15.0, "x", subdomains=2), solve=False)
    mesh, model = constant_case(3, 16, AbsorbingLayerSpec(PML, 3, 15.0), 8.0)
    case_fixture("pml3d_s", mesh, model, SmootherConfig(0.6, 2),
                 SweepOptions(3, 15.0, "x", subdomains=4))
    known_answers()
    c1_anchors()
    nx_fixture()
    exact_fixture()
    harness_fixture()


if __name__ == "__main__":
    main()
