"""The 1-D line (robin_level_1d) and factorize() of general sparse matrices:
the reference's line known-answer tests (test_sweepdd.py:192-210,
test_acceptance.py:52-71) and SuperLU solves (sparselin.py:40-68), against
golden vectors made by running the reference (tests/golden/make_line1d.py).

CPU: operator coefficients (bitwise), partition geometry, dense transmission
matrices.  GPU (through the C ABI): UD/X sweeps on the line vs the
reference's outputs (1e-10) and the line exactness property (residual
< 1e-10), general-matrix factorisations vs SuperLU (1e-10), zero pivots.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN, crand, rel

LINES = ["a", "b", "c", "d"]


@pytest.fixture(scope="module")
def g():
    with np.load(GOLDEN / "line1d.npz") as z:
        return {k: z[k] for k in z.files}


def _part(g, key, device=True):
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.sweepdd import build_partition
    n, J, tr = (int(v) for v in g[f"{key}_meta"])
    level = hb.robin_level_1d(float(g[f"{key}_k"]), 1.0 / n, n)
    return level, build_partition(level, J=J, tilde_right=bool(tr), device=device)


@pytest.mark.parametrize("key", LINES)
def test_line_setup_matches_reference(g, key):
    level, part = _part(g, key, device=False)
    for o in (-1, 0, 1):
        assert np.array_equal(level.op.coeffs[(o,)], g[f"{key}_op{o:+d}"])
    assert np.array_equal(part.beta, g[f"{key}_beta"])
    assert np.array_equal(part.beta_tilde, g[f"{key}_beta_tilde"])
    assert np.array_equal([[s.pt_lo, s.pt_hi] for s in part.subs], g[f"{key}_lohi"])
    import paper_1412_0464_b200 as hb
    assert np.array_equal(hb.extract_transmission(part, 2, "forward").dense(), g[f"{key}_tfwd2"])
    assert np.array_equal(hb.extract_transmission(part, 1, "backward").dense(), g[f"{key}_tbwd1"])


def test_line_transmission_known_answer():
    """test_sweepdd.py:68-77: forward block [[0, -1/h^2], [1/h^2, 0]], backward = -forward"""
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.sweepdd import build_partition
    n = 40
    level = hb.robin_level_1d(2 * np.pi * 4, 1.0 / n, n)
    part = build_partition(level, J=2, device=False)
    d = hb.extract_transmission(part, 2, "forward").dense()
    a01 = -(n * n)
    assert np.allclose(d, [[0, a01], [-a01, 0]])
    assert np.allclose(hb.extract_transmission(part, 1, "backward").dense(), -d)


def test_robin1d_operator_errors():
    import paper_1412_0464_b200 as hb
    with pytest.raises(ValueError, match="at least 2"):
        hb.robin1d_operator(1.0, 0.1, 1)
    with pytest.raises(ValueError, match="cannot carry"):
        hb.robin1d_operator(30.0, 0.1, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("key", LINES)
def test_line_sweeps_match_reference(g, key):
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.sparselin import to_csr
    level, part = _part(g, key)
    f = g[f"{key}_f"]
    a = to_csr(level.op)
    ux = hb.SweepingPreconditioner(part, "x")(f)
    uud = hb.SweepingPreconditioner(part, "ud")(f)
    assert rel(ux, g[f"{key}_ux"]) < 1e-10
    assert rel(uud, g[f"{key}_uud"]) < 1e-10
    # the line is exact for constant k (test_sweepdd.py:194-210)
    for u in (ux, uud):
        assert np.linalg.norm(f - a @ u) / np.linalg.norm(f) < 1e-10


@pytest.mark.gpu
def test_line_subdom_solve_and_transmission_apply(g):
    """public slab solve on the line + TransmissionMatrix.apply vs its dense form"""
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.sweepdd import forward_sweep, subdom_solve
    level, part = _part(g, "d")
    rng = np.random.default_rng(5)
    f = crand(rng, part.shape)
    u1 = np.zeros(part.shape, complex)
    forward_sweep(part, u1, f, 1, 1)
    u2 = np.zeros(part.shape, complex)
    subdom_solve(part, u2, f, 1, part.beta[0], part.beta[1], part.beta[0], part.beta[1])
    assert np.array_equal(u1, u2)
    assert u1[part.beta[1]:].any() == False  # noqa: E712  (locality)
    t = hb.extract_transmission(part, 3, "forward")
    buf = crand(rng, (2,))
    assert rel(t.apply(buf), t.dense() @ buf) < 1e-14


def _csr(g, p):
    a = sp.csr_matrix((g[p + "_data"], g[p + "_indices"], g[p + "_indptr"]))
    return a


@pytest.mark.gpu
def test_factorize_scipy_matrices_match_superlu(g):
    import paper_1412_0464_b200 as hb
    a = _csr(g, "fine")
    x = hb.factorize(a).solve(g["fine_b"])
    assert rel(x, g["fine_x"]) < 1e-10
    assert np.linalg.norm(a @ x - g["fine_b"]) / np.linalg.norm(g["fine_b"]) < 1e-10
    band = _csr(g, "band")
    xb = hb.solve_factored(hb.factorize(band), g["band_b"])
    assert rel(xb, g["band_x"]) < 1e-10


@pytest.mark.gpu
def test_factorize_scipy_known_answers():
    """test_sparselin.py:39-62: scalar, hand-solved tridiagonal, zero pivot"""
    import paper_1412_0464_b200 as hb
    f = hb.factorize(sp.csc_matrix(np.array([[2.0 + 0j]])))
    assert abs(f.solve(np.array([4.0 + 0j]))[0] - 2.0) < 1e-15
    tri = sp.diags([[-1.0] * 2, [2.0] * 3, [-1.0] * 2], [-1, 0, 1], format="csc")
    assert np.allclose(hb.factorize(tri).solve(np.ones(3, complex)), [1.5, 2.0, 1.5])
    with pytest.raises(ZeroDivisionError, match="zero pivot"):
        hb.factorize(sp.csc_matrix(np.array([[1.0, 1.0], [1.0, 1.0]], dtype=complex)))
    with pytest.raises(ValueError):
        hb.factorize(tri).solve(np.ones(4, complex))


@pytest.mark.gpu
def test_dense_solve_checker():
    import paper_1412_0464_b200 as hb
    op = hb.StencilOperator((3,), {(0,): np.ones(3)})
    assert np.allclose(hb.dense_solve(op, np.arange(3.0) + 0j), np.arange(3.0))
    big = hb.StencilOperator((101, 101), {(0, 0): np.ones((101, 101))})
    with pytest.raises(ValueError, match="capped"):
        hb.dense_solve(big, np.zeros(big.n))


@pytest.mark.gpu
def test_explicit_matrix_cycle(rng):
    """TwoGridCycle built from an explicit prolongation matrix (the reference's
    constructor, test_twogrid.py:104-118): identity P with the exact coarse
    solve is an exact solve; the tent matrix of a CoarseningMap gives the
    same cycle as the tent tables (1e-13)."""
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.mesh import PML, AbsorbingLayerSpec
    from paper_1412_0464_b200.sparselin import to_csr
    from paper_1412_0464_b200.twogrid import ExactCoarseSolver, TwoGridCycle
    mesh = hb.build_mesh(2, 12, 1 / 12, None)
    model = hb.WaveModel.constant(mesh, 2 * np.pi * 12 / 10.0)
    op = hb.assemble_fine(mesh, model)
    cyc = TwoGridCycle(op, op, sp.identity(op.n, format="csr"), hb.SmootherConfig(0.8, 0),
                       ExactCoarseSolver(hb.factorize(op), op.shape), restrict_scale=1.0)
    f = crand(rng, op.shape)
    u = cyc.vcycle(f)
    a = to_csr(op)
    assert np.linalg.norm(a @ u.ravel() - f.ravel()) < 1e-10 * np.linalg.norm(f)
    # explicit tent matrix == tent tables
    mesh = hb.build_mesh(2, 32, 1 / 32, AbsorbingLayerSpec(PML, 4, 20.0))
    model = hb.WaveModel.constant(mesh, 2 * np.pi * 32 / 10.0)
    cycle, _ = hb.build_two_grid(mesh, model, smoother=hb.SmootherConfig(0.8, 2), coarse="exact")
    gen = TwoGridCycle(cycle.fine_op, cycle.coarse_op, cycle.p_matrix, cycle.smoother,
                       cycle.coarse_solver, restrict_scale=cycle.restrict_scale)
    f = crand(rng, mesh.unknowns)
    assert rel(gen.vcycle(f), cycle.vcycle(f)) < 1e-13


@pytest.mark.gpu
def test_gmres_with_host_callables(rng):
    """gmres with numpy callables (the reference's contract, test_krylov.py):
    the operator runs on the host, the Krylov arithmetic on the device"""
    import paper_1412_0464_b200 as hb
    d = np.array([1.0] * 10 + [3.0] * 10, dtype=complex)
    b = crand(rng, 20)
    u, rep = hb.gmres(lambda v: d * v, None, b, hb.GmresConfig(tol=1e-12))
    assert rep.iterations == 2 and rep.converged and isinstance(u, np.ndarray)
    n = 60
    a = np.diag(np.linspace(1, 4, n)) + 0.1 * rng.standard_normal((n, n))
    bb = rng.standard_normal(n) + 0j
    u, rep = hb.gmres(lambda v: a @ v, None, bb, hb.GmresConfig(tol=1e-12, max_iter=n))
    assert np.linalg.norm(a @ u - bb) / np.linalg.norm(bb) < 1e-10
    assert np.all(np.diff(rep.residual_history) <= 1e-14)


@pytest.mark.gpu
def test_relay_plan_equals_x_sweep():
    """the X plan cut at sweep-axis shard boundaries (hs_sweep_plan_relay,
    the relay's critical path) gives the X sweep's result (bitwise with one
    face segment; with the two-level partition a front's first task after a
    cut reads its trace from global memory instead of the level-2 edge
    values: equal to rounding)"""
    import torch
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.configs import config
    from paper_1412_0464_b200.device import empty, ptr, to_device
    p = config(0)
    hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                            hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains))
    sw = hh.partition.device()
    f, _ = to_device(crand(np.random.default_rng(3), sw.n), sw.n)
    ux = sw.apply(f, "x")[0]
    for g in (2, 3, 8):
        u = sw.apply(f, sw.relay_variant(g))[0]
        if sw.segments == 1:
            assert torch.equal(u, ux), g
        else:
            assert float(torch.linalg.norm(u - ux) / torch.linalg.norm(ux)) < 1e-12, g
        assert sw.ctx.lib.hs_sweep_plan_launches(sw.h, sw.relay_variant(g)) >= \
            sw.ctx.lib.hs_sweep_plan_launches(sw.h, sw.variant_id("x")) + (g > 2)
    p = config(1)
    hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                            hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains))
    sw = hh.partition.device()
    f, _ = to_device(crand(np.random.default_rng(4), sw.n), sw.n)
    ux = sw.apply(f, "x")[0]
    for g in (2, 4):
        u = sw.apply(f, sw.relay_variant(g))[0]
        assert float(torch.linalg.norm(u - ux) / torch.linalg.norm(ux)) < 1e-12, g


@pytest.mark.gpu
@pytest.mark.parametrize("n", [7, 33, 300, 1000])
def test_dense_pivoted_factorisation(n):
    """the hand-written batched dense kernels (hs_dense.cu: panel LU with
    partial pivoting, trailing GEMM, blocked triangular inverse) through
    factorize() of a dense random matrix whose diagonal is tiny (pivoting is
    required), against numpy's LAPACK solve"""
    import paper_1412_0464_b200 as hb
    rng = np.random.default_rng(n)
    a = crand(rng, (n, n))
    a[np.diag_indices(n)] *= 1e-8
    b = crand(rng, (n, 2))
    x = hb.solve_factored(hb.factorize(sp.csr_matrix(a)), b)
    ref = np.linalg.solve(a, b)
    assert rel(x, ref) < 1e-10
