"""Pin the CPU oracle (oracle/tgsp_oracle.py) against vectors produced by the
reference itself (tests/golden/make_golden.py) and the reference's own
known-answer tests.  Runs on CPU."""

import numpy as np
import pytest

from conftest import CASES, NX_KEYS, SOLVED, c1_anchors, load_case, rel
from oracle import tgsp_oracle as orc


@pytest.fixture(scope="module", params=CASES)
def case(request):
    d = load_case(request.param)
    return request.param, d, orc.from_fixture(d)


def test_operator_applies(case):
    _, d, tg = case
    assert rel(tg.fine.apply(d["probe_x"]), d["apply_fine"]) < 1e-14
    assert rel(tg.part.op.apply(d["probe_xc"]), d["apply_coarse"]) < 1e-14
    # CSR and stencil forms agree (test_sparselin.py:28-36)
    assert rel(tg.fine.csr @ d["probe_x"].ravel(), d["apply_fine"].ravel()) < 1e-14


def test_jacobi(case):
    _, d, tg = case
    out = orc.jacobi(tg.fine, d["probe_x"], d["probe_f"], float(d["omega_jac"]), 2)
    assert rel(out, d["jacobi2"]) < 1e-13


def test_transfers(case):
    _, d, tg = case
    rc = float(d["restrict_scale"]) * (tg.p.T @ d["probe_f"].ravel())
    assert rel(rc, d["restrict"]) < 1e-14
    assert rel(tg.p @ d["probe_xc"].ravel(), d["prolong"]) < 1e-14


def test_sweeps(case):
    name, d, tg = case
    if tg.part.J % 2 == 0:
        ux = tg.part.prec_x(d["probe_xc"])
        assert rel(ux, d["sweep_x"]) < 1e-12
        tg.part.parallel = True    # two-thread X sweep (bench's CPU baseline): bitwise the serial
        try:
            assert np.array_equal(tg.part.prec_x(d["probe_xc"]), ux)
        finally:
            tg.part.parallel = False
    assert rel(tg.part.prec_ud(d["probe_xc"]), d["sweep_ud"]) < 1e-12
    for k in NX_KEYS:
        if f"sweep_{k}" in d:
            out = tg.part.prec_nx(d["probe_xc"], d[f"{k}_cells"], d[f"{k}_mid"])
            assert rel(out, d[f"sweep_{k}"]) < 1e-12, k


def test_nx_one_cell_is_x():
    """test_sweepdd.py:231-236: NX with one cell equals the X sweep."""
    d = load_case("nx2d")
    assert rel(d["sweep_nx1"], d["sweep_x"]) < 1e-14
    assert orc._nx_cells(8, 1) == (list(d["nx1_cells"]), list(d["nx1_mid"]))
    for n in (2, 3, 4):
        assert orc._nx_cells(8, n) == (list(d[f"nx{n}_cells"]), list(d[f"nx{n}_mid"]))


def test_tgsp_apply(case):
    _, d, tg = case
    assert rel(tg.vcycle(d["tgsp_z"]), d["tgsp_out"]) < 1e-12


@pytest.mark.parametrize("name", SOLVED)
def test_gmres_history(name):
    d = load_case(name)
    tg = orc.from_fixture(d)
    u, its, hist, conv, _ = orc.gmres(lambda v: tg.fine.csr @ v, tg.as_preconditioner(),
                                      d["rhs"].ravel(), tol=1e-6, max_iter=200, restart=20)
    assert its == int(d["gmres_iterations"]) and conv
    assert np.allclose(hist, d["gmres_history"], rtol=1e-8, atol=1e-14)
    assert rel(u, d["gmres_u"]) < 1e-9


def test_known_answers():
    ka = load_case("known_answers")
    # tridiagonal hand solve x = (1.5, 2, 1.5) (reference test_sparselin.py:44-47)
    op = orc.Op([(0,), (-1,), (1,)], [np.full(3, 2.0 + 0j), np.full(3, -1.0 + 0j),
                                       np.full(3, -1.0 + 0j)])
    import scipy.sparse.linalg as spla
    x = spla.splu(op.csr.tocsc()).solve(np.ones(3, complex))
    assert np.allclose(x, [1.5, 2.0, 1.5]) and np.allclose(x, ka["tridiag_solve"])
    # prolongation midpoint [0.5, 1, 0.5] (test_twogrid.py:68-73)
    p = orc.prolongation([np.array([0, 2, 4])], [np.array([True, True])])
    assert np.allclose(p @ np.array([1.0]), ka["prolong_mid"])
    # Jacobi mode damping 1 - w(1 - cos theta) (test_twogrid.py:36-47)
    n, h, w = 64, 1.0 / 64, 0.8
    lap = orc.Op([(0,), (-1,), (1,)], [np.full(n - 1, 2 / h**2, complex),
                                        np.full(n - 1, -1 / h**2, complex),
                                        np.full(n - 1, -1 / h**2, complex)])
    out = orc.jacobi(lap, ka["jacobi_mode_in"], np.zeros(n - 1, complex), w, 1)
    theta = np.pi * 17 * h
    assert np.abs(out - (1 - w * (1 - np.cos(theta))) * ka["jacobi_mode_in"]).max() < 1e-12
    assert rel(out, ka["jacobi_mode_out"]) < 1e-14


def test_oracle_zero_diagonal_error():
    op = orc.Op([(0,)], [np.array([1.0, 0.0, 1.0], complex)])
    with pytest.raises(ZeroDivisionError, match="1"):
        orc.jacobi(op, np.zeros(3, complex), np.ones(3, complex), 0.8, 1)


def test_oracle_gmres_small_known_answers(rng):
    # GMRES: identity -> 1 iteration; two eigenvalues -> 2 (test_krylov.py:9-21)
    b = rng.standard_normal(20) + 0j
    _, its, hist, conv, _ = orc.gmres(lambda v: v, None, b, tol=1e-10)
    assert its == 1 and conv and len(hist) == 2
    dd = np.array([1.0] * 10 + [3.0] * 10, dtype=complex)
    b = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    _, its, _, conv, _ = orc.gmres(lambda v: dd * v, None, b, tol=1e-12)
    assert its == 2 and conv


def test_c1_anchor_oracle():
    """BASELINE configs[0] through the package's host assembly + oracle:
    reproduces the reference's |tgsp_apply(z)| and GMRES iteration count."""
    from paper_1412_0464_b200.configs import config
    import paper_1412_0464_b200 as hb
    a = c1_anchors()
    p = config(0)
    hh = hb.build_hierarchy(p.mesh, p.model, None, hb.SmootherConfig(p.omega_jac, p.nu),
                            hb.SweepOptions(p.w_dd, p.s_dd, "x", subdomains=p.subdomains),
                            device=False)
    assert p.subdomains == a["J"]
    tg = orc.from_hierarchy(hh)
    z = np.random.default_rng(0).standard_normal(p.mesh.unknowns) \
        + 1j * np.random.default_rng(0).standard_normal(p.mesh.unknowns)
    rng = np.random.default_rng(0)
    z = rng.standard_normal(p.mesh.unknowns) + 1j * rng.standard_normal(p.mesh.unknowns)
    t = tg.vcycle(z)
    assert abs(np.linalg.norm(t) - a["x"]["tgsp_norm"]) <= 1e-12 * a["x"]["tgsp_norm"]
    idx = np.array(a["x"]["tgsp_sample_idx"])
    ref = np.array(a["x"]["tgsp_sample_re"]) + 1j * np.array(a["x"]["tgsp_sample_im"])
    assert np.abs(t.ravel()[idx] - ref).max() <= 1e-12 * np.abs(t).max()
    u, its, hist, conv, _ = orc.gmres(lambda v: tg.fine.csr @ v, tg.as_preconditioner(),
                                      p.f[0].ravel(), tol=1e-6, max_iter=400, restart=20)
    assert its == a["x"]["iterations"] and conv
    assert np.allclose(hist, a["x"]["history"], rtol=1e-8, atol=1e-14)


def test_exact_coarse_oracle():
    """Exact coarse solve (ExactCoarseSolver / factorize) vs the reference."""
    d = load_case("exact2d")
    tg = orc.from_exact_fixture(d)
    assert rel(tg.vcycle(d["vcycle_z"]), d["vcycle_out"]) < 1e-12
    assert rel(tg.part.solve(d["coarse_b"]), d["coarse_x"]) < 1e-12
    for p in ("c3", "l1"):
        ex = orc.Exact(orc.Op(d[f"{p}_offsets"], d[f"{p}_coeffs"]))
        assert rel(ex.solve(d[f"{p}_b"]), d[f"{p}_x"]) < 1e-12, p
    u, its, hist, conv, _ = orc.gmres(lambda v: tg.fine.csr @ v, tg.as_preconditioner(),
                                      d["rhs"].ravel(), tol=1e-6, max_iter=200, restart=20)
    assert its == int(d["gmres_iterations"]) and conv
    assert np.allclose(hist, d["gmres_history"], rtol=1e-8, atol=1e-14)
