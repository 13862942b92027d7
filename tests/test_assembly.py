"""Host-side assembly (setup) of this package vs the reference's coefficients
(golden fixtures produced by running the reference)."""

import numpy as np
import pytest

from conftest import CASES, load_case, rel
from cases import hierarchy


def _dict(d, prefix):
    offs = [tuple(int(v) for v in o) for o in d[prefix + "offsets"]]
    return dict(zip(offs, d[prefix + "coeffs"]))


def _check_op(op, ref, tol):
    assert set(op.coeffs) == set(ref)
    for off, c in ref.items():
        scale = np.abs(c).max() or 1.0
        assert np.abs(op.coeffs[off] - c).max() <= tol * scale, off


@pytest.mark.parametrize("name", CASES)
def test_hierarchy_matches_reference(name):
    d = load_case(name)
    hh = hierarchy(name)
    _check_op(hh.fine_op, _dict(d, "fine_"), 1e-15)
    _check_op(hh.coarse_op, _dict(d, "coarse_"), 1e-15)
    assert np.array_equal(hh.beta, d["beta"])
    assert np.array_equal(hh.beta_tilde, d["beta_tilde"])
    assert [lo for lo, _, _ in hh.slabs] == d["slab_lo"].tolist()
    assert [hi for _, hi, _ in hh.slabs] == d["slab_hi"].tolist()
    for j, (_, _, op) in enumerate(hh.slabs):
        _check_op(op, _dict(d, f"slab{j + 1}_"), 1e-15)
    for a in range(hh.mesh.dim):
        assert np.array_equal(hh.cmap.fine_point_of_coarse[a], d[f"fp{a}"])
        assert np.array_equal(hh.cmap.refined_cell[a], d[f"refined{a}"])
    assert hh.restrict_scale == pytest.approx(float(d["restrict_scale"]), rel=1e-15)
    assert np.allclose(hh.clevel.model.k, d["coarse_k"], rtol=1e-15, atol=0)
    if d["coarse_k_cells"].size:
        assert np.allclose(hh.clevel.k_cells, d["coarse_k_cells"], rtol=1e-15, atol=0)


def test_prolongation_matrix_matches_oracle():
    from oracle.tgsp_oracle import prolongation
    from paper_1412_0464_b200 import prolongation_matrix
    hh = hierarchy("pml2d")
    p1 = prolongation_matrix(hh.cmap)
    p2 = prolongation(hh.cmap.fine_point_of_coarse, hh.cmap.refined_cell)
    assert abs(p1 - p2).max() == 0
