"""Harness file formats (reference cli.py:83-143) against bytes the reference
itself wrote (tests/golden/harness.npz): field dumps, velocity ingestion,
results CSV."""

import numpy as np
import pytest

from conftest import load_case

from paper_1412_0464_b200 import harness as hz


def test_save_field_bytes_match_reference(tmp_path):
    d = load_case("harness")
    p = tmp_path / "u.bin"
    hz.save_field(p, d["field_u"])
    assert p.read_bytes() == d["field_bytes"].tobytes()
    back = hz.load_field(p, d["field_u"].shape)
    assert np.array_equal(back, d["field_u"])          # bit-exact round trip
    with pytest.raises(ValueError, match="wrong size"):
        hz.load_field(p, (5, 4, 4))


def test_load_model_matches_reference(tmp_path):
    d = load_case("harness")
    p = tmp_path / "v.bin"
    p.write_bytes(d["model_raw"].tobytes())
    v = hz.load_model(p, (6, 7))
    assert v.dtype == np.float64 and np.array_equal(v, d["model_loaded"])
    with pytest.raises(ValueError, match="samples"):
        hz.load_model(p, (6, 8))
    bad = np.frombuffer(d["model_raw"].tobytes(), dtype="<f4").copy()
    bad[5] = 0.0
    bad.tofile(p)
    with pytest.raises(ValueError, match="nonpositive velocity at flat index 5"):
        hz.load_model(p, (6, 7))


def test_results_csv_matches_reference(tmp_path):
    d = load_case("harness")
    rows = [hz.ResultRow("k1", "constant", 2, 64, 6.4, "pml", "tg-sweep", "x", 5, 6, "",
                         12, True, 7.5e-7, 0.1234567890123, 1.0 / 3.0, "k1.csv"),
            hz.ResultRow("k2", "wedge", 3, 32, 3.2, "sponge", "sweep-only", "nx", 3, 4, 7,
                         40, False, 2.5e-3, 10.0, 2.0 ** -40, "k2.csv")]
    p = tmp_path / "r.csv"
    hz.write_rows(p, rows)
    assert p.read_bytes() == d["csv_bytes"].tobytes()
    recs = hz.read_rows(p)
    assert recs[0]["iterations"] == 12 and recs[0]["converged"] is True
    assert recs[1]["solve_time"] == 2.0 ** -40 and recs[1]["converged"] is False
    hz.write_rows(p, rows[:1], append=True)
    assert len(hz.read_rows(p)) == 3


@pytest.mark.gpu
def test_save_field_from_device(tmp_path):
    import torch
    d = load_case("harness")
    p = tmp_path / "u.bin"
    hz.save_field(p, torch.from_numpy(d["field_u"]).cuda())
    assert p.read_bytes() == d["field_bytes"].tobytes()


def test_nx_cells_host_logic():
    """make_nx_cells / NxCells.validate (sweepdd.py:362-401) against the
    groupings the reference produced (nx2d.npz) and its error cases."""
    from conftest import NX_KEYS
    from paper_1412_0464_b200.sweepdd import NxCells, make_nx_cells
    d = load_case("nx2d")
    for n in (1, 2, 3, 4):
        c = make_nx_cells(8, n)
        assert list(c.j_cell) == list(d[f"nx{n}_cells"]) and list(c.j_mid) == list(d[f"nx{n}_mid"])
        assert c.n_cell == n
    NxCells(tuple(int(v) for v in d["nxc_cells"]), tuple(int(v) for v in d["nxc_mid"])).validate(8)
    assert "nxc" in NX_KEYS
    with pytest.raises(ValueError):
        make_nx_cells(8, 5)
    with pytest.raises(ValueError, match="sentinel|start at -1"):
        NxCells((0, 4, 9), (2, 6)).validate(8)
    with pytest.raises(ValueError, match="strictly increasing"):
        NxCells((-1, 4, 4, 9), (2, 3, 6)).validate(8)
    with pytest.raises(ValueError, match="meeting slab"):
        NxCells((-1, 4, 9), (5, 6)).validate(8)


def test_to_csr_matches_oracle():
    """sparselin.to_csr (sparselin.py:21-37) against the oracle's CSR of the
    same stencil (1-, 2- and 3-D, every compact offset, Dirichlet box)."""
    import itertools
    from oracle import tgsp_oracle as orc
    from paper_1412_0464_b200 import StencilOperator
    from paper_1412_0464_b200.sparselin import to_csr
    rng = np.random.default_rng(2)
    for shape in [(7,), (5, 6), (4, 5, 3)]:
        offs = list(itertools.product(*([(-1, 0, 1)] * len(shape))))
        co = {o: rng.standard_normal(shape) + 1j * rng.standard_normal(shape) for o in offs}
        a = to_csr(StencilOperator(shape, co))
        b = orc.stencil_csr(offs, [co[o] for o in offs], shape)
        assert abs(a - b).max() == 0 and a.nnz == b.nnz
