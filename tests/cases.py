"""The golden cases rebuilt through this package's API (same recipes as
tests/golden/make_golden.py, which ran them through the reference)."""

import numpy as np

import paper_1412_0464_b200 as hb
from paper_1412_0464_b200.configs import fe_fine_operator
from paper_1412_0464_b200.mesh import PML, SPONGE, AbsorbingLayerSpec


def constant_case(dim, interior, layer, ppw):
    h = 1.0 / interior
    mesh = hb.build_mesh(dim, interior, h, layer)
    model = hb.WaveModel.constant(mesh, 2 * np.pi * interior / ppw)
    return mesh, model


def hetero_case(interior, width, ppw, seed):
    h = 1.0 / interior
    mesh = hb.build_mesh(2, interior, h, AbsorbingLayerSpec(PML, width, 20.0, 2.0))
    rng = np.random.default_rng(seed)
    x = np.arange(1, interior) * h
    xx, yy = np.meshgrid(x, x, indexing="ij")
    c = np.where(yy < 0.4 + 0.2 * xx, 1.0, np.where(yy < 0.75 - 0.15 * xx, 1.5, 2.0))
    c = c * (1.0 + 0.05 * rng.random(c.shape))
    c_full = np.pad(c, width, mode="edge")
    model = hb.WaveModel.from_velocity(mesh, 2 * np.pi * c.min() * interior / ppw, c_full)
    return mesh, model


def case(name):
    """-> (mesh, model, fine_op or None, SmootherConfig, SweepOptions)"""
    if name == "pml2d":
        mesh, model = constant_case(2, 32, AbsorbingLayerSpec(PML, 4, 20.0), 10.0)
        return mesh, model, None, hb.SmootherConfig(0.8, 2), hb.SweepOptions(3, 15.0, "x",
                                                                             subdomains=4)
    if name == "wedge2d":
        mesh, model = hetero_case(48, 8, 8.0, seed=3)
        return mesh, model, None, hb.SmootherConfig(0.8, 2), hb.SweepOptions(5, 25.0, "x",
                                                                             subdomains=6)
    if name == "sponge2d":
        mesh, model = constant_case(2, 40, AbsorbingLayerSpec(SPONGE, 8, 1.0), 10.0)
        return mesh, model, None, hb.SmootherConfig(0.8, 3), hb.SweepOptions(4, 20.0, "ud",
                                                                             subdomains=4)
    if name == "fe9_2d":
        mesh, model = hetero_case(48, 8, 8.0, seed=4)
        return (mesh, model, fe_fine_operator(mesh, model), hb.SmootherConfig(0.8, 2),
                hb.SweepOptions(5, 25.0, "x", subdomains=6))
    if name == "pml3d":
        mesh, model = constant_case(3, 8, AbsorbingLayerSpec(PML, 3, 15.0), 6.0)
        return mesh, model, None, hb.SmootherConfig(0.6, 2), hb.SweepOptions(3, 15.0, "x",
                                                                             subdomains=2)
    if name == "pml3d_s":
        mesh, model = constant_case(3, 16, AbsorbingLayerSpec(PML, 3, 15.0), 8.0)
        return mesh, model, None, hb.SmootherConfig(0.6, 2), hb.SweepOptions(3, 15.0, "x",
                                                                             subdomains=4)
    if name == "nx2d":
        mesh, model = hetero_case(64, 8, 8.0, seed=5)
        return mesh, model, None, hb.SmootherConfig(0.8, 2), hb.SweepOptions(
            5, 25.0, "nx", n_cell=2, subdomains=8)
    raise KeyError(name)


def hierarchy(name, device=False):
    mesh, model, fine_op, sm, sw = case(name)
    return hb.build_hierarchy(mesh, model, fine_op, sm, sw, device=device)


def point_rhs(mesh):
    f = np.zeros(mesh.unknowns, complex)
    idx = tuple(mesh.layers[a][0].width + mesh.interior_cells(a) // 2 for a in range(mesh.dim))
    f[idx] = (1.0 / mesh.spacing[0][0]) ** mesh.dim
    return f
