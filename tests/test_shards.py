"""Sweep-axis sharding of the TGSP-GMRES solve (paper_1412_0464_b200/shards.py).

CPU: the shard geometry, and the sharded V-cycle / GMRES orchestration driven
over LocalComm (3 shards in-process) and over DistComm on a world_size-2
gloo group, with a numpy checker backend built on the oracle's operators --
against the oracle's single-domain cycle and solve.
GPU: the same orchestration with the CUDA backend (windowed stencils and
transfer maps) on G logical shards of one device, against the single-domain
GPU cycle and solve.
"""

import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import crand, rel
from cases import case, hierarchy, point_rhs

ROOT = Path(__file__).resolve().parents[1]


class NumpyShardBackend:
    """Checker backend: torch CPU tensors, numpy arithmetic through the
    oracle's stencil operators restricted to each shard's window."""

    def __init__(self, hh, plans, local):
        import torch
        from oracle import tgsp_oracle as orc
        self.torch = torch
        self.plans, self.local = plans, list(local)
        self.tg = orc.from_hierarchy(hh)
        offs = sorted(hh.fine_op.coeffs)
        self.fine = {}
        for g in self.local:
            p = plans[g]
            shape = (p.win_hi - p.win_lo,) + tuple(hh.fine_op.shape[1:])
            self.fine[g] = orc.Op(offs, [np.asarray(hh.fine_op.coeffs[o])
                                         .reshape(p.n0, p.row)[p.win_lo:p.win_hi].reshape(shape)
                                         for o in offs])
        self.fshape = hh.fine_op.shape
        self.cshape = hh.coarse_op.shape
        self.nc = int(np.prod(self.cshape))
        self.omega = float(hh.smoother.omega_jac)
        self.nu = int(hh.smoother.nu)
        self.scale = float(hh.restrict_scale)
        self.variant = hh.sweep.variant

    def _t(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a, dtype=complex))

    def zeros(self, g):
        return self.torch.zeros(self.plans[g].n_win, dtype=self.torch.complex128)

    def zeros_coarse(self):
        return self.torch.zeros(self.nc, dtype=self.torch.complex128)

    def small(self, n):
        return self.torch.zeros(n, dtype=self.torch.complex128)

    def basis(self, g, rows):
        return self.torch.zeros((rows, self.plans[g].n_win), dtype=self.torch.complex128)

    def to_host(self, t):
        return t.numpy().copy()

    def from_host(self, a):
        return self._t(a)

    def jacobi(self, g, u, f, steps, from_zero):
        from oracle import tgsp_oracle as orc
        op = self.fine[g]
        u0 = np.zeros(op.shape, complex) if from_zero else u.numpy().reshape(op.shape)
        u.copy_(self._t(orc.jacobi(op, u0, f.numpy().reshape(op.shape), self.omega, steps)
                        .reshape(-1)))

    def residual(self, g, f, u, out):
        op = self.fine[g]
        out.copy_(self._t(f.numpy() - op.apply(u.numpy()).reshape(-1)))

    def apply(self, g, x, out):
        out.copy_(self._t(self.fine[g].apply(x.numpy()).reshape(-1)))

    def restrict(self, g, r, rc):
        p = self.plans[g]
        full = np.zeros((p.n0, p.row), complex)
        full[p.win_lo:p.win_hi] = r.numpy().reshape(-1, p.row)
        rcf = (self.scale * (self.tg.p.T @ full.ravel())).reshape(p.nc0, p.crow)
        rc.numpy().reshape(p.nc0, p.crow)[p.c_lo:p.c_hi] = rcf[p.c_lo:p.c_hi]

    def prolong_add(self, g, uc, u):
        p = self.plans[g]
        pu = (self.tg.p @ uc.numpy()).reshape(p.n0, p.row)
        u.numpy()[p.own_slice] += pu[p.own_lo:p.own_hi].ravel()

    def coarse_solve(self, rc, uc):
        uc.copy_(self._t(self.tg.part.apply(rc.numpy().reshape(self.cshape), self.variant)
                         .reshape(-1)))

    def dots(self, g, V, k, w, out):
        s = self.plans[g].own_slice
        wv = w.numpy()[s]
        vals = [np.vdot(V[i].numpy()[s], wv) for i in range(k)] + [np.vdot(wv, wv)]
        out.copy_(self._t(vals))

    def update(self, g, V, k, h, w, out):
        s = self.plans[g].own_slice
        wv = w.numpy()
        hv = h.numpy()
        for i in range(k):
            wv[s] -= hv[i] * V[i].numpy()[s]
        out.copy_(self._t([np.vdot(wv[s], wv[s])]))

    def norm2(self, g, x, out):
        s = self.plans[g].own_slice
        xv = x.numpy()[s]
        out.copy_(self._t([np.vdot(xv, xv)]))

    def scale_(self, g, x, a):
        x.numpy()[:] *= a

    def lincomb(self, g, V, k, y, out):
        acc = np.zeros(out.shape[0], complex)
        for i in range(k):
            acc += y.numpy()[i] * V[i].numpy()
        out.copy_(self._t(acc))

    def axpby(self, g, a, x, b, y):
        y.copy_(self._t(a * x.numpy() + b * y.numpy()))


# ---------------------------------------------------------------------------
def test_plan_geometry():
    from paper_1412_0464_b200.shards import plan_shards
    hh = hierarchy("wedge2d")
    for world in (1, 2, 3, 5):
        plans = plan_shards(hh.fine_op.shape, hh.cmap, world)
        n0 = hh.fine_op.shape[0]
        assert plans[0].own_lo == 0 and plans[-1].own_hi == n0
        for a, b in zip(plans, plans[1:]):
            assert a.own_hi == b.own_lo and a.c_hi == b.c_lo
            assert a.win_hi == a.own_hi + 1 and b.win_lo == b.own_lo - 1
        assert plans[0].c_lo == 0 and plans[-1].c_hi == plans[0].nc0
        fp = np.asarray(hh.cmap.fine_point_of_coarse[0])
        for p in plans:   # restricted coarse rows: fine centre owned, +-1 inside the window
            for I in range(p.c_lo, p.c_hi):
                assert p.own_lo <= fp[I + 1] - 1 < p.own_hi
                assert p.win_lo <= max(fp[I + 1] - 2, 0) and min(fp[I + 1], p.n0 - 1) < p.win_hi
    with pytest.raises(ValueError):
        plan_shards(hh.fine_op.shape, hh.cmap, hh.fine_op.shape[0])


def _local_setup(name, world):
    from paper_1412_0464_b200.shards import LocalComm, ShardedTGSP, plan_shards
    hh = hierarchy(name)
    plans = plan_shards(hh.fine_op.shape, hh.cmap, world)
    comm = LocalComm(plans)
    be = NumpyShardBackend(hh, plans, comm.local)
    return hh, plans, be, ShardedTGSP(plans, be, comm)


@pytest.mark.parametrize("name,world", [("wedge2d", 3), ("pml3d", 2)])
def test_local_shards_vcycle_matches_oracle(name, world):
    from paper_1412_0464_b200.shards import gather_rows, scatter_rows
    hh, plans, be, st = _local_setup(name, world)
    z = crand(np.random.default_rng(7), hh.fine_op.shape)
    f = {g: be.from_host(scatter_rows(plans[g], z)) for g in st.local}
    u = {g: be.zeros(g) for g in st.local}
    st.vcycle(f, u)
    out = gather_rows(plans, [u[g].numpy() for g in st.local])
    assert rel(out, be.tg.vcycle(z)) < 1e-12


def test_local_shards_gmres_matches_oracle():
    import paper_1412_0464_b200 as hb
    from oracle import tgsp_oracle as orc
    from paper_1412_0464_b200.shards import gather_rows, scatter_rows
    hh, plans, be, st = _local_setup("wedge2d", 3)
    fh = point_rhs(case("wedge2d")[0])
    f = {g: be.from_host(scatter_rows(plans[g], fh)) for g in st.local}
    u, rep = st.gmres(f, hb.GmresConfig(1e-6, 100, 5))
    tg = be.tg
    _, its, _, _, _ = orc.gmres(lambda v: tg.fine.csr @ v, tg.as_preconditioner(), fh.ravel(),
                                tol=1e-6, max_iter=100, restart=5)
    assert rep.converged and abs(rep.iterations - its) <= 1
    uf = gather_rows(plans, [u[g].numpy() for g in st.local])
    assert np.linalg.norm(fh.ravel() - tg.fine.csr @ uf) / np.linalg.norm(fh) <= 1e-6


# ---------------------------------------------------------------------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.shards import DistComm, ShardedTGSP, plan_shards, scatter_rows
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hh = hierarchy("wedge2d")
    plans = plan_shards(hh.fine_op.shape, hh.cmap, world)
    comm = DistComm(plans, rank)
    be = NumpyShardBackend(hh, plans, comm.local)
    st = ShardedTGSP(plans, be, comm)
    z = crand(np.random.default_rng(7), hh.fine_op.shape)
    f = {rank: be.from_host(scatter_rows(plans[rank], z))}
    u = {rank: be.zeros(rank)}
    st.vcycle(f, u)
    fh = point_rhs(case("wedge2d")[0])
    fs = {rank: be.from_host(scatter_rows(plans[rank], fh))}
    us, rep = st.gmres(fs, hb.GmresConfig(1e-6, 100, 5))
    p = plans[rank]
    np.savez(Path(out_dir, f"r{rank}.npz"), v=u[rank].numpy()[p.own_slice],
             s=us[rank].numpy()[p.own_slice], its=rep.iterations, conv=rep.converged,
             hist=rep.residual_history)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_shards_match_oracle(tmp_path):
    import torch.multiprocessing as mp
    from oracle import tgsp_oracle as orc
    world = 2
    mp.start_processes(_gloo_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    hh = hierarchy("wedge2d")
    tg = orc.from_hierarchy(hh)
    z = crand(np.random.default_rng(7), hh.fine_op.shape)
    v = np.concatenate([r["v"] for r in res])
    assert rel(v, tg.vcycle(z)) < 1e-12
    fh = point_rhs(case("wedge2d")[0])
    _, its, _, _, _ = orc.gmres(lambda x: tg.fine.csr @ x, tg.as_preconditioner(), fh.ravel(),
                                tol=1e-6, max_iter=100, restart=5)
    assert int(res[0]["its"]) == int(res[1]["its"])          # ranks agree
    assert np.array_equal(res[0]["hist"], res[1]["hist"])
    assert bool(res[0]["conv"]) and abs(int(res[0]["its"]) - its) <= 1
    s = np.concatenate([r["s"] for r in res])
    assert np.linalg.norm(fh.ravel() - tg.fine.csr @ s) / np.linalg.norm(fh) <= 1e-6


# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("wedge2d", 2), ("wedge2d", 3), ("pml3d_s", 2)])
def test_gpu_local_shards_match_single_domain(name, world):
    """CUDA backend on G logical shards of one device: sharded TGSP apply vs
    the single-domain cycle (1e-12), sharded GMRES vs single-domain GMRES."""
    import paper_1412_0464_b200 as hb
    from paper_1412_0464_b200.shards import (CudaShardBackend, LocalComm, ShardedTGSP,
                                             gather_rows, plan_shards, scatter_rows)
    mesh, model, fine_op, sm, sw = case(name)
    cycle, _ = hb.build_two_grid(mesh, model, fine_op=fine_op, smoother=sm, coarse="sweep",
                                 sweep=sw)
    hh = cycle.hierarchy
    plans = plan_shards(hh.fine_op.shape, hh.cmap, world)
    comm = LocalComm(plans)
    be = CudaShardBackend(hh, plans, comm.local)
    st = ShardedTGSP(plans, be, comm)
    z = crand(np.random.default_rng(11), hh.fine_op.shape)
    f = {g: be.upload(g, scatter_rows(plans[g], z)) for g in st.local}
    u = {g: be.zeros(g) for g in st.local}
    st.vcycle(f, u)
    out = gather_rows(plans, [be.download(u[g]) for g in st.local])
    assert rel(out, hb.tgsp_apply(cycle, z)) < 1e-12
    fh = point_rhs(mesh)
    fs = {g: be.upload(g, scatter_rows(plans[g], fh)) for g in st.local}
    us, rep = st.gmres(fs, hb.GmresConfig(1e-6, 200, 20))
    u1, rep1 = hb.gmres(cycle.fine_csr, cycle.as_preconditioner(), fh.ravel(),
                        hb.GmresConfig(1e-6, 200, 20))
    assert rep.converged and abs(rep.iterations - rep1.iterations) <= 1
    uf = gather_rows(plans, [be.download(us[g]) for g in st.local])
    assert np.linalg.norm(fh.ravel() - cycle.fine_csr @ uf) / np.linalg.norm(fh) <= 1e-6
