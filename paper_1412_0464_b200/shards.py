"""Sweep-axis (x-slab) decomposition of the TGSP-GMRES solve over ranks.

SURVEY 8(e): the fine level shards naturally along axis 0 (the sweep axis).
Shard g owns fine rows [own_lo, own_hi) and keeps them in a *window* buffer
with one halo plane on each interior side.  Per V-cycle (reference
``TwoGridCycle.vcycle``, twogrid.py:150-159):

1. halo(f); pre-smoothing from zero (the fused two-step kernel reads f and
   1/diag one plane across the boundary, so the owned rows are exact);
2. halo(u); r = f - A u on the owned rows;  halo(r);
3. restriction of the coarse rows whose fine centre this shard owns, into a
   full-size coarse vector; all-gather of the owned coarse rows;
4. coarse X/UD sweep (replicated on every rank -- see below);
5. prolongation + correction of the owned fine rows from the full coarse
   vector; post-smoothing, one halo(u) per step.

GMRES (krylov.py:46-146) runs on the owned rows with every dot/norm
all-reduced (k+1 complex values per Gram-Schmidt pass); the Givens rotations
run on every rank's host on identical values.

The coarse level is replicated, not relayed: the sweep is a sequential chain
(J+2 slab solves) whatever the sharding, the coarse factors of every BASELINE
config fit one B200 (C5: 57 GB of 180 GB), and a replicated sweep needs one
all-gather of the coarse right-hand side (C3: 70 MB) instead of 2 x J/G
trace hand-offs inside the chain.  DESIGN.md section 7 has the numbers.

The orchestration here is backend-agnostic (``backend`` provides the
per-shard kernels, ``comm`` the halo / all-reduce / all-gather transport):
the product pairs :class:`CudaShardBackend` (libhsweep kernels) with
:class:`DistComm` (torch.distributed over NCCL, one rank per GPU) or
:class:`LocalComm` (G logical shards of one process on one device, halos as
stream-ordered device copies).  ``tests/`` drives the same code over gloo on
the CPU with a numpy checker backend.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .krylov import _DGKS, _KCHUNK, GmresConfig, SolveReport, _givens_column


# ---------------------------------------------------------------------------
# geometry

@dataclass(frozen=True)
class ShardPlan:
    """One shard of the sweep-axis decomposition (global 0-based row indices)."""

    rank: int
    world: int
    n0: int            # fine rows (axis 0)
    row: int           # fine elements per row (prod(shape[1:]))
    own_lo: int
    own_hi: int
    win_lo: int        # window = owned rows + halo planes
    win_hi: int
    c_lo: int          # coarse rows restricted here (fine centre owned)
    c_hi: int
    nc0: int           # coarse rows
    crow: int          # coarse elements per row

    @property
    def n_win(self) -> int:
        return (self.win_hi - self.win_lo) * self.row

    @property
    def own_slice(self) -> slice:
        a = (self.own_lo - self.win_lo) * self.row
        return slice(a, a + (self.own_hi - self.own_lo) * self.row)

    @property
    def window(self) -> tuple:
        """hs_transfer_create_window's {fw_lo, fw_hi, cr_lo, cr_hi, fr_lo, fr_hi}."""
        return (self.win_lo, self.win_hi, self.c_lo, self.c_hi, self.own_lo, self.own_hi)

    def halo_rows(self):
        """(left, right): (window row to receive into, neighbour rank) or None."""
        left = (0, self.rank - 1) if self.win_lo < self.own_lo else None
        right = (self.win_hi - self.win_lo - 1, self.rank + 1) if self.win_hi > self.own_hi \
            else None
        return left, right

    def edge_rows(self):
        """(first owned window row, last owned window row)."""
        return self.own_lo - self.win_lo, self.own_hi - 1 - self.win_lo


def plan_shards(fine_shape, cmap, world: int) -> list:
    """Split axis 0 into ``world`` contiguous shards of (nearly) equal row
    counts; coarse row I belongs to the shard owning its fine centre
    (``fine_point_of_coarse[0][I+1] - 1``)."""
    n0 = int(fine_shape[0])
    row = int(np.prod(fine_shape[1:]))
    if world < 1 or world > n0 // 2:
        raise ValueError(f"cannot split {n0} rows over {world} shards (need >= 2 rows each)")
    fp = np.asarray(cmap.fine_point_of_coarse[0], dtype=np.int64)
    centres = fp[1:-1] - 1                      # coarse row I -> fine row
    nc0 = len(centres)
    crow = int(np.prod([len(f) - 2 for f in cmap.fine_point_of_coarse[1:]]))
    bounds = [round(g * n0 / world) for g in range(world + 1)]
    plans = []
    for g in range(world):
        lo, hi = bounds[g], bounds[g + 1]
        owned = np.flatnonzero((centres >= lo) & (centres < hi))
        c_lo = int(owned[0]) if owned.size else int(np.searchsorted(centres, lo))
        c_hi = int(owned[-1]) + 1 if owned.size else c_lo
        plans.append(ShardPlan(g, world, n0, row, lo, hi, max(lo - 1, 0), min(hi + 1, n0),
                               c_lo, c_hi, nc0, crow))
    return plans


def scatter_rows(plan: ShardPlan, x_full) -> np.ndarray:
    """Window buffer of ``plan`` from a full fine field (host helper)."""
    x = np.asarray(x_full, dtype=complex).reshape(plan.n0, plan.row)
    return np.ascontiguousarray(x[plan.win_lo:plan.win_hi]).reshape(-1)


def gather_rows(plans, wins) -> np.ndarray:
    """Full fine field (flat) from the owned rows of every shard (host helper)."""
    parts = []
    for p, w in zip(plans, wins):
        w = np.asarray(w).reshape(-1)
        parts.append(w[p.own_slice])
    return np.concatenate(parts)


# ---------------------------------------------------------------------------
# transports

class LocalComm:
    """G logical shards in one process: halo planes and reductions are
    stream-ordered device copies / sums (no kernel waits on another shard)."""

    def __init__(self, plans):
        self.plans = list(plans)
        self.local = list(range(len(self.plans)))

    def exchange(self, bufs: dict):
        for g in self.local:
            p = self.plans[g]
            left, right = p.halo_rows()
            for side in (left, right):
                if side is None:
                    continue
                dst_row, nb = side
                q = self.plans[nb]
                first, last = q.edge_rows()
                src_row = last if nb < g else first
                bufs[g][dst_row * p.row:(dst_row + 1) * p.row].copy_(
                    bufs[nb][src_row * q.row:(src_row + 1) * q.row])

    def allreduce(self, parts: dict):
        total = parts[self.local[0]].clone()
        for g in self.local[1:]:
            total += parts[g]
        for g in self.local:
            parts[g].copy_(total)

    def allgather_coarse(self, coarse: dict):
        for g in self.local:
            p = self.plans[g]
            a, b = p.c_lo * p.crow, p.c_hi * p.crow
            for h in self.local:
                if h != g:
                    coarse[h][a:b].copy_(coarse[g][a:b])


class DistComm:
    """One shard per process over torch.distributed (NCCL on GPUs, gloo on
    CPUs): halo planes by point-to-point send/recv, dots by all_reduce, the
    owned coarse rows by all_gather (padded to equal length)."""

    def __init__(self, plans, rank: int):
        import torch.distributed as dist
        self.dist = dist
        self.plans = list(plans)
        self.rank = rank
        self.local = [rank]
        self._pad = max(p.c_hi - p.c_lo for p in self.plans) * self.plans[0].crow

    def exchange(self, bufs: dict):
        dist = self.dist
        p = self.plans[self.rank]
        buf = bufs[self.rank]
        left, right = p.halo_rows()
        first, last = p.edge_rows()
        ops = []
        for side, src_row in ((left, first), (right, last)):
            if side is None:
                continue
            dst_row, nb = side
            ops.append(dist.P2POp(dist.isend, buf[src_row * p.row:(src_row + 1) * p.row], nb))
            ops.append(dist.P2POp(dist.irecv, buf[dst_row * p.row:(dst_row + 1) * p.row], nb))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce(self, parts: dict):
        self.dist.all_reduce(parts[self.rank])

    def allgather_coarse(self, coarse: dict):
        import torch
        p = self.plans[self.rank]
        full = coarse[self.rank]
        mine = torch.zeros(self._pad, dtype=full.dtype, device=full.device)
        a, b = p.c_lo * p.crow, p.c_hi * p.crow
        mine[:b - a].copy_(full[a:b])
        outs = [torch.empty_like(mine) for _ in self.plans]
        self.dist.all_gather(outs, mine)
        for q, o in zip(self.plans, outs):
            if q.rank != self.rank:
                qa, qb = q.c_lo * q.crow, q.c_hi * q.crow
                full[qa:qb].copy_(o[:qb - qa])


# ---------------------------------------------------------------------------
# CUDA backend (libhsweep kernels on each shard's window)

class CudaShardBackend:
    """Per-shard device handles: the fine operator restricted to the window
    rows (true coefficients, halo rows included), the windowed transfer
    tables, and one replicated coarse sweep shared by the local shards."""

    def __init__(self, hh, plans, local, ctx=None):
        import torch
        from ._lib import context
        from .device import DeviceStencil, DeviceTransfer
        self.torch = torch
        self.ctx = ctx or context()
        self.hh = hh
        self.plans = plans
        self.local = list(local)
        op = hh.fine_op
        offs = sorted(op.coeffs)
        self.fine, self.transfer = {}, {}
        for g in self.local:
            p = plans[g]
            co = np.stack([np.asarray(op.coeffs[o]).reshape(p.n0, p.row)[p.win_lo:p.win_hi]
                           .reshape(-1) for o in offs])
            shape = (p.win_hi - p.win_lo,) + tuple(op.shape[1:])
            self.fine[g] = DeviceStencil(shape, offs, co, self.ctx)
            self.transfer[g] = DeviceTransfer(hh.cmap, self.ctx, window=p.window)
        self.sweep = hh.partition.device()
        cells = hh.sweep.n_cell
        if hh.sweep.variant == "nx" and isinstance(cells, (int, np.integer)):
            from .sweepdd import make_nx_cells
            cells = make_nx_cells(hh.partition.J, int(cells))
        self.variant = self.sweep.variant_id(hh.sweep.variant, cells)
        self.nc = int(np.prod(hh.coarse_op.shape))
        self.omega = float(hh.smoother.omega_jac)
        self.nu = int(hh.smoother.nu)
        self.scale = float(hh.restrict_scale)

    # vectors
    def zeros(self, g):
        return self.torch.zeros(self.plans[g].n_win, dtype=self.torch.complex128,
                                device=f"cuda:{self.ctx.device}")

    def zeros_coarse(self):
        return self.torch.zeros(self.nc, dtype=self.torch.complex128,
                                device=f"cuda:{self.ctx.device}")

    def upload(self, g, host_win):
        return self.torch.from_numpy(np.ascontiguousarray(host_win)).to(
            f"cuda:{self.ctx.device}")

    def download(self, x):
        return x.cpu().numpy()

    # kernels
    def _call(self, name, *a):
        self.ctx.call(name, *a)

    def jacobi(self, g, u, f, steps, from_zero):
        from .device import ptr
        self._call("hs_jacobi", self.fine[g].h, ptr(u), ptr(f), self.omega, int(steps),
                   int(bool(from_zero)), 1)

    def residual(self, g, f, u, out):
        from .device import ptr
        self._call("hs_stencil_residual", self.fine[g].h, ptr(f), ptr(u), ptr(out), 1)

    def apply(self, g, x, out):
        from .device import ptr
        self._call("hs_stencil_apply", self.fine[g].h, ptr(x), ptr(out), 1)

    def restrict(self, g, r, rc):
        from .device import ptr
        self._call("hs_restrict", self.transfer[g].h, ptr(r), ptr(rc), self.scale, 1)

    def prolong_add(self, g, uc, u):
        from .device import ptr
        self._call("hs_prolong_add", self.transfer[g].h, ptr(uc), ptr(u), 1, 1)

    def coarse_solve(self, rc, uc):
        from .device import ptr
        self._call("hs_sweep_apply", self.sweep.h, self.variant, ptr(rc), ptr(uc))

    def dots(self, g, V, k, w, out):
        """out[0:k] = V[0:k]^H w, out[k] = ||w||^2 over the owned rows."""
        from .device import ptr
        s = self.plans[g].own_slice
        n = s.stop - s.start
        done = 0
        while True:   # chunks of <= 32 vectors; the last one leaves ||w||^2 at out[k]
            kk = min(_KCHUNK, k - done)
            self._call("hs_block_dot", ptr(V[done, s]) if kk else ptr(w[s]), V.stride(0), kk,
                       ptr(w[s]), n, ptr(out[done:]))
            done += kk
            if done >= k:
                return

    def update(self, g, V, k, h, w, out):
        """w -= V[0:k] h on the owned rows, out[0] = ||w||^2 (owned)."""
        from .device import ptr
        s = self.plans[g].own_slice
        n = s.stop - s.start
        done = 0
        while True:
            kk = min(_KCHUNK, k - done)
            self._call("hs_block_update", ptr(V[done, s]) if kk else ptr(w[s]), V.stride(0),
                       kk, ptr(h[done:]), ptr(w[s]), n, ptr(out))
            done += kk
            if done >= k:
                return

    def norm2(self, g, x, out):
        from .device import ptr
        s = self.plans[g].own_slice
        self._call("hs_norm2", ptr(x[s]), s.stop - s.start, ptr(out))

    def scale_(self, g, x, a: complex):
        from .device import ptr
        self._call("hs_scale", ptr(x), x.numel(), float(a.real), float(a.imag))

    def lincomb(self, g, V, k, y, out):
        from .device import ptr
        done = 0
        while done < k:
            kk = min(_KCHUNK, k - done)
            part = out if done == 0 else self.zeros(g)
            self._call("hs_lincomb", ptr(V[done]), V.stride(0), kk, ptr(y[done:]), ptr(part),
                       out.numel())
            if done:
                self._call("hs_axpby", 1.0, 0.0, ptr(part), 1.0, 0.0, ptr(out), out.numel())
            done += kk

    def axpby(self, g, a: complex, x, b: complex, y):
        from .device import ptr
        self._call("hs_axpby", float(a.real), float(a.imag), ptr(x), float(b.real),
                   float(b.imag), ptr(y), y.numel())

    def small(self, n):
        return self.torch.zeros(n, dtype=self.torch.complex128,
                                device=f"cuda:{self.ctx.device}")

    def to_host(self, t):
        return t.cpu().numpy()

    def from_host(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{self.ctx.device}")

    def basis(self, g, rows):
        return self.torch.zeros((rows, self.plans[g].n_win), dtype=self.torch.complex128,
                                device=f"cuda:{self.ctx.device}")


# ---------------------------------------------------------------------------
# orchestration

class ShardedTGSP:
    """TGSP V-cycle and GMRES over the shards this process holds."""

    def __init__(self, plans, backend, comm):
        self.plans, self.be, self.comm = plans, backend, comm
        self.local = list(comm.local)
        self.nu = backend.nu
        self._r = {g: backend.zeros(g) for g in self.local}
        self._rc = {g: backend.zeros_coarse() for g in self.local}
        self._uc = backend.zeros_coarse()
        self._tmp = {g: backend.zeros(g) for g in self.local}

    # -- the preconditioner (twogrid.py:150-159)
    def vcycle(self, f: dict, u: dict):
        be, comm, L = self.be, self.comm, self.local
        comm.exchange(f)
        nu = self.nu
        if nu == 0:
            for g in L:
                u[g].zero_()
        else:
            first = min(nu, 2)      # 1 or 2 steps from zero need only f's halo
            for g in L:
                be.jacobi(g, u[g], f[g], first, True)
            for _ in range(nu - first):
                comm.exchange(u)
                for g in L:
                    be.jacobi(g, u[g], f[g], 1, False)
        comm.exchange(u)
        for g in L:
            be.residual(g, f[g], u[g], self._r[g])
        comm.exchange(self._r)
        for g in L:
            be.restrict(g, self._r[g], self._rc[g])
        comm.allgather_coarse(self._rc)
        # replicated coarse solve: every rank holds the full coarse vector
        # (LocalComm: one solve serves the process's shards)
        be.coarse_solve(self._rc[L[0]], self._uc)
        for g in L:
            be.prolong_add(g, self._uc, u[g])
        for _ in range(nu):
            comm.exchange(u)
            for g in L:
                be.jacobi(g, u[g], f[g], 1, False)
        return u

    def apply_a(self, x: dict, out: dict):
        self.comm.exchange(x)
        for g in self.local:
            self.be.apply(g, x[g], out[g])
        return out

    def op(self, v: dict, out: dict, z: dict | None = None):
        """out = A M v; ``z`` keeps M v (the GMRES driver's z_k)"""
        z = self._tmp if z is None else z
        self.vcycle(v, z)
        return self.apply_a(z, out)

    # -- reductions
    def _dots(self, V, k, w):
        parts = {g: self.be.small(k + 1) for g in self.local}
        for g in self.local:
            self.be.dots(g, V[g], k, w[g], parts[g])
        self.comm.allreduce(parts)
        return parts

    def _update(self, V, k, h, w):
        parts = {g: self.be.small(1) for g in self.local}
        for g in self.local:
            self.be.update(g, V[g], k, h[g], w[g], parts[g])
        self.comm.allreduce(parts)
        return self.be.to_host(parts[self.local[0]])[0].real

    def norm(self, x: dict) -> float:
        parts = {g: self.be.small(1) for g in self.local}
        for g in self.local:
            self.be.norm2(g, x[g], parts[g])
        self.comm.allreduce(parts)
        v = self.be.to_host(parts[self.local[0]])[0]
        if not math.isfinite(v.real) or v.imag != 0.0:
            raise FloatingPointError("non-finite values in a sharded vector")
        return math.sqrt(max(v.real, 0.0))

    # -- GMRES (krylov.py:46-146, CGS2 with the DGKS test)
    def gmres(self, f: dict, config: GmresConfig | None = None):
        config = config or GmresConfig()
        be, L = self.be, self.local
        t0 = time.perf_counter()
        bnorm = self.norm(f)
        u = {g: be.zeros(g) for g in L}
        if bnorm == 0.0:
            return u, SolveReport(0, np.array([0.0]), True, time.perf_counter() - t0)
        steps0 = config.max_iter if config.restart is None else min(config.restart,
                                                                     config.max_iter)
        V = {g: be.basis(g, steps0 + 1) for g in L}
        # z_k = M v_k kept (as in krylov.gmres): a cycle ends with u += Z y
        # instead of one more V-cycle on V y (M is linear and fixed)
        Z = {g: be.basis(g, steps0) for g in L}
        history = [1.0]
        res = {g: f[g].clone() for g in L}
        res_norm = bnorm
        converged = False
        while len(history) - 1 < config.max_iter and not converged:
            steps = config.max_iter - (len(history) - 1)
            if config.restart is not None:
                steps = min(steps, config.restart)
            mdv, converged = self._cycle(V, res, res_norm, bnorm, config.tol, steps, history, Z)
            if mdv is not None:
                for g in L:
                    be.axpby(g, 1.0, mdv[g], 1.0, u[g])
            # true residual between restarts
            self.comm.exchange(u)
            for g in L:
                be.residual(g, f[g], u[g], res[g])
            if config.restart is None:
                break
            res_norm = self.norm(res)
            converged = res_norm / bnorm <= config.tol
        hist = np.asarray(history)
        return u, SolveReport(len(history) - 1, hist, bool(hist[-1] <= config.tol),
                              time.perf_counter() - t0)

    def _cycle(self, V, r0, beta, bnorm, tol, max_steps, history, Z):
        be, L = self.be, self.local
        hess = np.zeros((max_steps + 1, max_steps), dtype=complex)
        cs = np.zeros(max_steps, dtype=complex)
        sn = np.zeros(max_steps, dtype=complex)
        g_ = np.zeros(max_steps + 1, dtype=complex)
        g_[0] = beta
        for g in L:
            V[g][0].copy_(r0[g])
            be.scale_(g, V[g][0], 1.0 / beta)
        k = 0
        converged = False
        for k in range(max_steps):
            vk = {g: V[g][k] for g in L}
            w = {g: V[g][k + 1] for g in L}
            self.op(vk, w, {g: Z[g][k] for g in L})
            h = self._dots(V, k + 1, w)
            hh = be.to_host(h[L[0]])
            hcol, w_norm0 = hh[:k + 1].copy(), hh[k + 1].real
            if not math.isfinite(w_norm0):
                raise FloatingPointError("operator produced non-finite values "
                                         f"at iteration {len(history)}")
            nrm2 = self._update(V, k + 1, h, w)
            if nrm2 < (_DGKS ** 2) * w_norm0:           # DGKS re-orthogonalisation
                h2 = self._dots(V, k + 1, w)
                hcol = hcol + be.to_host(h2[L[0]])[:k + 1]
                nrm2 = self._update(V, k + 1, h2, w)
            if not (math.isfinite(nrm2) and np.all(np.isfinite(hcol))):
                raise FloatingPointError("operator produced non-finite values "
                                         f"at iteration {len(history)}")
            hess[:k + 1, k] = hcol
            hess[k + 1, k] = math.sqrt(max(nrm2, 0.0))
            happy = hess[k + 1, k].real <= 1e-14 * beta
            if not happy:
                for g in L:
                    be.scale_(g, w[g], 1.0 / hess[k + 1, k].real)
            _givens_column(hess, cs, sn, g_, k)
            history.append(abs(g_[k + 1]) / bnorm)
            if history[-1] <= tol or happy:
                converged = True
                k += 1
                break
        else:
            k += 1
        if k == 0:
            return None, converged
        y = np.linalg.solve(hess[:k, :k], g_[:k])
        yd = be.from_host(y)
        mdv = {g: be.zeros(g) for g in L}   # M dv = Z y
        for g in L:
            be.lincomb(g, Z[g], k, yd, mdv[g])
        return mdv, converged
