"""Right-preconditioned restarted GMRES on the GPU (drop-in for reference
``krylov.py``: ``GmresConfig`` :17-30, ``SolveReport`` :32-43,
``_gmres_cycle`` :46-102, ``gmres`` :105-146).

Control flow is the reference's: Arnoldi on A M, complex Givens rotations on
the host (tiny), happy breakdown at H[k+1,k] <= 1e-14 beta, residual estimate
|g_{k+1}|/||f|| as the stopping test, restart with ``u += M dv`` and the TRUE
residual deciding convergence between cycles, ``iterations = len(history)-1``.

The vectors never leave the device.  Orthogonalisation defaults to classical
Gram-Schmidt with a conditional second pass (``orth="cgs2"``, threshold
``_DGKS``): one fused dot pass + one fused update pass over the basis
(the iteration count is unchanged vs MGS); ``orth="mgs"`` reproduces the reference's
modified Gram-Schmidt order exactly (one dot + one update per basis vector).
When ``apply_a``/``apply_m`` are this package's fine operator and TGSP
preconditioner, ``A M v`` runs as one fused device call.
"""

from __future__ import annotations

import gc
import math
import time
from dataclasses import dataclass

import numpy as np

from .device import empty, from_device, ptr, to_device
from ._lib import context

_KCHUNK = 32
import os as _os

# Re-orthogonalisation threshold of the CGS2 passes: a second Gram-Schmidt
# pass runs when ||w'|| < eta ||w|| after the first (decided on the device).
# eta = 0.1 is Rutishauser's criterion (re-orthogonalise when the projection
# cancelled more than one digit): one pass then leaves an orthogonality error
# of at most ~10 eps per step.  With w = A M v_k close to span(V) the DGKS
# choice eta = 1/sqrt(2) re-orthogonalised in 165 of C3's 196 steps (ratios
# 0.36-0.97 of the norm, tools/gate_stats.py) for no change in iteration
# counts or residual histories; HS_DGKS_ETA=0.7071 restores it.  (The
# reference's modified Gram-Schmidt never re-orthogonalises.)
_DGKS = float(_os.environ.get("HS_DGKS_ETA", 0.1))
# first-pass update fused with the second pass's dots (one read of the basis
# when the second pass runs; HS_FUSE_UPDATE_DOT=0: separate kernels, A/B)
_FUSE_UPDATE_DOT = _os.environ.get("HS_FUSE_UPDATE_DOT", "1") != "0"


@dataclass(frozen=True)
class GmresConfig:
    tol: float = 1e-6
    max_iter: int = 100
    restart: int | None = None

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tolerance must be positive")
        if self.max_iter < 1:
            raise ValueError("need at least one iteration")
        if self.restart is not None and self.restart < 1:
            raise ValueError("restart length must be >= 1")


@dataclass
class SolveReport:
    iterations: int
    residual_history: np.ndarray
    converged: bool
    wall_time: float

    def __str__(self):
        state = "converged" if self.converged else "stalled"
        return (f"{state} in {self.iterations} iterations, "
                f"final residual {self.residual_history[-1]:.3e}, {self.wall_time:.2f}s")


def on_device(fn):
    """Mark a user callable as taking and returning device (torch CUDA)
    vectors, so gmres passes it the device vector without a host copy."""
    fn._hs_device = True
    return fn


def _device_callable(fn) -> bool:
    """True for callables of this package that accept device (torch CUDA)
    vectors: operators, preconditioners, factorisation solves."""
    import torch
    if isinstance(fn, torch.nn.Module):
        return True
    if getattr(fn, "_hs_device", False):
        return True
    owner = getattr(fn, "__self__", None)
    if owner is not None and getattr(owner, "_hs_device", False):
        return True
    mod = getattr(type(fn), "__module__", "") or ""
    if mod.startswith(__name__.rsplit(".", 1)[0]):
        return True   # instances of this package's classes (FineOperator, _Prec, ...)
    return False


class _Ops:
    """Device-side operator bundle for one solve."""

    def __init__(self, apply_a, apply_m, n, ctx):
        self.ctx, self.n = ctx, n
        self.a, self.m = apply_a, apply_m
        self.cycle = None
        self.fine = None
        from .twogrid import FineOperator
        if isinstance(apply_a, FineOperator):
            self.fine = apply_a.op.device()
        cyc = getattr(apply_m, "cycle", None)
        lane = getattr(apply_m, "lane", None)
        if (cyc is not None and self.fine is not None and cyc.fine_op is apply_a.op
                and not getattr(cyc, "generic", False)):
            self.cycle = lane.dev if lane is not None else cyc.device()

    def _call(self, fn, v):
        """apply a user operator: this package's device callables take the
        device vector; any other callable is host code written for numpy
        (the reference's ``gmres`` contract): it gets a host copy, and its
        result is copied back to the device"""
        if _device_callable(fn):
            out = fn(v)
        else:
            out = fn(v.cpu().numpy())
        t, _ = to_device(out, self.n, self.ctx)
        return t

    def apply_m(self, v):
        if self.cycle is not None:
            return self.cycle.vcycle_dev(v)
        if self.m is None:
            return v.clone()
        return self._call(self.m, v)

    def apply_a(self, v, out=None):
        if self.fine is not None:
            y = out if out is not None else empty(self.n, self.ctx)
            self.ctx.call("hs_stencil_apply", self.fine.h, ptr(v), ptr(y), 1)
            return y
        t = self._call(self.a, v)
        if out is not None:
            out.copy_(t)
            return out
        return t

    def op(self, v, out):
        """out = A M v"""
        if self.cycle is not None:
            return self.cycle.apply_a_dev(v, out)
        return self.apply_a(self.apply_m(v), out)

    def residual(self, f, u):
        """f - A u"""
        if self.fine is not None:
            r = empty(self.n, self.ctx)
            self.ctx.call("hs_stencil_residual", self.fine.h, ptr(f), ptr(u), ptr(r), 1)
            return r
        r = f.clone()
        au = self.apply_a(u)
        self.ctx.call("hs_axpby", -1.0, 0.0, ptr(au), 1.0, 0.0, ptr(r), self.n)
        return r


class _Basis:
    """Arnoldi basis rows on the device, grown in chunks."""

    def __init__(self, n, rows, ctx):
        import torch
        self.n, self.ctx = n, ctx
        self.V = torch.empty((rows, n), dtype=torch.complex128, device=f"cuda:{ctx.device}")

    def ensure(self, rows):
        import torch
        if rows > self.V.shape[0]:
            new = torch.empty((max(rows, 2 * self.V.shape[0]), self.n), dtype=self.V.dtype,
                              device=self.V.device)
            new[: self.V.shape[0]].copy_(self.V)
            self.V = new

    def row(self, i):
        return self.V[i]


def _dot_pass(ctx, basis, k, w, n, hbuf, gate=None):
    """hbuf[0:k] = V[0:k]^H w, ||w||^2 at hbuf[k].  ``gate = (after, before)``:
    run only when after.re < DGKS^2 * before.re (decided on the device)."""
    lda = basis.V.stride(0)
    done = 0
    while True:
        kk = min(_KCHUNK, k - done)
        # the chunk writes kk dots then ||w||^2 at hbuf[done + kk]
        vp = ptr(basis.V[done]) if kk else ptr(w)
        if gate is None:
            ctx.call("hs_block_dot", vp, lda, kk, ptr(w), n, ptr(hbuf[done:]))
        else:
            ctx.call("hs_block_dot_gated", vp, lda, kk, ptr(w), n, ptr(hbuf[done:]),
                     ptr(gate[0]), ptr(gate[1]), _DGKS ** 2)
        done += kk
        if done >= k:
            return


def _update_pass(ctx, basis, k, h, w, n, nbuf, gate=None):
    """w -= V[0:k] h, ||w||^2 into nbuf[0] (a closed gate copies gate[0] there)."""
    lda = basis.V.stride(0)
    done = 0
    while True:
        kk = min(_KCHUNK, k - done)
        vp = ptr(basis.V[done]) if kk else ptr(w)
        if gate is None:
            ctx.call("hs_block_update", vp, lda, kk, ptr(h[done:]), ptr(w), n, ptr(nbuf))
        else:
            ctx.call("hs_block_update_gated", vp, lda, kk, ptr(h[done:]), ptr(w), n, ptr(nbuf),
                     ptr(gate[0]), ptr(gate[1]), _DGKS ** 2)
        done += kk
        if done >= k:
            return


def _update_dot_pass(ctx, basis, k, h, w, n, nbuf, h2):
    """First-pass update fused with the second pass's dots (one read of the
    basis; bitwise the update then the dot pass): w -= V[0:k] h, h2[0:k] =
    V[0:k]^H w, ||w||^2 into nbuf[0] and h2[k].  False when k exceeds one
    kernel chunk (the caller then runs the two passes)."""
    if k > _KCHUNK or not _FUSE_UPDATE_DOT:
        return False
    ctx.call("hs_block_update_dot", ptr(basis.V[0]), basis.V.stride(0), k, ptr(h), ptr(w), n,
             ptr(nbuf), ptr(h2))
    return True


def _givens_column(hess, cs, sn, g, k):
    """Apply the previous rotations to column k, form rotation k, update g
    (krylov.py:74-88)."""
    for i in range(k):
        t = cs[i] * hess[i, k] + sn[i] * hess[i + 1, k]
        hess[i + 1, k] = -np.conj(sn[i]) * hess[i, k] + np.conj(cs[i]) * hess[i + 1, k]
        hess[i, k] = t
    denom = np.sqrt(abs(hess[k, k]) ** 2 + abs(hess[k + 1, k]) ** 2)
    if denom == 0.0:
        cs[k], sn[k] = 1.0, 0.0
    else:
        cs[k] = np.conj(hess[k, k]) / denom
        sn[k] = np.conj(hess[k + 1, k]) / denom
    hess[k, k] = cs[k] * hess[k, k] + sn[k] * hess[k + 1, k]
    hess[k + 1, k] = 0.0
    g[k + 1] = -np.conj(sn[k]) * g[k]
    g[k] = cs[k] * g[k]


def _basis_update(ctx, basis, hess, g, k, n, dev):
    """dv = sum_i y_i v_i with y = H[:k,:k]^-1 g[:k] (krylov.py:96-101)."""
    import torch
    y = np.linalg.solve(hess[:k, :k], g[:k])
    yd = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
    upd = empty(n, ctx)
    done = 0
    while done < k:
        kk = min(_KCHUNK, k - done)
        part = upd if done == 0 else empty(n, ctx)
        ctx.call("hs_lincomb", ptr(basis.row(done)), basis.V.stride(0), kk, ptr(yd[done:]),
                 ptr(part), n)
        if done:
            ctx.call("hs_axpby", 1.0, 0.0, ptr(part), 1.0, 0.0, ptr(upd), n)
        done += kk
    return upd


def _gmres_cycle_pipelined(ops: _Ops, basis: _Basis, r0, r0_norm, bnorm, tol, max_steps,
                           history, zb=None):
    """CGS2 Arnoldi cycle for this package's TGSP operator with the host one
    step behind the device.  Everything the next step needs is decided on the
    device (the DGKS second pass is gated there, v_{k+1} = w / ||w|| is scaled
    there), so while the host reads Hessenberg column k and applies the
    Givens rotations, A M v_{k+1} up to and including the sweep's first launch
    (~1 ms of device work) is already queued.  The arithmetic is the
    synchronous cycle's, operation for operation; a converged cycle discards
    that queued part."""
    import torch
    ctx, n = ops.ctx, ops.n
    cyc = ops.cycle
    dev = torch.device(f"cuda:{ctx.device}")
    hess = np.zeros((max_steps + 1, max_steps), dtype=complex)
    cs = np.zeros(max_steps, dtype=complex)
    sn = np.zeros(max_steps, dtype=complex)
    beta = r0_norm
    basis.ensure(max_steps + 1)
    v0 = basis.row(0)
    v0.copy_(r0)
    ctx.call("hs_scale", ptr(v0), n, 1.0 / beta, 0.0)
    g = np.zeros(max_steps + 1, dtype=complex)
    g[0] = beta
    W = max_steps + 2
    col = torch.zeros(2 * W + 2, dtype=torch.complex128, device=dev)
    hb, h2b, nb = col[:W], col[W:2 * W], col[2 * W:]
    pin = torch.empty((max_steps, 2 * W + 2), dtype=torch.complex128, pin_memory=True)
    stream = torch.cuda.current_stream(dev)
    events = [torch.cuda.Event() for _ in range(max_steps)]

    def orthonormalise(k):
        w = basis.row(k + 1)
        _dot_pass(ctx, basis, k + 1, w, n, hb)
        gate = (nb[0:], hb[k + 1:])
        if not _update_dot_pass(ctx, basis, k + 1, hb, w, n, nb[0:], h2b):
            _update_pass(ctx, basis, k + 1, hb, w, n, nb[0:])
            _dot_pass(ctx, basis, k + 1, w, n, h2b, gate)
        _update_pass(ctx, basis, k + 1, h2b, w, n, nb[1:], gate)
        ctx.call("hs_scale_inv_sqrt", ptr(w), n, ptr(nb[1:]))
        pin[k].copy_(col, non_blocking=True)
        events[k].record(stream)

    # z_k = M v_k is kept (zb): the cycle ends with u += Z y, no extra V-cycle
    zb.ensure(max_steps)
    cyc.apply_az_part(basis.row(0), zb.row(0), basis.row(1), 3)
    orthonormalise(0)
    k = 0
    converged = False
    for k in range(max_steps):
        ahead = k + 1 < max_steps
        if ahead:   # ~1 ms of the next step queued while the host trails
            cyc.apply_az_part(basis.row(k + 1), zb.row(k + 1), None, 0)
            cyc.apply_az_part(basis.row(k + 1), zb.row(k + 1), None, 1)
        events[k].synchronize()
        host = pin[k].numpy()
        hcol, w_norm0, nrm1 = host[:k + 1].copy(), host[k + 1].real, host[2 * W].real
        if not math.isfinite(w_norm0):
            raise FloatingPointError("operator produced non-finite values "
                                     f"at iteration {len(history)}")
        if nrm1 < (_DGKS ** 2) * w_norm0:          # the device ran the DGKS pass
            hcol = hcol + host[W:W + k + 1]
        nrm2 = host[2 * W + 1].real
        if not (math.isfinite(nrm2) and np.all(np.isfinite(hcol))):
            raise FloatingPointError("operator produced non-finite values "
                                     f"at iteration {len(history)}")
        hess[:k + 1, k] = hcol
        hess[k + 1, k] = math.sqrt(max(nrm2, 0.0))
        happy = hess[k + 1, k].real <= 1e-14 * beta
        _givens_column(hess, cs, sn, g, k)
        history.append(abs(g[k + 1]) / bnorm)
        if history[-1] <= tol or happy:
            converged = True
            k += 1
            break
        if ahead:
            cyc.apply_az_part(basis.row(k + 1), zb.row(k + 1), basis.row(k + 2), 2)
            orthonormalise(k + 1)
    else:
        k += 1
    if k == 0:
        return None, converged
    return _basis_update(ctx, zb, hess, g, k, n, dev), converged   # M dv = Z y


def _gmres_cycle(ops: _Ops, basis: _Basis, r0, r0_norm, bnorm, tol, max_steps, history, orth,
                 zb=None):
    """Synchronous Arnoldi cycle (the reference's _gmres_cycle, krylov.py:46-102).
    Returns (update, converged): with ``zb`` (this package's TGSP operator)
    the update is M dv = Z y from the kept z_k = M v_k, else dv = V y."""
    import torch
    ctx, n = ops.ctx, ops.n
    hess = np.zeros((max_steps + 1, max_steps), dtype=complex)
    cs = np.zeros(max_steps, dtype=complex)
    sn = np.zeros(max_steps, dtype=complex)
    beta = r0_norm
    basis.ensure(max_steps + 1)
    v0 = basis.row(0)
    v0.copy_(r0)
    ctx.call("hs_scale", ptr(v0), n, 1.0 / beta, 0.0)
    g = np.zeros(max_steps + 1, dtype=complex)
    g[0] = beta
    dev = torch.device(f"cuda:{ctx.device}")
    hbuf = torch.zeros(max_steps + 2, dtype=torch.complex128, device=dev)
    h2buf = torch.zeros(max_steps + 2, dtype=torch.complex128, device=dev)
    nbuf = torch.zeros(2, dtype=torch.complex128, device=dev)
    k = 0
    converged = False
    if zb is not None:
        zb.ensure(max_steps)
    for k in range(max_steps):
        w = basis.row(k + 1)
        if zb is not None:
            ops.cycle.apply_az_part(basis.row(k), zb.row(k), w, 3)
        else:
            ops.op(basis.row(k), w)
        if orth == "mgs":
            for i in range(k + 1):
                ctx.call("hs_block_dot", ptr(basis.row(i)), basis.V.stride(0), 1, ptr(w), n,
                         ptr(h2buf[2 * 0:]))
                hbuf[i:i + 1].copy_(h2buf[0:1])
                ctx.call("hs_block_update", ptr(basis.row(i)), basis.V.stride(0), 1,
                         ptr(hbuf[i:]), ptr(w), n, ptr(nbuf))
            host = torch.cat([hbuf[:k + 1], nbuf[:1]]).cpu().numpy()
            hcol, nrm2 = host[:k + 1], host[k + 1].real
            w_norm0 = None
        else:
            _dot_pass(ctx, basis, k + 1, w, n, hbuf)
            fused = _update_dot_pass(ctx, basis, k + 1, hbuf, w, n, nbuf, h2buf)
            if not fused:
                _update_pass(ctx, basis, k + 1, hbuf, w, n, nbuf)
            host = torch.cat([hbuf[:k + 2], nbuf[:1]]).cpu().numpy()
            hcol, w_norm0, nrm2 = host[:k + 1], host[k + 1].real, host[k + 2].real
            if not math.isfinite(w_norm0):
                raise FloatingPointError("operator produced non-finite values "
                                         f"at iteration {len(history)}")
            if nrm2 < (_DGKS ** 2) * w_norm0:      # DGKS: re-orthogonalise once
                if not fused:
                    _dot_pass(ctx, basis, k + 1, w, n, h2buf)
                _update_pass(ctx, basis, k + 1, h2buf, w, n, nbuf)
                host2 = torch.cat([h2buf[:k + 1], nbuf[:1]]).cpu().numpy()
                hcol = hcol + host2[:k + 1]
                nrm2 = host2[k + 1].real
        if not (math.isfinite(nrm2) and np.all(np.isfinite(hcol))):
            raise FloatingPointError("operator produced non-finite values "
                                     f"at iteration {len(history)}")
        hess[:k + 1, k] = hcol
        hess[k + 1, k] = math.sqrt(max(nrm2, 0.0))
        happy = hess[k + 1, k].real <= 1e-14 * beta
        if not happy:
            ctx.call("hs_scale", ptr(w), n, 1.0 / hess[k + 1, k].real, 0.0)
        _givens_column(hess, cs, sn, g, k)
        history.append(abs(g[k + 1]) / bnorm)
        if history[-1] <= tol or happy:
            converged = True
            k += 1
            break
    else:
        k += 1
    if k == 0:
        return None, converged
    return _basis_update(ctx, zb if zb is not None else basis, hess, g, k, n, dev), converged


def _norm(ctx, x, n):
    import torch
    out = torch.zeros(1, dtype=torch.complex128, device=x.device)
    ctx.call("hs_norm2", ptr(x), n, ptr(out))
    v = out.cpu().numpy()[0]
    return math.sqrt(max(v.real, 0.0)), v.imag


def gmres(apply_a, apply_m, f, config: GmresConfig | None = None, orth: str = "cgs2",
          pipelined: bool = True):
    """Solve A u = f with right preconditioning (see :func:`_gmres`).  The
    cyclic garbage collector is paused for the solve: a generation-2 pass
    over torch's object graph was measured to stall the launching thread for
    30-50 ms in one of ~6 solves (C2, 157 ms each)."""
    was = gc.isenabled()
    gc.disable()
    try:
        return _gmres(apply_a, apply_m, f, config, orth, pipelined)
    finally:
        if was:
            gc.enable()


def _gmres(apply_a, apply_m, f, config: GmresConfig | None = None, orth: str = "cgs2",
           pipelined: bool = True):
    """Solve A u = f with right preconditioning (GMRES on A M v = f, u = M v).

    ``f`` numpy -> ``u`` numpy; ``f`` torch CUDA -> ``u`` torch.  Stops on
    the true relative residual between restarts, like the reference.
    ``pipelined`` (CGS2 with this package's TGSP operator): the host trails
    the device by one Arnoldi step; same arithmetic as the synchronous loop.
    """
    if config is None:
        config = GmresConfig()
    if orth not in ("cgs2", "mgs"):
        raise ValueError(f"orth must be 'cgs2' or 'mgs', got {orth!r}")
    lane = getattr(apply_m, "lane", None)
    ctx = lane.ctx if lane is not None else context()
    t0 = time.perf_counter()
    ft, was_np = to_device(f, None, ctx)
    n = ft.numel()
    bnorm, bad = _norm(ctx, ft, n)
    if bad or not math.isfinite(bnorm):
        raise FloatingPointError("right-hand side contains non-finite values")
    if bnorm == 0.0:
        u = empty(n, ctx).zero_()
        return (from_device(u, was_np), SolveReport(0, np.array([0.0]), True,
                                                    time.perf_counter() - t0))
    ops = _Ops(apply_a, apply_m, n, ctx)
    steps0 = config.max_iter if config.restart is None else min(config.restart, config.max_iter)
    basis = _Basis(n, min(steps0, 64) + 1, ctx)
    # the TGSP operator keeps z_k = M v_k (FGMRES-style storage of a fixed
    # preconditioner): each cycle ends with u += Z y instead of one more
    # V-cycle on V y -- the same update (M linear), one sweep fewer per cycle
    zb = _Basis(n, min(steps0, 64), ctx) if ops.cycle is not None else None
    history = [1.0]
    u = empty(n, ctx).zero_()
    res = ft
    res_norm = bnorm
    converged = False
    while len(history) - 1 < config.max_iter and not converged:
        steps = config.max_iter - (len(history) - 1)
        if config.restart is not None:
            steps = min(steps, config.restart)
        if pipelined and orth == "cgs2" and ops.cycle is not None:
            dv, converged = _gmres_cycle_pipelined(ops, basis, res, res_norm, bnorm,
                                                   config.tol, steps, history, zb)
        else:
            dv, converged = _gmres_cycle(ops, basis, res, res_norm, bnorm, config.tol, steps,
                                         history, orth, zb)
        if dv is not None:
            mdv = dv if zb is not None else ops.apply_m(dv)
            ctx.call("hs_axpby", 1.0, 0.0, ptr(mdv), 1.0, 0.0, ptr(u), n)
        res = ops.residual(ft, u)
        if config.restart is None:
            break
        res_norm, _ = _norm(ctx, res, n)
        converged = res_norm / bnorm <= config.tol
    hist = np.asarray(history)
    report = SolveReport(len(history) - 1, hist, bool(hist[-1] <= config.tol),
                         time.perf_counter() - t0)
    out = from_device(u, was_np)
    if not was_np:
        out = out.reshape(f.shape)
    return out, report


class _View:
    """A right-hand side's rows of a shared (nrhs, rows, n) basis tensor."""

    def __init__(self, V):
        self.V = V

    def ensure(self, rows):
        if rows > self.V.shape[0]:
            raise ValueError("lockstep basis too short")

    def row(self, i):
        return self.V[i]


def _runs(idx):
    """consecutive runs of a sorted index list: [(first, count)]"""
    out = []
    for i in idx:
        if out and out[-1][0] + out[-1][1] == i:
            out[-1][1] += 1
        else:
            out.append([i, 1])
    return [(a, b) for a, b in out]


def gmres_many(apply_a, apply_m, rhs, config: GmresConfig | None = None):
    """Independent restarted GMRES solves of several right-hand sides in
    lockstep on one stream: at every Arnoldi step the preconditioner of all
    unconverged right-hand sides is ONE ``hs_vcycle_many`` call, so their
    coarse sweeps share one pass over the slab factors (several right-hand
    sides per chain of slab solves).  Everything else -- the fine matvec, the
    CGS2 orthogonalisation with the device-gated DGKS pass, the host Givens
    rotations, the restart logic of ``gmres`` (krylov.py:105-146) -- runs per
    right-hand side with the kernels and operation order of ``gmres``: each
    solution, iteration count and residual history is bitwise the
    single-right-hand-side solve's.  Needs this package's fine operator and
    TGSP preconditioner with a finite restart; anything else falls back to
    one ``gmres`` per right-hand side.  Returns [(u, SolveReport)]."""
    import torch
    if config is None:
        config = GmresConfig()
    rhs = list(rhs)
    lane = getattr(apply_m, "lane", None)
    ctx = lane.ctx if lane is not None else context()
    probe = None
    if rhs:
        ft0, _ = to_device(rhs[0], None, ctx)
        probe = _Ops(apply_a, apply_m, ft0.numel(), ctx)
    if len(rhs) < 2 or probe.cycle is None or config.restart is None:
        return [gmres(apply_a, apply_m, f, config) for f in rhs]
    was = gc.isenabled()
    gc.disable()
    try:
        return _gmres_many(probe, rhs, config)
    finally:
        if was:
            gc.enable()


def _gmres_many(ops: _Ops, rhs, config: GmresConfig):
    import torch
    ctx, n, cyc = ops.ctx, ops.n, ops.cycle
    dev = torch.device(f"cuda:{ctx.device}")
    R = len(rhs)
    t0 = time.perf_counter()
    steps0 = min(config.restart, config.max_iter)
    rows = steps0 + 1
    W = steps0 + 2
    fts, was_np = [], []
    for f in rhs:
        t, w = to_device(f, n, ctx)
        fts.append(t)
        was_np.append(w)
    Vall = torch.empty((R, rows, n), dtype=torch.complex128, device=dev)
    Zall = torch.empty((R, rows, n), dtype=torch.complex128, device=dev)   # (same stride as Vall)
    cols = torch.zeros((R, 2 * W + 2), dtype=torch.complex128, device=dev)
    pins = torch.empty((R, 2 * W + 2), dtype=torch.complex128, pin_memory=True)
    stream = torch.cuda.current_stream(dev)
    event = torch.cuda.Event()
    bases = [_View(Vall[r]) for r in range(R)]
    zbs = [_View(Zall[r]) for r in range(R)]
    us = [empty(n, ctx).zero_() for _ in range(R)]
    hist = [[1.0] for _ in range(R)]
    done = [False] * R
    bnorm = [0.0] * R
    res, res_norm = list(fts), [0.0] * R
    for r in range(R):
        bnorm[r], bad = _norm(ctx, fts[r], n)
        if bad or not math.isfinite(bnorm[r]):
            raise FloatingPointError("right-hand side contains non-finite values")
        res_norm[r] = bnorm[r]
        if bnorm[r] == 0.0:
            hist[r] = [0.0]
            done[r] = True

    def orthonormalise(r, k):
        basis, col = bases[r], cols[r]
        hb, h2b, nb = col[:W], col[W:2 * W], col[2 * W:]
        w = basis.row(k + 1)
        _dot_pass(ctx, basis, k + 1, w, n, hb)
        gate = (nb[0:], hb[k + 1:])
        if not _update_dot_pass(ctx, basis, k + 1, hb, w, n, nb[0:], h2b):
            _update_pass(ctx, basis, k + 1, hb, w, n, nb[0:])
            _dot_pass(ctx, basis, k + 1, w, n, h2b, gate)
        _update_pass(ctx, basis, k + 1, h2b, w, n, nb[1:], gate)
        ctx.call("hs_scale_inv_sqrt", ptr(w), n, ptr(nb[1:]))

    while True:
        live = [r for r in range(R) if not done[r] and len(hist[r]) - 1 < config.max_iter]
        if not live:
            break
        # ---- one restart cycle of every live right-hand side, in lockstep
        steps = {r: min(config.max_iter - (len(hist[r]) - 1), config.restart) for r in live}
        hess = {r: np.zeros((steps[r] + 1, steps[r]), dtype=complex) for r in live}
        cs = {r: np.zeros(steps[r], dtype=complex) for r in live}
        sn = {r: np.zeros(steps[r], dtype=complex) for r in live}
        g = {r: np.zeros(steps[r] + 1, dtype=complex) for r in live}
        kdone = {}
        for r in live:
            v0 = bases[r].row(0)
            v0.copy_(res[r])
            ctx.call("hs_scale", ptr(v0), n, 1.0 / res_norm[r], 0.0)
            g[r][0] = res_norm[r]
        active = list(live)
        k = 0
        while active:
            for first, count in _runs(active):   # z_k = M v_k: one chain for the run
                ctx.call("hs_vcycle_many", cyc.h, count, ptr(Vall[first, k]), ptr(Zall[first, k]),
                         rows * n)
            for r in active:
                ctx.call("hs_stencil_apply", ops.fine.h, ptr(Zall[r, k]), ptr(Vall[r, k + 1]), 1)
                orthonormalise(r, k)
            for r in active:
                pins[r].copy_(cols[r], non_blocking=True)
            event.record(stream)
            event.synchronize()
            nxt = []
            for r in active:
                host = pins[r].numpy()
                hcol, w_norm0, nrm1 = host[:k + 1].copy(), host[k + 1].real, host[2 * W].real
                if not math.isfinite(w_norm0):
                    raise FloatingPointError("operator produced non-finite values "
                                             f"at iteration {len(hist[r])}")
                if nrm1 < (_DGKS ** 2) * w_norm0:          # the device ran the DGKS pass
                    hcol = hcol + host[W:W + k + 1]
                nrm2 = host[2 * W + 1].real
                if not (math.isfinite(nrm2) and np.all(np.isfinite(hcol))):
                    raise FloatingPointError("operator produced non-finite values "
                                             f"at iteration {len(hist[r])}")
                hess[r][:k + 1, k] = hcol
                hess[r][k + 1, k] = math.sqrt(max(nrm2, 0.0))
                happy = hess[r][k + 1, k].real <= 1e-14 * res_norm[r]
                _givens_column(hess[r], cs[r], sn[r], g[r], k)
                hist[r].append(abs(g[r][k + 1]) / bnorm[r])
                if hist[r][-1] <= config.tol or happy:
                    kdone[r] = k + 1
                elif k + 1 >= steps[r]:
                    kdone[r] = k + 1
                else:
                    nxt.append(r)
            active = nxt
            k += 1
        # ---- u += Z y, true residual (gmres' restart logic per right-hand side)
        for r in live:
            mdv = _basis_update(ctx, zbs[r], hess[r], g[r], kdone[r], n, dev)
            ctx.call("hs_axpby", 1.0, 0.0, ptr(mdv), 1.0, 0.0, ptr(us[r]), n)
            res[r] = ops.residual(fts[r], us[r])
            res_norm[r], _ = _norm(ctx, res[r], n)
            done[r] = res_norm[r] / bnorm[r] <= config.tol   # the true residual decides
    out = []
    wall = time.perf_counter() - t0
    for r in range(R):
        h = np.asarray(hist[r])
        rep = SolveReport(len(h) - 1, h, bool(h[-1] <= config.tol), wall)
        u = from_device(us[r], was_np[r])
        if not was_np[r]:
            u = u.reshape(rhs[r].shape)
        out.append((u, rep))
    return out
