"""CPU ORACLE for the TGSP-GMRES hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference algorithm
(``/root/reference/pkg/src/helmsweep``) used as the parity checker.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package never imports
it and has no CPU fallback.

Pinning: ``tests/test_oracle.py`` checks every function here against golden
vectors produced by running the reference itself
(``tests/golden/make_golden.py``): operator applies, smoother, transfers,
X/UD sweeps, TGSP apply (1e-12) and GMRES histories/iteration counts.

The slab solves use scipy's SuperLU exactly as the reference does
(``sparselin.py:49``); the operator arithmetic is scipy sparse CSR like the
reference (``twogrid.py:140-141``), so ``cpu_baseline`` times the same
third-party kernels the reference spends its time in.

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


# ---------------------------------------------------------------------------
# operators  (reference discretize.py:110-117, sparselin.py:21-37)

def stencil_apply(offsets, coeffs, u):
    """out[i] = sum_s coeffs[s][i] * u[i + off_s], Dirichlet outside the box."""
    u = np.asarray(u, dtype=complex)
    out = np.zeros(u.shape, dtype=complex)
    for off, c in zip(offsets, coeffs):
        dst, src = [], []
        for o, n in zip(off, u.shape):
            o = int(o)
            dst.append(slice(max(0, -o), n - max(0, o)))
            src.append(slice(max(0, o), n - max(0, -o)))
        out[tuple(dst)] += c[tuple(dst)] * u[tuple(src)]
    return out


def stencil_csr(offsets, coeffs, shape):
    """CSR matrix of a stencil operator, row-major unknown ordering."""
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape))
    index = np.arange(n).reshape(shape)
    rows, cols, vals = [], [], []
    for off, c in zip(offsets, coeffs):
        dst, src = [], []
        for o, m in zip(off, shape):
            o = int(o)
            dst.append(slice(max(0, -o), m - max(0, o)))
            src.append(slice(max(0, o), m - max(0, -o)))
        rows.append(index[tuple(dst)].ravel())
        cols.append(index[tuple(src)].ravel())
        vals.append(np.asarray(c)[tuple(dst)].ravel())
    a = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n), dtype=complex)
    a.sum_duplicates()
    a.sort_indices()
    return a


class Op:
    """Stencil operator held as (offsets, coeffs) plus its CSR matrix."""

    def __init__(self, offsets, coeffs):
        self.offsets = [tuple(int(o) for o in off) for off in offsets]
        self.coeffs = [np.asarray(c, dtype=complex) for c in coeffs]
        self.shape = self.coeffs[0].shape
        self.dim = len(self.shape)
        self._csr = None

    @classmethod
    def from_dict(cls, coeffs: dict):
        offs = sorted(coeffs)
        return cls(offs, [coeffs[o] for o in offs])

    @property
    def csr(self):
        if self._csr is None:
            self._csr = stencil_csr(self.offsets, self.coeffs, self.shape)
        return self._csr

    def coeff(self, off):
        off = tuple(off)
        for o, c in zip(self.offsets, self.coeffs):
            if o == off:
                return c
        return None

    def diagonal(self):
        return self.coeff((0,) * self.dim)

    def apply(self, u):
        return stencil_apply(self.offsets, self.coeffs, np.asarray(u).reshape(self.shape))


# ---------------------------------------------------------------------------
# smoother and transfers  (reference twogrid.py:41-93, 140-159)

def jacobi(op: Op, u, f, omega, steps):
    """u <- u + omega (f - A u) / diag, ``steps`` times (twogrid.py:41-50)."""
    diag = op.diagonal()
    if (diag == 0).any():
        node = tuple(np.argwhere(diag == 0)[0])
        raise ZeroDivisionError(f"zero operator diagonal at node {node}")
    u = np.array(u, dtype=complex)
    for _ in range(steps):
        u = u + omega * (f - (op.csr @ u.ravel()).reshape(op.shape)) / diag
    return u


def prolongation_1d(fp, refined):
    """Tent prolongation along one axis (twogrid.py:53-71): 1 at the coarse
    image, 1/2 at the midpoint of every refined (merged) cell."""
    fp = np.asarray(fp)
    n_f, n_c = int(fp[-1]) - 1, len(fp) - 2
    r, c, v = [], [], []
    for i in range(1, n_c + 1):
        r.append(fp[i] - 1)
        c.append(i - 1)
        v.append(1.0)
    for cell, merged in enumerate(refined):
        if merged:
            mid = fp[cell] + 1
            for cp in (cell, cell + 1):
                if 1 <= cp <= n_c:
                    r.append(mid - 1)
                    c.append(cp - 1)
                    v.append(0.5)
    return sp.csr_matrix((v, (r, c)), shape=(n_f, n_c))


def prolongation(fps, refineds):
    """Tensor product over axes (twogrid.py:74-79)."""
    p = prolongation_1d(fps[0], refineds[0])
    for a in range(1, len(fps)):
        p = sp.kron(p, prolongation_1d(fps[a], refineds[a]), format="csr")
    return p


# ---------------------------------------------------------------------------
# sweeping preconditioner  (reference sweepdd.py:98-359)

class Slab:
    def __init__(self, lo, hi, op: Op):
        self.lo, self.hi, self.op = int(lo), int(hi), op
        self.lu = spla.splu(sp.csc_matrix(op.csr))


class Partition:
    """Coarse operator + slabs with staggered interfaces beta / beta_tilde."""

    def __init__(self, coarse: Op, beta, beta_tilde, slabs):
        self.op = coarse
        self.shape = coarse.shape
        self.beta = np.asarray(beta, dtype=int)
        self.bt = np.asarray(beta_tilde, dtype=int)
        self.J = len(self.beta) - 1
        self.slabs = slabs

    def transmit(self, point, sign, buf):
        """Two-layer interface sources from the global operator couplings
        (sweepdd.py:113-118, 133-141): src0 = +-A[b,b+1] buf1, src1 = -+A[b+1,b] buf0."""
        x0 = point - 1
        src0 = np.zeros(buf[0].shape, complex)
        src1 = np.zeros(buf[0].shape, complex)
        face = self.op.dim - 1
        for off, c in zip(self.op.offsets, self.op.coeffs):
            if off[0] == 1:
                src0 += stencil_apply([off[1:]], [c[x0]], buf[1]) if face else c[x0] * buf[1]
            elif off[0] == -1:
                src1 += stencil_apply([off[1:]], [c[x0 + 1]], buf[0]) if face else c[x0 + 1] * buf[0]
        return sign * src0, -sign * src1

    def solve(self, u, f, j, a, b, ta, tb, B1=None, B3=None, out2=False, out4=False):
        """Generic slab solve (sweepdd.py:236-268)."""
        s = self.slabs[j - 1]
        lo = s.lo
        fd = np.zeros(s.op.shape, complex)
        fd[a + 1 - lo:b + 1 - lo] = f[a:b]
        if B1 is not None and j > 1:
            p = int(self.beta[j - 1])
            s0, s1 = self.transmit(p, +1, B1)
            fd[p - lo] += s0
            fd[p + 1 - lo] += s1
        if B3 is not None and j < self.J:
            p = int(self.bt[j])
            s0, s1 = self.transmit(p, -1, B3)
            fd[p - lo] += s0
            fd[p + 1 - lo] += s1
        ud = s.lu.solve(fd.ravel()).reshape(s.op.shape)
        u[ta:tb] += ud[ta + 1 - lo:tb + 1 - lo]
        r2 = r4 = None
        if out2 and j < self.J:
            p = int(self.beta[j])
            r2 = ud[p - lo:p - lo + 2].copy()
        if out4 and j > 1:
            p = int(self.bt[j - 1])
            r4 = ud[p - lo:p - lo + 2].copy()
        return r2, r4

    def forward(self, u, f, j0, j1, B=None):
        """sweepdd.py:271-282."""
        for j in range(j0, j1 + 1):
            if 1 <= j <= self.J:
                out, _ = self.solve(u, f, j, self.beta[j - 1], self.beta[j], self.beta[j - 1],
                                    self.beta[j], B1=B if j > 1 else None, out2=j < self.J)
                if out is not None:
                    B = out
        return B

    def backward(self, u, f, j0, j1, B=None):
        """sweepdd.py:285-294."""
        for j in range(j0, j1 - 1, -1):
            if 1 <= j <= self.J:
                _, out = self.solve(u, f, j, self.bt[j - 1], self.bt[j], self.bt[j - 1],
                                    self.bt[j], B3=B if j < self.J else None, out4=j > 1)
                if out is not None:
                    B = out
        return B

    def residual(self, u, f):
        return f - (self.op.csr @ u.ravel()).reshape(self.shape)

    def prec_ud(self, f):
        """sweepdd.py:312-319."""
        f = np.asarray(f, complex).reshape(self.shape)
        u = np.zeros(self.shape, complex)
        B = self.forward(u, f, 1, self.J)
        self.backward(u, self.residual(u, f), self.J, 1, B)
        return u

    parallel = False   # run the X sweep's two half-sweeps on two threads

    def prec_x(self, f):
        """sweepdd.py:322-359; with ``parallel`` the two half-sweeps of each
        pass run on two threads like the reference's ``parallel=True``
        (:336-358; disjoint rows of u, results bitwise the serial ones)."""
        if self.J % 2:
            raise ValueError(f"X-sweep needs an even subdomain count, got {self.J}")
        f = np.asarray(f, complex).reshape(self.shape)
        u = np.zeros(self.shape, complex)
        jm = self.J // 2 + 1
        if self.parallel:
            return self._prec_x_parallel(f, u, jm)
        B1 = self.forward(u, f, 1, jm - 1)
        B2 = self.backward(u, f, self.J, jm + 1)
        self.solve(u, f, jm, self.beta[jm - 1], self.bt[jm], self.beta[jm - 1], self.bt[jm],
                   B1=B1, B3=B2)
        g = self.residual(u, f)
        B2, B1 = self.solve(u, g, jm, self.bt[jm - 1], self.beta[jm], self.bt[jm - 1],
                            self.beta[jm], out2=True, out4=True)
        self.backward(u, g, jm - 1, 1, B1)
        self.forward(u, g, jm + 1, self.J, B2)
        return u

    def _prec_x_parallel(self, f, u, jm):
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=2) as ex:
            fa = ex.submit(self.forward, u, f, 1, jm - 1)
            fb = ex.submit(self.backward, u, f, self.J, jm + 1)
            B1, B2 = fa.result(), fb.result()
            self.solve(u, f, jm, self.beta[jm - 1], self.bt[jm], self.beta[jm - 1],
                       self.bt[jm], B1=B1, B3=B2)
            g = self.residual(u, f)
            B2, B1 = self.solve(u, g, jm, self.bt[jm - 1], self.beta[jm], self.bt[jm - 1],
                                self.beta[jm], out2=True, out4=True)
            fa = ex.submit(self.backward, u, g, jm - 1, 1, B1)
            fb = ex.submit(self.forward, u, g, jm + 1, self.J, B2)
            fa.result(), fb.result()
        return u

    def mid_in(self, u, f, j, B1, B3):
        """midsolve_in (sweepdd.py:297-300)."""
        self.solve(u, f, j, self.beta[j - 1], self.bt[j], self.beta[j - 1], self.bt[j],
                   B1=B1, B3=B3)

    def mid_out(self, u, f, j):
        """midsolve_out (sweepdd.py:303-306): returns (out2, out4)."""
        return self.solve(u, f, j, self.bt[j - 1], self.beta[j], self.bt[j - 1], self.beta[j],
                          out2=True, out4=True)

    def prec_nx(self, f, j_cell, j_mid):
        """NX sweep over cell groups (sweepdd.py:403-434): j_cell has the -1 / J+1
        sentinels; buffer k of the reference is buf[k] here."""
        f = np.asarray(f, complex).reshape(self.shape)
        u = np.zeros(self.shape, complex)
        jc, jm = list(j_cell), list(j_mid)
        nc = len(jm)
        buf = {i: None for i in range(1, 2 * nc + 2)}
        for m in range(1, nc + 1):
            if m < nc:
                bf, bb = self.mid_out(u, f, jc[m])
                buf[2 * m + 1], buf[2 * m] = bf, bb
            buf[2 * m - 1] = self.forward(u, f, jc[m - 1] + 1, jm[m - 1] - 1, buf[2 * m - 1])
            buf[2 * m] = self.backward(u, f, jc[m] - 1, jm[m - 1] + 1, buf[2 * m])
            self.mid_in(u, f, jm[m - 1], buf[2 * m - 1], buf[2 * m])
        g = self.residual(u, f)
        for m in range(1, nc + 1):
            bf, bb = self.mid_out(u, g, jm[m - 1])
            buf[2 * m], buf[2 * m - 1] = bf, bb
            buf[2 * m - 1] = self.backward(u, g, jm[m - 1] - 1, jc[m - 1] + 1, buf[2 * m - 1])
            buf[2 * m] = self.forward(u, g, jm[m - 1] + 1, jc[m] - 1, buf[2 * m])
            if m > 1:
                self.mid_in(u, g, jc[m - 1], buf[2 * m - 2], buf[2 * m - 1])
        return u

    def apply(self, f, variant="x", cells=None):
        if variant == "nx":
            return self.prec_nx(f, *cells)
        return self.prec_x(f) if variant == "x" else self.prec_ud(f)


class Exact:
    """ExactCoarseSolver (twogrid.py:99-105): SuperLU of the whole operator
    (sparselin.py:40-62), as a stand-in for a partition in TwoGrid."""

    def __init__(self, op: Op):
        self.op = op
        self.shape = op.shape
        self.lu = spla.splu(sp.csc_matrix(op.csr))

    def solve(self, b):
        return self.lu.solve(np.asarray(b, complex).ravel())

    def apply(self, f, variant=None, cells=None):
        return self.solve(f).reshape(self.shape)


# ---------------------------------------------------------------------------
# two-grid cycle  (reference twogrid.py:119-176)

class TwoGrid:
    def __init__(self, fine: Op, p_matrix, partition: Partition, omega_jac, nu,
                 restrict_scale, variant="x", cells=None):
        self.fine, self.p, self.part = fine, p_matrix, partition
        self.cells = cells          # NX: (j_cell, j_mid)
        self.omega_jac, self.nu = float(omega_jac), int(nu)
        self.restrict_scale = float(restrict_scale)
        self.variant = variant
        self.diag = fine.diagonal()

    def _smooth(self, u, f):
        for _ in range(self.nu):
            u = u + self.omega_jac * (f - (self.fine.csr @ u.ravel()).reshape(f.shape)) / self.diag
        return u

    def vcycle(self, f):
        """u = S_post(S_pre(0) + P Sweep(h^d P^T (f - A S_pre(0))))."""
        f = np.asarray(f, complex).reshape(self.fine.shape)
        u = self._smooth(np.zeros_like(f), f) if self.nu else np.zeros_like(f)
        r = f - (self.fine.csr @ u.ravel()).reshape(f.shape)
        rc = self.restrict_scale * (self.p.T @ r.ravel())
        uc = self.part.apply(rc.reshape(self.part.shape), self.variant, self.cells)
        u = u + (self.p @ uc.ravel()).reshape(f.shape)
        if self.nu:
            u = self._smooth(u, f)
        return u

    def as_preconditioner(self):
        return lambda v: self.vcycle(v).ravel()


# ---------------------------------------------------------------------------
# GMRES  (reference krylov.py:46-146)

def _gmres_cycle(op, r0, bnorm, tol, max_steps, history):
    n = r0.shape[0]
    H = np.zeros((max_steps + 1, max_steps), complex)
    cs = np.zeros(max_steps, complex)
    sn = np.zeros(max_steps, complex)
    beta = np.linalg.norm(r0)
    V = [r0 / beta]
    g = np.zeros(max_steps + 1, complex)
    g[0] = beta
    k = 0
    done = False
    for k in range(max_steps):
        w = op(V[k])
        if not np.all(np.isfinite(w)):
            raise FloatingPointError(f"operator produced non-finite values at iteration "
                                     f"{len(history)}")
        for i in range(k + 1):            # modified Gram-Schmidt
            H[i, k] = np.vdot(V[i], w)
            w = w - H[i, k] * V[i]
        H[k + 1, k] = np.linalg.norm(w)
        happy = H[k + 1, k].real <= 1e-14 * beta
        if not happy:
            V.append(w / H[k + 1, k])
        for i in range(k):                 # previous rotations
            t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
            H[i + 1, k] = -np.conj(sn[i]) * H[i, k] + np.conj(cs[i]) * H[i + 1, k]
            H[i, k] = t
        den = np.sqrt(abs(H[k, k]) ** 2 + abs(H[k + 1, k]) ** 2)
        if den == 0.0:
            cs[k], sn[k] = 1.0, 0.0
        else:
            cs[k], sn[k] = np.conj(H[k, k]) / den, np.conj(H[k + 1, k]) / den
        H[k, k] = cs[k] * H[k, k] + sn[k] * H[k + 1, k]
        H[k + 1, k] = 0.0
        g[k + 1] = -np.conj(sn[k]) * g[k]
        g[k] = cs[k] * g[k]
        history.append(abs(g[k + 1]) / bnorm)
        if history[-1] <= tol or happy:
            done = True
            k += 1
            break
    else:
        k += 1
    if k == 0:
        return np.zeros(n, complex), done
    y = np.linalg.solve(H[:k, :k], g[:k])
    upd = np.zeros(n, complex)
    for i in range(k):
        upd += y[i] * V[i]
    return upd, done


def gmres(apply_a, apply_m, f, tol=1e-6, max_iter=100, restart=None):
    """Right-preconditioned restarted GMRES; returns (u, iterations, history,
    converged, seconds).  Control flow of krylov.py:105-146."""
    f = np.asarray(f, complex).ravel()
    if not np.all(np.isfinite(f)):
        raise FloatingPointError("right-hand side contains non-finite values")
    if apply_m is None:
        apply_m = lambda v: v  # noqa: E731
    t0 = time.perf_counter()
    bnorm = np.linalg.norm(f)
    if bnorm == 0.0:
        return np.zeros_like(f), 0, np.array([0.0]), True, time.perf_counter() - t0
    op = lambda v: np.asarray(apply_a(apply_m(v)), complex).ravel()  # noqa: E731
    history = [1.0]
    u = np.zeros_like(f)
    res = f.copy()
    done = False
    while len(history) - 1 < max_iter and not done:
        steps = max_iter - (len(history) - 1)
        if restart is not None:
            steps = min(steps, restart)
        dv, done = _gmres_cycle(op, res, bnorm, tol, steps, history)
        u = u + np.asarray(apply_m(dv), complex).ravel()
        res = f - np.asarray(apply_a(u), complex).ravel()
        if restart is None:
            break
        done = np.linalg.norm(res) / bnorm <= tol
    hist = np.asarray(history)
    return u, len(history) - 1, hist, bool(hist[-1] <= tol), time.perf_counter() - t0


# ---------------------------------------------------------------------------
# builders

def from_fixture(d, variant=None):
    """Oracle objects from a golden fixture (tests/golden/*.npz)."""
    fine = Op(d["fine_offsets"], d["fine_coeffs"])
    coarse = Op(d["coarse_offsets"], d["coarse_coeffs"])
    J = len(d["beta"]) - 1
    slabs = [Slab(d["slab_lo"][j], d["slab_hi"][j],
                  Op(d[f"slab{j + 1}_offsets"], d[f"slab{j + 1}_coeffs"])) for j in range(J)]
    part = Partition(coarse, d["beta"], d["beta_tilde"], slabs)
    dim = len(d["fine_shape"])
    p = prolongation([d[f"fp{a}"] for a in range(dim)], [d[f"refined{a}"] for a in range(dim)])
    v = variant or str(d["variant"])
    cells = (d["nx2_cells"], d["nx2_mid"]) if v == "nx" else None   # the nx2d case's NX(2)
    return TwoGrid(fine, p, part, d["omega_jac"], d["nu"], d["restrict_scale"], v, cells)


def from_exact_fixture(d):
    """Two-grid cycle with the exact coarse solve from tests/golden/exact2d.npz."""
    fine = Op(d["fine_offsets"], d["fine_coeffs"])
    coarse = Op(d["coarse_offsets"], d["coarse_coeffs"])
    dim = len(d["fine_shape"])
    p = prolongation([d[f"fp{a}"] for a in range(dim)], [d[f"refined{a}"] for a in range(dim)])
    return TwoGrid(fine, p, Exact(coarse), d["omega_jac"], d["nu"], d["restrict_scale"], "exact")


def from_hierarchy(h):
    """Oracle objects from the package's host-side hierarchy (``HostHierarchy``):
    the same coefficient arrays the GPU consumes."""
    fine = Op.from_dict(h.fine_op.coeffs)
    coarse = Op.from_dict(h.coarse_op.coeffs)
    slabs = [Slab(lo, hi, Op.from_dict(op.coeffs)) for (lo, hi, op) in h.slabs]
    part = Partition(coarse, h.beta, h.beta_tilde, slabs)
    p = prolongation(h.cmap.fine_point_of_coarse, h.cmap.refined_cell)
    cells = None
    if h.sweep.variant == "nx":
        c = h.sweep.n_cell
        cells = (list(c.j_cell), list(c.j_mid)) if hasattr(c, "j_cell") else \
            _nx_cells(h.partition.J, int(c))
    return TwoGrid(fine, p, part, h.smoother.omega_jac, h.smoother.nu, h.restrict_scale,
                   h.sweep.variant, cells)


def _nx_cells(J, n_cell):
    """make_nx_cells (sweepdd.py:392-401) as (j_cell, j_mid)."""
    bounds = [-1] + [round(m * J / n_cell) for m in range(1, n_cell)] + [J + 1]
    mids = [(max(1, bounds[m - 1] + 1) + min(J, bounds[m] - 1) + 1) // 2
            for m in range(1, n_cell + 1)]
    return bounds, mids
