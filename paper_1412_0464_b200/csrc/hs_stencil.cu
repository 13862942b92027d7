// Compact-stencil kernels: matvec, residual, fused omega-Jacobi smoothing.
//
// Reference semantics: stencil_apply (discretize.py:110-117), the fine CSR
// matvec (twogrid.py:140-141), jacobi_smooth / TwoGridCycle._smooth
// (twogrid.py:41-50, 143-148).  All HBM-bound: per DOF a matvec
// moves (S+2)*16 B, a Jacobi step (S+3)*16 B.  Layout: coefficients stored
// per offset ([S][n] complex128, SoA) so every offset's load is a coalesced
// 16-B/lane stream; neighbour values of x come through L1/L2 (rows of x are
// small enough to stay L2-resident while a sweep of the grid passes them).
//
// Grid: x = column blocks over the fastest axis n2, y = rows (i0*n1 + i1),
// z = right-hand side.  No 64-bit division per element.

#include "hs_common.cuh"

namespace hs {

namespace {

constexpr int kThreads = 256;

enum Mode : int {
  kApply = 0,      // y = A x
  kResidual = 1,   // y = f - A x
  kJacobi = 2,     // y = x + w (f - A x) / diag
  kJacobi2Z = 3,   // y = two Jacobi steps from x = 0 (x unused)
};

template <int S, int MODE>
__global__ void __launch_bounds__(kThreads)
k_stencil(StencilDesc d, const double2* __restrict__ x, const double2* __restrict__ f,
          double2* __restrict__ y, double omega) {
  const int64_t i2 = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i2 >= d.n2) return;
  const int64_t row = blockIdx.y;            // i0 * n1 + i1
  const int64_t i1 = row % d.n1;
  const int64_t i0 = row / d.n1;
  const int64_t i = row * d.n2 + i2;
  const int64_t rhs = (int64_t)blockIdx.z * d.n;
  const double2* __restrict__ C = d.coeffs;

  double2 acc = czero();
  double2 diag = make_double2(1.0, 0.0);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int o0 = d.off[s][0], o1 = d.off[s][1], o2 = d.off[s][2];
    const bool ok = (uint64_t)(i0 + o0) < (uint64_t)d.n0 && (uint64_t)(i1 + o1) < (uint64_t)d.n1 &&
                    (uint64_t)(i2 + o2) < (uint64_t)d.n2;
    const double2 c = __ldg(C + (int64_t)s * d.n + i);
    if (MODE >= kJacobi && s == d.diag) diag = c;
    if (ok) {
      const int64_t j = i + ((int64_t)o0 * d.n1 + o1) * d.n2 + o2;
      double2 xv;
      if (MODE == kJacobi2Z) {
        // first pre-smoothing step from zero, evaluated at the neighbour:
        // u1[j] = w f[j] / diag[j]
        const double2 dj = __ldg(C + (int64_t)d.diag * d.n + j);
        xv = cscale(omega, cdiv(__ldg(f + rhs + j), dj));
      } else {
        xv = __ldg(x + rhs + j);
      }
      acc = cfma(c, xv, acc);
    }
  }
  if (MODE == kApply) {
    y[rhs + i] = acc;
  } else if (MODE == kResidual) {
    y[rhs + i] = csub(__ldg(f + rhs + i), acc);
  } else {
    const double2 fi = __ldg(f + rhs + i);
    double2 ui;
    if (MODE == kJacobi2Z) ui = cscale(omega, cdiv(fi, diag));
    else ui = __ldg(x + rhs + i);
    const double2 corr = cdiv(cscale(omega, csub(fi, acc)), diag);
    y[rhs + i] = cadd(ui, corr);
  }
}

template <int MODE>
int launch_mode(Ctx* c, const Stencil* op, const double2* x, const double2* f, double2* y,
                double omega, int nrhs) {
  const StencilDesc& d = op->d;
  dim3 grid((unsigned)((d.n2 + kThreads - 1) / kThreads), (unsigned)(d.n0 * d.n1),
            (unsigned)nrhs);
  if (d.n0 * d.n1 > 65535) return set_error(c, HS_E_SHAPE, "stencil grid too large");
  const int cls = MODE == kApply ? K_STENCIL
                  : MODE == kResidual ? K_RESIDUAL
                  : MODE == kJacobi ? K_JACOBI : K_JACOBI2Z;
  const double nb = (double)d.n * nrhs * 16.0;
  ProfScope ps(c, cls, nb * (d.S + ((MODE == kApply || MODE == kJacobi2Z) ? 2 : 3)));
  switch (d.S) {
#define HS_CASE(SS) \
  case SS: k_stencil<SS, MODE><<<grid, kThreads, 0, c->stream>>>(d, x, f, y, omega); break;
    HS_CASE(1) HS_CASE(2) HS_CASE(3) HS_CASE(4) HS_CASE(5) HS_CASE(6) HS_CASE(7) HS_CASE(8)
    HS_CASE(9) HS_CASE(10) HS_CASE(11) HS_CASE(12) HS_CASE(13) HS_CASE(14) HS_CASE(15)
    HS_CASE(16) HS_CASE(17) HS_CASE(18) HS_CASE(19) HS_CASE(20) HS_CASE(21) HS_CASE(22)
    HS_CASE(23) HS_CASE(24) HS_CASE(25) HS_CASE(26) HS_CASE(27)
#undef HS_CASE
    default:
      return set_error(c, HS_E_SHAPE, "stencil with unsupported offset count");
  }
  HS_LAUNCH_CHECK(c, "stencil kernel");
  return HS_OK;
}

}  // namespace

int stencil_apply(Ctx* c, const Stencil* op, const double2* x, double2* y, int nrhs,
                  const double2* f_minus) {
  if (f_minus) return launch_mode<kResidual>(c, op, x, f_minus, y, 0.0, nrhs);
  return launch_mode<kApply>(c, op, x, nullptr, y, 0.0, nrhs);
}

int stencil_jacobi(Ctx* c, const Stencil* op, double2* u, const double2* f, double omega,
                   int steps, int u_is_zero, int nrhs) {
  if (steps <= 0) return HS_OK;
  if (op->d.diag < 0 || op->has_zero_diag) {
    char buf[160];
    snprintf(buf, sizeof buf, "zero operator diagonal at node %lld", op->zero_diag_node);
    return set_error(c, HS_E_ZERO_DIAG, buf, op->zero_diag_node);
  }
  const size_t bytes = (size_t)op->d.n * nrhs * sizeof(double2);
  double2* tmp = (double2*)scratch(c, bytes, 1);
  if (!tmp) return set_error(c, HS_E_CUDA, "scratch allocation failed");
  // ping-pong between u and tmp; the last step must land in u
  int done = 0;
  double2* cur = u;
  double2* nxt = tmp;
  // with an odd number of remaining steps start by writing into u directly
  if (u_is_zero) {
    if (steps >= 2) {
      // fused: two steps from zero in one pass
      int rem = steps - 2;
      double2* dst = (rem % 2 == 0) ? u : tmp;
      int r = launch_mode<kJacobi2Z>(c, op, nullptr, f, dst, omega, nrhs);
      if (r) return r;
      done = 2;
      cur = dst;
      nxt = (dst == u) ? tmp : u;
    } else {
      // one step from zero: u = w f / diag == Jacobi2Z's inner value; use a
      // residual-free formulation through kJacobi with x = 0 (memset)
      HS_CUDA(c, cudaMemsetAsync(u, 0, bytes, c->stream), "memset");
      int r = launch_mode<kJacobi>(c, op, u, f, tmp, omega, nrhs);
      if (r) return r;
      HS_CUDA(c, cudaMemcpyAsync(u, tmp, bytes, cudaMemcpyDeviceToDevice, c->stream), "copy");
      return HS_OK;
    }
  } else {
    if (steps % 2 == 1) {
      // odd: copy u into tmp first so that the final write lands in u
      HS_CUDA(c, cudaMemcpyAsync(tmp, u, bytes, cudaMemcpyDeviceToDevice, c->stream), "copy");
      cur = tmp;
      nxt = u;
    }
  }
  for (int s = done; s < steps; ++s) {
    int r = launch_mode<kJacobi>(c, op, cur, f, nxt, omega, nrhs);
    if (r) return r;
    double2* t = cur;
    cur = nxt;
    nxt = t;
  }
  return HS_OK;
}

}  // namespace hs
