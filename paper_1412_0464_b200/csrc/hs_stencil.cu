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

#include <algorithm>

namespace hs {

namespace {

constexpr int kThreads = 256;

enum Mode : int {
  kApply = 0,      // y = A x
  kResidual = 1,   // y = f - A x
  kJacobi = 2,     // y = x + w (f - A x) / diag
  kJacobi2Z = 3,   // y = two Jacobi steps from x = 0 (x unused)
};

// Persistent grid-stride form: one wave of resident blocks (no tail), flat
// 32-bit point index decomposed per point; blockIdx.y = right-hand side.
template <int S, int MODE>
__global__ void __launch_bounds__(kThreads)
k_stencil(StencilDesc d, const double2* __restrict__ x, const double2* __restrict__ f,
          double2* __restrict__ y, double omega) {
  const uint32_t n = (uint32_t)d.n, n1 = (uint32_t)d.n1, n2 = (uint32_t)d.n2;
  const int64_t rhs = (int64_t)blockIdx.y * d.n;
  const double2* __restrict__ C = d.coeffs;
  int64_t delta[S];
#pragma unroll
  for (int s = 0; s < S; ++s)
    delta[s] = ((int64_t)d.off[s][0] * d.n1 + d.off[s][1]) * d.n2 + d.off[s][2];
  for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) {
    const uint32_t row = i / n2, i2 = i - row * n2;
    const uint32_t i0 = row / n1, i1 = row - i0 * n1;
    double2 acc = czero();
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int o0 = d.off[s][0], o1 = d.off[s][1], o2 = d.off[s][2];
      const bool ok = (uint32_t)(i0 + o0) < (uint32_t)d.n0 && (uint32_t)(i1 + o1) < n1 &&
                      (uint32_t)(i2 + o2) < n2;
      const double2 c = __ldg(C + (int64_t)s * d.n + i);
      if (ok) {
        const int64_t j = (int64_t)i + delta[s];
        double2 xv;
        if (MODE == kJacobi2Z) {
          // first pre-smoothing step from zero, evaluated at the neighbour:
          // u1[j] = w f[j] / diag[j]
          xv = cscale(omega, cmul(__ldg(f + rhs + j), __ldg(d.invd + j)));
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
      const double2 inv = __ldg(d.invd + i);
      double2 ui;
      if (MODE == kJacobi2Z) ui = cscale(omega, cmul(fi, inv));
      else ui = __ldg(x + rhs + i);
      const double2 corr = cmul(cscale(omega, csub(fi, acc)), inv);
      y[rhs + i] = cadd(ui, corr);
    }
  }
}

// one wave of resident blocks of this kernel (grid-stride loop, no tail)
template <int S, int MODE>
int wave_of() {
  static int wave = 0;
  if (!wave) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stencil<S, MODE>, kThreads, 0);
    wave = std::max(1, sms * std::max(1, per));
  }
  return wave;
}

template <int MODE>
int launch_mode(Ctx* c, const Stencil* op, const double2* x, const double2* f, double2* y,
                double omega, int nrhs) {
  const StencilDesc& d = op->d;
  if (d.n >= (int64_t)1 << 31) return set_error(c, HS_E_SHAPE, "stencil grid too large");
  const int64_t need = (d.n + kThreads - 1) / kThreads;
  const int cls = MODE == kApply ? K_STENCIL
                  : MODE == kResidual ? K_RESIDUAL
                  : MODE == kJacobi ? K_JACOBI : K_JACOBI2Z;
  const double nb = (double)d.n * nrhs * 16.0;
  ProfScope ps(c, cls, nb * (d.S + ((MODE == kApply || MODE == kJacobi2Z) ? 2 : 3)));
  switch (d.S) {
#define HS_CASE(SS)                                                                    \
  case SS: {                                                                           \
    dim3 grid((unsigned)std::min<int64_t>(need, wave_of<SS, MODE>()), (unsigned)nrhs); \
    k_stencil<SS, MODE><<<grid, kThreads, 0, c->stream>>>(d, x, f, y, omega);          \
    break;                                                                             \
  }
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
