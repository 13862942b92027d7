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

// 3-D compact 27-point operators (2.5-D blocking): a block owns a TY x TX
// tile of the (i1, i2) plane and marches over a run of i0 planes, keeping
// three planes of the input (with a one-point ring) in shared memory, so each
// x value is loaded once per run instead of 27 times per point; the 27
// coefficient streams are read once.  Per point the arithmetic is
// k_stencil's, in the same order (bitwise the same).
constexpr int k3TX = 32, k3TY = 8, k3Run = 16;
// residency: the matvec keeps its 27 coefficient loads in flight with 2
// blocks per SM; the smoother / residual modes run best at 3 (measured)
template <int MODE>
__global__ void __launch_bounds__(256, MODE == kApply ? 2 : 3)
k_stencil27(StencilDesc d, const double2* __restrict__ x, const double2* __restrict__ f,
            double2* __restrict__ y, double omega) {
  constexpr int W = k3TX + 2, H = k3TY + 2;
  __shared__ double2 P[3][H * W];
  const int n0 = (int)d.n0, n1 = (int)d.n1, n2 = (int)d.n2;
  const int t1 = blockIdx.y * k3TY, t2 = blockIdx.x * k3TX;
  const int p0 = blockIdx.z * k3Run, p1 = min(n0, p0 + k3Run);
  const int tx = threadIdx.x % k3TX, ty = threadIdx.x / k3TX;
  const int g1 = t1 + ty, g2 = t2 + tx;
  const bool mine = g1 < n1 && g2 < n2;
  const int64_t plane = (int64_t)n1 * n2;
  // neighbour value at flat index j (x, or the first smoothing step from zero)
  auto val = [&](int64_t j) {
    if (MODE == kJacobi2Z) return cscale(omega, cmul(__ldg(f + j), __ldg(d.invd + j)));
    return __ldg(x + j);
  };
  auto load_plane = [&](int i0, double2* dst) {
    for (int k = threadIdx.x; k < H * W; k += 256) {
      const int ly = k / W, lx = k - ly * W;
      const int a = t1 + ly - 1, b = t2 + lx - 1;
      double2 v = czero();
      if (i0 >= 0 && i0 < n0 && (unsigned)a < (unsigned)n1 && (unsigned)b < (unsigned)n2)
        v = val((int64_t)i0 * plane + (int64_t)a * n2 + b);
      dst[k] = v;
    }
  };
  load_plane(p0 - 1, P[0]);
  load_plane(p0, P[1]);
  for (int i0 = p0; i0 < p1; ++i0) {
    const int cur = (i0 - p0 + 1) % 3, nxt = (i0 - p0 + 2) % 3, prv = (i0 - p0) % 3;
    load_plane(i0 + 1, P[nxt]);
    __syncthreads();
    if (mine) {
      const int64_t i = (int64_t)i0 * plane + (int64_t)g1 * n2 + g2;
      double2 acc = czero();
#pragma unroll
      for (int s = 0; s < 27; ++s) {
        const int o0 = d.off[s][0], o1 = d.off[s][1], o2 = d.off[s][2];
        const bool ok = (unsigned)(i0 + o0) < (unsigned)n0 && (unsigned)(g1 + o1) < (unsigned)n1 &&
                        (unsigned)(g2 + o2) < (unsigned)n2;
        const double2 c = __ldg(d.coeffs + (int64_t)s * d.n + i);
        if (ok) {
          const double2* pl = P[o0 < 0 ? prv : o0 > 0 ? nxt : cur];
          acc = cfma(c, pl[(ty + 1 + o1) * W + tx + 1 + o2], acc);
        }
      }
      if (MODE == kApply) {
        y[i] = acc;
      } else if (MODE == kResidual) {
        y[i] = csub(__ldg(f + i), acc);
      } else {
        const double2 fi = __ldg(f + i);
        const double2 inv = __ldg(d.invd + i);
        double2 ui;
        if (MODE == kJacobi2Z) ui = cscale(omega, cmul(fi, inv));
        else ui = __ldg(x + i);
        y[i] = cadd(ui, cmul(cscale(omega, csub(fi, acc)), inv));
      }
    }
    __syncthreads();   // plane `prv` is overwritten by the next iteration's load
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
  static const bool flat27 = getenv("HS_STENCIL27_FLAT") != nullptr;   // A/B switch
  if (d.S == 27 && d.n0 > 1 && nrhs == 1 && !flat27) {   // 3-D compact: 2.5-D blocking
    dim3 grid((unsigned)((d.n2 + k3TX - 1) / k3TX), (unsigned)((d.n1 + k3TY - 1) / k3TY),
              (unsigned)((d.n0 + k3Run - 1) / k3Run));
    k_stencil27<MODE><<<grid, 256, 0, c->stream>>>(d, x, f, y, omega);
    HS_LAUNCH_CHECK(c, "stencil kernel");
    return HS_OK;
  }
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

// ---------------------------------------------------------------------------
// Fused fine-level halves of the V-cycle on 2-D levels (twogrid.py:150-159
// with nu = 2): temporal blocking over a BY x BX tile with a two-point halo,
// the intermediate smoother iterates in shared memory.
//   pre:  u1 = w f / d (ring 2), u2 = u1 + w (f - A u1) / d (ring 1),
//         r = f - A u2 (tile)                    -> u2, r
//   post: u3 = u2 + P uc (ring 2), u4 = Jacobi(u3) (ring 1),
//         u5 = Jacobi(u4) (tile)                 -> u5
// Per point the arithmetic is that of the unfused kernels (k_stencil modes,
// k_prolong), in the same order: the results are bitwise the same.  HBM
// bytes per DOF (5-point): pre 16 f + 8 d + 80 A + 32 out = 136 (vs 256
// unfused); post 16 u2 + 4 uc + 16 f + 8 d + 80 A + 16 out = 140 (vs 288);
// halo re-reads hit L2.

#include "hs_transfer.cuh"

namespace hs {
namespace {

#ifndef HS_FUSED_MINB
#define HS_FUSED_MINB 6   // 40 registers: 6 blocks per SM (measured best of 1 / 6 / 8)
#endif
#ifndef HS_FUSED_UNROLL
#define HS_FUSED_UNROLL _Pragma("unroll")
#endif
#ifndef HS_FUSED_BX
#define HS_FUSED_BX 32
#endif
#ifndef HS_FUSED_BY
#define HS_FUSED_BY 16
#endif
constexpr int kBX = HS_FUSED_BX, kBY = HS_FUSED_BY;   // tile (fastest axis x rows)
constexpr int kR2X = kBX + 4, kR2Y = kBY + 4;  // tile + 2-point ring
constexpr int kR1X = kBX + 2, kR1Y = kBY + 2;  // tile + 1-point ring

// A x at global (g1, g2) = flat i from a shared-memory field V (row length
// W, the point at (vy, vx)); couplings leaving the box are dropped.  The
// coefficients are re-read per stage (L1/L2 hits for the tile's second
// stage: keeping them in registers was measured slower -- occupancy).
template <int S>
__device__ __forceinline__ double2 apply_at(const StencilDesc& d, int64_t i, int g1, int g2,
                                            const double2* V, int W, int vy, int vx) {
  double2 acc = czero();
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int o1 = d.off[s][1], o2 = d.off[s][2];
    const bool ok = (uint32_t)(g1 + o1) < (uint32_t)d.n1 && (uint32_t)(g2 + o2) < (uint32_t)d.n2;
    const double2 c = __ldg(d.coeffs + (int64_t)s * d.n + i);
    if (ok) acc = cfma(c, V[(vy + o1) * W + vx + o2], acc);
  }
  return acc;
}

template <int S>
__global__ void __launch_bounds__(256, HS_FUSED_MINB)
k_pre2d(StencilDesc d, const double2* __restrict__ f, double2* __restrict__ u2,
        double2* __restrict__ r, double omega) {
  __shared__ double2 U1[kR2Y * kR2X];
  __shared__ double2 U2[kR1Y * kR1X];
  const int n1 = (int)d.n1, n2 = (int)d.n2;
  const int t1 = blockIdx.y * kBY, t2 = blockIdx.x * kBX;
  HS_FUSED_UNROLL
  for (int k = threadIdx.x; k < kR2Y * kR2X; k += 256) {   // u1 = w f / d, ring 2
    const int ly = k / kR2X, lx = k - ly * kR2X;
    const int g1 = t1 + ly - 2, g2 = t2 + lx - 2;
    double2 v = czero();
    if ((unsigned)g1 < (unsigned)n1 && (unsigned)g2 < (unsigned)n2) {
      const int64_t j = (int64_t)g1 * n2 + g2;
      v = cscale(omega, cmul(__ldg(f + j), __ldg(d.invd + j)));
    }
    U1[k] = v;
  }
  __syncthreads();
  HS_FUSED_UNROLL
  for (int k = threadIdx.x; k < kR1Y * kR1X; k += 256) {   // u2, ring 1
    const int ly = k / kR1X, lx = k - ly * kR1X;
    const int g1 = t1 + ly - 1, g2 = t2 + lx - 1;
    double2 v = czero();
    if ((unsigned)g1 < (unsigned)n1 && (unsigned)g2 < (unsigned)n2) {
      const int64_t i = (int64_t)g1 * n2 + g2;
      const double2 acc = apply_at<S>(d, i, g1, g2, U1, kR2X, ly + 1, lx + 1);
      const double2 fi = __ldg(f + i), inv = __ldg(d.invd + i);
      const double2 ui = cscale(omega, cmul(fi, inv));
      v = cadd(ui, cmul(cscale(omega, csub(fi, acc)), inv));
    }
    U2[k] = v;
  }
  __syncthreads();
  HS_FUSED_UNROLL
  for (int k = threadIdx.x; k < kBY * kBX; k += 256) {   // r = f - A u2, tile
    const int ly = k / kBX, lx = k - ly * kBX;
    const int g1 = t1 + ly, g2 = t2 + lx;
    if (g1 >= n1 || g2 >= n2) continue;
    const int64_t i = (int64_t)g1 * n2 + g2;
    const double2 acc = apply_at<S>(d, i, g1, g2, U2, kR1X, ly + 1, lx + 1);
    u2[i] = U2[(ly + 1) * kR1X + lx + 1];
    r[i] = csub(__ldg(f + i), acc);
  }
}

// (P uc)[g1, g2] on a 2-D level: k_prolong's gather (axis 0 of the canonical
// shape is the singleton)
__device__ __forceinline__ double2 prolong_at(const TransferDesc& t, const double2* uc, int g1,
                                              int g2) {
  double2 acc = czero();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int p0 = t.par[0][a];
    if (p0 < 0) continue;
    const double w0 = t.pw[0][a];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int p1 = t.par[1][2 * g1 + b];
      if (p1 < 0) continue;
      const double w01 = w0 * t.pw[1][2 * g1 + b];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int p2 = t.par[2][2 * g2 + c];
        if (p2 < 0) continue;
        const double w = w01 * t.pw[2][2 * g2 + c];
        const double2 v = __ldg(uc + ((int64_t)p0 * t.nc[1] + p1) * t.nc[2] + p2);
        acc.x = fma(w, v.x, acc.x);
        acc.y = fma(w, v.y, acc.y);
      }
    }
  }
  return acc;
}

template <int S>
__global__ void __launch_bounds__(256, HS_FUSED_MINB)
k_post2d(StencilDesc d, TransferDesc t, const double2* __restrict__ uc,
         const double2* __restrict__ f, const double2* __restrict__ u2,
         double2* __restrict__ u, double omega) {
  __shared__ double2 U3[kR2Y * kR2X];
  __shared__ double2 U4[kR1Y * kR1X];
  const int n1 = (int)d.n1, n2 = (int)d.n2;
  const int t1 = blockIdx.y * kBY, t2 = blockIdx.x * kBX;
  HS_FUSED_UNROLL
  for (int k = threadIdx.x; k < kR2Y * kR2X; k += 256) {   // u3 = u2 + P uc, ring 2
    const int ly = k / kR2X, lx = k - ly * kR2X;
    const int g1 = t1 + ly - 2, g2 = t2 + lx - 2;
    double2 v = czero();
    if ((unsigned)g1 < (unsigned)n1 && (unsigned)g2 < (unsigned)n2)
      v = cadd(__ldg(u2 + (int64_t)g1 * n2 + g2), prolong_at(t, uc, g1, g2));
    U3[k] = v;
  }
  __syncthreads();
  HS_FUSED_UNROLL
  for (int k = threadIdx.x; k < kR1Y * kR1X; k += 256) {   // u4, ring 1
    const int ly = k / kR1X, lx = k - ly * kR1X;
    const int g1 = t1 + ly - 1, g2 = t2 + lx - 1;
    double2 v = czero();
    if ((unsigned)g1 < (unsigned)n1 && (unsigned)g2 < (unsigned)n2) {
      const int64_t i = (int64_t)g1 * n2 + g2;
      const double2 acc = apply_at<S>(d, i, g1, g2, U3, kR2X, ly + 1, lx + 1);
      const double2 fi = __ldg(f + i), inv = __ldg(d.invd + i);
      v = cadd(U3[(ly + 1) * kR2X + lx + 1], cmul(cscale(omega, csub(fi, acc)), inv));
    }
    U4[k] = v;
  }
  __syncthreads();
  HS_FUSED_UNROLL
  for (int k = threadIdx.x; k < kBY * kBX; k += 256) {   // u5, tile
    const int ly = k / kBX, lx = k - ly * kBX;
    const int g1 = t1 + ly, g2 = t2 + lx;
    if (g1 >= n1 || g2 >= n2) continue;
    const int64_t i = (int64_t)g1 * n2 + g2;
    const double2 acc = apply_at<S>(d, i, g1, g2, U4, kR1X, ly + 1, lx + 1);
    const double2 fi = __ldg(f + i), inv = __ldg(d.invd + i);
    u[i] = cadd(U4[(ly + 1) * kR1X + lx + 1], cmul(cscale(omega, csub(fi, acc)), inv));
  }
}

}  // namespace

bool fused2d_ok(const Stencil* op, const Transfer* t, int nu) {
  const StencilDesc& d = op->d;
  if (nu != 2 || op->dim != 2 || d.n0 != 1 || d.diag < 0 || op->has_zero_diag || !d.invd) return false;
  if (d.S != 5 && d.S != 9) return false;
  for (int s = 0; s < d.S; ++s)
    if (d.off[s][0] != 0) return false;
  if (d.n >= ((int64_t)1 << 31)) return false;
  if (t) {
    const TransferDesc& q = t->d;
    for (int a = 0; a < 3; ++a)
      if (q.fw_lo[a] != 0 || q.fw_cnt[a] != q.nf[a] || q.fr_lo[a] != 0 || q.fr_cnt[a] != q.nf[a])
        return false;
    if (q.nf[0] != 1 || q.nf[1] != d.n1 || q.nf[2] != d.n2) return false;
  }
  return true;
}

int stencil_pre2d(Ctx* c, const Stencil* op, const double2* f, double2* u2, double2* r,
                  double omega) {
  const StencilDesc& d = op->d;
  dim3 grid((unsigned)((d.n2 + kBX - 1) / kBX), (unsigned)((d.n1 + kBY - 1) / kBY));
  // algorithmic bytes: f, 1/d, coefficients once; u2 and r written
  ProfScope ps(c, K_PRE_FUSED, (double)d.n * (16.0 * d.S + 16.0 + 8.0 + 32.0));
  if (d.S == 5) k_pre2d<5><<<grid, 256, 0, c->stream>>>(d, f, u2, r, omega);
  else k_pre2d<9><<<grid, 256, 0, c->stream>>>(d, f, u2, r, omega);
  HS_LAUNCH_CHECK(c, "fused pre-smoothing kernel");
  return HS_OK;
}

int stencil_post2d(Ctx* c, const Stencil* op, const Transfer* t, const double2* uc,
                   const double2* f, const double2* u2, double2* u, double omega) {
  const StencilDesc& d = op->d;
  dim3 grid((unsigned)((d.n2 + kBX - 1) / kBX), (unsigned)((d.n1 + kBY - 1) / kBY));
  const double nc = (double)(t->d.nc[0] * t->d.nc[1] * t->d.nc[2]);
  // algorithmic bytes: u2, f, 1/d, coefficients, uc once; u written
  ProfScope ps(c, K_POST_FUSED, (double)d.n * (16.0 * d.S + 16.0 + 16.0 + 8.0 + 16.0) + 16.0 * nc);
  if (d.S == 5) k_post2d<5><<<grid, 256, 0, c->stream>>>(d, t->d, uc, f, u2, u, omega);
  else k_post2d<9><<<grid, 256, 0, c->stream>>>(d, t->d, uc, f, u2, u, omega);
  HS_LAUNCH_CHECK(c, "fused post-smoothing kernel");
  return HS_OK;
}

}  // namespace hs
