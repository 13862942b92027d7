// 3-D coarse sweep (SURVEY §8 A9/A11 for 3-D levels, config C5).
//
// A 3-D slab (T layers x n1 x n2 face, 27-point operator) is block
// tridiagonal along face axis 1: block i1 holds the T*n2 unknowns (t, i2)
// of plane i1 (NB = T*n2, up to ~1000).  Setup factorises every slab by
// block LU along i1 with dense NB x NB blocks (cuSOLVER getrf/getrs for the
// pivot blocks, cuBLAS ZGEMM for the Schur updates):
//   D'_0 = D_0,  D'_i = D_i - L_i X_{i-1},  Dinv_i = D'_i^{-1},  X_i = Dinv_i U_i,
// so a slab solve (subdom_solve's LU_j^{-1}, sweepdd.py:236-268) is
//   y_i = Dinv_i (f_i - L_i y_{i-1})   (L_i applied from the stencil coefficients)
//   x_i = y_i - X_i x_{i+1}.
// Storage: 2 dense blocks per plane (C5: ~2.5 GB per slab, 71 GB in all).
// Right-hand side (restriction rows + the 9-offset transmission terms of
// TransmissionMatrix.apply, sweepdd.py:98-141) and the output scatter are
// small kernels; the schedules (tasks, traces) are shared with the 2-D sweep.

#include "hs_common.cuh"
#include "hs_sweep.cuh"

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <array>
#include <vector>

namespace hs {

struct Sweep3 {
  int n1 = 0, n2 = 0;
  std::vector<int> T;                  // slab thickness
  std::vector<double2*> dinv, xf;      // per slab: [n1][NB^2], [n1-1][NB^2] (column-major)
  std::vector<double2*> coef;          // per slab: stencil coefficients [S][T n1 n2] (owned copy)
  std::vector<std::array<int, 27>> slot;   // per slab: (o0+1)*9 + (o1+1)*3 + (o2+1) -> slot
  std::array<int, 27> cslot{};         // coarse operator slots
  cublasHandle_t blas = nullptr;
  double2* F = nullptr;                // [n1][NBmax] right-hand side / forward solution
  double2* W = nullptr;                // [NBmax] work
  long long bytes = 0;
};

namespace {

constexpr int kT3 = 256;

__host__ __device__ inline int oid(int o0, int o1, int o2) { return (o0 + 1) * 9 + (o1 + 1) * 3 + (o2 + 1); }

struct Slots { int s[27]; };

// dense block (o1 = -1, 0, +1 of plane i1) of a slab, column-major NB x NB:
// row (t, i2) couples to column (t + o0, i2 + o2) of plane i1 + o1
__global__ void k3_block(const double2* __restrict__ coef, Slots sl, int T, int n1, int n2, int i1,
                         int o1, double2* __restrict__ A) {
  const int NB = T * n2;
  const int r = blockIdx.x * kT3 + threadIdx.x;
  if (r >= NB) return;
  const int t = r / n2, i2 = r - t * n2;
  const int64_t n = (int64_t)T * n1 * n2;
  if (i1 + o1 < 0 || i1 + o1 >= n1) return;
  for (int o0 = -1; o0 <= 1; ++o0)
    for (int o2 = -1; o2 <= 1; ++o2) {
      const int s = sl.s[oid(o0, o1, o2)];
      if (s < 0 || t + o0 < 0 || t + o0 >= T || i2 + o2 < 0 || i2 + o2 >= n2) continue;
      const int c = (t + o0) * n2 + (i2 + o2);
      A[r + (int64_t)c * NB] = coef[(int64_t)s * n + ((int64_t)t * n1 + i1) * n2 + i2];
    }
}

__global__ void k3_eye(double2* __restrict__ A, int NB) {
  const int64_t i = (int64_t)blockIdx.x * kT3 + threadIdx.x;
  if (i >= (int64_t)NB * NB) return;
  A[i] = make_double2(i % NB == i / NB ? 1.0 : 0.0, 0.0);
}

// F[i1][t n2 + i2] = restriction rows of src + transmission terms (subdom_solve steps 1-2)
__global__ void k3_rhs(SweepTask t, int n0, int n1, int n2, const double2* __restrict__ src,
                       const double2* __restrict__ cco, int64_t cn, Slots cs,
                       const double2* __restrict__ trace, double2* __restrict__ F) {
  const int NB = t.T * n2;
  const int64_t e = (int64_t)blockIdx.x * kT3 + threadIdx.x;
  if (e >= (int64_t)n1 * NB) return;
  const int i1 = (int)(e / NB), r = (int)(e - (int64_t)i1 * NB);
  const int x = r / n2, i2 = r - x * n2;
  const int64_t M = (int64_t)n1 * n2;
  const int gr = x + t.lo - 1;
  double2 v = make_double2(0.0, 0.0);
  if (gr >= t.a && gr < t.b) v = src[(int64_t)gr * M + (int64_t)i1 * n2 + i2];
  for (int k = 0; k < 2; ++k) {
    const int buf = k ? t.tin3 : t.tin1, row = k ? t.row3 : t.row1;
    const double sign = k ? -1.0 : 1.0;
    if (buf < 0 || (x != row && x != row + 1)) continue;
    const int which = x - row, p = row + t.lo;
    const int o0 = which == 0 ? 1 : -1, crow = which == 0 ? p - 1 : p;
    const double2* Bt = trace + (int64_t)buf * 2 * M + (which == 0 ? M : 0);
    double2 acc = make_double2(0.0, 0.0);
    for (int o1 = -1; o1 <= 1; ++o1)
      for (int o2 = -1; o2 <= 1; ++o2) {
        const int s = cs.s[oid(o0, o1, o2)];
        if (s < 0 || i1 + o1 < 0 || i1 + o1 >= n1 || i2 + o2 < 0 || i2 + o2 >= n2) continue;
        const double2 c = cco[(int64_t)s * cn + (int64_t)crow * M + (int64_t)i1 * n2 + i2];
        acc = cfma(c, Bt[(int64_t)(i1 + o1) * n2 + (i2 + o2)], acc);
      }
    v = cadd(v, cscale(which == 0 ? sign : -sign, acc));
  }
  F[(int64_t)i1 * NB + r] = v;
}

// W = F_i1 - L_i1 y_{i1-1}   (L from the stencil's o1 = -1 offsets)
__global__ void k3_lsub(const double2* __restrict__ coef, Slots sl, int T, int n1, int n2, int i1,
                        const double2* __restrict__ Fi, const double2* __restrict__ yprev,
                        double2* __restrict__ W) {
  const int NB = T * n2;
  const int r = blockIdx.x * kT3 + threadIdx.x;
  if (r >= NB) return;
  const int t = r / n2, i2 = r - t * n2;
  const int64_t n = (int64_t)T * n1 * n2;
  double2 acc = Fi[r];
  if (i1 > 0)
    for (int o0 = -1; o0 <= 1; ++o0)
      for (int o2 = -1; o2 <= 1; ++o2) {
        const int s = sl.s[oid(o0, -1, o2)];
        if (s < 0 || t + o0 < 0 || t + o0 >= T || i2 + o2 < 0 || i2 + o2 >= n2) continue;
        const double2 c = coef[(int64_t)s * n + ((int64_t)t * n1 + i1) * n2 + i2];
        acc = csub(acc, cmul(c, yprev[(t + o0) * n2 + (i2 + o2)]));
      }
  W[r] = acc;
}

// u rows [ta, tb) and the outgoing traces (subdom_solve steps 4-5)
__global__ void k3_out(SweepTask t, int n1, int n2, const double2* __restrict__ X,
                       double2* __restrict__ u, double2* __restrict__ trace) {
  const int NB = t.T * n2;
  const int64_t e = (int64_t)blockIdx.x * kT3 + threadIdx.x;
  if (e >= (int64_t)n1 * NB) return;
  const int i1 = (int)(e / NB), r = (int)(e - (int64_t)i1 * NB);
  const int x = r / n2, i2 = r - x * n2;
  const int64_t M = (int64_t)n1 * n2, f = (int64_t)i1 * n2 + i2;
  const double2 v = X[e];
  if (x >= t.ta + 1 - t.lo && x < t.tb + 1 - t.lo) u[(int64_t)(x + t.lo - 1) * M + f] = v;
  if (t.out2 >= 0 && (x == t.orow2 || x == t.orow2 + 1))
    trace[((int64_t)t.out2 * 2 + (x - t.orow2)) * M + f] = v;
  if (t.out4 >= 0 && (x == t.orow4 || x == t.orow4 + 1))
    trace[((int64_t)t.out4 * 2 + (x - t.orow4)) * M + f] = v;
}

Slots to_slots(const std::array<int, 27>& a) {
  Slots s;
  for (int i = 0; i < 27; ++i) s.s[i] = a[i];
  return s;
}

int slots3(const Stencil* op, std::array<int, 27>& a, Ctx* c) {
  a.fill(-1);
  for (int s = 0; s < op->d.S; ++s) {
    const int o0 = op->d.off[s][0], o1 = op->d.off[s][1], o2 = op->d.off[s][2];
    if (o0 < -1 || o0 > 1 || o1 < -1 || o1 > 1 || o2 < -1 || o2 > 1)
      return set_error(c, HS_E_SHAPE, "3-D sweep needs compact 27-point operators");
    a[oid(o0, o1, o2)] = s;
  }
  return HS_OK;
}

#define S3_TRY(expr, what)                                                   \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) return check_cuda(c, _e, what);                   \
  } while (0)
#define S3_BLAS(expr, what)                                                  \
  do {                                                                       \
    if ((expr) != 0) return set_error(c, HS_E_CUDA, std::string(what) + " failed"); \
  } while (0)

}  // namespace

void sweep3_destroy(Sweep3* s3) {
  if (!s3) return;
  for (auto* p : s3->dinv) cudaFree(p);
  for (auto* p : s3->xf) cudaFree(p);
  for (auto* p : s3->coef) cudaFree(p);
  cudaFree(s3->F);
  cudaFree(s3->W);
  if (s3->blas) cublasDestroy(s3->blas);
  delete s3;
}

// Factorise every slab (block LU along face axis 1).  `s` already holds J,
// n0, M and the schedules.
int sweep3_create(Ctx* c, Sweep* s, const Stencil* coarse, const Stencil* const* slabs,
                  const int64_t* lo, const int64_t* hi) {
  Sweep3* s3 = new Sweep3();
  s->s3 = s3;
  s3->n1 = (int)coarse->shape[1];
  s3->n2 = (int)coarse->shape[2];
  const int J = s->J, n1 = s3->n1, n2 = s3->n2;
  if (int r = slots3(coarse, s3->cslot, c)) return r;
  if (cublasCreate(&s3->blas) != CUBLAS_STATUS_SUCCESS)
    return set_error(c, HS_E_CUDA, "cublasCreate failed");
  cusolverDnHandle_t sol = nullptr;
  if (cusolverDnCreate(&sol) != CUSOLVER_STATUS_SUCCESS)
    return set_error(c, HS_E_CUDA, "cusolverDnCreate failed");
  cublasSetStream(s3->blas, c->stream);
  cusolverDnSetStream(sol, c->stream);
  int NBmax = 0;
  for (int j = 0; j < J; ++j) NBmax = std::max(NBmax, (int)(hi[j] - lo[j] + 1) * n2);
  double2 *D = nullptr, *Lb = nullptr, *U = nullptr, *work = nullptr;
  int *ipiv = nullptr, *info = nullptr;
  const size_t blk = (size_t)NBmax * NBmax * sizeof(double2);
  int lwork = 0;
  auto done = [&](int rc) {
    cudaFree(D); cudaFree(Lb); cudaFree(U); cudaFree(work); cudaFree(ipiv); cudaFree(info);
    if (sol) cusolverDnDestroy(sol);
    return rc;
  };
  if (cudaMalloc((void**)&D, blk) || cudaMalloc((void**)&Lb, blk) || cudaMalloc((void**)&U, blk) ||
      cudaMalloc((void**)&ipiv, NBmax * sizeof(int)) ||
      cudaMalloc((void**)&info, (size_t)n1 * J * sizeof(int)) ||
      cudaMalloc((void**)&s3->F, (size_t)n1 * NBmax * sizeof(double2)) ||
      cudaMalloc((void**)&s3->W, (size_t)NBmax * sizeof(double2)))
    return done(set_error(c, HS_E_CUDA, "3-D sweep work allocation failed"));
  if (cusolverDnZgetrf_bufferSize(sol, NBmax, NBmax, (cuDoubleComplex*)D, NBmax, &lwork) != 0 ||
      cudaMalloc((void**)&work, (size_t)std::max(1, lwork) * sizeof(double2)))
    return done(set_error(c, HS_E_CUDA, "getrf workspace failed"));
  cudaMemsetAsync(info, 0, (size_t)n1 * J * sizeof(int), c->stream);
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), mone = make_cuDoubleComplex(-1.0, 0.0),
                        zero = make_cuDoubleComplex(0.0, 0.0);
  s3->T.resize(J);
  s3->slot.resize(J);
  for (int j = 0; j < J; ++j) {
    const Stencil* op = slabs[j];
    const int T = (int)(hi[j] - lo[j] + 1), NB = T * n2;
    if (op->dim != 3 || op->shape[0] != T || op->shape[1] != n1 || op->shape[2] != n2)
      return done(set_error(c, HS_E_SHAPE, "slab operator shape does not match the partition"));
    s3->T[j] = T;
    if (int r = slots3(op, s3->slot[j], c)) return done(r);
    double2* cf = nullptr;
    const size_t cb = (size_t)op->d.S * op->d.n * sizeof(double2);
    S3_TRY(cudaMalloc((void**)&cf, cb), "slab coefficients");
    s3->coef.push_back(cf);
    S3_TRY(cudaMemcpyAsync(cf, op->d.coeffs, cb, cudaMemcpyDeviceToDevice, c->stream), "copy");
    double2 *dv = nullptr, *xv = nullptr;
    const size_t nb2 = (size_t)NB * NB;
    S3_TRY(cudaMalloc((void**)&dv, n1 * nb2 * sizeof(double2)), "3-D slab factors (Dinv)");
    s3->dinv.push_back(dv);
    S3_TRY(cudaMalloc((void**)&xv, std::max(1, n1 - 1) * nb2 * sizeof(double2)),
           "3-D slab factors (X)");
    s3->xf.push_back(xv);
    s3->bytes += (long long)(2 * n1 - 1) * nb2 * sizeof(double2);
    const Slots sl = to_slots(s3->slot[j]);
    const unsigned gb = (unsigned)((NB + kT3 - 1) / kT3);
    for (int i1 = 0; i1 < n1; ++i1) {
      double2* Di = dv + i1 * nb2;
      S3_TRY(cudaMemsetAsync(D, 0, nb2 * sizeof(double2), c->stream), "memset");
      k3_block<<<gb, kT3, 0, c->stream>>>(cf, sl, T, n1, n2, i1, 0, D);
      c->launches++;
      if (i1 > 0) {   // D' = D - L_i X_{i-1}
        S3_TRY(cudaMemsetAsync(Lb, 0, nb2 * sizeof(double2), c->stream), "memset");
        k3_block<<<gb, kT3, 0, c->stream>>>(cf, sl, T, n1, n2, i1, -1, Lb);
        c->launches++;
        S3_BLAS(cublasZgemm(s3->blas, CUBLAS_OP_N, CUBLAS_OP_N, NB, NB, NB, &mone,
                            (cuDoubleComplex*)Lb, NB, (cuDoubleComplex*)(xv + (i1 - 1) * nb2), NB,
                            &one, (cuDoubleComplex*)D, NB), "zgemm");
      }
      // Dinv = D'^{-1} (partial pivoting inside the block)
      S3_BLAS(cusolverDnZgetrf(sol, NB, NB, (cuDoubleComplex*)D, NB, (cuDoubleComplex*)work, ipiv,
                               info + j * n1 + i1), "getrf");
      k3_eye<<<(unsigned)((nb2 + kT3 - 1) / kT3), kT3, 0, c->stream>>>(Di, NB);
      c->launches++;
      S3_BLAS(cusolverDnZgetrs(sol, CUBLAS_OP_N, NB, NB, (cuDoubleComplex*)D, NB, ipiv,
                               (cuDoubleComplex*)Di, NB, info + j * n1 + i1), "getrs");
      if (i1 + 1 < n1) {   // X_i = Dinv_i U_i
        S3_TRY(cudaMemsetAsync(U, 0, nb2 * sizeof(double2), c->stream), "memset");
        k3_block<<<gb, kT3, 0, c->stream>>>(cf, sl, T, n1, n2, i1, 1, U);
        c->launches++;
        S3_BLAS(cublasZgemm(s3->blas, CUBLAS_OP_N, CUBLAS_OP_N, NB, NB, NB, &one,
                            (cuDoubleComplex*)Di, NB, (cuDoubleComplex*)U, NB, &zero,
                            (cuDoubleComplex*)(xv + i1 * nb2), NB), "zgemm");
      }
    }
    S3_TRY(cudaGetLastError(), "3-D factor kernels");
  }
  std::vector<int> hinfo((size_t)n1 * J);
  S3_TRY(cudaMemcpyAsync(hinfo.data(), info, hinfo.size() * sizeof(int), cudaMemcpyDeviceToHost,
                         c->stream), "info");
  S3_TRY(cudaStreamSynchronize(c->stream), "3-D factor sync");
  for (int j = 0; j < J; ++j)
    for (int i1 = 0; i1 < n1; ++i1)
      if (hinfo[(size_t)j * n1 + i1] > 0) {
        const long long row = (long long)i1 * s3->T[j] * n2 + hinfo[(size_t)j * n1 + i1] - 1;
        char buf[128];
        snprintf(buf, sizeof buf, "zero pivot at row %lld (slab %d)", row, j + 1);
        return done(set_error(c, HS_E_ZERO_PIVOT, buf, row));
      }
  s->factor_bytes = s3->bytes;
  return done(HS_OK);
}

// One slab solve of the schedule (subdom_solve, sweepdd.py:236-268).
int sweep3_task(Ctx* c, Sweep* s, const SweepTask& t, const double2* src, double2* const* u,
                const double2* coarse_coeffs, int64_t coarse_n) {
  Sweep3* s3 = s->s3;
  const int n1 = s3->n1, n2 = s3->n2, j = t.slab, T = s3->T[j], NB = T * n2;
  const size_t nb2 = (size_t)NB * NB;
  cublasSetStream(s3->blas, c->stream);
  const Slots sl = to_slots(s3->slot[j]);
  const int64_t tot = (int64_t)n1 * NB;
  k3_rhs<<<(unsigned)((tot + kT3 - 1) / kT3), kT3, 0, c->stream>>>(
      t, s->n0, n1, n2, src, coarse_coeffs, coarse_n, to_slots(s3->cslot), s->trace, s3->F);
  HS_LAUNCH_CHECK(c, "3-D rhs");
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), mone = make_cuDoubleComplex(-1.0, 0.0),
                        zero = make_cuDoubleComplex(0.0, 0.0);
  const unsigned gb = (unsigned)((NB + kT3 - 1) / kT3);
  for (int i1 = 0; i1 < n1; ++i1) {   // y_i = Dinv_i (f_i - L_i y_{i-1})
    double2* Fi = s3->F + (int64_t)i1 * NB;
    k3_lsub<<<gb, kT3, 0, c->stream>>>(s3->coef[j], sl, T, n1, n2, i1, Fi,
                                        i1 ? Fi - NB : nullptr, s3->W);
    HS_LAUNCH_CHECK(c, "3-D forward");
    S3_BLAS(cublasZgemv(s3->blas, CUBLAS_OP_N, NB, NB, &one,
                        (const cuDoubleComplex*)(s3->dinv[j] + i1 * nb2), NB,
                        (const cuDoubleComplex*)s3->W, 1, &zero, (cuDoubleComplex*)Fi, 1), "zgemv");
    c->launches++;
  }
  for (int i1 = n1 - 2; i1 >= 0; --i1) {   // x_i = y_i - X_i x_{i+1}
    double2* Fi = s3->F + (int64_t)i1 * NB;
    S3_BLAS(cublasZgemv(s3->blas, CUBLAS_OP_N, NB, NB, &mone,
                        (const cuDoubleComplex*)(s3->xf[j] + i1 * nb2), NB,
                        (const cuDoubleComplex*)(Fi + NB), 1, &one, (cuDoubleComplex*)Fi, 1),
            "zgemv");
    c->launches++;
  }
  k3_out<<<(unsigned)((tot + kT3 - 1) / kT3), kT3, 0, c->stream>>>(t, n1, n2, s3->F, u[t.dst],
                                                                   s->trace);
  HS_LAUNCH_CHECK(c, "3-D outputs");
  return HS_OK;
}

}  // namespace hs
