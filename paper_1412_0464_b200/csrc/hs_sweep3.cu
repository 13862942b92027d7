// 3-D coarse sweep (SURVEY §8 A9/A11 for 3-D levels, config C5).
//
// A 3-D slab (T layers x n1 x n2 face, 27-point operator) is block
// tridiagonal along face axis 1: block i1 holds the T*n2 unknowns (t, i2)
// of plane i1 (NB = T*n2, up to ~1000).  Setup factorises every slab by
// block LU along i1 with dense NB x NB blocks (cuSOLVER getrf/getrs for the
// pivot blocks, cuBLAS ZGEMM for the Schur updates):
//   D'_0 = D_0,  D'_i = D_i - L_i X_{i-1},  Dinv_i = D'_i^{-1},  X_i = Dinv_i U_i,
// so a slab solve (subdom_solve's LU_j^{-1}, sweepdd.py:236-268) is
//   y_i = Dinv_i (f_i - L_i y_{i-1}) = w_i - G_i y_{i-1},  w_i = Dinv_i f_i,  G_i = Dinv_i L_i
//   x_i = y_i - X_i x_{i+1}.
// w for every plane is one batched GEMV ahead of the chain (independent of
// it); the chain is then one dense GEMV per plane in both directions.
// Storage: 3 dense blocks per plane (C5: ~3 GB per slab, 86 GB in all).
// Right-hand side (restriction rows + the 9-offset transmission terms of
// TransmissionMatrix.apply, sweepdd.py:98-141) and the output scatter are
// small kernels; the schedules (tasks, traces) are shared with the 2-D sweep.

#include "hs_common.cuh"
#include "hs_sweep.cuh"

#include "hs_dense.cuh"

#include <algorithm>
#include <array>
#include <vector>

#ifndef HS_S3_EXP   // timing experiments: 1 no GEMV, 2 no rhs stencil, 4 no grid barrier
#define HS_S3_EXP 0
#endif

namespace hs {

struct Sweep3 {
  int n1 = 0, n2 = 0;
  std::vector<int> T;                  // slab thickness
  std::vector<double2*> dinv, xf, gf;  // per slab: [n1][NB^2], [n1-1][NB^2], [n1][NB^2] (row-major;
                                       // gf[0] unused: G_i = Dinv_i L_i for i >= 1)
  std::vector<double2*> coef;          // per slab: stencil coefficients [S][T n1 n2] (owned copy)
  std::vector<std::array<int, 27>> slot;   // per slab: (o0+1)*9 + (o1+1)*3 + (o2+1) -> slot
  std::array<int, 27> cslot{};         // coarse operator slots
  double2* F[2] = {nullptr, nullptr};  // per concurrent chain: [nrcap][n1][NBmax] right-hand side
  double2* Y[2] = {nullptr, nullptr};  // [nrcap][n1][NBmax] forward solution, then x
  int nrcap = 1;                       // right-hand sides F / Y hold (grown by sweep3_reserve)
  unsigned* gbar = nullptr;            // [2] grid barrier counters of the solve kernel
  int optin = 0;                       // opt-in shared memory per block
  int grid = 0;                        // CTAs of the solve kernel (one per SM)
  int nbuf = 1;                        // staging buffers of the solve kernel
  int nbmax = 0;                       // largest plane block
  int gemv_grid = 0;                   // resident CTAs of k3_gemv (set on first use)
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

// dense block (o1 = -1, 0, +1 of block row i1) of a general sparse matrix
// given in CSR, as the exact solver of factorize(scipy matrix) sees it: a
// banded matrix cut into NB x NB blocks is block tridiagonal (NB >= the
// bandwidth).  Rows past n (padding of the last block) are identity rows.
// One thread per row of the block (no write races); duplicates summed.
__global__ void k3_csr_block(const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices,
                             const double2* __restrict__ vals, int64_t n, int NB, int n1, int i1,
                             int o1, double2* __restrict__ A) {
  const int r = blockIdx.x * kT3 + threadIdx.x;
  if (r >= NB || i1 + o1 < 0 || i1 + o1 >= n1) return;
  const int64_t row = (int64_t)i1 * NB + r;
  if (row >= n) {
    if (o1 == 0) A[r + (int64_t)r * NB] = make_double2(1.0, 0.0);
    return;
  }
  const int64_t cb0 = (int64_t)(i1 + o1) * NB;
  for (int64_t e = indptr[row]; e < indptr[row + 1]; ++e) {
    const int64_t col = indices[e] - cb0;
    if (col < 0 || col >= NB) continue;
    double2& a = A[r + col * NB];
    a = cadd(a, vals[e]);
  }
}


// F[i1][t n2 + i2] = restriction rows of src + transmission terms (subdom_solve steps 1-2)
// (blockIdx.y: the right-hand side; its vectors at src + y * vs_src, trace +
// y * ts, F + y * fs)
__global__ void k3_rhs(SweepTask t, int n0, int n1, int n2, const double2* __restrict__ src,
                       const double2* __restrict__ cco, int64_t cn, Slots cs,
                       const double2* __restrict__ trace, double2* __restrict__ F,
                       int64_t vs_src, int64_t ts, int64_t fs) {
  const int NB = t.T * n2;
  const int64_t e = (int64_t)blockIdx.x * kT3 + threadIdx.x;
  if (e >= (int64_t)n1 * NB) return;
  src += blockIdx.y * vs_src;
  trace += blockIdx.y * ts;
  F += blockIdx.y * fs;
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

// w_i = Dinv_i f_i for every plane i1 (row-major Dinv) of one or two slab
// solves (the two fronts' tasks): the slab solve's first step, independent
// of the block recursion.  Persistent grid (a whole number of resident
// waves) striding over (task, plane, 32-row block) items -- a launch of one
// CTA per item left a 20%-full third wave; each warp owns 4 rows (4
// independent accumulators, 16-B lane loads of contiguous row segments), the
// plane's f is staged in shared memory.  HBM-bound: n1 NB^2 16 B per task.
// Fixed reduction order (bitwise reproducible, the same sums as before).
constexpr int kGvRows = 32;
// NR right-hand sides (template): the plane's NR vectors f + q * fs are staged
// together and every matrix element is loaded once for all of them; per
// right-hand side the sums are the single kernel's (bitwise the same).
struct GemvTask {
  const double2* Dinv;
  const double2* F;
  double2* Y;
  int NB, nrb;   // rows per plane, 32-row blocks per plane
};
template <int NR>
__global__ void __launch_bounds__(256) k3_gemv(GemvTask t0, GemvTask t1, int n1, int64_t items0,
                                              int64_t items, int64_t fs) {
  extern __shared__ __align__(16) double2 fv[];   // [NR][NB]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const bool second = it >= items0;
    const GemvTask& t = second ? t1 : t0;
    const int64_t loc = second ? it - items0 : it;
    const int i1 = (int)(loc / t.nrb), rb = (int)(loc - (int64_t)i1 * t.nrb);
    const int NB = t.NB;
    const int64_t nb2 = (int64_t)NB * NB;
    __syncthreads();   // the previous item's readers of fv are done
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const double2* f = t.F + q * fs + (int64_t)i1 * NB;
      for (int c = threadIdx.x; c < NB; c += blockDim.x) fv[q * NB + c] = __ldg(f + c);
    }
    __syncthreads();
    const int r0 = rb * kGvRows + warp * 4;
    const double2* A = t.Dinv + (int64_t)i1 * nb2;
    double2 acc[4][NR];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < NR; ++q) acc[k][q] = czero();
    const int nr = max(0, min(4, NB - r0));
    if (nr == 4) {
      const double2* a0 = A + (int64_t)r0 * NB;
      for (int c = lane; c < NB; c += 32) {
        const double2 m0 = __ldcs(a0 + c), m1 = __ldcs(a0 + NB + c);
        const double2 m2 = __ldcs(a0 + 2 * NB + c), m3 = __ldcs(a0 + 3 * NB + c);
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const double2 v = fv[q * NB + c];
          acc[0][q] = cfma(m0, v, acc[0][q]);
          acc[1][q] = cfma(m1, v, acc[1][q]);
          acc[2][q] = cfma(m2, v, acc[2][q]);
          acc[3][q] = cfma(m3, v, acc[3][q]);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= nr) break;
        const double2* ar = A + (int64_t)(r0 + k) * NB;
        for (int c = lane; c < NB; c += 32) {
          const double2 m = __ldcs(ar + c);
#pragma unroll
          for (int q = 0; q < NR; ++q) acc[k][q] = cfma(m, fv[q * NB + c], acc[k][q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        for (int m = 16; m > 0; m >>= 1) acc[k][q] = cadd(acc[k][q], shfl_xor_c(acc[k][q], m));
      // (lane k stores row k: pick it without a dynamically indexed register array)
      double2 mine = acc[0][q];
      if (lane == 1) mine = acc[1][q];
      if (lane == 2) mine = acc[2][q];
      if (lane == 3) mine = acc[3][q];
      if (lane < nr) t.Y[q * fs + (int64_t)i1 * NB + r0 + lane] = mine;
    }
  }
}

// u rows [ta, tb) and the outgoing traces (subdom_solve steps 4-5)
__global__ void k3_out(SweepTask t, int n1, int n2, const double2* __restrict__ X,
                       double2* __restrict__ u, double2* __restrict__ trace, int64_t fs,
                       int64_t vs_u, int64_t ts) {
  const int NB = t.T * n2;
  const int64_t e = (int64_t)blockIdx.x * kT3 + threadIdx.x;
  if (e >= (int64_t)n1 * NB) return;
  X += blockIdx.y * fs;
  u += blockIdx.y * vs_u;
  trace += blockIdx.y * ts;
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

// ---- the whole block recursion of one slab solve in one cooperative launch:
// every CTA rebuilds the step's right-hand vector in shared memory and owns
// rows r = blockIdx.x + k * gridDim.x of every plane's dense block.  Those
// rows do not depend on the chain, so they are staged by TMA bulk copies
// (one per row, completing on an mbarrier) into shared memory one plane
// ahead: the copy of plane i+1's rows is issued as soon as plane i's GEMV
// has read its buffer and lands while the CTA writes its rows, crosses the
// grid barrier and rebuilds the next right-hand vector.  The GEMV then reads
// shared memory only.  Grid barrier split into arrive / wait.
constexpr int kW3 = 16;   // warps per CTA

__device__ __forceinline__ uint32_t s3_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void s3_mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(s3_smem(bar)), "r"(phase)
        : "memory");
  }
}

#ifndef HS_S3_RED
#define HS_S3_RED 1
#endif
__device__ __forceinline__ void barrier_arrive(unsigned* bar) {
  __syncthreads();
  if (HS_S3_EXP & 4) return;
  if (threadIdx.x == 0) {
    if (HS_S3_RED) {   // release-add: orders the CTA's writes (bar.sync + cumulativity)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    } else {
      __threadfence();
      atomicAdd(bar, 1u);
    }
  }
}
__device__ __forceinline__ void barrier_wait(unsigned* bar, unsigned target) {
  if (!(HS_S3_EXP & 4) && threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar));
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// this CTA's rows of a plane matrix -> shared memory (thread 0; one bulk copy per row)
__device__ __forceinline__ void stage_rows(const double2* __restrict__ A, int NB, int nrow,
                                           double2* dst, uint64_t* bar, int lb, int G) {
  const uint32_t bytes = (uint32_t)NB * 16u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s3_smem(bar)),
               "r"(bytes * (uint32_t)nrow)
               : "memory");
  for (int k = 0; k < nrow; ++k) {
    const double2* src = A + (int64_t)(lb + k * G) * NB;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(s3_smem(dst + (int64_t)k * NB)), "l"(src), "r"(bytes), "r"(s3_smem(bar))
        : "memory");
  }
}

constexpr int kR3 = 16;  // rows per CTA at most (NB <= 16 * CTAs of the task)

// rows k < nrow of (staged rows) x v: (row, column segment) items go round
// the warps (4 independent partial sums per lane); partial sums land in
// acc[k][segment], summed in a fixed order by the caller: bitwise
// reproducible.  (A column-slice variant -- each warp all rows of a slice of
// v -- measured 12% slower at C5; 2 segments per row cost 0.7% over the
// earlier rows-per-CTA-dependent split, 4 segments 3.5%, 8 segments 24%.)
// Every row is cut into kSeg3 fixed column segments (boundaries depend on NB
// only): (row, segment) items go round the warps, so a row's sum does not
// depend on how many rows the CTA owns -- the same bits whether a chain runs
// alone on every CTA or paired on a CTA group, for any number of
// right-hand sides.
#ifndef HS_S3_SEG
#define HS_S3_SEG 2
#endif
constexpr int kSeg3 = HS_S3_SEG;
static_assert(kSeg3 >= 1 && kSeg3 <= kW3, "partial sums: kW3 slots per row");
// NR right-hand sides: vectors v + q * NB, sums acc + q * as; every staged
// matrix element is read once for all of them.
template <int NR>
__device__ __forceinline__ void cta_rows(const double2* A, const double2* v, int NB, int nrow,
                                         double2* acc, int as) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (nrow == 0 || (HS_S3_EXP & 1)) return;
  const int seg = (NB + kSeg3 - 1) / kSeg3;
  for (int it = warp; it < nrow * kSeg3; it += kW3) {
    const int k = it / kSeg3, part = it - k * kSeg3;
    const int c0 = part * seg, c1 = min(NB, c0 + seg);
    const double2* row = A + (int64_t)k * NB;
    double2 a0[NR], a1[NR], a2[NR], a3[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) a0[q] = a1[q] = a2[q] = a3[q] = czero();
    int c = c0 + lane;
    for (; c + 96 < c1; c += 128) {
      const double2 m0 = row[c], m1 = row[c + 32], m2 = row[c + 64], m3 = row[c + 96];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const double2* vq = v + q * NB;
        a0[q] = cfma(m0, vq[c], a0[q]);
        a1[q] = cfma(m1, vq[c + 32], a1[q]);
        a2[q] = cfma(m2, vq[c + 64], a2[q]);
        a3[q] = cfma(m3, vq[c + 96], a3[q]);
      }
    }
    for (; c < c1; c += 32) {
      const double2 m0 = row[c];
#pragma unroll
      for (int q = 0; q < NR; ++q) a0[q] = cfma(m0, v[q * NB + c], a0[q]);
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      double2 t = cadd(cadd(a0[q], a1[q]), cadd(a2[q], a3[q]));
      for (int m = 16; m > 0; m >>= 1) t = cadd(t, shfl_xor_c(t, m));
      if (lane == 0) acc[q * as + k * kSeg3 + part] = t;
    }
  }
}

// One chain of a slab solve: its slab thickness, factors, vector and grid
// barrier.  A launch runs one chain on every CTA or two independent chains
// (the two sweep fronts' slabs) on disjoint CTA groups [0, g0) and
// [g0, grid), each with its own barrier: the per-step latency (barrier,
// vector load) is paid once for both.
struct K3Chain {
  int T;
  const double2* gT;
  const double2* xT;
  double2* Y;
  unsigned* bar;
  int nbuf;
};

// NR right-hand sides per chain (template): Y + q * fs; the staged rows are
// shared, the step's vector and the partial sums hold NR copies.
template <int NR>
__global__ void __launch_bounds__(kW3 * 32, 1)
k3_solve(K3Chain c0, K3Chain c1, int g0, int n1, int n2, int64_t fs) {
  extern __shared__ __align__(128) double2 v3[];   // [NR][NB] vectors | [nbuf][rmax][NB] rows | sums
  const bool second = (int)blockIdx.x >= g0;
  const K3Chain& ch = second ? c1 : c0;
  const int lb = second ? (int)blockIdx.x - g0 : (int)blockIdx.x;   // CTA within the chain
  const int G = second ? (int)gridDim.x - g0 : g0;                 // CTAs of the chain
  const int T = ch.T, nbuf = ch.nbuf;
  const double2* __restrict__ gT = ch.gT;
  const double2* __restrict__ xT = ch.xT;
  double2* Y = ch.Y;
  unsigned* bar = ch.bar;
  const int NB = T * n2;
  const int64_t nb2 = (int64_t)NB * NB;
  const int nrow = lb < NB ? (NB - 1 - lb) / G + 1 : 0;
  const int rmax = (NB + G - 1) / G;
  double2* rows = v3 + NR * NB;                     // nbuf (1 or 2) staging buffers
  double2* racc = rows + nbuf * (int64_t)rmax * NB; // [NR][rows][warps per row] partial row sums
  uint64_t* rbar = (uint64_t*)(racc + NR * rmax * kW3);  // [2] staging barriers
  const int as = rmax * kW3;
  auto row_sum = [&](int q, int k) {
    double2 a = czero();
#pragma unroll
    for (int p = 0; p < kSeg3; ++p) a = cadd(a, racc[q * as + k * kSeg3 + p]);
    return a;
  };
  // step s: forward plane i = s + 1 (y_i = w_i - G_i y_{i-1}, Y_i holds w_i), then
  // back substitution plane i = 2 n1 - 3 - s (x_i = y_i - X_i x_{i+1})
  const int nsteps = 2 * (n1 - 1);
  auto mat = [&](int st) {
    return st < n1 - 1 ? gT + (int64_t)(st + 1) * nb2 : xT + (int64_t)(2 * n1 - 3 - st) * nb2;
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s3_smem(rbar)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s3_smem(rbar + 1)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && nrow > 0)   // nbuf steps ahead
    for (int st = 0; st < nbuf && st < nsteps; ++st)
      stage_rows(mat(st), NB, nrow, rows + (int64_t)st * rmax * NB, rbar + st, lb, G);
  for (int st = 0; st < nsteps; ++st) {
    const bool fwd = st < n1 - 1;
    const int i1 = fwd ? st + 1 : 2 * n1 - 3 - st;
    double2* Yi = Y + (int64_t)i1 * NB;
    const double2* Yin = fwd ? Yi - NB : Yi + NB;
    if (st > 0) barrier_wait(bar, (unsigned)st * G);
    if (!(HS_S3_EXP & 2)) {
#pragma unroll
      for (int q = 0; q < NR; ++q)
        for (int r = threadIdx.x; r < NB; r += blockDim.x) v3[q * NB + r] = __ldcg(Yin + q * fs + r);
    }
    __syncthreads();
    const int b = nbuf == 2 ? (st & 1) : 0;
    double2* buf = rows + (int64_t)b * rmax * NB;
    if (nrow > 0) s3_mbar_wait(rbar + b, (uint32_t)(st / nbuf) & 1);
    cta_rows<NR>(buf, v3, NB, nrow, racc, as);
    __syncthreads();   // this buffer is consumed: stage the step after next into it
    if (threadIdx.x == 0 && nrow > 0 && st + nbuf < nsteps)
      stage_rows(mat(st + nbuf), NB, nrow, buf, rbar + b, lb, G);
    for (int kk = threadIdx.x; kk < NR * nrow; kk += blockDim.x) {
      const int q = NR == 1 ? 0 : kk / nrow, k = kk - q * nrow;
      const int r = lb + k * G;
      Yi[q * fs + r] = csub(__ldcg(Yi + q * fs + r), row_sum(q, k));
    }
    barrier_arrive(bar);
  }
}

size_t k3_smem(int NB, int grid, int nbuf, int nr = 1) {
  const int rmax = (NB + grid - 1) / grid;
  return (size_t)((size_t)nr * NB + nbuf * (size_t)rmax * NB + (size_t)nr * rmax * kW3) *
             sizeof(double2) + 16;
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

}  // namespace

void sweep3_destroy(Sweep3* s3) {
  if (!s3) return;
  for (auto* p : s3->dinv) cudaFree(p);
  for (auto* p : s3->xf) cudaFree(p);
  for (auto* p : s3->gf) cudaFree(p);
  for (auto* p : s3->coef) cudaFree(p);
  for (int i = 0; i < 2; ++i) {
    cudaFree(s3->F[i]);
    cudaFree(s3->Y[i]);
  }
  cudaFree(s3->gbar);
  delete s3;
}

// Factorise every slab (block LU along face axis 1).  `s` already holds J,
// n0, M and the schedules.
int sweep3_create(Ctx* c, Sweep* s, const Stencil* coarse, const Stencil* const* slabs,
                  const int64_t* lo, const int64_t* hi, const CsrSource* csr) {
  Sweep3* s3 = new Sweep3();
  s->s3 = s3;
  s3->n1 = (int)coarse->shape[1];
  s3->n2 = (int)coarse->shape[2];
  const int J = s->J, n1 = s3->n1, n2 = s3->n2;
  if (int r = slots3(coarse, s3->cslot, c)) return r;
  int NBmax = 0;
  for (int j = 0; j < J; ++j) NBmax = std::max(NBmax, (int)(hi[j] - lo[j] + 1) * n2);
  s3->nbmax = NBmax;
  // the solve kernel's limits first (nothing is factorised for a plane it cannot solve)
  s3->grid = c->num_sms;
  int optin = 0;
  S3_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device),
         "smem attr");
  if ((NBmax + s3->grid - 1) / s3->grid > kR3 || k3_smem(NBmax, s3->grid, 1) > (size_t)optin)
    return set_error(c, HS_E_SHAPE, "3-D slab planes too large for the solve kernel");
  // per-slab work blocks (column-major NB x NB): D (factorised in place), L, U, Dinv
  std::vector<double2*> Dw(J, nullptr), Lw(J, nullptr), Uw(J, nullptr), Iw(J, nullptr);
  std::vector<int*> Pw(J, nullptr);
  int* info = nullptr;
  auto done = [&](int rc) {
    for (int j = 0; j < J; ++j) {
      cudaFree(Dw[j]); cudaFree(Lw[j]); cudaFree(Uw[j]); cudaFree(Iw[j]); cudaFree(Pw[j]);
    }
    cudaFree(info);
    return rc;
  };
  if (cudaMalloc((void**)&s3->gbar, 2 * sizeof(unsigned)) ||
      cudaMalloc((void**)&info, ((size_t)n1 * J + 1) * sizeof(int)) ||
      cudaMalloc((void**)&s3->F[0], (size_t)n1 * NBmax * sizeof(double2)) ||
      cudaMalloc((void**)&s3->Y[0], (size_t)n1 * NBmax * sizeof(double2)) ||
      cudaMalloc((void**)&s3->F[1], (size_t)n1 * NBmax * sizeof(double2)) ||
      cudaMalloc((void**)&s3->Y[1], (size_t)n1 * NBmax * sizeof(double2)))
    return done(set_error(c, HS_E_CUDA, "3-D sweep work allocation failed"));
  S3_TRY(cudaMemsetAsync(info, 0, (size_t)n1 * J * sizeof(int), c->stream), "memset");
  s3->T.resize(J);
  s3->slot.resize(J);
  // dense blocks of a slab: from its stencil coefficients, or (exact solve of
  // a general sparse matrix) from the CSR rows of the block row
  auto block = [&](const double2* cf, const Slots& sl, int T, int NB, int i1, int o1, double2* A) {
    const unsigned gb = (unsigned)((NB + kT3 - 1) / kT3);
    if (csr)
      k3_csr_block<<<gb, kT3, 0, c->stream>>>(csr->indptr, csr->indices, csr->vals, csr->n, NB, n1,
                                              i1, o1, A);
    else
      k3_block<<<gb, kT3, 0, c->stream>>>(cf, sl, T, n1, n2, i1, o1, A);
    c->launches++;
  };
  std::vector<int> NBs(J);
  for (int j = 0; j < J; ++j) {
    const Stencil* op = slabs[j];
    const int T = (int)(hi[j] - lo[j] + 1), NB = T * n2;
    if (op->dim != 3 || op->shape[0] != T || op->shape[1] != n1 || op->shape[2] != n2)
      return done(set_error(c, HS_E_SHAPE, "slab operator shape does not match the partition"));
    s3->T[j] = T;
    NBs[j] = NB;
    if (int r = slots3(op, s3->slot[j], c)) return done(r);
    double2* cf = nullptr;
    const size_t cb = (size_t)op->d.S * op->d.n * sizeof(double2);
    if (cb) {
      S3_TRY(cudaMalloc((void**)&cf, cb), "slab coefficients");
      S3_TRY(cudaMemcpyAsync(cf, op->d.coeffs, cb, cudaMemcpyDeviceToDevice, c->stream), "copy");
    }
    s3->coef.push_back(cf);
    double2 *dv = nullptr, *xv = nullptr, *gv = nullptr;
    const size_t nb2 = (size_t)NB * NB;
    S3_TRY(cudaMalloc((void**)&dv, n1 * nb2 * sizeof(double2)), "3-D slab factors (Dinv)");
    s3->dinv.push_back(dv);
    S3_TRY(cudaMalloc((void**)&xv, std::max(1, n1 - 1) * nb2 * sizeof(double2)),
           "3-D slab factors (X)");
    s3->xf.push_back(xv);
    S3_TRY(cudaMalloc((void**)&gv, n1 * nb2 * sizeof(double2)), "3-D slab factors (G)");
    s3->gf.push_back(gv);
    s3->bytes += (long long)(3 * n1 - 2) * nb2 * sizeof(double2);
    S3_TRY(cudaMalloc((void**)&Dw[j], nb2 * sizeof(double2)), "factor work");
    S3_TRY(cudaMalloc((void**)&Lw[j], nb2 * sizeof(double2)), "factor work");
    S3_TRY(cudaMalloc((void**)&Uw[j], nb2 * sizeof(double2)), "factor work");
    S3_TRY(cudaMalloc((void**)&Iw[j], nb2 * sizeof(double2)), "factor work");
    S3_TRY(cudaMalloc((void**)&Pw[j], (size_t)NB * sizeof(int)), "factor work");
  }
  // Block LU along the planes, every slab at once (hand-written batched dense
  // kernels, hs_dense.cu), per plane i:
  //   D' = D_i - L_i X_{i-1};  LU(D') with partial pivoting, Dinv_i = D'^{-1};
  //   G_i = Dinv_i L_i;  X_i = Dinv_i U_i   (all stored row-major)
  std::vector<GemmJob> gj;
  std::vector<LuJob> lj(J);
  std::vector<TransposeJob> tj(J);
  for (int i1 = 0; i1 < n1; ++i1) {
    for (int j = 0; j < J; ++j) {
      const int NB = NBs[j];
      const size_t nb2 = (size_t)NB * NB;
      const Slots sl = to_slots(s3->slot[j]);
      S3_TRY(cudaMemsetAsync(Dw[j], 0, nb2 * sizeof(double2), c->stream), "memset");
      block(s3->coef[j], sl, s3->T[j], NB, i1, 0, Dw[j]);
      if (i1 > 0) {
        S3_TRY(cudaMemsetAsync(Lw[j], 0, nb2 * sizeof(double2), c->stream), "memset");
        block(s3->coef[j], sl, s3->T[j], NB, i1, -1, Lw[j]);
      }
      if (i1 + 1 < n1) {
        S3_TRY(cudaMemsetAsync(Uw[j], 0, nb2 * sizeof(double2), c->stream), "memset");
        block(s3->coef[j], sl, s3->T[j], NB, i1, 1, Uw[j]);
      }
    }
    if (i1 > 0) {   // D' = D - L_i X_{i-1} (X_{i-1} stored row-major: op T)
      gj.clear();
      for (int j = 0; j < J; ++j) {
        const int NB = NBs[j];
        GemmJob q{};
        q.m = q.n = q.k = NB;
        q.A = Lw[j]; q.lda = NB;
        q.B = s3->xf[j] + (size_t)(i1 - 1) * NB * NB; q.ldb = NB; q.opB = 1;
        q.C = Dw[j]; q.ldc = NB;
        q.alpha = make_double2(-1.0, 0.0); q.beta = make_double2(1.0, 0.0);
        gj.push_back(q);
      }
      if (int r = dense_gemm(c, gj.data(), J)) return done(r);
    }
    for (int j = 0; j < J; ++j) {
      lj[j] = LuJob{Dw[j], NBs[j], NBs[j], Pw[j], info + (size_t)j * n1 + i1, Iw[j], NBs[j]};
      tj[j] = TransposeJob{Iw[j], NBs[j], s3->dinv[j] + (size_t)i1 * NBs[j] * NBs[j], NBs[j], NBs[j]};
    }
    if (int r = dense_lu_inverse(c, lj.data(), J)) return done(r);
    if (int r = dense_transpose(c, tj.data(), J)) return done(r);
    gj.clear();
    for (int j = 0; j < J; ++j) {
      const int NB = NBs[j];
      GemmJob q{};
      q.m = q.n = q.k = NB;
      q.A = Iw[j]; q.lda = NB;
      q.ldb = NB;
      q.ldc = NB;
      q.transC = 1;
      if (i1 > 0) {   // G_i = Dinv_i L_i
        q.B = Lw[j];
        q.C = s3->gf[j] + (size_t)i1 * NB * NB;
        gj.push_back(q);
      }
      if (i1 + 1 < n1) {   // X_i = Dinv_i U_i
        q.B = Uw[j];
        q.C = s3->xf[j] + (size_t)i1 * NB * NB;
        gj.push_back(q);
      }
    }
    if (int r = dense_gemm(c, gj.data(), (int)gj.size())) return done(r);
  }
  S3_TRY(cudaGetLastError(), "3-D factor kernels");
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
  {   // the solve kernel: one CTA per SM, co-resident (cooperative launch); the
      // staged rows double-buffered when two planes' rows fit shared memory
    s3->nbuf = k3_smem(NBmax, s3->grid, 2) <= (size_t)optin ? 2 : 1;
    s3->optin = optin;
    S3_TRY(cudaFuncSetAttribute(k3_solve<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "attr");
    S3_TRY(cudaFuncSetAttribute(k3_solve<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "attr");
    S3_TRY(cudaFuncSetAttribute(k3_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "attr");
    S3_TRY(cudaFuncSetAttribute(k3_gemv<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "attr");
    S3_TRY(cudaFuncSetAttribute(k3_gemv<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "attr");
    int per = 0;
    S3_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k3_solve<1>, kW3 * 32, optin), "occ");
    if (per < 1) return done(set_error(c, HS_E_CUDA, "3-D solve kernel does not fit an SM"));
    // widest chain kernel (right-hand sides per chain): its vectors and sums
    // must fit beside one staging buffer, co-resident on every SM
    s->max_nr = 1;
    for (int w : {2, 4}) {
      int pw = 0;
      const bool fits = k3_smem(NBmax, s3->grid, 1, w) <= (size_t)optin;
      if (!fits) break;
      cudaError_t e = w == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pw, k3_solve<2>, kW3 * 32, optin)
                             : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pw, k3_solve<4>, kW3 * 32, optin);
      if (e != cudaSuccess || pw < 1) { cudaGetLastError(); break; }
      s->max_nr = w;
    }
  }
  return done(HS_OK);
}

// One slab solve of the schedule (subdom_solve, sweepdd.py:236-268).
// Slab solves of one or two independent tasks (two sweep fronts): right-hand
// sides, the batched w = Dinv f GEMVs, then ONE cooperative chain launch --
// two chains on disjoint CTA groups when both fit the group's shared memory
// (CTAs split by NB^2, the per-step bytes) -- and the outputs.
// F / Y of both chains for nr right-hand sides (grown on demand)
static int sweep3_reserve(Ctx* c, Sweep3* s3, int nr) {
  if (nr <= s3->nrcap) return HS_OK;
  S3_TRY(cudaStreamSynchronize(c->stream), "sync");
  const size_t bytes = (size_t)nr * s3->n1 * s3->nbmax * sizeof(double2);
  for (int i = 0; i < 2; ++i) {
    cudaFree(s3->F[i]);
    cudaFree(s3->Y[i]);
    s3->F[i] = s3->Y[i] = nullptr;
  }
  s3->nrcap = 0;
  for (int i = 0; i < 2; ++i) {
    S3_TRY(cudaMalloc((void**)&s3->F[i], bytes), "3-D right-hand sides");
    S3_TRY(cudaMalloc((void**)&s3->Y[i], bytes), "3-D solutions");
  }
  s3->nrcap = nr;
  return HS_OK;
}

int sweep3_tasks(Ctx* c, Sweep* s, const SweepTask* const* ts, int nt, const double2* src,
                 double2* const* u, const double2* coarse_coeffs, int64_t coarse_n,
                 const Sweep3Rhs* mr) {
  Sweep3* s3 = s->s3;
  const int n1 = s3->n1, n2 = s3->n2;
  const int G = s3->grid;
  // nr right-hand sides through the chains (1 unless mr): strides of src,
  // of the two u destinations and of the trace buffers
  const int nr = mr ? mr->nr : 1;
  const int64_t vs_src = mr ? mr->vs_src : 0, ts_ = mr ? mr->ts : 0;
  const int64_t vs_u[2] = {mr ? mr->vs_u[0] : 0, mr ? mr->vs_u[1] : 0};
  double2* trace = mr ? mr->trace : s->trace;
  const int64_t fs = (int64_t)n1 * s3->nbmax;   // F / Y stride between right-hand sides
  if (nr != 1 && nr != 2 && nr != 4) return set_error(c, HS_E_ARG, "3-D chains carry 1, 2 or 4 right-hand sides");
  if (int r = sweep3_reserve(c, s3, nr)) return r;
  int NB[2] = {0, 0}, g0 = G, nbuf[2] = {1, 1};
  for (int k = 0; k < nt; ++k) NB[k] = s3->T[ts[k]->slab] * n2;
  if (nt == 2) {   // CTA split by per-step bytes; both groups must fit
    const double a = (double)NB[0] * NB[0], b = (double)NB[1] * NB[1];
    g0 = std::min(G - 1, std::max(1, (int)std::lround(G * a / (a + b))));
    bool ok = true;
    for (int k = 0; k < 2; ++k) {
      const int gk = k ? G - g0 : g0;
      nbuf[k] = k3_smem(NB[k], gk, 2, nr) <= (size_t)s3->optin ? 2 : 1;
      ok = ok && (NB[k] + gk - 1) / gk <= kR3 &&
           k3_smem(NB[k], gk, nbuf[k], nr) <= (size_t)s3->optin;
    }
    if (!ok) {   // one chain at a time
      for (int k = 0; k < 2; ++k)
        if (int r = sweep3_tasks(c, s, ts + k, 1, src, u, coarse_coeffs, coarse_n, mr)) return r;
      return HS_OK;
    }
  } else {
    nbuf[0] = k3_smem(NB[0], G, 2, nr) <= (size_t)s3->optin ? std::min(2, std::max(1, s3->nbuf)) : 1;
  }
  size_t smem = 0;
  K3Chain ch[2] = {};
  GemvTask gv[2] = {};
  double gemv_bytes = 0;
  for (int k = 0; k < nt; ++k) {
    const SweepTask& t = *ts[k];
    const int j = t.slab, nb = NB[k];
    const size_t nb2 = (size_t)nb * nb;
    const int64_t tot = (int64_t)n1 * nb;
    k3_rhs<<<dim3((unsigned)((tot + kT3 - 1) / kT3), nr), kT3, 0, c->stream>>>(
        t, s->n0, n1, n2, src, coarse_coeffs, coarse_n, to_slots(s3->cslot), trace, s3->F[k],
        vs_src, ts_, fs);
    HS_LAUNCH_CHECK(c, "3-D rhs");
    gv[k] = GemvTask{s3->dinv[j], s3->F[k], s3->Y[k], nb, (nb + kGvRows - 1) / kGvRows};
    gemv_bytes += (double)n1 * nb2 * 16.0;
    ch[k] = K3Chain{s3->T[j], s3->gf[j], s3->xf[j], s3->Y[k], s3->gbar + k, nbuf[k]};
    smem = std::max(smem, k3_smem(nb, nt == 2 ? (k ? G - g0 : g0) : G, nbuf[k], nr));
  }
  if (nt == 1) ch[1] = ch[0];
  {   // w_i = Dinv_i f_i for every plane of both tasks: one persistent GEMV launch
    ProfScope ps(c, K_SWEEP_GATHER, gemv_bytes);
    const int64_t items0 = (int64_t)n1 * gv[0].nrb;
    const int64_t items = items0 + (nt == 2 ? (int64_t)n1 * gv[1].nrb : 0);
    if (nt == 1) gv[1] = gv[0];
    const int nbm = std::max(gv[0].NB, gv[1].NB);
    if (!s3->gemv_grid) {   // resident CTAs of the GEMV at the largest plane
      int per = 0;
      S3_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k3_gemv<1>, 256,
                                                           (size_t)s3->nbmax * sizeof(double2)),
             "gemv occupancy");
      s3->gemv_grid = std::max(1, per) * c->num_sms;
    }
    int ggrid = s3->gemv_grid;
    const size_t gsm = (size_t)nr * nbm * sizeof(double2);
    if (nr > 1) {   // (wider kernels: their own residency)
      int per = 0;
      S3_TRY(nr == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k3_gemv<2>, 256, gsm)
                     : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k3_gemv<4>, 256, gsm),
             "gemv occupancy");
      ggrid = std::max(1, per) * c->num_sms;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(items, ggrid);
    if (nr == 1) k3_gemv<1><<<grid, 256, gsm, c->stream>>>(gv[0], gv[1], n1, items0, items, fs);
    else if (nr == 2) k3_gemv<2><<<grid, 256, gsm, c->stream>>>(gv[0], gv[1], n1, items0, items, fs);
    else k3_gemv<4><<<grid, 256, gsm, c->stream>>>(gv[0], gv[1], n1, items0, items, fs);
    HS_LAUNCH_CHECK(c, "3-D batched GEMV");
  }
  // profiler: the chain kernel (and the output scatter) as sweep_front, with
  // its algorithmic bytes -- both factor planes of every step + Y in/out
  double chain_bytes = 0;
  for (int k = 0; k < nt; ++k)
    chain_bytes += (2.0 * (n1 - 1)) * (double)NB[k] * NB[k] * 16.0 + 48.0 * n1 * (double)NB[k];
  ProfScope pf(c, K_SWEEP_FRONT, chain_bytes);
  {   // the chains: one cooperative launch
    S3_TRY(cudaMemsetAsync(s3->gbar, 0, 2 * sizeof(unsigned), c->stream), "memset");
    int g0_ = g0, n1_ = n1, n2_ = n2;
    int64_t fs_ = fs;
    void* args[] = {(void*)&ch[0], (void*)&ch[1], (void*)&g0_, (void*)&n1_, (void*)&n2_, (void*)&fs_};
    const void* kern = nr == 1 ? (const void*)k3_solve<1> : nr == 2 ? (const void*)k3_solve<2>
                                                                   : (const void*)k3_solve<4>;
    S3_TRY(cudaLaunchCooperativeKernel(kern, dim3(G), dim3(kW3 * 32), args, smem, c->stream),
           "3-D solve launch");
    HS_LAUNCH_CHECK(c, "3-D solve kernel");
  }
  for (int k = 0; k < nt; ++k) {
    const SweepTask& t = *ts[k];
    const int64_t tot = (int64_t)n1 * NB[k];
    k3_out<<<dim3((unsigned)((tot + kT3 - 1) / kT3), nr), kT3, 0, c->stream>>>(
        t, n1, n2, s3->Y[k], u[t.dst], trace, fs, vs_u[t.dst], ts_);
    HS_LAUNCH_CHECK(c, "3-D outputs");
  }
  return HS_OK;
}

int sweep3_task(Ctx* c, Sweep* s, const SweepTask& t, const double2* src, double2* const* u,
                const double2* coarse_coeffs, int64_t coarse_n) {
  const SweepTask* ts[1] = {&t};
  return sweep3_tasks(c, s, ts, 1, src, u, coarse_coeffs, coarse_n, nullptr);
}

// ---------------------------------------------------------------------------
// exact solver: the operator viewed as a single slab.  Canonical shapes are
// (1, a, b) for 2-D and (1, 1, a) for 1-D; the view puts the user's first
// axis on the slab's layer axis so that the blocks are planes of the
// second axis: 2-D (a, b) -> (T = a, n1 = b, n2 = 1), NB = a; 3-D keeps
// (a, b, c), NB = a c; 1-D (a) -> (1, a, 1).  Same memory layout in every
// case (only the axis bookkeeping changes).
int exact_create(Ctx* c, const Stencil* op, Sweep** out) {
  Stencil* v = new Stencil(*op);
  v->coeffs = nullptr;   // borrowed: the operator owns its coefficients
  v->invd = nullptr;
  v->dim = 3;
  const StencilDesc& d = op->d;
  int64_t sh[3];
  if (op->dim == 3) {
    sh[0] = d.n0; sh[1] = d.n1; sh[2] = d.n2;
  } else if (op->dim == 2) {
    sh[0] = d.n1; sh[1] = d.n2; sh[2] = 1;
  } else {
    sh[0] = 1; sh[1] = d.n2; sh[2] = 1;
  }
  for (int s_ = 0; s_ < d.S; ++s_) {
    int8_t o[3] = {d.off[s_][0], d.off[s_][1], d.off[s_][2]};
    if (op->dim == 2) { o[0] = d.off[s_][1]; o[1] = d.off[s_][2]; o[2] = 0; }
    if (op->dim == 1) { o[0] = 0; o[1] = d.off[s_][2]; o[2] = 0; }
    for (int k = 0; k < 3; ++k) v->d.off[s_][k] = o[k];
  }
  for (int k = 0; k < 3; ++k) v->shape[k] = sh[k];
  v->d.n0 = sh[0]; v->d.n1 = sh[1]; v->d.n2 = sh[2];
  Sweep* s = new Sweep();
  s->view = v;
  s->J = 1;
  s->n0 = (int)sh[0];
  s->M = (int)(sh[1] * sh[2]);
  s->coarse = v;
  const int64_t lo = 1, hi = sh[0];
  SweepTask t{};
  t.slab = 0;
  t.lo = 1;
  t.T = (int)sh[0];
  t.a = 0;
  t.b = (int)sh[0];
  t.ta = 0;
  t.tb = (int)sh[0];
  t.tin1 = t.tin3 = t.out2 = t.out4 = -1;
  t.row1 = t.row3 = t.orow2 = t.orow4 = -1;
  t.dst = 0;
  s->tasks.push_back(t);
  SweepLaunch fl{};
  fl.kind = SweepLaunch::kSolve;
  fl.src = 0;
  fl.nfront = 1;
  fl.ffirst[0] = 0;
  fl.fcount[0] = 1;
  const Stencil* slabs[1] = {v};
  int r = sweep3_create(c, s, v, slabs, &lo, &hi, nullptr);
  if (r) {
    sweep_destroy(s);
    return r;
  }
  fl.bytes = (2.0 * sh[1] - 1.0) * (double)sh[0] * sh[2] * (double)sh[0] * sh[2] * 16.0 +
             32.0 * (double)sh[0] * sh[1] * sh[2];
  s->plan[HS_VARIANT_UD].push_back(fl);
  *out = s;
  return HS_OK;
}

// exact solver of a general sparse n x n matrix (factorize(scipy matrix),
// sparselin.py:65-68): CSR rows on the device, cut into NB x NB blocks with
// NB >= the matrix bandwidth, so the matrix is block tridiagonal over
// nb = ceil(n / NB) block rows; the same block LU and chain kernel as a
// slab, on the view (T = 1, n1 = nb, n2 = NB) padded with identity rows.
// Vectors passed to the solve hold nb * NB entries.
int exact_create_csr(Ctx* c, int64_t n, int64_t nnz, const int64_t* indptr, const int64_t* indices,
                     const double2* vals, int NB, Sweep** out) {
  if (n < 1 || NB < 1 || nnz < 0) return set_error(c, HS_E_ARG, "empty matrix");
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      const int64_t j = indices[e];
      if (j < 0 || j >= n) return set_error(c, HS_E_SHAPE, "column index out of range");
      if (j / NB - i / NB > 1 || i / NB - j / NB > 1)
        return set_error(c, HS_E_SHAPE, "matrix bandwidth exceeds the block size");
    }
  const int64_t nb = (n + NB - 1) / NB;
  if (nb > (int64_t)1 << 30) return set_error(c, HS_E_SHAPE, "too many block rows");
  CsrSource src{};
  src.n = n;
  cudaError_t e = cudaMalloc((void**)&src.indptr, (n + 1) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc((void**)&src.indices, std::max<int64_t>(1, nnz) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc((void**)&src.vals, std::max<int64_t>(1, nnz) * sizeof(double2));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync((void*)src.indptr, indptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                        c->stream);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpyAsync((void*)src.indices, indices, nnz * sizeof(int64_t), cudaMemcpyHostToDevice,
                        c->stream);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpyAsync((void*)src.vals, vals, nnz * sizeof(double2), cudaMemcpyHostToDevice, c->stream);
  auto release = [&]() {
    cudaStreamSynchronize(c->stream);
    cudaFree((void*)src.indptr);
    cudaFree((void*)src.indices);
    cudaFree((void*)src.vals);
  };
  if (e != cudaSuccess) {
    release();
    return check_cuda(c, e, "CSR upload");
  }
  Stencil* v = new Stencil();
  v->dim = 3;
  v->shape[0] = 1; v->shape[1] = nb; v->shape[2] = NB;
  v->d.n0 = 1; v->d.n1 = nb; v->d.n2 = NB;
  v->d.n = nb * NB;
  v->d.S = 0;
  v->d.diag = -1;
  Sweep* s = new Sweep();
  s->view = v;
  s->J = 1;
  s->n0 = 1;
  s->M = (int)(nb * NB);
  s->coarse = v;
  const int64_t lo = 1, hi = 1;
  SweepTask t{};
  t.slab = 0;
  t.lo = 1;
  t.T = 1;
  t.a = 0;
  t.b = 1;
  t.ta = 0;
  t.tb = 1;
  t.tin1 = t.tin3 = t.out2 = t.out4 = -1;
  t.row1 = t.row3 = t.orow2 = t.orow4 = -1;
  t.dst = 0;
  s->tasks.push_back(t);
  SweepLaunch fl{};
  fl.kind = SweepLaunch::kSolve;
  fl.src = 0;
  fl.nfront = 1;
  fl.ffirst[0] = 0;
  fl.fcount[0] = 1;
  const Stencil* slabs[1] = {v};
  int r = sweep3_create(c, s, v, slabs, &lo, &hi, &src);
  release();
  if (r) {
    sweep_destroy(s);
    return r;
  }
  fl.bytes = (2.0 * nb - 1.0) * (double)NB * NB * 16.0 + 32.0 * (double)nb * NB;
  s->plan[HS_VARIANT_UD].push_back(fl);
  *out = s;
  return HS_OK;
}

}  // namespace hs
