// Coarse-level sweeping preconditioner on B200: slab solves by block cyclic
// reduction (BCR) over the face axis, one thread-block cluster per sweep front.
//
// Reference: build_partition + Factorization (sweepdd.py:192-218,
// sparselin.py:40-68), subdom_solve (sweepdd.py:236-268), TransmissionMatrix
// (sweepdd.py:98-141), forward/backward/mid sweeps, prec_ud / prec_x
// (sweepdd.py:271-359).
//
// Slab system.  A slab of T <= 32 layers along the sweep axis and M face points
// is block tridiagonal along the face: block y couples to y-1 (L_y), y (D_y),
// y+1 (U_y), blocks tm x tm (tm = 16 or 32, T padded with identity rows).
// SuperLU's sparse LU is a chain of ~2*M*T dependent rows per solve; a block
// Thomas chain still has 2M dependent steps.  BCR has 2*ceil(log2 M)
// dependent levels, each a batch of independent dense tm x tm mat-vecs:
//   level l (stride s = 2^l): blocks y = odd multiples of s are eliminated,
//     y_y = Dinv_y f_y;  kept blocks (even multiples) update
//     f_y -= alpha_y f_{y-s} + gamma_y f_{y+s}   (alpha = L Dinv_{y-s}, gamma = U Dinv_{y+s})
//   top: x_0 = Dinv_0 f_0
//   back substitution, level L-1 .. 0: x_y = y_y - (Dinv L)_y x_{y-s} - (Dinv U)_y x_{y+s}.
// Setup computes every level's Schur complements on the device, batched over
// all slabs (k_bcr_elim / k_bcr_keep per level; Gauss-Jordan with partial
// pivoting inside each block, no pivoting across blocks -- SURVEY H2).
//
// Apply: one cluster of C CTAs per front (C <= 16, non-portable size), CTA k
// owns face points [kM/C, (k+1)M/C); the right-hand side / solution blocks
// live in shared memory and neighbours in other CTAs are read through DSMEM;
// levels are separated by cluster barriers.  Dense blocks are stored
// "lane-major" so each of a warp's 16-byte loads is one contiguous 512-byte
// line.  Transmission (sweepdd.py:113-118) is applied by the consumer when it
// builds its right-hand side, from the producer's two trace rows in global
// memory and the global coarse operator's interface couplings.

#include "hs_common.cuh"
#include "hs_sweep.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace hs {

namespace {

constexpr int kMaxLevels = 20;
constexpr int kWarps = 16;
constexpr int kMaxTasks = 1024;   // slab solves per front per launch

template <int TM>
struct Geo {
  static constexpr int TM2 = TM * TM;
  static constexpr int NH = 32 / TM;   // lanes sharing one row
  static constexpr int CPL = TM / NH;  // columns per lane
};

// lane-major position of element (r, c): lane = (c / CPL) * TM + r, k = c % CPL
template <int TM>
__host__ __device__ __forceinline__ int lm(int r, int c) {
  return (c % Geo<TM>::CPL) * 32 + (c / Geo<TM>::CPL) * TM + r;
}

struct SlabInfo {
  const double2* coeffs;   // slab operator [S][T*M]
  int T;
  int slot[3][3];          // (o0+1, o1+1) -> coefficient slot or -1
};

// ---------------------------------------------------------------------------
// setup kernels (thread (r, c) of a tm x tm block; batched over slabs)

template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_bcr_init(const SlabInfo* __restrict__ slabs, int M, double2* __restrict__ D,
           double2* __restrict__ Lc, double2* __restrict__ Uc) {
  const int y = blockIdx.x, s = blockIdx.y;
  const SlabInfo si = slabs[s];
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  const int T = si.T;
  const int64_t n = (int64_t)T * M;
  auto coef = [&](int o0, int o1) -> double2 {
    // coupling (r, y) -> (r + o0, y + o1) with c = r + o0
    if (o0 < -1 || o0 > 1) return czero();
    const int sl = si.slot[o0 + 1][o1 + 1];
    if (sl < 0 || r >= T || c >= T || y + o1 < 0 || y + o1 >= M) return czero();
    return si.coeffs[(int64_t)sl * n + (int64_t)r * M + y];
  };
  const int64_t off = ((int64_t)s * M + y) * Geo<TM>::TM2 + r * TM + c;
  double2 d = coef(c - r, 0);
  if (r >= T || c >= T) d = make_double2(r == c ? 1.0 : 0.0, 0.0);
  D[off] = d;
  Lc[off] = coef(c - r, -1);
  Uc[off] = coef(c - r, 1);
}

// In-place Gauss-Jordan inversion with partial pivoting of A (smem, pitch TM+1)
// into Inv.  All TM*TM threads participate.
template <int TM>
__device__ void gj_invert(double2 (*A)[TM + 1], double2 (*Inv)[TM + 1], int* piv_row,
                          double* piv_abs, unsigned long long* err, unsigned long long code) {
  const int tid = threadIdx.x;
  const int r = tid / TM, c = tid % TM;
  Inv[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  __syncthreads();
  for (int p = 0; p < TM; ++p) {
    if (tid < 32) {
      double v = (tid >= p && tid < TM) ? cabs2(A[tid][p]) : -1.0;
      int idx = tid;
      for (int m = 16; m > 0; m >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, m);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, m);
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
      }
      if (tid == 0) { *piv_row = idx; *piv_abs = v; }
    }
    __syncthreads();
    const int pr = *piv_row;
    if (*piv_abs <= 0.0) {
      if (tid == 0) atomicMin(err, code + (unsigned long long)p);
      if (r == p && c == p) A[p][p] = make_double2(1.0, 0.0);
      __syncthreads();
    } else if (pr != p) {
      if (r == p) {
        double2 t = A[p][c]; A[p][c] = A[pr][c]; A[pr][c] = t;
        t = Inv[p][c]; Inv[p][c] = Inv[pr][c]; Inv[pr][c] = t;
      }
      __syncthreads();
    }
    const double2 app = A[p][p];
    const double2 apc = A[p][c], ipc = Inv[p][c];
    const double2 arp = A[r][p];
    double2 arc = A[r][c], irc = Inv[r][c];
    __syncthreads();
    const double2 inv_p = cdiv(make_double2(1.0, 0.0), app);
    const double2 np = cmul(apc, inv_p), ni = cmul(ipc, inv_p);
    if (r == p) {
      arc = np;
      irc = ni;
    } else {
      arc = csub(arc, cmul(arp, np));
      irc = csub(irc, cmul(arp, ni));
    }
    A[r][c] = arc;
    Inv[r][c] = irc;
    __syncthreads();
  }
}

template <int TM>
__device__ __forceinline__ void load_mat(double2 (*S)[TM + 1], const double2* __restrict__ g) {
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  S[r][c] = g[r * TM + c];
}

template <int TM>
__device__ __forceinline__ double2 mm_rc(double2 (*A)[TM + 1], double2 (*B)[TM + 1]) {
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  double2 acc = czero();
#pragma unroll 8
  for (int k = 0; k < TM; ++k) acc = cfma(A[r][k], B[k][c], acc);
  return acc;
}

// Eliminated blocks of level l (odd multiples of s): Dinv, Dinv L, Dinv U.
// D[y] is overwritten with Dinv (natural layout) for the keep kernel.
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_bcr_elim(int level, int M, int top, double2* __restrict__ D, const double2* __restrict__ Lc,
           const double2* __restrict__ Uc, double2* __restrict__ ef, double2* __restrict__ eb,
           unsigned long long* __restrict__ err) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int s_ = 1 << level;
  const int y = top ? 0 : (2 * blockIdx.x + 1) * s_;
  const int slab = blockIdx.y;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*A)[TM + 1] = reinterpret_cast<double2(*)[TM + 1]>(smraw);
  double2(*Inv)[TM + 1] = A + TM;
  double2(*B)[TM + 1] = Inv + TM;
  __shared__ int piv_row;
  __shared__ double piv_abs;
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  const int64_t base = ((int64_t)slab * M + y) * TM2;
  load_mat<TM>(A, D + base);
  __syncthreads();
  const unsigned long long code =
      ((unsigned long long)slab << 40) | ((unsigned long long)y * TM & 0xffffffffffull);
  gj_invert<TM>(A, Inv, &piv_row, &piv_abs, err, code);
  ef[base + lm<TM>(r, c)] = Inv[r][c];
  D[base + r * TM + c] = Inv[r][c];
  if (top) return;
  load_mat<TM>(B, Lc + base);
  __syncthreads();
  eb[2 * base + lm<TM>(r, c)] = mm_rc<TM>(Inv, B);
  __syncthreads();
  load_mat<TM>(B, Uc + base);
  __syncthreads();
  eb[2 * base + TM2 + lm<TM>(r, c)] = mm_rc<TM>(Inv, B);
}

// Kept blocks of level l (multiples of 2s): alpha, gamma and the next level's
// D, L, U (in place).
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_bcr_keep(int level, int M, int koff, double2* __restrict__ D, double2* __restrict__ Lc,
           double2* __restrict__ Uc, double2* __restrict__ kr, int ktot) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int s_ = 1 << level;
  const int j = blockIdx.x;
  const int y = j * 2 * s_;
  const int slab = blockIdx.y;
  const int left = y - s_, right = y + s_;
  const bool hl = left >= 0, hr = right < M;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*S0)[TM + 1] = reinterpret_cast<double2(*)[TM + 1]>(smraw);
  double2(*S1)[TM + 1] = S0 + TM;
  double2(*Al)[TM + 1] = S1 + TM;
  double2(*Ga)[TM + 1] = Al + TM;
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  auto at = [&](int yy) { return ((int64_t)slab * M + yy) * TM2; };
  double2* kout = kr + ((int64_t)slab * ktot + koff + j) * 2 * TM2;
  // alpha = L_y Dinv_left, gamma = U_y Dinv_right
  Al[r][c] = czero();
  Ga[r][c] = czero();
  if (hl) {
    load_mat<TM>(S0, Lc + at(y));
    load_mat<TM>(S1, D + at(left));
    __syncthreads();
    Al[r][c] = mm_rc<TM>(S0, S1);
  }
  __syncthreads();
  if (hr) {
    load_mat<TM>(S0, Uc + at(y));
    load_mat<TM>(S1, D + at(right));
    __syncthreads();
    Ga[r][c] = mm_rc<TM>(S0, S1);
  }
  __syncthreads();
  kout[lm<TM>(r, c)] = Al[r][c];
  kout[TM2 + lm<TM>(r, c)] = Ga[r][c];
  // D' = D - alpha U_left - gamma L_right
  double2 d = D[at(y) + r * TM + c];
  if (hl) {
    load_mat<TM>(S0, Uc + at(left));
    __syncthreads();
    d = csub(d, mm_rc<TM>(Al, S0));
    __syncthreads();
  }
  if (hr) {
    load_mat<TM>(S1, Lc + at(right));
    __syncthreads();
    d = csub(d, mm_rc<TM>(Ga, S1));
    __syncthreads();
  }
  D[at(y) + r * TM + c] = d;
  // L' = -alpha L_left, U' = -gamma U_right
  double2 lnew = czero(), unew = czero();
  if (hl) {
    load_mat<TM>(S0, Lc + at(left));
    __syncthreads();
    lnew = cscale(-1.0, mm_rc<TM>(Al, S0));
  }
  if (hr) {
    load_mat<TM>(S1, Uc + at(right));
    __syncthreads();
    unew = cscale(-1.0, mm_rc<TM>(Ga, S1));
  }
  Lc[at(y) + r * TM + c] = lnew;
  Uc[at(y) + r * TM + c] = unew;
}

// ---------------------------------------------------------------------------
// apply

struct SolveArgs {
  const SweepTask* tasks;
  int ffirst[2], fcount[2];
  int C, M, L, ktot, nloc_max, nslot;
  int koff[kMaxLevels];
  const double2* ef;
  const double2* eb;
  const double2* kr;
  const double2* src;      // right-hand side field (n0 x M)
  const double2* coarse;   // global coarse operator [S][n0*M] (transmission couplings)
  int64_t ncoarse;
  int cslot[3][3];
  double2* trace;          // [ntrace][2][M]
  double2* u[2];
  unsigned long long* dbg;   // optional phase timestamps (HS_SWEEP_TRACE)
};

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  // TMA bulk prefetch into L2 (sizes are multiples of 16 bytes here)
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes)
                          : "memory");
}

// Prefetch this CTA's share of slab `slab`'s BCR records into L2.
template <int TM>
__device__ void prefetch_slab(const SolveArgs& a, int slab, int Y0, int Y1) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int M = a.M;
  const uint32_t mb = TM2 * 16;
  const double2* ef = a.ef + (int64_t)slab * M * TM2;
  const double2* eb = a.eb + (int64_t)slab * M * 2 * TM2;
  const double2* kr = a.kr + (int64_t)slab * a.ktot * 2 * TM2;
  prefetch_l2(ef + (int64_t)Y0 * TM2, (uint32_t)(Y1 - Y0) * mb);
  prefetch_l2(eb + (int64_t)Y0 * 2 * TM2, (uint32_t)(Y1 - Y0) * 2 * mb);
  for (int l = 0; l < a.L; ++l) {
    const int s2 = 2 << l;
    const int j0 = (Y0 + s2 - 1) / s2, j1 = (Y1 - 1) / s2;
    if (j1 >= j0)
      prefetch_l2(kr + (int64_t)(a.koff[l] + j0) * 2 * TM2, (uint32_t)(j1 - j0 + 1) * 2 * mb);
  }
}

// y = Mat v for a tm x tm lane-major block; every lane returns row (lane % tm)
template <int TM>
__device__ __forceinline__ double2 mv(const double2* __restrict__ mat, const double2* v,
                                      int lane) {
  constexpr int CPL = Geo<TM>::CPL;
  const int hh = lane / TM;
  double2 a0 = czero(), a1 = czero();
#pragma unroll
  for (int k = 0; k < CPL; k += 2) {
    a0 = cfma(__ldg(mat + k * 32 + lane), v[CPL * hh + k], a0);
    a1 = cfma(__ldg(mat + (k + 1) * 32 + lane), v[CPL * hh + k + 1], a1);
  }
  double2 acc = cadd(a0, a1);
  if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
  return acc;
}

// Ring of shared-memory slots fed by TMA bulk copies: the BCR items (one
// block's 1-2 matrices) of this CTA in consumption order, across phases and
// tasks.  The warp that consumes item i refills its slot with item i+NSLOT, so
// copies run up to NSLOT items ahead of the dependency chain and never sit on
// a thread's scoreboard across a cluster barrier (a global load in flight
// delays barrier.cluster completion; an async-proxy copy does not).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  const uint32_t a = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// y = Mat v, Mat a lane-major tm x tm block in shared memory; every lane
// returns row (lane % tm)
template <int TM>
__device__ __forceinline__ double2 mvs(const double2* mat, const double2* v, int lane) {
  constexpr int CPL = Geo<TM>::CPL;
  const int hh = lane / TM;
  double2 vv[CPL];   // issue every operand load first (DSMEM round trips overlap)
#pragma unroll
  for (int k = 0; k < CPL; ++k) vv[k] = v[CPL * hh + k];
  double2 a0 = czero(), a1 = czero();
#pragma unroll
  for (int k = 0; k < CPL; k += 2) {
    a0 = cfma(mat[k * 32 + lane], vv[k], a0);
    a1 = cfma(mat[(k + 1) * 32 + lane], vv[k + 1], a1);
  }
  double2 acc = cadd(a0, a1);
  if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
  return acc;
}

// acc = A0 v0 + A1 v1 (either term may be absent); both operand vectors are
// fetched before any arithmetic so remote (DSMEM) round trips overlap
template <int TM>
__device__ __forceinline__ double2 mvs2(const double2* m0, const double2* v0, const double2* m1,
                                        const double2* v1, int lane, double2* stage) {
  constexpr int CPL = Geo<TM>::CPL;
  const int hh = lane / TM;
  // one coalesced (possibly remote) read per operand element into this warp's
  // staging area, then broadcast reads from local shared memory
  if (lane < TM) {
    if (v0) stage[lane] = v0[lane];
    if (v1) stage[TM + lane] = v1[lane];
  }
  __syncwarp();
  double2 va[CPL], vb[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    va[k] = v0 ? stage[CPL * hh + k] : czero();
    vb[k] = v1 ? stage[TM + CPL * hh + k] : czero();
  }
  __syncwarp();
  double2 a0 = czero(), a1 = czero();
  if (v0) {
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
      a0 = cfma(m0[k * 32 + lane], va[k], a0);
      a1 = cfma(m0[(k + 1) * 32 + lane], va[k + 1], a1);
    }
  }
  if (v1) {
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
      a0 = cfma(m1[k * 32 + lane], vb[k], a0);
      a1 = cfma(m1[(k + 1) * 32 + lane], vb[k + 1], a1);
    }
  }
  double2 acc = cadd(a0, a1);
  if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
  return acc;
}

template <int TM>
struct Ring {
  static constexpr int SLOT = 2 * Geo<TM>::TM2;   // double2 per slot (two matrices)
  static int nslot(int nloc_max) {
    const int vec = 2 * nloc_max * TM * 16;
    const int avail = 225 * 1024 - vec - 1024 - kMaxTasks * 4 - kWarps * 2 * TM * 16;
    return std::max(2, std::min(32, avail / (SLOT * 16 + 12)));
  }
  static int smem(int nloc_max) {
    const int n = nslot(nloc_max);
    return 2 * nloc_max * TM * 16 + n * SLOT * 16 + n * 12 + (64 + kMaxTasks) * 4 + 64 +
           kWarps * 2 * TM * 16 + 16;
  }
};

template <int TM>
__global__ void __launch_bounds__(kWarps * 32, 1) k_bcr_solve(SolveArgs a) {
  constexpr int TM2 = Geo<TM>::TM2;
  constexpr int SLOT = Ring<TM>::SLOT;
  constexpr int YPW = 32 / TM;   // face points per warp pass in row-wise loops
  cg::cluster_group cl = cg::this_cluster();
  const int C = a.C, M = a.M, L = a.L;
  const int rank = (int)cl.block_rank();
  const int front = blockIdx.x / C;
  const int Y0 = (int)((int64_t)rank * M / C), Y1 = (int)((int64_t)(rank + 1) * M / C);
  const int nloc = Y1 - Y0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int x = lane % TM, hh = lane / TM;
  const int NS = a.nslot;
  extern __shared__ __align__(128) double2 sm[];
  double2* F = sm;                          // [nloc_max][TM] right-hand side / reduced rhs
  double2* Yv = sm + a.nloc_max * TM;       // [nloc_max][TM] Dinv f, then the solution
  double2* ring = Yv + a.nloc_max * TM;     // [NS][SLOT]
  uint64_t* bars = (uint64_t*)(ring + (int64_t)NS * SLOT);
  volatile int* seq = (volatile int*)(bars + NS);   // [NS] item currently issued into a slot
  int* pfx = (int*)(bars + NS) + NS;        // [2L+1] items before each phase
  int* slabs = pfx + 64;                    // [fcount] slab of each task of this front
  double2* stage = (double2*)(((uintptr_t)(slabs + kMaxTasks) + 15) & ~(uintptr_t)15) +
                   warp * 2 * TM;             // [2][TM] per warp (16-byte aligned)

  // owner CTA of face point y: local test first, else a search of the
  // partition table (no 64-bit division on the chain)
  auto owner = [&](int y, int& base) -> int {
    if (y >= Y0 && y < Y1) { base = Y0; return rank; }
    const int r = ((y + 1) * C - 1) / M;   // 32-bit: (y+1)*C < 2^31
    base = r * M / C;
    return r;
  };
  auto Fany = [&](int y) -> const double2* {
    int base;
    const int o = owner(y, base);
    const double2* p = F + (y - base) * TM;
    return o == rank ? p : cl.map_shared_rank(p, o);
  };
  auto Yany = [&](int y) -> const double2* {
    int base;
    const int o = owner(y, base);
    const double2* p = Yv + (y - base) * TM;
    return o == rank ? p : cl.map_shared_rank(p, o);
  };
  auto cc = [&](int o0, int o1, int row, int y) -> double2 {
    const int sl = a.cslot[o0 + 1][o1 + 1];
    if (sl < 0 || y + o1 < 0 || y + o1 >= M) return czero();
    return __ldg(a.coarse + (int64_t)sl * a.ncoarse + (int64_t)row * M + y);
  };
  // transmission source into slab row p-lo (which 0) / p+1-lo (which 1)
  auto trans = [&](int buf, int p, int sign, int which, int y) -> double2 {
    const double2* B = a.trace + (int64_t)buf * 2 * M + (which == 0 ? M : 0);
    const int o0 = which == 0 ? 1 : -1;
    const int row = which == 0 ? p - 1 : p;
    double2 cv[3], bv[3];
#pragma unroll
    for (int o = -1; o <= 1; ++o) {   // all six loads in flight together
      const bool ok = y + o >= 0 && y + o < M;
      cv[o + 1] = ok ? cc(o0, o, row, y) : czero();
      bv[o + 1] = ok ? B[y + o] : czero();
    }
    double2 acc = cmul(cv[0], bv[0]);
    acc = cfma(cv[1], bv[1], acc);
    acc = cfma(cv[2], bv[2], acc);
    return cscale(which == 0 ? (double)sign : (double)-sign, acc);
  };

  // Phases of one slab solve: p < L forward level p, p >= L backward level
  // 2L-1-p; items of a phase are this CTA's active blocks, item j -> warp j%16.
  const int NP = 2 * L;
  auto ph_level = [&](int p) { return p < L ? p : NP - 1 - p; };
  auto ph_first = [&](int p) -> int {
    const int s = 1 << ph_level(p);
    int first = ((Y0 + s - 1) / s) * s;
    if (p >= L && ((first / s) & 1) == 0) first += s;
    return first;
  };
  auto ph_step = [&](int p) { return (p < L ? 1 : 2) << ph_level(p); };
  const int ffirst = front ? a.ffirst[1] : a.ffirst[0];
  const int fcount = front ? a.fcount[1] : a.fcount[0];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int p = 0; p < NP; ++p) {
      pfx[p] = acc;
      const int f = ph_first(p);
      if (f < Y1) acc += (Y1 - 1 - f) / ph_step(p) + 1;
    }
    pfx[NP] = acc;
    for (int i = 0; i < NS; ++i) {
      mbar_init(&bars[i], 1);
      seq[i] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < fcount; i += blockDim.x) slabs[i] = a.tasks[ffirst + i].slab;
  __syncthreads();
  const int ITEMS = pfx[NP];
  const int total = fcount * ITEMS;

  // matrices of item (task ti, phase p, y): up to two 16/32-square blocks
  auto item_src = [&](int ti, int p, int y, const double2*& m0, const double2*& m1) {
    const int slab = slabs[ti];
    const int l = ph_level(p), s = 1 << l;
    m0 = m1 = nullptr;
    if (p < L) {
      if ((y / s) & 1) {
        m0 = a.ef + ((int64_t)slab * M + y) * TM2;
      } else {
        const double2* k2 =
            a.kr + ((int64_t)slab * a.ktot + a.koff[l] + y / (2 * s)) * 2 * TM2;
        if (y - s >= 0) m0 = k2;
        if (y + s < M) m1 = k2 + TM2;
        if (y == 0 && l == L - 1) m0 = a.ef + (int64_t)slab * M * TM2;   // top block Dinv
      }
    } else {
      const double2* e2 = a.eb + ((int64_t)slab * M + y) * 2 * TM2;
      if (y - s >= 0) m0 = e2;
      if (y + s < M) m1 = e2 + TM2;
    }
  };
  auto issue = [&](int i) {   // one lane
    const int ti = i / ITEMS;
    const int r = i - ti * ITEMS;
    int p = 0;
    while (pfx[p + 1] <= r) ++p;
    const int y = ph_first(p) + (r - pfx[p]) * ph_step(p);
    const double2 *m0, *m1;
    item_src(ti, p, y, m0, m1);
    const int sl = i % NS;
    double2* slot = ring + sl * SLOT;
    uint64_t* bar = &bars[sl];
    const uint32_t mb = TM2 * 16;
    mbar_expect_tx(bar, (m0 ? mb : 0) + (m1 ? mb : 0));
    if (m0) bulk_g2s(slot, m0, mb, bar);
    if (m1) bulk_g2s(slot + TM2, m1, mb, bar);
    seq[sl] = i;
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < total && i < NS; ++i) issue(i);
  if (L == 0 && rank == 0 && warp == 0 && lane == 0 && fcount) {
    // M == 1: the only block is the top; its Dinv is read directly
  }

  // optional instrumentation: timestamps of task 1 kept in shared memory (a
  // global store would hold the next cluster-barrier arrive), dumped at exit
  __shared__ unsigned long long tsm[512];
  auto stamp = [&](int ti, int k) {
    if (a.dbg && threadIdx.x == 0 && ti == 1 && k < 64) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tsm[k] = tt;
    }
  };
  auto stamp2 = [&](int ti, int p, int k) {
    if (a.dbg && threadIdx.x == 0 && ti == 1 && p < 56) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tsm[64 + p * 8 + k] = tt;
    }
  };
  if (a.dbg && threadIdx.x == 0)
    for (int k = 0; k < 512; ++k) tsm[k] = 0;
  for (int ti = 0; ti < fcount; ++ti) {
    stamp(ti, 0);
    const SweepTask t = a.tasks[ffirst + ti];
    if (threadIdx.x == 0 && ti + 1 < fcount)
      prefetch_slab<TM>(a, slabs[ti + 1], Y0, Y1);
    // ---- right-hand side of the owned blocks (restriction + transmission)
    for (int yl = warp * YPW + hh; yl < nloc; yl += kWarps * YPW) {
      const int y = Y0 + yl;
      double2 v = czero();
      const int g = x + t.lo - 1;
      if (x < t.T && g >= t.a && g < t.b) v = __ldg(a.src + (int64_t)g * M + y);
      if (t.tin1 >= 0 && (x == t.row1 || x == t.row1 + 1))
        v = cadd(v, trans(t.tin1, t.row1 + t.lo, 1, x - t.row1, y));
      if (t.tin3 >= 0 && (x == t.row3 || x == t.row3 + 1))
        v = cadd(v, trans(t.tin3, t.row3 + t.lo, -1, x - t.row3, y));
      F[yl * TM + x] = v;
    }
    cl.sync();
    stamp(ti, 1);
    if (L == 0) {   // M == 1: x_0 = Dinv_0 f_0
      if (rank == 0 && warp == 0) {
        const double2 r = mv<TM>(a.ef + (int64_t)t.slab * M * TM2, F, lane);
        if (hh == 0) Yv[x] = r;
      }
      __syncthreads();
    }
    // ---- forward reduction, top solve, back substitution
    const int base = ti * ITEMS;
    int defer0 = -1, defer = -1;
    for (int p = 0; p < NP; ++p) {
      const int l = ph_level(p), s = 1 << l;
      const int f0 = ph_first(p), st = ph_step(p);
      const int cnt = pfx[p + 1] - pfx[p];
      for (int j = warp; j < cnt; j += kWarps) {
        const int y = f0 + j * st;
        const int i = base + pfx[p] + j;
        // a parity wait is only valid once the slot's previous use completed:
        // wait until this item has been issued into the slot (which happens
        // after its previous occupant was consumed)
        if (j == 0) stamp2(ti, p, 0);
        while (seq[i % NS] != (int)i) {
        }
        if (j == 0) stamp2(ti, p, 1);
        mbar_wait(&bars[i % NS], (uint32_t)((i / NS) & 1));
        if (j == 0) stamp2(ti, p, 2);
        const double2* m0 = ring + (i % NS) * SLOT;
        const double2* m1 = m0 + TM2;
        if (p < L) {
          if ((y / s) & 1) {   // eliminated at this level: y = Dinv f
            const double2 r = mvs<TM>(m0, F + (y - Y0) * TM, lane);
            if (hh == 0) Yv[(y - Y0) * TM + x] = r;
          } else {             // kept: f -= alpha f_{y-s} + gamma f_{y+s}
            double2 acc = czero();
            acc = mvs2<TM>(y - s >= 0 ? m0 : nullptr, y - s >= 0 ? Fany(y - s) : nullptr,
                           y + s < M ? m1 : nullptr, y + s < M ? Fany(y + s) : nullptr, lane,
                           stage);
            if (hh == 0) F[(y - Y0) * TM + x] = csub(F[(y - Y0) * TM + x], acc);
            if (y == 0 && l == L - 1) {   // top of the reduction: x_0 = Dinv_0 f_0
              __syncwarp();
              const double2 r = mvs<TM>(m0, F, lane);
              if (hh == 0) Yv[x] = r;
            }
          }
        } else {               // x_y = Dinv f - (Dinv L) x_{y-s} - (Dinv U) x_{y+s}
          double2 acc = czero();
          acc = mvs2<TM>(y - s >= 0 ? m0 : nullptr, y - s >= 0 ? Yany(y - s) : nullptr,
                         y + s < M ? m1 : nullptr, y + s < M ? Yany(y + s) : nullptr, lane,
                         stage);
          if (hh == 0) Yv[(y - Y0) * TM + x] = csub(Yv[(y - Y0) * TM + x], acc);
        }
        __syncwarp();
        if (j == 0) stamp2(ti, p, 3);
        if (i + NS < total) {
          if (i + NS < base + pfx[p + 1]) {   // needed within this phase: refill now
            if (lane == 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue(i + NS);
            }
          } else {
            if (defer0 < 0) defer0 = i + NS;
            defer = i + NS;   // refill after arriving at the barrier (off the chain)
          }
        }
        if (j == 0) stamp2(ti, p, 4);
      }
      asm volatile("barrier.cluster.arrive.release;" ::: "memory");
      if (defer0 >= 0 && lane == 0) {   // refills deferred from this phase
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int d = defer0; d <= defer; d += kWarps) issue(d);
      }
      defer0 = defer = -1;
      asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
      stamp(ti, 2 + p);
    }
    // ---- outputs: solution rows into u (one producer per row and pass), traces
    const int ur0 = t.ta + 1 - t.lo, ur1 = t.tb + 1 - t.lo;
    for (int yl = warp * YPW + hh; yl < nloc; yl += kWarps * YPW) {
      const int y = Y0 + yl;
      const double2 xv = Yv[yl * TM + x];
      if (x >= ur0 && x < ur1) a.u[t.dst][(int64_t)(x + t.lo - 1) * M + y] = xv;
      if (t.out2 >= 0 && (x == t.orow2 || x == t.orow2 + 1))
        a.trace[((int64_t)t.out2 * 2 + (x - t.orow2)) * M + y] = xv;
      if (t.out4 >= 0 && (x == t.orow4 || x == t.orow4 + 1))
        a.trace[((int64_t)t.out4 * 2 + (x - t.orow4)) * M + y] = xv;
    }
    cl.sync();   // traces visible to the cluster; F / Yv free for the next task
    stamp(ti, 63);
  }
  if (a.dbg && threadIdx.x == 0 && blockIdx.x < 16)
    for (int k = 0; k < 512; ++k) a.dbg[blockIdx.x * 512 + k] = tsm[k];
  {
  }
}

__global__ void k_combine(double2* __restrict__ u, const double2* __restrict__ u2, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[i] = cadd(u[i], __ldg(u2 + i));
}

template <int TM>
int solve_smem(int nloc_max) { return Ring<TM>::smem(nloc_max); }

template <int TM>
cudaError_t launch_solve(const SolveArgs& a, int nfront, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nfront * a.C, 1, 1);
  cfg.blockDim = dim3(kWarps * 32, 1, 1);
  cfg.dynamicSmemBytes = solve_smem<TM>(a.nloc_max);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_bcr_solve<TM>, a);
}

template <int TM>
cudaError_t prepare_solve(int C, int nloc_max, int* max_clusters) {
  cudaError_t e = cudaFuncSetAttribute(k_bcr_solve<TM>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_bcr_solve<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           std::max(solve_smem<TM>(nloc_max), 1024));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(kWarps * 32, 1, 1);
  cfg.dynamicSmemBytes = solve_smem<TM>(nloc_max);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(max_clusters, k_bcr_solve<TM>, &cfg);
}

template <int TM>
int factorize(Ctx* c, Sweep* s, const std::vector<SlabInfo>& info) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int J = s->J, M = s->M, L = s->L;
  const size_t wbytes = (size_t)J * M * TM2 * sizeof(double2);
  double2 *D = nullptr, *Lc = nullptr, *Uc = nullptr;
  SlabInfo* d_info = nullptr;
  unsigned long long* d_err = nullptr;
  int rc = HS_OK;
  auto cleanup = [&]() {
    cudaFree(D); cudaFree(Lc); cudaFree(Uc); cudaFree(d_info); cudaFree(d_err);
  };
#define HS_TRYF(call, what)                                            \
  do {                                                                 \
    cudaError_t _e = (call);                                           \
    if (_e != cudaSuccess) { rc = check_cuda(c, _e, what); cleanup(); return rc; } \
  } while (0)
  HS_TRYF(cudaMalloc((void**)&D, wbytes), "bcr work alloc");
  HS_TRYF(cudaMalloc((void**)&Lc, wbytes), "bcr work alloc");
  HS_TRYF(cudaMalloc((void**)&Uc, wbytes), "bcr work alloc");
  HS_TRYF(cudaMalloc((void**)&d_info, J * sizeof(SlabInfo)), "alloc");
  HS_TRYF(cudaMalloc((void**)&d_err, sizeof(unsigned long long)), "alloc");
  HS_TRYF(cudaMemcpyAsync(d_info, info.data(), J * sizeof(SlabInfo), cudaMemcpyHostToDevice,
                          c->stream), "upload");
  HS_TRYF(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), c->stream), "memset");
  HS_TRYF(cudaMemsetAsync(s->eb, 0, (size_t)J * M * 2 * TM2 * sizeof(double2), c->stream),
          "memset");
  const int smem3 = 3 * TM * (TM + 1) * (int)sizeof(double2);
  const int smem4 = 4 * TM * (TM + 1) * (int)sizeof(double2);
  HS_TRYF(cudaFuncSetAttribute(k_bcr_elim<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem3), "attr");
  HS_TRYF(cudaFuncSetAttribute(k_bcr_keep<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem4), "attr");
  k_bcr_init<TM><<<dim3(M, J), TM * TM, 0, c->stream>>>(d_info, M, D, Lc, Uc);
  c->launches++;
  HS_TRYF(cudaGetLastError(), "bcr init");
  std::vector<int> koff(L + 1, 0);
  for (int l = 0; l < L; ++l) {
    const int sl = 1 << l;
    const int nel = (M - 1 - sl) / (2 * sl) + 1;   // odd multiples of s below M
    const int nkeep = (M - 1) / (2 * sl) + 1;      // even multiples (incl. 0)
    k_bcr_elim<TM><<<dim3(nel, J), TM * TM, smem3, c->stream>>>(l, M, 0, D, Lc, Uc, s->ef,
                                                                   s->eb, d_err);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "bcr elim");
    k_bcr_keep<TM><<<dim3(nkeep, J), TM * TM, smem4, c->stream>>>(l, M, koff[l], D, Lc, Uc,
                                                                     s->kr, s->ktot);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "bcr keep");
    koff[l + 1] = koff[l] + nkeep;
  }
  k_bcr_elim<TM><<<dim3(1, J), TM * TM, smem3, c->stream>>>(L, M, 1, D, Lc, Uc, s->ef, s->eb,
                                                              d_err);
  c->launches++;
  HS_TRYF(cudaGetLastError(), "bcr top");
  unsigned long long err = 0;
  HS_TRYF(cudaMemcpyAsync(&err, d_err, sizeof err, cudaMemcpyDeviceToHost, c->stream), "err");
  HS_TRYF(cudaStreamSynchronize(c->stream), "factor sync");
#undef HS_TRYF
  cleanup();
  if (err != ~0ull) {
    const int slab = (int)(err >> 40);
    const long long row = (long long)(err & 0xffffffffffull);
    char buf[128];
    snprintf(buf, sizeof buf, "zero pivot at row %lld (slab %d)", row, slab + 1);
    return set_error(c, HS_E_ZERO_PIVOT, buf, row);
  }
  return HS_OK;
}

int slot_table(const Stencil* op, int slot[3][3], Ctx* c) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) slot[i][j] = -1;
  for (int s = 0; s < op->d.S; ++s) {
    const int o0 = op->d.off[s][1], o1 = op->d.off[s][2];
    if (op->d.off[s][0] != 0) return set_error(c, HS_E_SHAPE, "sweep needs 2-D operators");
    slot[o0 + 1][o1 + 1] = s;
  }
  return HS_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

int sweep_create(Ctx* c, const Stencil* coarse, int J, const int64_t* beta, const int64_t* bt,
                 const int64_t* lo, const int64_t* hi, const Stencil* const* slabs,
                 Sweep** out) {
  if (coarse->dim != 2)
    return set_error(c, HS_E_SHAPE, "the device sweep supports 2-D levels (3-D: not yet)");
  if (J < 2) return set_error(c, HS_E_SHAPE, "the sweep needs at least 2 subdomains");
  Sweep* s = new Sweep();
  s->J = J;
  s->n0 = (int)coarse->shape[0];
  s->M = (int)coarse->shape[1];
  s->coarse = coarse;
  const int M = s->M;
  std::vector<SlabInfo> info(J);
  for (int j = 0; j < J; ++j) {
    const Stencil* op = slabs[j];
    const int T = (int)(hi[j] - lo[j] + 1);
    if (T > 32) {
      delete s;
      return set_error(c, HS_E_SHAPE, "slab thicker than 32 layers: not supported by the sweep");
    }
    if (T > 16) s->tm = 32;
    if (op->dim != 2 || op->shape[0] != T || op->shape[1] != M) {
      delete s;
      return set_error(c, HS_E_SHAPE, "slab operator shape does not match the partition");
    }
    info[j].coeffs = op->d.coeffs;
    info[j].T = T;
    if (int r = slot_table(op, info[j].slot, c)) { delete s; return r; }
  }
  const int TM = s->tm, TM2 = TM * TM;
  s->L = 0;
  while ((1 << s->L) < M) ++s->L;
  if (s->L > kMaxLevels) { delete s; return set_error(c, HS_E_SHAPE, "face too long"); }
  s->ktot = 0;
  for (int l = 0; l < s->L; ++l) s->ktot += (M - 1) / (2 << l) + 1;
  // cluster size: ~32 face points per CTA, at most 16 CTAs, schedulable twice
  int C = std::min(16, std::max(1, (M + 31) / 32));
  for (;;) {
    const int nloc = (M + C - 1) / C + 1;
    int maxc = 0;
    cudaError_t e = TM == 16 ? prepare_solve<16>(C, nloc, &maxc) : prepare_solve<32>(C, nloc, &maxc);
    if (e == cudaSuccess && maxc >= 2) break;
    cudaGetLastError();
    if (C == 1) {
      delete s;
      return set_error(c, HS_E_CUDA, "no schedulable cluster for the sweep kernel");
    }
    C = C > 8 ? 8 : C / 2;
  }
  s->C = C;
  s->nloc_max = (M + C - 1) / C + 1;

  const size_t efb = (size_t)J * M * TM2 * sizeof(double2);
  const size_t ebb = 2 * efb;
  const size_t krb = (size_t)J * s->ktot * 2 * TM2 * sizeof(double2);
  s->factor_bytes = (long long)(efb + ebb + krb);
  cudaError_t e = cudaMalloc((void**)&s->ef, efb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->eb, ebb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->kr, krb);
  if (e != cudaSuccess) {
    sweep_destroy(s);
    return check_cuda(c, e, "factor alloc");
  }
  int r = TM == 16 ? factorize<16>(c, s, info) : factorize<32>(c, s, info);
  if (r) {
    sweep_destroy(s);
    return r;
  }

  // ---- schedules (task lists) ----
  int ntin = 0;
  auto mk = [&](int j, int a_, int b_) {
    SweepTask t{};
    t.slab = j - 1;
    t.lo = (int)lo[j - 1];
    t.T = (int)(hi[j - 1] - lo[j - 1] + 1);
    t.a = a_;
    t.b = b_;
    t.ta = a_;
    t.tb = b_;
    t.tin1 = t.tin3 = t.out2 = t.out4 = -1;
    t.row1 = t.row3 = t.orow2 = t.orow4 = -1;
    return t;
  };
  auto want1 = [&](SweepTask& t, int j) {   // tau1 (forward in), gated j > 1
    if (j <= 1) return -1;
    t.tin1 = ntin++;
    t.row1 = (int)beta[j - 1] - t.lo;
    return t.tin1;
  };
  auto want3 = [&](SweepTask& t, int j) {   // tau3 (backward in), gated j < J
    if (j >= J) return -1;
    t.tin3 = ntin++;
    t.row3 = (int)bt[j] - t.lo;
    return t.tin3;
  };
  auto give2 = [&](SweepTask& t, int j, int buf) {   // tau2 (forward out), gated j < J
    if (j >= J || buf < 0) return;
    t.out2 = buf;
    t.orow2 = (int)beta[j] - t.lo;
  };
  auto give4 = [&](SweepTask& t, int j, int buf) {   // tau4 (backward out), gated j > 1
    if (j <= 1 || buf < 0) return;
    t.out4 = buf;
    t.orow4 = (int)bt[j - 1] - t.lo;
  };
  auto fwd_task = [&](int j) { return mk(j, (int)beta[j - 1], (int)beta[j]); };
  auto bwd_task = [&](int j) { return mk(j, (int)bt[j - 1], (int)bt[j]); };
  std::vector<SweepTask>& T = s->tasks;
  auto fwd_chain = [&](int j0, int j1, std::vector<SweepTask>& pass) {
    for (int j = j0; j <= j1; ++j) {
      if (j < 1 || j > J) continue;
      SweepTask t = fwd_task(j);
      want1(t, j);
      if (!pass.empty() && j > 1 && pass.back().slab == j - 2 && pass.back().out2 == -2)
        give2(pass.back(), j - 1, t.tin1);
      if (j < J) t.out2 = -2;   // placeholder until a consumer appears
      pass.push_back(t);
    }
  };
  auto bwd_chain = [&](int j0, int j1, std::vector<SweepTask>& pass) {
    for (int j = j0; j >= j1; --j) {
      if (j < 1 || j > J) continue;
      SweepTask t = bwd_task(j);
      want3(t, j);
      if (!pass.empty() && j < J && pass.back().slab == j && pass.back().out4 == -2)
        give4(pass.back(), j + 1, t.tin3);
      if (j > 1) t.out4 = -2;
      pass.push_back(t);
    }
  };
  auto clear_placeholders = [&](std::vector<SweepTask>& v) {
    for (auto& t : v) {
      if (t.out2 == -2) t.out2 = -1;
      if (t.out4 == -2) t.out4 = -1;
    }
  };
  const double rec_bytes = (double)(3 * M + 2 * s->ktot) * TM2 * 16.0;
  // one solve launch per stage (up to two concurrent fronts)
  auto emit_pass = [&](std::vector<SweepLaunch>& plan, int src,
                       std::vector<std::vector<std::vector<SweepTask>>> stages) {
    for (auto& st : stages) {
      SweepLaunch fl{};
      fl.kind = SweepLaunch::kSolve;
      fl.src = src;
      for (auto& fr : st) {
        if (fr.empty()) continue;
        fl.ffirst[fl.nfront] = (int)T.size();
        fl.fcount[fl.nfront] = (int)fr.size();
        fl.nfront++;
        for (auto t : fr) {
          t.dst = src;
          double b = rec_bytes + (double)M * 16.0 * ((t.b - t.a) + (t.tb - t.ta));
          b += (double)M * 32.0 * ((t.tin1 >= 0) + (t.tin3 >= 0) + (t.out2 >= 0) + (t.out4 >= 0));
          fl.bytes += b;
          T.push_back(t);
        }
      }
      if (fl.nfront) plan.push_back(fl);
    }
  };
  // ---- UD: forward 1..J on f; g = f - A u; backward J..1 on g ----
  {
    std::vector<SweepLaunch>& plan = s->plan[HS_VARIANT_UD];
    std::vector<SweepTask> F, B;
    fwd_chain(1, J, F);
    clear_placeholders(F);
    bwd_chain(J, 1, B);
    clear_placeholders(B);
    emit_pass(plan, 0, {{F}});
    plan.push_back(SweepLaunch{SweepLaunch::kResidual});
    emit_pass(plan, 1, {{B}});
    plan.push_back(SweepLaunch{SweepLaunch::kCombine});
    s->has_plan[HS_VARIANT_UD] = true;
  }
  // ---- X: simultaneous half sweeps meeting at jm = J/2 + 1 ----
  if (J % 2 == 0) {
    std::vector<SweepLaunch>& plan = s->plan[HS_VARIANT_X];
    const int jm = J / 2 + 1;
    std::vector<SweepTask> F, B, MI;
    fwd_chain(1, jm - 1, F);
    bwd_chain(J, jm + 1, B);
    SweepTask mi = mk(jm, (int)beta[jm - 1], (int)bt[jm]);
    want1(mi, jm);
    want3(mi, jm);
    if (!F.empty() && F.back().out2 == -2) give2(F.back(), jm - 1, mi.tin1);
    if (!B.empty() && B.back().out4 == -2) give4(B.back(), jm + 1, mi.tin3);
    clear_placeholders(F);
    clear_placeholders(B);
    MI.push_back(mi);
    emit_pass(plan, 0, {{F, B}, {MI}});
    plan.push_back(SweepLaunch{SweepLaunch::kResidual});
    std::vector<SweepTask> MO, BB, FF;
    SweepTask mo = mk(jm, (int)bt[jm - 1], (int)beta[jm]);
    bwd_chain(jm - 1, 1, BB);
    fwd_chain(jm + 1, J, FF);
    if (!FF.empty()) give2(mo, jm, FF.front().tin1);
    if (!BB.empty()) give4(mo, jm, BB.front().tin3);
    clear_placeholders(BB);
    clear_placeholders(FF);
    MO.push_back(mo);
    emit_pass(plan, 1, {{MO}, {BB, FF}});
    plan.push_back(SweepLaunch{SweepLaunch::kCombine});
    s->has_plan[HS_VARIANT_X] = true;
  }
  const size_t tb = T.size() * sizeof(SweepTask);
  e = cudaMalloc((void**)&s->d_tasks, tb);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_tasks, T.data(), tb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMalloc((void**)&s->trace, (size_t)std::max(1, ntin) * 2 * M * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->g, (size_t)s->n0 * M * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->u2, (size_t)s->n0 * M * sizeof(double2));
  if (e != cudaSuccess) {
    sweep_destroy(s);
    return check_cuda(c, e, "sweep buffers");
  }
  *out = s;
  return HS_OK;
}

void sweep_destroy(Sweep* s) {
  if (!s) return;
  cudaFree(s->ef);
  cudaFree(s->eb);
  cudaFree(s->kr);
  cudaFree(s->trace);
  cudaFree(s->g);
  cudaFree(s->u2);
  cudaFree(s->d_tasks);
  delete s;
}

int sweep_apply(Ctx* c, Sweep* s, int variant, const double2* f, double2* u) {
  if (variant < 0 || variant > 1 || !s->has_plan[variant])
    return set_error(c, HS_E_ARG,
                     variant == HS_VARIANT_X ? "X-sweep needs an even subdomain count"
                                             : "unknown sweep variant");
  const int M = s->M;
  for (const SweepLaunch& Lh : s->plan[variant]) {
    switch (Lh.kind) {
      case SweepLaunch::kCombine: {
        // u = u_pass1 + u_pass2 (the order of the reference's u[ta:tb] += ud)
        const int64_t n = (int64_t)s->n0 * M;
        ProfScope ps(c, K_SWEEP_GATHER, 48.0 * n);
        k_combine<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(u, s->u2, n);
        HS_LAUNCH_CHECK(c, "combine kernel");
        break;
      }
      case SweepLaunch::kResidual: {
        int r = stencil_apply(c, s->coarse, u, s->g, 1, f);
        if (r) return r;
        break;
      }
      case SweepLaunch::kSolve: {
        SolveArgs a{};
        a.tasks = s->d_tasks;
        for (int i = 0; i < 2; ++i) {
          a.ffirst[i] = i < Lh.nfront ? Lh.ffirst[i] : 0;
          a.fcount[i] = i < Lh.nfront ? Lh.fcount[i] : 0;
        }
        a.C = s->C;
        a.M = M;
        a.L = s->L;
        a.ktot = s->ktot;
        a.nloc_max = s->nloc_max;
        a.nslot = s->tm == 16 ? Ring<16>::nslot(s->nloc_max) : Ring<32>::nslot(s->nloc_max);
        int acc = 0;
        for (int l = 0; l < s->L; ++l) {
          a.koff[l] = acc;
          acc += (M - 1) / (2 << l) + 1;
        }
        a.ef = s->ef;
        a.eb = s->eb;
        a.kr = s->kr;
        a.src = Lh.src ? s->g : f;
        a.coarse = s->coarse->d.coeffs;
        a.ncoarse = s->coarse->d.n;
        if (int r = slot_table(s->coarse, a.cslot, c)) return r;
        a.trace = s->trace;
        a.u[0] = u;
        a.u[1] = s->u2;
        static const char* trace_path = getenv("HS_SWEEP_TRACE");
        static bool traced = false;
        unsigned long long* dbg = nullptr;
        if (trace_path && !traced && Lh.nfront == 2) {
          cudaMalloc((void**)&dbg, 16 * 512 * sizeof(unsigned long long));
          cudaMemsetAsync(dbg, 0, 16 * 512 * sizeof(unsigned long long), c->stream);
        }
        a.dbg = dbg;

        ProfScope ps(c, K_SWEEP_FRONT, Lh.bytes);
        cudaError_t e = s->tm == 16 ? launch_solve<16>(a, Lh.nfront, c->stream)
                                    : launch_solve<32>(a, Lh.nfront, c->stream);
        if (e != cudaSuccess) return check_cuda(c, e, "sweep solve launch");
        HS_LAUNCH_CHECK(c, "sweep solve kernel");
        if (dbg) {
          std::vector<unsigned long long> h(16 * 512);
          cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, c->stream);
          cudaStreamSynchronize(c->stream);
          cudaFree(dbg);
          traced = true;
          if (FILE* fp = fopen(trace_path, "w")) {
            // per CTA of cluster 0: 512 stamps (task 1): [0] start, [1] after rhs barrier,
            // [2+p] after phase p barrier, [63] end, [64+8p+k] item 0 of phase p:
            // k = 0 start, 1 seq, 2 mbar, 3 compute, 4 refill   (ns, relative to CTA 0 [0])
            fprintf(fp, "# C=%d M=%d L=%d\n", s->C, M, s->L);
            const unsigned long long t0 = h[0];
            for (int b = 0; b < std::min(16, s->C); ++b) {
              for (int k = 0; k < 512; ++k)
                fprintf(fp, "%lld ", h[b * 512 + k] ? (long long)(h[b * 512 + k] - t0) : -1LL);
              fprintf(fp, "\n");
            }
            fclose(fp);
          }
        }
        break;
      }
    }
  }
  return HS_OK;
}

}  // namespace hs
