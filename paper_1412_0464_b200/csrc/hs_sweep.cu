// Coarse-level sweeping preconditioner on B200: partitioned slab solves
// (SPIKE with block cyclic reduction inside each partition), one thread-block
// cluster per sweep front.
//
// Reference: build_partition + Factorization (sweepdd.py:192-218,
// sparselin.py:40-68), subdom_solve (sweepdd.py:236-268), TransmissionMatrix
// (sweepdd.py:98-141), forward/backward/mid sweeps, prec_ud / prec_x
// (sweepdd.py:271-359).
//
// Slab system.  A slab of T <= 32 layers along the sweep axis and M face points
// is block tridiagonal along the face: block y couples to y-1 (L_y), y (D_y),
// y+1 (U_y), blocks tm x tm (tm = 16 or 32, T padded with identity rows).
// SuperLU's sparse LU is a chain of ~2*M*T dependent rows per solve.  Here the
// face is cut into C chunks, one per CTA of a cluster (C <= 16):
//   A x = f  <=>  x_k = g_k - W_k x_{first(k)-1} - V_k x_{last(k)+1},
//   g_k = A_k^{-1} f_k (chunk-local), W_k / V_k the chunk's spikes
//   (A_k^{-1} applied to the couplings leaving the chunk).
// 1. every CTA solves its chunk by block cyclic reduction (BCR): 2*ceil(log2 m)
//    phases of independent tm x tm mat-vecs separated by __syncthreads only;
// 2. the chunk-end values of g (the "tips") are pushed to every CTA (DSMEM
//    stores) and one cluster barrier later each CTA applies its two rows of the
//    precomputed inverse of the 2(C-1)-block interface system (R) to them;
// 3. x_k = g_k - W_k alpha - V_k beta for every block (independent mat-vecs).
// Two cluster barriers per slab instead of one per BCR level.
//
// Setup (all on the device, batched over slabs and chunks): chunk-local BCR
// Schur complements (k_bcr_elim / k_bcr_keep per level, Gauss-Jordan with
// partial pivoting inside each block, no pivoting across blocks -- SURVEY H2),
// spikes by a block-Thomas pass per chunk (k_spikes), and R by block-Thomas
// elimination of the interface system with identity right-hand sides
// (k_reduced).
//
// Apply: every matrix a CTA needs (BCR records, R column blocks, spikes) is
// streamed into a shared-memory ring by TMA bulk copies in consumption order,
// up to NSLOT items ahead, also across slab solves; vectors stay in shared
// memory.  Dense blocks are stored "lane-major" so a warp's 16-byte loads are
// contiguous 512-byte lines.  Transmission (sweepdd.py:113-118) is applied by
// the consumer when it builds its right-hand side, from the producer's two
// trace rows in global memory and the global operator's interface couplings.

#include "hs_common.cuh"
#include "hs_sweep.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace hs {

namespace {

constexpr int kMaxLevels = 16;     // local BCR levels: chunks up to 65536 points
constexpr int kWarps = 16;        // 15 consumer warps + 1 TMA producer warp
constexpr int kCW = kWarps - 1;
#ifndef HS_SWEEP_NA
#define HS_SWEEP_NA 8
#endif
constexpr int kNA = HS_SWEEP_NA;   // consumer warps of the back substitution while the rest
                                   // run the interface GEMV (group B = kCW - kNA warps)
static_assert(HS_SWEEP_NA >= 1 && HS_SWEEP_NA <= 8,
              "group B's partial-sum slots also hold the dense top's 15 partials");
#ifndef HS_SWEEP_PREFETCH
#define HS_SWEEP_PREFETCH 0
#endif
#ifndef HS_SWEEP_HALF      // tm 16: one ring item per half warp
#define HS_SWEEP_HALF 0
#endif
#ifndef HS_SWEEP_L2NEXT    // consumers prefetch the next slab's stream into L2
#define HS_SWEEP_L2NEXT 0
#endif
#ifndef HS_SWEEP_EXP       // timing experiments: 1 no item arithmetic, 2 no factor copies
#define HS_SWEEP_EXP 0
#endif
#if (HS_SWEEP_EXP & 8) && !(HS_SWEEP_EXP & 2)
#error "HS_SWEEP_EXP bit 8 (no ring reuse wait) needs bit 2 (no copies)"
#endif
#ifndef HS_SWEEP_DIRECT    // experiment: consumers read factor blocks straight from global memory
#define HS_SWEEP_DIRECT 0
#endif
#ifndef HS_SWEEP_G16       // tm 16: blocks per ring chunk (bulk copy)
#define HS_SWEEP_G16 4
#endif
constexpr int kMaxC = 16;         // chunks (CTAs) per cluster
constexpr int kMaxG = 8;          // face segments (clusters) per front
constexpr int kMaxCh = 64;        // chunks over the whole face
constexpr int kNR = 8;             // rows of a restricted (last-level / spike) update
constexpr int kMaxTasks = 1024;    // slab solves per front per launch

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

// chunk geometry: the face is cut into G segments of C chunks each (chunk
// K = seg * C + rank covers face points [y0s[K], y0s[K+1])); one cluster of
// C CTAs solves one segment, the G clusters of a front couple through a
// second-level interface system (two-level SPIKE, see k_level2).
struct Chunks {
  int M, C, L, kstride;
  int G;                   // segments (clusters) per front
  int q;                   // dense top: blocks per chunk left after L levels
  int nr;                  // restricted level-0 / spike updates (kNR rows) or 0
  int cpl0;                // level-0 kept updates from the sparse stencil couplings (one
                           // streamed block of 6 tm values) instead of alpha / gamma blocks
  int koff[kMaxLevels];
  int y0s[kMaxCh + 1];     // chunk K covers face points [y0s[K], y0s[K+1])
  int mmax;                // longest chunk
  __host__ __device__ int nch() const { return C * G; }
  __host__ __device__ int xstride() const { return G > 1 ? 1 + 4 * (G - 1) + 4 : 0; }
  __host__ __device__ int y0(int k) const { return y0s[k]; }
  __host__ __device__ int len(int k) const { return y0s[k + 1] - y0s[k]; }
  __host__ __device__ int chunk_of(int y) const {
    int k = 0;
    while (y >= y0s[k + 1]) ++k;
    return k;
  }
};

// ---------------------------------------------------------------------------
// setup kernels (thread (r, c) of a tm x tm block)

// Dense D, L, U of every block; couplings that leave a chunk are moved to
// EL / EU (the spikes' right-hand sides) and zeroed in L / U.
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_bcr_init(const SlabInfo* __restrict__ slabs, Chunks g, double2* __restrict__ D,
           double2* __restrict__ Lc, double2* __restrict__ Uc, double2* __restrict__ EL,
           double2* __restrict__ EU) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int y = blockIdx.x, s = blockIdx.y, M = g.M;
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
  const int64_t off = ((int64_t)s * M + y) * TM2 + r * TM + c;
  double2 d = coef(c - r, 0);
  if (r >= T || c >= T) d = make_double2(r == c ? 1.0 : 0.0, 0.0);
  D[off] = d;
  double2 l = coef(c - r, -1), u = coef(c - r, 1);
  const int k = g.chunk_of(y);
  if (y == g.y0(k)) {
    EL[((int64_t)s * g.nch() + k) * TM2 + r * TM + c] = l;
    l = czero();
  }
  if (y == g.y0(k + 1) - 1) {
    EU[((int64_t)s * g.nch() + k) * TM2 + r * TM + c] = u;
    u = czero();
  }
  Lc[off] = l;
  Uc[off] = u;
}

// Level-0 couplings of every face point to its two face neighbours (the
// tridiagonal thin-axis stencil of the slab operator), for the solve's
// level-0 kept updates: cpl[slab][y][side][o0 + 1][row], side 0 = y - 1.
template <int TM>
__global__ void __launch_bounds__(256)
k_cpl0(const SlabInfo* __restrict__ slabs, int M, double2* __restrict__ cpl) {
  const int y = blockIdx.x, s = blockIdx.y;
  const SlabInfo si = slabs[s];
  const int64_t n = (int64_t)si.T * M;
  for (int e = threadIdx.x; e < 2 * 3 * TM; e += blockDim.x) {
    const int side = e / (3 * TM), o0 = (e / TM) % 3 - 1, r = e % TM;
    const int o1 = side ? 1 : -1, sl = si.slot[o0 + 1][o1 + 1];
    double2 v = czero();
    if (sl >= 0 && r < si.T && r + o0 >= 0 && r + o0 < si.T && y + o1 >= 0 && y + o1 < M)
      v = si.coeffs[(int64_t)sl * n + (int64_t)r * M + y];
    cpl[((int64_t)s * M + y) * TM * TM + e] = v;   // one (padded) block per face point
  }
}

// In-place Gauss-Jordan inversion with partial pivoting of an N x N matrix A
// (smem, pitch N+1) into Inv; any block size, threads loop over elements
// (blockDim.x >= 256 assumed for the register staging below).
template <int N, int NT = 256>
__device__ void gj_invert(double2 (*A)[N + 1], double2 (*Inv)[N + 1], int* piv_row,
                          double* piv_abs, unsigned long long* err, unsigned long long code) {
  const int tid = threadIdx.x, nt = blockDim.x;   // nt >= NT
  constexpr int PER = (N * N + NT - 1) / NT;
  for (int e = tid; e < N * N; e += nt) Inv[e / N][e % N] = make_double2(e / N == e % N, 0.0);
  __syncthreads();
  for (int p = 0; p < N; ++p) {
    if (tid < 32) {
      double v = -1.0;
      int idx = 0;
      for (int i = tid; i < N; i += 32) {
        const double av = i >= p ? cabs2(A[i][p]) : -1.0;
        if (av > v) { v = av; idx = i; }
      }
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
      if (tid == 0) {
        atomicMin(err, code + (unsigned long long)p);
        A[p][p] = make_double2(1.0, 0.0);
      }
      __syncthreads();
    } else if (pr != p) {
      for (int cc = tid; cc < N; cc += nt) {
        double2 t = A[p][cc]; A[p][cc] = A[pr][cc]; A[pr][cc] = t;
        t = Inv[p][cc]; Inv[p][cc] = Inv[pr][cc]; Inv[pr][cc] = t;
      }
      __syncthreads();
    }
    const double2 inv_p = cdiv(make_double2(1.0, 0.0), A[p][p]);
    double2 na[PER], ni[PER];   // read phase
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * nt;
      if (e >= N * N) continue;
      const int r = e / N, cc = e % N;
      const double2 npc = cmul(A[p][cc], inv_p), nic = cmul(Inv[p][cc], inv_p);
      if (r == p) {
        na[q] = npc;
        ni[q] = nic;
      } else {
        const double2 arp = A[r][p];
        na[q] = csub(A[r][cc], cmul(arp, npc));
        ni[q] = csub(Inv[r][cc], cmul(arp, nic));
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q) {   // write phase
      const int e = tid + q * nt;
      if (e >= N * N) continue;
      A[e / N][e % N] = na[q];
      Inv[e / N][e % N] = ni[q];
    }
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

// Eliminated blocks of level l in every chunk (local odd multiples of s):
// Dinv, Dinv L, Dinv U.  D[y] is overwritten with Dinv for the keep kernel.
// top != 0: the last block standing in each chunk (local 0).
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_bcr_elim(int level, Chunks g, int top, double2* __restrict__ D,
           const double2* __restrict__ Lc, const double2* __restrict__ Uc,
           double2* __restrict__ ef, double2* __restrict__ eb,
           unsigned long long* __restrict__ err) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int s_ = 1 << level;
  const int slab = blockIdx.y / g.nch(), k = blockIdx.y % g.nch();
  const int yl = top ? 0 : (2 * blockIdx.x + 1) * s_;
  if (yl >= g.len(k)) return;
  const int y = g.y0(k) + yl, M = g.M;
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

// Kept blocks of level l (local multiples of 2s): alpha, gamma and the next
// level's D, L, U (in place).
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_bcr_keep(int level, Chunks g, double2* __restrict__ D, double2* __restrict__ Lc,
           double2* __restrict__ Uc, double2* __restrict__ kr) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int s_ = 1 << level;
  const int slab = blockIdx.y / g.nch(), k = blockIdx.y % g.nch();
  const int j = blockIdx.x;
  const int yl = j * 2 * s_, m = g.len(k);
  if (yl >= m) return;
  const int y = g.y0(k) + yl, M = g.M;
  const int left = y - s_, right = y + s_;
  const bool hl = yl - s_ >= 0, hr = yl + s_ < m;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*S0)[TM + 1] = reinterpret_cast<double2(*)[TM + 1]>(smraw);
  double2(*S1)[TM + 1] = S0 + TM;
  double2(*Al)[TM + 1] = S1 + TM;
  double2(*Ga)[TM + 1] = Al + TM;
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  auto at = [&](int yy) { return ((int64_t)slab * M + yy) * TM2; };
  double2* kout = kr + (((int64_t)slab * g.nch() + k) * g.kstride + g.koff[level] + j) * 2 * TM2;
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

// Dense top of every chunk (one CTA per slab x chunk): after L cyclic-reduction
// levels the chunk's kept blocks (local multiples of S = 2^L, q_k of them)
// form a block-tridiagonal system D, L, U; its inverse (padded to Q blocks
// with identity) is stored lane-major per block: qd[slab][k][r][c].
template <int TM, int Q>
__global__ void __launch_bounds__(1024)
k_dense_top(Chunks g, const double2* __restrict__ D, const double2* __restrict__ Lc,
            const double2* __restrict__ Uc, double2* __restrict__ qd,
            unsigned long long* __restrict__ err) {
  constexpr int TM2 = Geo<TM>::TM2;
  constexpr int N = Q * TM;
  const int slab = blockIdx.x / g.nch(), k = blockIdx.x % g.nch(), M = g.M;
  const int S = 1 << g.L, Y0 = g.y0(k);
  const int qk = (g.len(k) - 1) / S + 1;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*A)[N + 1] = reinterpret_cast<double2(*)[N + 1]>(smraw);
  double2(*Inv)[N + 1] = A + N;
  __shared__ int piv_row;
  __shared__ double piv_abs;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int R = e / N, Cc = e % N;
    const int br = R / TM, bc = Cc / TM, r = R % TM, c = Cc % TM;
    double2 v = make_double2(R == Cc ? 1.0 : 0.0, 0.0);
    if (br < qk && bc < qk) {
      const int64_t at = ((int64_t)slab * M + Y0 + br * S) * TM2 + r * TM + c;
      v = bc == br ? D[at] : bc == br - 1 ? Lc[at] : bc == br + 1 ? Uc[at] : czero();
    }
    A[R][Cc] = v;
  }
  __syncthreads();
  const unsigned long long code =
      ((unsigned long long)slab << 40) | ((unsigned long long)Y0 * TM & 0xffffffffffull);
  gj_invert<N, 1024>(A, Inv, &piv_row, &piv_abs, err, code);
  double2* out = qd + ((int64_t)slab * g.nch() + k) * Q * Q * TM2;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int R = e / N, Cc = e % N;
    out[((R / TM) * Q + Cc / TM) * TM2 + lm<TM>(R % TM, Cc % TM)] = Inv[R][Cc];
  }
}

// Spikes of every chunk by one block-Thomas pass (one CTA per slab x chunk):
//   W = A_k^{-1} [EL; 0 ...],  V = A_k^{-1} [... 0; EU]
// stored lane-major per block (sp[y] = {W_y, V_y}) plus the four tips
// (W_first, W_last, V_first, V_last; natural layout) for the interface system.
// Uses pristine D, L, U (run before the BCR levels).  Hw / Zw: work [J][M][tm^2].
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_spikes(Chunks g, const double2* __restrict__ D, const double2* __restrict__ Lc,
         const double2* __restrict__ Uc, const double2* __restrict__ EL,
         const double2* __restrict__ EU, double2* __restrict__ Hw, double2* __restrict__ Zw,
         double2* __restrict__ sp, double2* __restrict__ tips,
         unsigned long long* __restrict__ err) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int slab = blockIdx.x / g.nch(), k = blockIdx.x % g.nch(), M = g.M;
  const int Y0 = g.y0(k), Y1 = g.y0(k + 1);
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*A)[TM + 1] = reinterpret_cast<double2(*)[TM + 1]>(smraw);
  double2(*Inv)[TM + 1] = A + TM;
  double2(*Hp)[TM + 1] = Inv + TM;   // H_{y-1}
  double2(*Zp)[TM + 1] = Hp + TM;    // Z_{y-1} (W forward)
  double2(*B)[TM + 1] = Zp + TM;
  double2(*Wn)[TM + 1] = B + TM;     // W_{y+1}
  double2(*Vn)[TM + 1] = Wn + TM;    // V_{y+1}
  __shared__ int piv_row;
  __shared__ double piv_abs;
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  auto at = [&](int yy) { return ((int64_t)slab * M + yy) * TM2; };
  const double2* el = EL + ((int64_t)slab * g.nch() + k) * TM2;
  const double2* eu = EU + ((int64_t)slab * g.nch() + k) * TM2;
  double2* tp = tips + ((int64_t)slab * g.nch() + k) * 4 * TM2;
  Hp[r][c] = czero();
  Zp[r][c] = czero();
  double2 zv_last = czero();
  for (int y = Y0; y < Y1; ++y) {
    // D~ = D - L H_{y-1} (L zero at the chunk start)
    load_mat<TM>(B, Lc + at(y));
    __syncthreads();
    double2 d = D[at(y) + r * TM + c];
    d = csub(d, mm_rc<TM>(B, Hp));
    A[r][c] = d;
    __syncthreads();
    const unsigned long long code =
        ((unsigned long long)slab << 40) | ((unsigned long long)y * TM & 0xffffffffffull);
    gj_invert<TM>(A, Inv, &piv_row, &piv_abs, err, code);
    // Z_y = Inv (rhs_y - L Z_{y-1}); rhs = EL at the chunk start, else 0
    double2 t = cscale(-1.0, mm_rc<TM>(B, Zp));
    if (y == Y0) t = el[r * TM + c];
    __syncthreads();
    A[r][c] = t;
    __syncthreads();
    const double2 z = mm_rc<TM>(Inv, A);
    __syncthreads();
    // H_y = Inv U_y
    load_mat<TM>(B, Uc + at(y));
    __syncthreads();
    const double2 h = mm_rc<TM>(Inv, B);
    __syncthreads();
    if (y == Y1 - 1) {   // V forward: nonzero only at the chunk end, Inv EU
      load_mat<TM>(B, eu);
      __syncthreads();
      zv_last = mm_rc<TM>(Inv, B);
    }
    __syncthreads();
    Hp[r][c] = h;
    Zp[r][c] = z;
    Hw[at(y) + r * TM + c] = h;
    Zw[at(y) + r * TM + c] = z;
    __syncthreads();
  }
  // backward: W_y = Z_y - H_y W_{y+1}, V_y = Zv_y - H_y V_{y+1}
  Wn[r][c] = czero();
  Vn[r][c] = czero();
  __syncthreads();
  for (int y = Y1 - 1; y >= Y0; --y) {
    load_mat<TM>(A, Hw + at(y));
    __syncthreads();
    const double2 w = csub(Zw[at(y) + r * TM + c], mm_rc<TM>(A, Wn));
    double2 v = cscale(-1.0, mm_rc<TM>(A, Vn));
    if (y == Y1 - 1) v = zv_last;
    __syncthreads();
    Wn[r][c] = w;
    Vn[r][c] = v;
    sp[2 * at(y) + lm<TM>(r, c)] = w;
    sp[2 * at(y) + TM2 + lm<TM>(r, c)] = v;
    if (y == Y0) {
      tp[0 * TM2 + r * TM + c] = w;
      tp[2 * TM2 + r * TM + c] = v;
    }
    if (y == Y1 - 1) {
      tp[1 * TM2 + r * TM + c] = w;
      tp[3 * TM2 + r * TM + c] = v;
    }
    __syncthreads();
  }
}

// Inverse of an interface system (one CTA per slab x group of C chunks: the
// segment's chunks at level 1, the G segments of the face at level 2).
// Unknowns per boundary b (between chunks b and b+1 of the group): xi_b =
// (alpha_b = x at the last point of chunk b, beta_b = x at the first point of
// chunk b+1); right-hand side tau_b = (g_b[last], g_{b+1}[first]):
//   alpha_b + Vb[last] beta_b + Wb[last] alpha_{b-1}            = g_b[last]
//   beta_b + W_{b+1}[first] alpha_b + V_{b+1}[first] beta_{b+1} = g_{b+1}[first]
// Block Thomas over b with identity right-hand sides gives R = S^{-1}; chunk k
// keeps rows alpha_{k-1} and beta_k, stored per column block q (tm columns) as
// 2tm x tm with the row index fastest.  tips: [slab][ngrp * C][4][tm^2],
// rk: [slab][ngrp * C][2(C-1)][2 tm^2].
template <int TM>
__global__ void __launch_bounds__(1024)
k_reduced(int C, int ngrp, const double2* __restrict__ tips, double2* __restrict__ Gw,
          double2* __restrict__ Zr, double2* __restrict__ rk,
          unsigned long long* __restrict__ err) {
  constexpr int TM2 = Geo<TM>::TM2;
  constexpr int N = 2 * TM;
  const int grp = blockIdx.x, slab = grp / ngrp, B = C - 1, NR = B * N;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*A)[N + 1] = reinterpret_cast<double2(*)[N + 1]>(smraw);
  double2(*Inv)[N + 1] = A + N;
  __shared__ int piv_row;
  __shared__ double piv_abs;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double2* tp = tips + (int64_t)grp * C * 4 * TM2;
  auto tip = [&](int k, int which, int r, int c) -> double2 {   // 0 Wf 1 Wl 2 Vf 3 Vl
    return tp[((int64_t)k * 4 + which) * TM2 + r * TM + c];
  };
  double2* G = Gw + (int64_t)grp * B * N * N;    // G_b = Dt_b^{-1} Up_b
  double2* Z = Zr + (int64_t)grp * NR * NR;      // block row b: rows b*N.., all NR columns
  for (int b = 0; b < B; ++b) {
    // D~_b = D_b - Lo_b G_{b-1};  D_b = [[I, V_b[l]], [W_{b+1}[f], I]]; Lo_b = [[W_b[l], 0],[0,0]]
    for (int e = tid; e < N * N; e += nt) {
      const int r = e / N, c = e % N;
      double2 d = make_double2(r == c ? 1.0 : 0.0, 0.0);
      if (r < TM && c >= TM) d = tip(b, 3, r, c - TM);
      if (r >= TM && c < TM) d = tip(b + 1, 0, r - TM, c);
      if (b > 0 && r < TM) {
        for (int q = 0; q < TM; ++q)
          d = csub(d, cmul(tip(b, 1, r, q), G[((int64_t)(b - 1) * N + q) * N + c]));
      }
      A[r][c] = d;
    }
    __syncthreads();
    gj_invert<N>(A, Inv, &piv_row, &piv_abs, err, ((unsigned long long)slab << 40));
    // G_b = Inv Up_b, Up_b = [[0,0],[0, V_{b+1}[first]]] (coupling to beta_{b+1})
    for (int e = tid; e < N * N; e += nt) {
      const int r = e / N, c = e % N;
      double2 acc = czero();
      if (b + 1 < B && c >= TM)
        for (int q = 0; q < TM; ++q) acc = cfma(Inv[r][TM + q], tip(b + 1, 2, q, c - TM), acc);
      G[((int64_t)b * N + r) * N + c] = acc;
    }
    // Z_b = Inv (E_b - Lo_b Z_{b-1})
    for (int e = tid; e < N * NR; e += nt) {
      const int r = e / NR, col = e % NR;
      double2 acc = czero();
      for (int q = 0; q < N; ++q) {
        double2 rhs = make_double2(col == b * N + q ? 1.0 : 0.0, 0.0);
        if (b > 0 && q < TM)
          for (int w = 0; w < TM; ++w)
            rhs = csub(rhs, cmul(tip(b, 1, q, w), Z[((int64_t)(b - 1) * N + w) * NR + col]));
        acc = cfma(Inv[r][q], rhs, acc);
      }
      Z[((int64_t)b * N + r) * NR + col] = acc;
    }
    __syncthreads();
  }
  // backward: X_b = Z_b - G_b X_{b+1}; X overwrites Z block rows
  for (int b = B - 2; b >= 0; --b) {
    for (int e = tid; e < N * NR; e += nt) {
      const int r = e / NR, col = e % NR;
      double2 acc = Z[((int64_t)b * N + r) * NR + col];
      for (int q = TM; q < N; ++q)   // G_b has nonzero columns only in the beta half
        acc = csub(acc, cmul(G[((int64_t)b * N + r) * N + q],
                             Z[((int64_t)(b + 1) * N + q) * NR + col]));
      Z[((int64_t)b * N + r) * NR + col] = acc;
    }
    __syncthreads();
  }
  // rows of chunk k: alpha_{k-1} (block k-1, rows 0..TM-1), beta_k (block k,
  // rows TM..2TM-1); column block q of tm columns
  for (int e = tid; e < C * N * NR; e += nt) {
    const int k = e / (N * NR), rem = e % (N * NR);
    const int r = rem / NR, col = rem % NR;
    double2 v = czero();
    if (r < TM && k > 0) v = Z[((int64_t)(k - 1) * N + r) * NR + col];
    if (r >= TM && k < B) v = Z[((int64_t)k * N + r) * NR + col];
    const int q = col / TM, cq = col % TM;
    rk[(((int64_t)grp * C + k) * (2 * B) + q) * (2 * TM2) + cq * N + r] = v;
  }
}

// Second level of the two-level partition (one CTA of tm x tm threads per
// slab x segment, C >= 2 chunks per segment).  With P_s = x at the last
// point of segment s-1 and Q_s = x at the first point of segment s+1 the
// segment's level-1 unknowns are affine in them:
//   (alpha_{k-1}, beta_k) = R_k tau - Pk P_s - Qk Q_s,
//   Pk = R_k[:, alpha_0] W_{K0}[last],  Qk = R_k[:, beta_{C-2}] V_{KL}[first]
// (K0 / KL the segment's first / last chunk), and its end values are
//   x_last  = c_s + E_s P_s + F_s Q_s,   c_s = g_KL[last] - W_KL[last] (R tau)_alpha
//   x_first = d_s + E'_s P_s + F'_s Q_s, d_s = g_K0[first] - V_K0[first] (R tau)_beta
// which is the chunk-level relation x = g - W alpha - V beta one level up, with
// segment "tips" Wf = -E', Wl = -E, Vf = -F', Vl = -F: k_reduced on them
// gives every segment its rows (P_s, Q_s) of the G-segment interface inverse.
// Writes tips2 [slab][G][4][tm^2] (natural layout) and, per chunk K, the
// level-2 stream blocks x2[slab][K][xstride][tm^2]: block 0 the c / d tip
// (W_KL[last] for the last chunk, V_K0[first] for the first, lane-major),
// blocks 1 + 4(G-1) .. the column blocks of [Pk | Qk] (2tm x tm, row index
// fastest, like R).  Blocks 1 .. 4(G-1) (the level-2 inverse rows of the
// segment's first chunk) are copied in after k_reduced of level 2.
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_level2(Chunks g, const double2* __restrict__ tips, const double2* __restrict__ rk,
         double2* __restrict__ tips2, double2* __restrict__ x2) {
  constexpr int TM2 = Geo<TM>::TM2;
  constexpr int N = 2 * TM;
  const int C = g.C, G = g.G, B = C - 1, nch = g.nch(), xs = g.xstride();
  const int slab = blockIdx.x / G, seg = blockIdx.x % G;
  const int K0 = seg * C, KL = K0 + C - 1;
  const int r = threadIdx.x / TM, c = threadIdx.x % TM;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*S0)[TM + 1] = reinterpret_cast<double2(*)[TM + 1]>(smraw);
  double2(*S1)[TM + 1] = S0 + TM;
  double2(*S2)[TM + 1] = S1 + TM;
  double2(*S3)[TM + 1] = S2 + TM;
  auto tip = [&](int K, int which) {   // 0 Wf 1 Wl 2 Vf 3 Vl, natural layout
    return tips + (((int64_t)slab * nch + K) * 4 + which) * TM2;
  };
  // R column block q of chunk K, element (row rr of 2tm, column cq)
  auto R = [&](int K, int q, int rr, int cq) {
    return rk[(((int64_t)slab * nch + K) * (2 * B) + q) * (2 * TM2) + cq * N + rr];
  };
  auto mm = [&](double2 (*A)[TM + 1], double2 (*Bm)[TM + 1]) {
    double2 acc = czero();
    for (int k = 0; k < TM; ++k) acc = cfma(A[r][k], Bm[k][c], acc);
    return acc;
  };
  const double2 wl0 = tip(K0, 1)[r * TM + c], vfL = tip(KL, 2)[r * TM + c];
  // (P_{C-1})_alpha = R_KL[alpha rows, col 0] W_K0[last]; E = W_KL[last] (P_{C-1})_alpha
  S0[r][c] = R(KL, 0, r, c);
  S1[r][c] = wl0;
  __syncthreads();
  S2[r][c] = mm(S0, S1);
  S3[r][c] = tip(KL, 1)[r * TM + c];
  __syncthreads();
  const double2 E = mm(S3, S2);
  __syncthreads();
  // (Q_{C-1})_alpha = R_KL[alpha rows, col 2B-1] V_KL[first]; F = W_KL[last] (.) - V_KL[last]
  S0[r][c] = R(KL, 2 * B - 1, r, c);
  S1[r][c] = vfL;
  __syncthreads();
  S2[r][c] = mm(S0, S1);
  __syncthreads();
  const double2 F = csub(mm(S3, S2), tip(KL, 3)[r * TM + c]);
  __syncthreads();
  // (P_0)_beta = R_K0[beta rows, col 0] W_K0[last]; E' = V_K0[first] (.) - W_K0[first]
  S0[r][c] = R(K0, 0, TM + r, c);
  S1[r][c] = wl0;
  S3[r][c] = tip(K0, 2)[r * TM + c];
  __syncthreads();
  S2[r][c] = mm(S0, S1);
  __syncthreads();
  const double2 Ep = csub(mm(S3, S2), tip(K0, 0)[r * TM + c]);
  __syncthreads();
  // (Q_0)_beta = R_K0[beta rows, col 2B-1] V_KL[first]; F' = V_K0[first] (.)
  S0[r][c] = R(K0, 2 * B - 1, TM + r, c);
  S1[r][c] = vfL;
  __syncthreads();
  S2[r][c] = mm(S0, S1);
  __syncthreads();
  const double2 Fp = mm(S3, S2);
  double2* t2 = tips2 + ((int64_t)slab * G + seg) * 4 * TM2;
  t2[0 * TM2 + r * TM + c] = cscale(-1.0, Ep);
  t2[1 * TM2 + r * TM + c] = cscale(-1.0, E);
  t2[2 * TM2 + r * TM + c] = cscale(-1.0, Fp);
  t2[3 * TM2 + r * TM + c] = cscale(-1.0, F);
  // per chunk: the c / d tip block and [Pk | Qk]
  for (int k = 0; k < C; ++k) {
    const int K = K0 + k;
    double2* xb = x2 + ((int64_t)slab * nch + K) * xs * TM2;
    double2 tv = czero();
    if (k == C - 1 && seg < G - 1) tv = tip(KL, 1)[r * TM + c];   // c_s: W_KL[last]
    if (k == 0 && seg > 0) tv = tip(K0, 2)[r * TM + c];           // d_s: V_K0[first]
    xb[lm<TM>(r, c)] = tv;
    double2* pq = xb + (int64_t)(1 + 4 * (G - 1)) * TM2;
    for (int h = 0; h < 2; ++h) {       // rows h*TM + r of the 2tm x tm column blocks
      const int rr = h * TM + r;
      double2 pa = czero(), qa = czero();
      for (int q = 0; q < TM; ++q) {
        pa = cfma(R(K, 0, rr, q), tip(K0, 1)[q * TM + c], pa);
        qa = cfma(R(K, 2 * B - 1, rr, q), tip(KL, 2)[q * TM + c], qa);
      }
      pq[c * N + rr] = pa;
      pq[2 * TM2 + c * N + rr] = qa;
    }
  }
}

// ---------------------------------------------------------------------------
// apply

struct SolveArgs {
  const SweepTask* tasks;
  int ffirst[kMaxFront], fcount[kMaxFront];
  Chunks g;
  int nchunk;              // ring slots (16-KB chunks)
  const double2* stream;   // [J][C][nbs] factor blocks in item order
  int64_t nbs;
  const uint32_t* plan;    // [C][plan_words] item / chunk tables (chunk_plan)
  const int* rows;         // [J][kNR] rows of the restricted updates (g.nr != 0)
  const double2* cpl;      // (unused: the level-0 couplings travel in the stream)
  const double2* src;      // right-hand side field (n0 x M)
  const double2* coarse;   // global coarse operator [S][n0*M] (transmission couplings)
  int64_t ncoarse;
  int cslot[3][3];
  double2* trace;          // [ntrace][2][M]
  double2* u[2];
  unsigned long long* dbg; // optional per-phase timestamps (HS_SWEEP_TRACE)
  // two-level partition (g.G > 1): per front f, segment s the c_s / d_s
  // vectors of the level-2 system, xbuf[f][task parity][s][c, d][tm], and
  // their arrival counters xflag[f][c, d][s] (monotone; this launch's task ti
  // posts value xbase[f] + ti + 1)
  double2* xbuf;
  unsigned* xflag;
  unsigned xbase[kMaxFront];
  // several right-hand sides through one chain (k_part_solve<TM, NR>): element
  // strides from one right-hand side's vectors to the next
  int64_t vs_src, vs_u[2];   // src, u[0], u[1]
  int64_t ts, xs;            // trace buffers, level-2 exchange buffers
};

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
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  const uint32_t a = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}
// 16-B global -> shared copy that does not block the thread (zero-fill when !ok)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ uint32_t map_rank(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// 16-B store into another CTA's shared memory, completing bytes on its mbarrier
__device__ __forceinline__ void st_async_c(uint32_t dst, double2 v, uint32_t bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
      ::"r"(dst), "d"(v.x), "d"(v.y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  if (bytes)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// acc = A0 v0 + A1 v1 (either term may be absent); A lane-major in shared
// memory, v in shared memory; every lane returns row (lane % tm)
template <int TM>
__device__ __forceinline__ double2 mvs2(const double2* m0, const double2* v0, const double2* m1,
                                        const double2* v1, int lane) {
  if (HS_SWEEP_EXP & 1) return czero();
  constexpr int CPL = Geo<TM>::CPL;
  const int hh = lane / TM;
  double2 a0 = czero(), a1 = czero(), a2 = czero(), a3 = czero();
  if (v0) {
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
      a0 = cfma(m0[k * 32 + lane], v0[CPL * hh + k], a0);
      a1 = cfma(m0[(k + 1) * 32 + lane], v0[CPL * hh + k + 1], a1);
    }
  }
  if (v1) {
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
      a2 = cfma(m1[k * 32 + lane], v1[CPL * hh + k], a2);
      a3 = cfma(m1[(k + 1) * 32 + lane], v1[CPL * hh + k + 1], a3);
    }
  }
  double2 acc = cadd(cadd(a0, a1), cadd(a2, a3));
  if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
  return acc;
}

// ---------------------------------------------------------------------------
// Item plan of one chunk solve, shared by the packing kernel (setup), the host
// (stream sizes) and the solve kernel.  Phases: p < L forward cyclic-reduction
// level p (eliminated points first, then kept ones); p == L the dense top,
// items (row r, column pair cp); L < p < NP back substitution of level 2L-p;
// then the 2B column blocks of R, the level-2 items (G > 1: the c / d tip,
// the first chunk's 2(G-1) column blocks of the segment inverse, the two
// column blocks of [Pk | Qk]) and the m spike blocks.
struct ItemPlan {
  int m, L, S, qk, QP, B, NP;
  int rank, seg, G;
  int ct, zq, pqn;               // level-2 items: c / d tip, inverse rows, [Pk | Qk]
  int plast;                     // phase after which the right tip g[m-1] is final
  int pfx[2 * kMaxLevels + 4];   // items before each phase (NP + 2 = total)
};

__host__ __device__ inline int plan_level(const ItemPlan& P, int p) {
  return p <= P.L ? p : 2 * P.L - p;
}
__host__ __device__ inline int plan_first(const ItemPlan& P, int p) {
  return p > P.L ? (1 << plan_level(P, p)) : 0;
}
__host__ __device__ inline int plan_step(const ItemPlan& P, int p) {
  return (p < P.L ? 1 : 2) << plan_level(P, p);
}
__host__ __device__ inline void plan_items(const Chunks& g, int K, ItemPlan& P) {
  P.m = g.len(K);
  P.L = g.L;
  P.S = 1 << g.L;
  P.qk = (P.m - 1) / P.S + 1;
  P.QP = (P.qk + 1) / 2;
  P.B = g.C - 1;
  P.NP = 2 * P.L + 1;
  P.rank = K % g.C;
  P.seg = K / g.C;
  P.G = g.G;
  P.ct = g.G > 1 && ((P.rank == 0 && P.seg > 0) || (P.rank == P.B && P.seg < g.G - 1)) ? 1 : 0;
  P.zq = g.G > 1 && P.rank == 0 ? 2 * (g.G - 1) : 0;
  P.pqn = g.G > 1 ? 2 : 0;
  int acc = 0;
  for (int p = 0; p < P.NP; ++p) {
    P.pfx[p] = acc;
    const int f = plan_first(P, p);
    if (p == P.L) acc += P.qk * P.QP;
    else if (f < P.m) acc += (P.m - 1 - f) / plan_step(P, p) + 1;
  }
  P.pfx[P.NP] = acc;
  P.pfx[P.NP + 1] = acc + (P.B > 0 ? 2 * P.B : 0) + P.ct + P.zq + P.pqn;
  P.pfx[P.NP + 2] = P.pfx[P.NP + 1] + (P.B > 0 ? P.m : 0);
  // the dense top, or the back-substitution level of m-1 (its lowest set bit)
  int tz = 0;
  while (P.m > 1 && (((P.m - 1) >> tz) & 1) == 0) ++tz;
  P.plast = (P.m == 1 || (P.m - 1) % P.S == 0) ? P.L : 2 * P.L - tz;
}
__host__ __device__ inline int plan_phase(const ItemPlan& P, int r) {
  int p = 0;
  while (P.pfx[p + 1] <= r) ++p;
  return p;
}

// Stream (= ring) order of one chunk solve's items, as (item, segment); a new
// segment starts a new copy chunk.  Phases up to the dense top in order; then
// the back substitution (warp group A) and the interface GEMV (group B) in
// interleaved runs -- the first A run holds every level the right tip needs,
// so group B's data never blocks it -- then the spikes.
constexpr int kRunA = 4, kRunB = 4;
template <class Fn>
__host__ __device__ inline void for_stream(const ItemPlan& P, Fn&& fn) {
  const int L = P.L, NP = P.NP;
  for (int r = 0; r < P.pfx[L + 1]; ++r) fn(r, plan_phase(P, r));
  int a = P.pfx[L + 1], b = P.pfx[NP];
  const int a_end = P.pfx[NP], b_end = P.pfx[NP + 1];
  const int first = P.pfx[(P.plast > L + 1 ? P.plast : L + 1) + 1];
  for (; a < first && a < a_end; ++a) fn(a, 64 + plan_phase(P, a));
  int seg = 128;
  bool turn_b = true;
  while (a < a_end || b < b_end) {
    if (turn_b && b < b_end) {
      for (int k = 0; k < kRunB && b < b_end; ++k) fn(b++, seg);
    } else if (a < a_end) {
      const int ph = plan_phase(P, a);
      for (int k = 0; k < kRunA && a < a_end && plan_phase(P, a) == ph; ++k) fn(a++, seg);
    }
    ++seg;
    turn_b = !turn_b;
  }
  for (int r = P.pfx[NP + 1]; r < P.pfx[NP + 2]; ++r) fn(r, 1 << 20);
}
// face point of item j of a cyclic-reduction phase
__host__ __device__ inline int plan_yl(const ItemPlan& P, int p, int j) {
  if (p > P.L) return plan_first(P, p) + j * plan_step(P, p);
  const int ne = (P.pfx[p + 1] - P.pfx[p]) / 2;
  return (j < ne ? 2 * j + 1 : 2 * (j - ne)) << p;
}

// Factor arrays of one slab before packing (setup only).
enum ItemArray : uint32_t {
  kArrEf = 0, kArrEb = 1, kArrKr = 2, kArrRk = 3, kArrSp = 4, kArrQd = 5, kArrEbr = 6, kArrSpr = 7,
  kArrX2 = 8, kArrCpl = 9
};
constexpr uint32_t kOffMask = (1u << 28) - 1;
__host__ __device__ constexpr uint32_t item_enc(uint32_t arr, int64_t off) {
  return (arr << 28) | (uint32_t)off;
}

// Source blocks of item r (array + offset from the slab base, in stream
// order); *hasx: the first block is the item's "x" operand (alpha / Dinv L /
// left), not only the right one.  Returns the block count (0..2).
template <int TM>
__host__ __device__ inline int item_sources(const Chunks& g, int rank, const ItemPlan& P, int r,
                                            uint32_t src[2], bool* hasx) {
  constexpr int TM2 = TM * TM;
  int p = 0;
  while (P.pfx[p + 1] <= r) ++p;
  const int j = r - P.pfx[p];
  const int Y0 = g.y0(rank), m = P.m;
  int n = 0;
  *hasx = true;
  if (p == P.L) {            // dense top: Q[row][c0], Q[row][c0 + 1]
    const int row = j / P.QP, c0 = 2 * (j % P.QP);
    const int64_t o = (((int64_t)rank * g.q + row) * g.q + c0) * TM2;
    src[n++] = item_enc(kArrQd, o);
    if (c0 + 1 < P.qk) src[n++] = item_enc(kArrQd, o + TM2);
  } else if (p < P.NP) {
    const int l = plan_level(P, p), s = 1 << l;
    const int yl = plan_yl(P, p, j);
    const int64_t y = Y0 + yl;
    if (p < P.L) {
      if ((yl >> l) & 1) {
        src[n++] = item_enc(kArrEf, y * TM2);
      } else if (g.cpl0 && l == 0) {   // F -= L Yv[y-1] + U Yv[y+1]: the sparse couplings'
        *hasx = false;                 // block (6 TM values) instead of alpha, gamma
        src[n++] = item_enc(kArrCpl, y * TM2);
      } else {
        const int64_t k2 = ((int64_t)rank * g.kstride + g.koff[l] + (yl >> (l + 1))) * 2 * TM2;
        *hasx = yl - s >= 0;
        if (yl - s >= 0) src[n++] = item_enc(kArrKr, k2);
        if (yl + s < m) src[n++] = item_enc(kArrKr, k2 + TM2);
      }
    } else if (g.nr && l == 0 && yl != m - 1) {   // restricted level-0 update (one block)
      src[n++] = item_enc(kArrEbr, y * TM2);
    } else {
      if (yl - s >= 0) src[n++] = item_enc(kArrEb, y * 2 * TM2);
      if (yl + s < m) src[n++] = item_enc(kArrEb, y * 2 * TM2 + TM2);
    }
  } else if (p == P.NP && j < 2 * P.B) {   // R column block j (2tm x tm, two blocks)
    const int64_t o = ((int64_t)rank * (2 * P.B) + j) * (2 * TM2);
    src[n++] = item_enc(kArrRk, o);
    src[n++] = item_enc(kArrRk, o + TM2);
  } else if (p == P.NP) {    // level 2: c / d tip, inverse rows, [Pk | Qk]
    const int jj = j - 2 * P.B;
    const int64_t xb = (int64_t)rank * g.xstride() * TM2;
    if (jj < P.ct) {
      src[n++] = item_enc(kArrX2, xb);
    } else if (jj < P.ct + P.zq) {
      const int64_t o = xb + (1 + 2 * (int64_t)(jj - P.ct)) * TM2;
      src[n++] = item_enc(kArrX2, o);
      src[n++] = item_enc(kArrX2, o + TM2);
    } else {
      const int64_t o = xb + (1 + 4 * (int64_t)(g.G - 1) + 2 * (jj - P.ct - P.zq)) * TM2;
      src[n++] = item_enc(kArrX2, o);
      src[n++] = item_enc(kArrX2, o + TM2);
    }
  } else if (g.nr) {         // spikes W, V of block j, restricted to the kNR rows
    src[n++] = item_enc(kArrSpr, (int64_t)(Y0 + j) * TM2);
  } else {                   // spikes W, V of block j
    const int64_t o = (int64_t)(Y0 + j) * 2 * TM2;
    src[n++] = item_enc(kArrSp, o);
    src[n++] = item_enc(kArrSp, o + TM2);
  }
  return n;
}

constexpr int kMaxItems = 1024;   // items of one chunk solve (checked at sweep_create)

// items of one chunk solve: <= 3m + 2L local, 15 dense, 2(C-1) R blocks,
// <= 2G + 1 level-2 items, m spike blocks
__host__ __device__ inline int itab_len(int mmax) {
  return 4 * mmax + 2 * kMaxLevels + 2 * kMaxC + 2 * kMaxG + 24;
}

// blocks of one chunk's slab-solve stream
template <int TM>
__host__ __device__ inline int stream_blocks(const Chunks& g, int rank) {
  ItemPlan P;
  plan_items(g, rank, P);
  int nb = 0;
  uint32_t src[2];
  bool hx;
  for (int r = 0; r < P.pfx[P.NP + 2]; ++r) nb += item_sources<TM>(g, rank, P, r, src, &hx);
  return nb;
}

template <int TM>
__host__ __device__ constexpr int ring_g() { return TM == 16 ? HS_SWEEP_G16 : 2; }

// Words of one rank's solve plan: ItemPlan, ib[itab_len], ctab[itab_len], nchk.
__host__ __device__ inline int plan_words(int mmax) {
  return (int)(sizeof(ItemPlan) / 4) + 2 * itab_len(mmax) + 1;
}
// The solve kernel's item and chunk tables of one rank (built on the host
// once per sweep).  Chunks: runs of whole items of one phase, up to G blocks
// (one bulk copy each); a ring slot is released as soon as its items are
// consumed, so a chunk never waits for a later phase.
//   ib[r]   = chunk << 12 | offset in chunk << 3 | blocks << 1 | hasx
//   ctab[c] = first stream block << 8 | blocks
template <int TM>
__host__ __device__ inline void chunk_plan(const Chunks& g, int rank, int mmax, uint32_t* w) {
  constexpr int G = ring_g<TM>();
  ItemPlan& P = *(ItemPlan*)w;
  uint32_t* ib = w + sizeof(ItemPlan) / 4;
  uint32_t* ctab = ib + itab_len(mmax);
  plan_items(g, rank, P);
  int acc = 0, nc = -1, cfill = G, last_seg = -1;
  for_stream(P, [&](int r, int seg) {   // stream order (k_pack's)
    uint32_t src[2];
    bool hx;
    const int n = item_sources<TM>(g, rank, P, r, src, &hx);
    if (seg != last_seg || cfill + n > G) {
      ++nc;
      ctab[nc] = (uint32_t)acc << 8;
      cfill = 0;
      last_seg = seg;
    }
    ib[r] = (uint32_t)nc << 12 | (uint32_t)cfill << 3 | (uint32_t)n << 1 | (hx ? 1u : 0u);
    ctab[nc] += (uint32_t)n;
    cfill += n;
    acc += n;
  });
  ctab[itab_len(mmax)] = (uint32_t)(nc + 1);   // nchk
}

struct FactorArrays {
  const double2 *ef, *eb, *kr, *rk, *sp, *qd, *ebr, *spr, *x2, *cpl;
};

// Restricted updates (setup): for the kNR rows R of each slab, one block per
// face point holding [A0[R, :] | A1[R, :]] laid out for a 32-lane GEMV:
// element (k, q, r) at k*32 + q*8 + r, q = 2*matrix + column half,
// column = k + (q & 1) * tm/2.  ebr: (Dinv L, Dinv U); spr: (W, V).
template <int TM>
__global__ void __launch_bounds__(256) k_rows(Chunks g, const int* __restrict__ rows,
                                              const double2* __restrict__ eb,
                                              const double2* __restrict__ sp,
                                              double2* __restrict__ ebr, double2* __restrict__ spr) {
  constexpr int TM2 = TM * TM, H = TM / 2;
  const int y = blockIdx.x, slab = blockIdx.y, M = g.M;
  const int64_t b = ((int64_t)slab * M + y);
  for (int e = threadIdx.x; e < H * 32; e += blockDim.x) {
    const int k = e / 32, q = (e % 32) / 8, r = e % 8;
    const int row = rows[slab * kNR + r], col = k + (q & 1) * H, mat = q >> 1;
    ebr[b * TM2 + e] = eb[(b * 2 + mat) * TM2 + lm<TM>(row, col)];
    spr[b * TM2 + e] = sp[(b * 2 + mat) * TM2 + lm<TM>(row, col)];
  }
}

// Repack every slab's factors into per-chunk streams in item order (one CTA
// per slab x chunk), so the solve kernel fetches 16-KB runs with single bulk
// copies: stream[slab][k][nbs] blocks.
template <int TM>
__global__ void __launch_bounds__(256) k_pack(Chunks g, FactorArrays f, double2* __restrict__ stream,
                                              int nbs) {
  constexpr int TM2 = TM * TM;
  const int C = g.nch(), slab = blockIdx.x / C, k = blockIdx.x % C, M = g.M;
  __shared__ ItemPlan P;
  __shared__ int boff[kMaxItems];
  if (threadIdx.x == 0) {
    plan_items(g, k, P);
    int acc = 0;
    for_stream(P, [&](int r, int) {
      uint32_t src[2];
      bool hx;
      boff[r] = acc;
      acc += item_sources<TM>(g, k, P, r, src, &hx);
    });
  }
  __syncthreads();
  const double2* base[10] = {
      f.ef + (int64_t)slab * M * TM2,           f.eb + (int64_t)slab * M * 2 * TM2,
      f.kr + (int64_t)slab * C * g.kstride * 2 * TM2,
      f.rk + (int64_t)slab * C * (2 * (g.C - 1)) * 2 * TM2,
      f.sp + (int64_t)slab * M * 2 * TM2,       f.qd + (int64_t)slab * C * g.q * g.q * TM2,
      f.ebr ? f.ebr + (int64_t)slab * M * TM2 : nullptr,
      f.spr ? f.spr + (int64_t)slab * M * TM2 : nullptr,
      f.x2 ? f.x2 + (int64_t)slab * C * g.xstride() * TM2 : nullptr,
      f.cpl ? f.cpl + (int64_t)slab * M * TM2 : nullptr};
  double2* out = stream + ((int64_t)slab * C + k) * nbs * TM2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int r = warp; r < P.pfx[P.NP + 2]; r += 8) {
    uint32_t src[2];
    bool hx;
    const int n = item_sources<TM>(g, k, P, r, src, &hx);
    for (int b = 0; b < n; ++b) {
      const double2* s = base[src[b] >> 28] + (src[b] & kOffMask);
      double2* d = out + (int64_t)(boff[r] + b) * TM2;
      for (int e = lane; e < TM2; e += 32) d[e] = s[e];
    }
  }
}

// One item per half warp for tm = 16 (lane row x = lane % 16 of the half's
// item, all 16 columns), the whole warp for tm = 32: row x of A0 v0 + A1 v1.
template <int TM, int HW>
__device__ __forceinline__ double2 mvx(const double2* m0, const double2* v0, const double2* m1,
                                       const double2* v1, int lane) {
  if constexpr (HW == 1) {
    return mvs2<TM>(m0, v0, m1, v1, lane);
  } else {
    const int x = lane % 16;
    double2 a0 = czero(), a1 = czero(), a2 = czero(), a3 = czero();
    if (v0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {   // lm<16>(x, c) = (c % 8) * 32 + (c / 8) * 16 + x
        a0 = cfma(m0[k * 32 + x], v0[k], a0);
        a1 = cfma(m0[k * 32 + 16 + x], v0[k + 8], a1);
      }
    }
    if (v1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a2 = cfma(m1[k * 32 + x], v1[k], a2);
        a3 = cfma(m1[k * 32 + 16 + x], v1[k + 8], a3);
      }
    }
    return cadd(cadd(a0, a1), cadd(a2, a3));
  }
}


// Shared-memory ring of stream chunks: G blocks (16 KB) per bulk copy.
// Restricted update (k_rows layout): lanes 0..7 return row r = lane of
// A0[R, :] v0 + A1[R, :] v1 (a term with a null vector is skipped).
template <int TM>
__device__ __forceinline__ double2 mvr(const double2* blk, const double2* v0, const double2* v1,
                                       int lane) {
  if (HS_SWEEP_EXP & 1) return czero();
  constexpr int H = TM / 2;
  const int q = lane / 8;
  const double2* v = q < 2 ? v0 : v1;
  double2 a0 = czero(), a1 = czero();
  if (v) {
    v += (q & 1) * H;
#pragma unroll
    for (int k = 0; k < H; k += 2) {
      a0 = cfma(blk[k * 32 + lane], v[k], a0);
      a1 = cfma(blk[(k + 1) * 32 + lane], v[k + 1], a1);
    }
  }
  double2 acc = cadd(a0, a1);
  acc = cadd(acc, shfl_xor_c(acc, 8));
  return cadd(acc, shfl_xor_c(acc, 16));
}

// The same mat-vecs for NR right-hand sides at once: vectors of right-hand
// side r at v + r * vs; each matrix element is read from shared memory once
// per group of <= 4 right-hand sides (register budget) and every right-hand
// side's sums are accumulated in mvs2 / mvr's order, so a batched solve is
// bitwise the single one.
template <int TM, int NR>
__device__ __forceinline__ void mvs2n(const double2* m0, const double2* v0, const double2* m1,
                                      const double2* v1, int vs, int lane, double2 (&out)[NR]) {
  if constexpr (NR == 1) {
    out[0] = mvs2<TM>(m0, v0, m1, v1, lane);
  } else {
    constexpr int CPL = Geo<TM>::CPL;
    constexpr int GR = NR < 4 ? NR : 4;
    const int hh = lane / TM;
#pragma unroll
    for (int r0 = 0; r0 < NR; r0 += GR) {
      double2 a0[GR], a1[GR], a2[GR], a3[GR];
#pragma unroll
      for (int r = 0; r < GR; ++r) a0[r] = a1[r] = a2[r] = a3[r] = czero();
      if (v0) {
#pragma unroll
        for (int k = 0; k < CPL; k += 2) {
          const double2 ma = m0[k * 32 + lane], mb = m0[(k + 1) * 32 + lane];
#pragma unroll
          for (int r = 0; r < GR; ++r) {
            a0[r] = cfma(ma, v0[(r0 + r) * vs + CPL * hh + k], a0[r]);
            a1[r] = cfma(mb, v0[(r0 + r) * vs + CPL * hh + k + 1], a1[r]);
          }
        }
      }
      if (v1) {
#pragma unroll
        for (int k = 0; k < CPL; k += 2) {
          const double2 ma = m1[k * 32 + lane], mb = m1[(k + 1) * 32 + lane];
#pragma unroll
          for (int r = 0; r < GR; ++r) {
            a2[r] = cfma(ma, v1[(r0 + r) * vs + CPL * hh + k], a2[r]);
            a3[r] = cfma(mb, v1[(r0 + r) * vs + CPL * hh + k + 1], a3[r]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < GR; ++r) {
        double2 acc = cadd(cadd(a0[r], a1[r]), cadd(a2[r], a3[r]));
        if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
        out[r0 + r] = (HS_SWEEP_EXP & 1) ? czero() : acc;
      }
    }
  }
}

template <int TM, int NR>
__device__ __forceinline__ void mvrn(const double2* blk, const double2* v0, const double2* v1,
                                     int vs, int lane, double2 (&out)[NR]) {
  if constexpr (NR == 1) {
    out[0] = mvr<TM>(blk, v0, v1, lane);
  } else {
    constexpr int H = TM / 2;
    constexpr int GR = NR < 4 ? NR : 4;
    const int q = lane / 8;
    const double2* v = q < 2 ? v0 : v1;
#pragma unroll
    for (int r0 = 0; r0 < NR; r0 += GR) {
      double2 a0[GR], a1[GR];
#pragma unroll
      for (int r = 0; r < GR; ++r) a0[r] = a1[r] = czero();
      if (v) {
        const double2* vv = v + (q & 1) * H;
#pragma unroll
        for (int k = 0; k < H; k += 2) {
          const double2 ma = blk[k * 32 + lane], mb = blk[(k + 1) * 32 + lane];
#pragma unroll
          for (int r = 0; r < GR; ++r) {
            a0[r] = cfma(ma, vv[(r0 + r) * vs + k], a0[r]);
            a1[r] = cfma(mb, vv[(r0 + r) * vs + k + 1], a1[r]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < GR; ++r) {
        double2 acc = cadd(a0[r], a1[r]);
        acc = cadd(acc, shfl_xor_c(acc, 8));
        acc = cadd(acc, shfl_xor_c(acc, 16));
        out[r0 + r] = (HS_SWEEP_EXP & 1) ? czero() : acc;
      }
    }
  }
}


template <int TM, int HW, int NR>
__device__ __forceinline__ void mvxn(const double2* m0, const double2* v0, const double2* m1,
                                     const double2* v1, int vs, int lane, double2 (&out)[NR]) {
  if constexpr (NR == 1) out[0] = mvx<TM, HW>(m0, v0, m1, v1, lane);
  else mvs2n<TM, NR>(m0, v0, m1, v1, vs, lane, out);
}

template <int TM>
struct Ring {
  static constexpr int TM2 = TM * TM;
  static constexpr int G = ring_g<TM>();           // blocks per chunk copy (>= 2: whole items)
  static constexpr int CHUNK = G * TM2;            // double2 per chunk
  // F, Yv vectors + tau + halo + R partials + couplings + bookkeeping, then the ring
  // (nr right-hand sides: every vector array holds nr copies)
  // (C chunks per cluster; F, Yv; tau2; halo2; part + ab; t2v + pqv)
  static int fixed(int mmax, int C, int nr) {
    return nr * (2 * (mmax + 1) * TM * 16 + 4 * C * TM * 16 + 4 * TM * 16 +
                 (kCW - kNA + 2) * 2 * TM * 16 + (2 * kMaxG * TM + 4 * TM) * 16) +
           12 * mmax * 16 + 64 + (int)sizeof(ItemPlan) +
           kMaxTasks * 4 + itab_len(mmax) * 12 + 512 + 16;
  }
  static int nchunk(int mmax, int C, int nr) {
    const int avail = 225 * 1024 - fixed(mmax, C, nr);
    return std::max(2, std::min(32, avail / (CHUNK * 16 + 16)));   // one producer lane per slot
  }
  static int smem(int mmax, int C, int nr) {
    return fixed(mmax, C, nr) + nchunk(mmax, C, nr) * (CHUNK * 16 + 16);
  }
};

template <int TM, int NR>
__global__ void __launch_bounds__(kWarps * 32, 1) k_part_solve(SolveArgs a) {
  constexpr int TM2 = Geo<TM>::TM2;
  constexpr int CHUNK = Ring<TM>::CHUNK;
  constexpr int YPW = 32 / TM;   // face points per warp pass in row-wise loops
  constexpr int N2 = 2 * TM;     // interface unknowns per chunk (alpha, beta)
  cg::cluster_group cl = cg::this_cluster();
  const Chunks& g = a.g;
  const int C = g.C, M = g.M, B = C - 1, G = g.G, NCH = g.nch();
  const int rank = (int)cl.block_rank();
  const int front = blockIdx.x / (C * G);
  const int seg = (blockIdx.x / C) % G;   // face segment of this cluster (two-level partition)
  const int K = seg * C + rank;           // global chunk index
  const int Y0 = g.y0(K), Y1 = g.y0(K + 1);
  // the last chunk of a segment with a right neighbour segment keeps its own
  // right tip g[m-1] for c_s (pushed to itself, tau slot 2B)
  const bool lastpush = G > 1 && rank == B && seg < G - 1;
  const int m = Y1 - Y0;
  const int mmax = g.mmax;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int x = lane % TM, hh = lane / TM;
  constexpr int HW = (TM == 16 && HS_SWEEP_HALF && NR == 1) ? 2 : 1;   // items per warp pass
  const int sub = HW == 2 ? hh : 0;      // this lane's item within the pass
  const bool wr = HW == 2 || hh == 0;    // lane owns the result row it computed
  const int NC = a.nchunk;
  extern __shared__ __align__(128) double2 sm[];
  // vector arrays hold NR right-hand sides (strides FS, TS, HS, PS, N2, T2S)
  const int FS = (mmax + 1) * TM;
  const int TS = 2 * C * TM;
  constexpr int HS = 2 * TM, PS = (kCW - kNA + 1) * N2, T2S = 2 * kMaxG * TM;
  double2* F = sm;                                  // [NR][mmax+1][TM] rhs / reduced rhs
  double2* Yv = F + NR * FS;                        // [NR][mmax+1][TM] Dinv f, then x
  double2* tau2 = Yv + NR * FS;                     // [2][NR][2 C][TM] interface rhs (by task parity)
  double2* halo2 = tau2 + 2 * NR * TS;              // [2][NR][2][TM] neighbours' edge blocks of x
  double2* part = halo2 + 2 * NR * HS;              // [NR][group-B warps + 1][2TM] R / dense-top partial sums
  double2* ab = part + NR * PS;                     // [NR][2TM] alpha_{k-1}, beta_k
  double2* stc = ab + NR * N2;                      // [2 tin][2 rows][3 offsets][mmax] couplings
  double2* t2v = stc + 12 * mmax;                   // [NR][2(G-1)][TM] level-2 right-hand side
  double2* pqv = t2v + NR * T2S;                    // [2][NR][2TM] (P_s, Q_s) by task parity
  uint64_t* xbar = (uint64_t*)(pqv + 2 * NR * N2);  // [6] tips (2), halo (2), (P_s, Q_s) (2)
  uint64_t* cbar = xbar + 6;                        // [NC] chunk arrival
  volatile int* cseq = (volatile int*)(cbar + NC);  // [NC] chunk issued into a slot
  int* ccnt = (int*)(cseq + NC);                    // [NC] blocks of the slot's chunk consumed
  uint32_t* plan = (uint32_t*)(ccnt + NC);          // this rank's plan (chunk_plan layout)
  ItemPlan* Pp = (ItemPlan*)plan;
  uint32_t* ib = plan + sizeof(ItemPlan) / 4;       // [ITEMS] chunk | offset in chunk | nblk | hasx
  uint32_t* ctab = ib + itab_len(mmax);             // [<= ITEMS] chunk: first block | blocks
  int* nchk = (int*)(ctab + itab_len(mmax));        // chunks per slab solve
  int* slabs = nchk + 1;                            // [fcount]
  uint32_t* cmq = (uint32_t*)(slabs + kMaxTasks);   // [chunks] c % NC | (c / NC) << 16
  // (offset from sm keeps the shared-space provenance: LDS, not generic loads)
  double2* ring = sm + ((((char*)(cmq + itab_len(mmax)) - (char*)sm) + 127) & ~(ptrdiff_t)127) / 16;
  const ItemPlan& P = *Pp;

  const int ffirst = a.ffirst[front];
  const int fcount = a.fcount[front];
  {
    const int pw = plan_words(mmax);
    const uint32_t* src = a.plan + (int64_t)K * pw;
    for (int i = threadIdx.x; i < pw; i += blockDim.x) plan[i] = __ldg(src + i);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NC; ++i) {
      mbar_init(&cbar[i], 1);
      cseq[i] = -1;
      ccnt[i] = 0;
    }
    for (int i = 0; i < 6; ++i) mbar_init(&xbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < fcount; i += blockDim.x) slabs[i] = a.tasks[ffirst + i].slab;
  cl.sync();   // every CTA's barriers initialised before any remote arrival
  const int NP = P.NP, L = P.L, S = P.S, qk = P.qk, QP = P.QP;
  const int ITEMS = P.pfx[NP + 2];
  const int CPT = *nchk;   // chunk copies per slab solve
  for (int c = threadIdx.x; c < CPT; c += blockDim.x) cmq[c] = (uint32_t)(c % NC) | (uint32_t)(c / NC) << 16;
  __syncthreads();
  // ring position of the current task's chunk 0 (set per task: no divisions per item)
  int task_q = 0, task_r = 0;
  bool trace_task = false;   // HS_SWEEP_TRACE: per-item stamps of task 1

  __shared__ int rr[kNR];   // the current task's restricted-update rows
  // optional instrumentation: task 1 timestamps kept in shared memory, dumped at exit
  __shared__ unsigned long long tsm[128];
  auto stamp = [&](int ti, int k) {   // k >= 40: group B's first thread stamps
    if (a.dbg && threadIdx.x == (k >= 40 && k < 48 ? kNA * 32 : 0) && ti == 1 && k < 64) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tsm[k] = tt;
    }
  };
  if (a.dbg && threadIdx.x == 0)
    for (int k = 0; k < 128; ++k) tsm[k] = 0;
  // per-item timestamps of task 1 (cluster 0): chunk issue, item data ready, item consumed
  auto istamp = [&](int r, int k) {
    if (a.dbg && blockIdx.x < 16 && r >= 0 && r < 256) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      a.dbg[blockIdx.x * 1024 + 256 + 3 * r + k] = tt;
    }
  };
  auto csync = [&]() {   // consumer warps only (the producer never joins)
    asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
  };

  const int total_chunks = fcount * CPT;
  // issue chunk cs into its ring slot (the slot's previous chunk is consumed)
  auto fill = [&](int cs) {
    const int sl = cs % NC;
    const int ti = cs / CPT, c = cs - ti * CPT;
    const uint32_t ce = ctab[c];
    const int nbk = (int)(ce & 0xff);
    *(volatile int*)&ccnt[sl] = 0;   // ordered before cseq (same thread, volatile)
    // (timing experiment bit 16: every task streams slab 0's data -> L2-resident)
    const double2* sbase = a.stream + ((int64_t)((HS_SWEEP_EXP & 16) ? 0 : slabs[ti]) * NCH + K) *
                                          a.nbs * TM2;
    mbar_expect_tx(&cbar[sl], (HS_SWEEP_EXP & 2) ? 0u : (uint32_t)nbk * TM2 * 16);
    if (!(HS_SWEEP_EXP & 2))
      bulk_g2s(ring + (int64_t)sl * CHUNK, sbase + (int64_t)(ce >> 8) * TM2,
               (uint32_t)nbk * TM2 * 16, &cbar[sl]);
    cseq[sl] = cs;
    if (ti == 1) istamp(c, 0);
  };
  if (warp == kCW) {
    // ---- TMA producer warp: lane l owns ring slot l (l < NC) and streams
    // chunks cs = l, l + NC, l + 2 NC, ... of the launch's slab solves, each as
    // soon as the slot's previous chunk has been fully consumed.  Lanes run
    // independently (no batch lockstep).
    if (lane < NC && !HS_SWEEP_DIRECT) {
      const int sl = lane;
      int prev_n = -1;
      for (int cs = sl; cs < total_chunks; cs += NC) {
        if (prev_n >= 0 && !(HS_SWEEP_EXP & 8)) {   // the slot's previous chunk fully consumed
          while (*(volatile int*)&ccnt[sl] != prev_n) {
          }
        }
        prev_n = (int)(ctab[cs % CPT] & 0xff);
        fill(cs);
      }
    }
    __syncwarp();
    cl.sync();   // matches the consumers' exit barrier
    return;
  }

  // ---- consumers: item r of task ti -> its (one or two) blocks in the ring
  auto wait_chunk = [&](int cs, int sl, int q) {
    if (HS_SWEEP_EXP & 8) {   // experiment: no slot reuse hazard (no data), only issue order
      while ((int)(cseq[sl] - cs) < 0) {
      }
      return;
    }
    while (cseq[sl] != cs) {
    }
    mbar_wait(&cbar[sl], (uint32_t)(q & 1));
  };
  struct Item { const double2* m0; const double2* m1; int sl, n, r; };
  // slot and phase parity of chunk c of the current task
  auto slot_of = [&](int c, int& sl, int& q) {
    const uint32_t t = cmq[c];
    sl = task_r + (int)(t & 0xffff);
    q = task_q + (int)(t >> 16);
    if (sl >= NC) { sl -= NC; ++q; }
  };
  auto acquire = [&](int ti, int r) -> Item {
    const uint32_t e = ib[r];
    const int cs = ti * CPT + (int)(e >> 12);
    const bool hx = e & 1;
    const int n = (int)((e >> 1) & 3);
    if (HS_SWEEP_DIRECT) {
      const double2* p0 = a.stream + (((int64_t)slabs[ti] * NCH + K) * a.nbs +
                                      (ctab[e >> 12] >> 8) + ((e >> 3) & 0x1ff)) * TM2;
      return hx ? Item{p0, p0 + TM2, 0, n, r} : Item{nullptr, p0, 0, n, r};
    }
    int sl, q;
    slot_of((int)(e >> 12), sl, q);
    wait_chunk(cs, sl, q);
    if (ti == 1 && lane % (32 / HW) == 0) istamp(r, 1);
    const double2* p0 = ring + (int64_t)sl * CHUNK + (int)((e >> 3) & 0x1ff) * TM2;
    return hx ? Item{p0, p0 + TM2, sl, n, r} : Item{nullptr, p0, sl, n, r};
  };
  // The warp's reads of the blocks have returned (their values are consumed
  // before the __syncwarp), so the producer's async-proxy refill cannot race.
  auto release = [&](const Item& it, bool has) {
    __syncwarp();
    if (!HS_SWEEP_DIRECT && has && lane % (32 / HW) == 0) {
      atomicAdd(&ccnt[it.sl], it.n);
      if (trace_task) istamp(it.r, 2);
    }
  };
  // Right-hand-side inputs of task tn, copied asynchronously while the
  // previous task finishes: restriction rows straight into F (free after the
  // previous task's dense top) and the transmission couplings into stc.
  auto prefetch_rhs = [&](const SweepTask& t, int w0, int nw) {   // warps [w0, w0 + nw)
    for (int yl = (warp - w0) * YPW + hh; yl < m; yl += nw * YPW) {
      const int y = Y0 + yl;
      const int gr = x + t.lo - 1;
      const bool ok = x < t.T && gr >= t.a && gr < t.b;
#pragma unroll
      for (int rh = 0; rh < NR; ++rh)
        cp_async16(&F[rh * FS + yl * TM + x],
                   a.src + (ok ? rh * a.vs_src + (int64_t)gr * M + y : 0), ok);
#pragma unroll
      for (int tn_i = 0; tn_i < 2; ++tn_i) {
        const int tin = tn_i ? t.tin3 : t.tin1, row = tn_i ? t.row3 : t.row1;
        if (tin < 0 || (x != row && x != row + 1)) continue;
        const int which = x - row, p = row + t.lo;
        const int o0 = which == 0 ? 1 : -1, crow = which == 0 ? p - 1 : p;
#pragma unroll
        for (int o = -1; o <= 1; ++o) {
          const int sl = a.cslot[o0 + 1][o + 1];
          const bool okc = sl >= 0 && y + o >= 0 && y + o < M;
          cp_async16(&stc[((tn_i * 2 + which) * 3 + o + 1) * mmax + yl],
                     a.coarse + (okc ? (int64_t)sl * a.ncoarse + (int64_t)crow * M + y : 0), okc);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // Transmission into slab row `which` of an incoming trace: from the previous
  // task of this front without a trip through global memory (its x is still in
  // Yv, the neighbours' edge blocks arrive in halo by st.async), else from the
  // trace buffer written by an earlier launch.
  auto transx = [&](int rh, int tn_i, bool local, const double2* halo, int buf, int prow, int sign,
                    int which, int yl) -> double2 {
    const int y = Y0 + yl;
    const int xr = prow + (which == 0 ? 1 : 0);   // trace row 1 feeds which 0, row 0 which 1
    const double2* Bt = a.trace + rh * a.ts + (int64_t)buf * 2 * M + (which == 0 ? M : 0);   // L2 reads (__ldcg)
    double2 acc = czero();
#pragma unroll
    for (int o = -1; o <= 1; ++o) {
      if (y + o < 0 || y + o >= M) continue;
      const int q = yl + o;
      const double2 bv = !local ? __ldcg(Bt + y + o)
                         : q < 0 ? halo[rh * HS + xr] : q >= m ? halo[rh * HS + TM + xr]
                                                               : Yv[rh * FS + q * TM + xr];
      acc = cfma(stc[((tn_i * 2 + which) * 3 + o + 1) * mmax + yl], bv, acc);
    }
    return cscale(which == 0 ? (double)sign : (double)-sign, acc);
  };
  const uint32_t halo_bytes = (rank > 0 ? TM * 16 : 0) + (rank < B ? TM * 16 : 0);
  // tips g[first], g[last] of this chunk go to every CTA's tau:
  // tau block b = (g_b[last], g_{b+1}[first]) -> tm-slots 2b, 2b+1
  auto push_tip = [&](double2* tau, int par, int slot, const double2* v, int w, int nw) {
#pragma unroll
    for (int rh = 0; rh < NR; ++rh) {
      const double2 val = v[rh * FS + lane];   // lanes < TM; warp w of nw pushing warps
      for (int d = w; d < C; d += nw)
        st_async_c(map_rank(&tau[rh * TS + slot + lane], d), val, map_rank(&xbar[par], d));
    }
  };

  SweepTask prev{}, t = fcount > 0 ? a.tasks[ffirst] : SweepTask{};
  if (fcount > 0) prefetch_rhs(t, 0, kCW);
  SweepTask tn = t;
  for (int ti = 0; ti < fcount; ++ti) {
    if (ti > 0) t = tn;   // loaded during the previous task
    trace_task = a.dbg != nullptr && ti == 1;
    task_q = ti * CPT / NC;
    task_r = ti * CPT - task_q * NC;
    if (ti + 1 < fcount) tn = a.tasks[ffirst + ti + 1];   // in flight early
    const int par = ti & 1;
    double2* tau = tau2 + par * NR * TS;
    const double2* halo = halo2 + par * NR * HS;
    // previous task's traces consumed here straight from shared memory
    const bool loc1 = ti > 0 && t.tin1 >= 0 && prev.out2 == t.tin1;
    const bool loc3 = ti > 0 && t.tin3 >= 0 && prev.out4 == t.tin3;
    if (threadIdx.x == 0) {
      if (ti > 0) mbar_expect_tx(&xbar[2 + par], NR * halo_bytes);
      if (B > 0) mbar_expect_tx(&xbar[par], NR * (2 * B * TM * 16 + (lastpush ? TM * 16 : 0)));
      if (G > 1) mbar_expect_tx(&xbar[4 + par], NR * N2 * 16);
    }
    stamp(ti, 0);
    if (HS_SWEEP_L2NEXT && ti + 1 < fcount) {   // next slab's stream into L2 (LSU path, not TMA)
      const char* nb = (const char*)(a.stream + ((int64_t)slabs[ti + 1] * NCH + K) * a.nbs * TM2);
      const int64_t bytes = (int64_t)((ctab[CPT - 1] >> 8) + (ctab[CPT - 1] & 0xff)) * TM2 * 16;
      for (int64_t o = (int64_t)threadIdx.x * 128; o < bytes; o += kCW * 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nb + o));
    }
    if (g.nr && threadIdx.x < kNR) rr[threadIdx.x] = a.rows[t.slab * kNR + threadIdx.x];
    // ---- right-hand side of the owned blocks: restriction rows (already in
    // F) plus the transmission terms of the incoming traces
    asm volatile("cp.async.wait_all;" ::: "memory");
    // (always: the neighbours' previous task is then complete, which also
    // orders the double-buffered tau/halo reuse across the cluster)
    if (ti > 0) mbar_wait(&xbar[2 + par], (uint32_t)((ti - 1) >> 1) & 1);
    csync();
    for (int yl = warp * YPW + hh; yl < m; yl += kCW * YPW) {
      const bool r1 = t.tin1 >= 0 && (x == t.row1 || x == t.row1 + 1);
      const bool r3 = t.tin3 >= 0 && (x == t.row3 || x == t.row3 + 1);
      if (!r1 && !r3) continue;
#pragma unroll
      for (int rh = 0; rh < NR; ++rh) {
        double2 v = F[rh * FS + yl * TM + x];
        if (r1) v = cadd(v, transx(rh, 0, loc1, halo, t.tin1, prev.orow2, 1, x - t.row1, yl));
        if (r3) v = cadd(v, transx(rh, 1, loc3, halo, t.tin3, prev.orow4, -1, x - t.row3, yl));
        F[rh * FS + yl * TM + x] = v;
      }
    }
    csync();
    stamp(ti, 1);
    // ---- chunk-local solve: L cyclic-reduction levels, the dense top, back substitution
    // item j of phase p (warp-uniform `has`)
    // phase constants in registers (P lives in shared memory and the ring's
    // waits are memory clobbers: per-item reloads would be on the critical path)
    struct Ph { int p, l, s, pf0, cnt, ne, first, step; };
    auto phase = [&](int p) {
      Ph h;
      h.p = p;
      h.l = plan_level(P, p);
      h.s = 1 << h.l;
      h.pf0 = P.pfx[p];
      h.cnt = P.pfx[p + 1] - h.pf0;
      h.ne = h.cnt / 2;
      h.first = plan_first(P, p);
      h.step = plan_step(P, p);
      return h;
    };
    auto do_item = [&](const Ph& h, int j, bool has) {
      const int p = h.p, l = h.l, s = h.s;
      const int yl = !has || p == L ? 0
                     : p > L        ? h.first + j * h.step
                                    : (j < h.ne ? 2 * j + 1 : 2 * (j - h.ne)) << p;
      const int r = h.pf0 + j;
      // level-0 kept items with sparse couplings: one block of 6 TM coupling values
      const bool sparse0 = g.cpl0 && p == 0 && !(yl & 1);
      const Item it = has ? acquire(ti, r) : Item{nullptr, nullptr};
      const double2* m0 = it.m0;
      const double2* m1 = it.m1;
      if (has) {
        double2 acc[NR];
        if (p == L) {            // partial x_r += Q[r][c0] f_c0 + Q[r][c0+1] f_c0+1
          const int c0 = 2 * (j % QP);
          const bool two = c0 + 1 < qk;
          mvxn<TM, HW, NR>(m0, F + c0 * S * TM, two ? m1 : nullptr,
                           two ? F + (c0 + 1) * S * TM : nullptr, FS, lane, acc);
          if (wr) {
#pragma unroll
            for (int rh = 0; rh < NR; ++rh) part[rh * PS + j * TM + x] = acc[rh];
          }
        } else if (p < L) {
          if ((yl >> l) & 1) {   // eliminated at this level: y = Dinv f
            mvxn<TM, HW, NR>(m0, F + yl * TM, nullptr, nullptr, FS, lane, acc);
            if (wr) {
#pragma unroll
              for (int rh = 0; rh < NR; ++rh) Yv[rh * FS + yl * TM + x] = acc[rh];
            }
          } else if (sparse0) {  // kept, level 0: f -= L Yv[y-1] + U Yv[y+1]
            // (alpha f_{y-1} = L Dinv_{y-1} f_{y-1} = L Yv[y-1], Yv from this
            // phase's first half; L, U the slab stencil's thin-axis couplings)
            const double2* cp = m1;   // (hasx = false: the item's block)
#pragma unroll
            for (int rh = 0; rh < NR; ++rh) {
            double2 acc0 = czero();
#pragma unroll
            for (int sd = 0; sd < 2; ++sd) {
              const int q = yl + (sd ? 1 : -1);
              if (q < 0 || q >= m) continue;
#pragma unroll
              for (int o0 = -1; o0 <= 1; ++o0) {
                const int xx = x + o0;
                if (xx < 0 || xx >= TM) continue;
                acc0 = cfma(cp[(sd * 3 + o0 + 1) * TM + x], Yv[rh * FS + q * TM + xx], acc0);
              }
            }
            if (wr) F[rh * FS + yl * TM + x] = csub(F[rh * FS + yl * TM + x], acc0);
            }
          } else {               // kept: f -= alpha f_{y-s} + gamma f_{y+s}
            const bool hl = yl - s >= 0, hr = yl + s < m;
            mvxn<TM, HW, NR>(hl ? m0 : nullptr, hl ? F + (yl - s) * TM : nullptr,
                             hr ? m1 : nullptr, hr ? F + (yl + s) * TM : nullptr, FS, lane, acc);
            if (wr) {
#pragma unroll
              for (int rh = 0; rh < NR; ++rh)
                F[rh * FS + yl * TM + x] = csub(F[rh * FS + yl * TM + x], acc[rh]);
            }
          }
        } else if (g.nr && l == 0 && yl != m - 1) {   // level 0: only the rows read later
          mvrn<TM, NR>(m0, Yv + (yl - 1) * TM, Yv + (yl + 1) * TM, FS, lane, acc);
          if (lane < kNR) {
#pragma unroll
            for (int rh = 0; rh < NR; ++rh)
              Yv[rh * FS + yl * TM + rr[lane]] = csub(Yv[rh * FS + yl * TM + rr[lane]], acc[rh]);
          }
        } else {                 // x_y = Dinv f - (Dinv L) x_{y-s} - (Dinv U) x_{y+s}
          const bool hl = yl - s >= 0, hr = yl + s < m;
          mvxn<TM, HW, NR>(hl ? m0 : nullptr, hl ? Yv + (yl - s) * TM : nullptr,
                           hr ? m1 : nullptr, hr ? Yv + (yl + s) * TM : nullptr, FS, lane, acc);
          if (wr) {
#pragma unroll
            for (int rh = 0; rh < NR; ++rh)
              Yv[rh * FS + yl * TM + x] = csub(Yv[rh * FS + yl * TM + x], acc[rh]);
          }
        }
      }
      release(it, has);
    };
    // phase p over warps [w0, w0 + nw)
    auto run_phase = [&](int p, int w0, int nw) {
      const Ph h = phase(p);
      for (int jp = (warp - w0) * HW; jp < h.cnt; jp += nw * HW) do_item(h, jp + sub, jp + sub < h.cnt);
    };
    for (int p = 0; p <= L; ++p) {   // forward levels and the dense top: all warps
      if (p == 0 && g.cpl0) {        // level 0: eliminated points, then the kept points' updates
        const Ph h = phase(0);
        for (int jp = warp * HW; jp < h.ne; jp += kCW * HW) do_item(h, jp + sub, jp + sub < h.ne);
        csync();
        for (int jp = h.ne + warp * HW; jp < h.cnt; jp += kCW * HW)
          do_item(h, jp + sub, jp + sub < h.cnt);
      } else {
        run_phase(p, 0, kCW);
      }
      csync();
      stamp(ti, 2 + p);
    }
    {   // x at the level-L points = sum of the column-pair partials
      for (int t = threadIdx.x; t < NR * qk * TM; t += kCW * 32) {
        const int rh = NR == 1 ? 0 : t / (qk * TM), t1 = t - rh * qk * TM;
        const int r = t1 / TM, xx = t1 % TM;
        double2 acc = czero();
        for (int cp = 0; cp < QP; ++cp) acc = cadd(acc, part[rh * PS + (r * QP + cp) * TM + xx]);
        Yv[rh * FS + r * S * TM + xx] = acc;
      }
      csync();
    }
    if (B == 0) {
      if (ti + 1 < fcount) prefetch_rhs(tn, 0, kCW);   // F is free from here on
      for (int p = L + 1; p < NP; ++p) {
        run_phase(p, 0, kCW);
        csync();
      }
    } else if (warp < kNA) {
      // ---- group A: back substitution (its own named barrier)
      for (int p = L + 1; p < NP; ++p) {
        run_phase(p, 0, kNA);
        asm volatile("bar.sync 2, %0;" ::"r"(kNA * 32) : "memory");
        if (p == P.plast && rank < B && lane < TM)
          push_tip(tau, par, 2 * rank * TM, Yv + (m - 1) * TM, warp, kNA);
        if (p == P.plast && lastpush && warp == 0 && lane < TM) {   // own g[m-1] for c_s
#pragma unroll
          for (int rh = 0; rh < NR; ++rh)
            st_async_c(map_rank(&tau[rh * TS + 2 * B * TM + lane], rank),
                       Yv[rh * FS + (m - 1) * TM + lane], map_rank(&xbar[par], rank));
        }
      }
      stamp(ti, 48);
    } else {
      // ---- group B: tips out (as soon as final), the next task's rhs inputs
      // (F is free from here on), then alpha_{k-1}, beta_k = (rows of R) tau
      if (lane < TM) {
        if (rank > 0) push_tip(tau, par, (2 * (rank - 1) + 1) * TM, Yv, warp - kNA, kCW - kNA);
        if (P.plast == L && rank < B)
          push_tip(tau, par, 2 * rank * TM, Yv + (m - 1) * TM, warp - kNA, kCW - kNA);
        if (P.plast == L && lastpush && warp == kNA) {
#pragma unroll
          for (int rh = 0; rh < NR; ++rh)
            st_async_c(map_rank(&tau[rh * TS + 2 * B * TM + lane], rank),
                       Yv[rh * FS + (m - 1) * TM + lane], map_rank(&xbar[par], rank));
        }
      }
      if (ti + 1 < fcount) prefetch_rhs(tn, kNA, kCW - kNA);
      mbar_wait(&xbar[par], (uint32_t)(ti >> 1) & 1);
      stamp(ti, 40);
      // column-block GEMV over group B: out (2tm) = sum_j blocks_j vec_j, or
      // out -= it (subtract); items rfirst.. of 2tm x tm column blocks (row index
      // fastest over two ring blocks), rows r0 = lane (tm 32) or x (tm 16)
      // and r0 + 32 / r0 + 16
      // (right-hand side rh: vec + rh * vstr, out + rh * ostr)
      auto cgemv = [&](int rfirst, int nq, const double2* vec, int vstr, double2* out, int ostr,
                       bool subtract) {
        double2 acc0[NR], acc1[NR];
#pragma unroll
        for (int rh = 0; rh < NR; ++rh) acc0[rh] = acc1[rh] = czero();
        const int r0 = HW == 1 ? lane : x, r1 = r0 + (HW == 1 ? 32 : 16);   // r1 unused: tm 16, HW 1
        for (int jp = (warp - kNA) * HW; jp < nq; jp += (kCW - kNA) * HW) {
          const int j = jp + sub;
          const bool has = j < nq;
          Item it{};
          if (has) {
            it = acquire(ti, rfirst + j);
            const double2* tq = vec + j * TM;
#pragma unroll 4
            for (int c = 0; c < TM / 2; ++c) {
              const double2 ma = it.m0[c * N2 + r0];
              const double2 mb = (HW == 2 || TM == 32) ? it.m0[c * N2 + r1] : czero();
#pragma unroll
              for (int rh = 0; rh < NR; ++rh) {
                const double2 tv = tq[rh * vstr + c];
                acc0[rh] = cfma(ma, tv, acc0[rh]);
                if (HW == 2 || TM == 32) acc1[rh] = cfma(mb, tv, acc1[rh]);
              }
            }
#pragma unroll 4
            for (int c = 0; c < TM / 2; ++c) {
              const double2 ma = it.m1[c * N2 + r0];
              const double2 mb = (HW == 2 || TM == 32) ? it.m1[c * N2 + r1] : czero();
#pragma unroll
              for (int rh = 0; rh < NR; ++rh) {
                const double2 tv = tq[rh * vstr + TM / 2 + c];
                acc0[rh] = cfma(ma, tv, acc0[rh]);
                if (HW == 2 || TM == 32) acc1[rh] = cfma(mb, tv, acc1[rh]);
              }
            }
          }
          release(it, has);
        }
        if (HW == 2) {   // both halves' items hold rows x and x + 16
          acc0[0] = cadd(acc0[0], shfl_xor_c(acc0[0], 16));
          acc1[0] = cadd(acc1[0], shfl_xor_c(acc1[0], 16));
        }
        if (lane < 32 / HW) {
#pragma unroll
          for (int rh = 0; rh < NR; ++rh) {
            part[rh * PS + (warp - kNA) * N2 + r0] = acc0[rh];
            if (HW == 2 || TM == 32) part[rh * PS + (warp - kNA) * N2 + r1] = acc1[rh];
          }
        }
        asm volatile("bar.sync 3, %0;" ::"r"((kCW - kNA) * 32) : "memory");
        static_assert((kCW - kNA) * 32 >= N2, "one reduction thread per interface unknown");
        for (int tt = threadIdx.x - kNA * 32; tt < NR * N2; tt += NR == 1 ? 1 << 20 : (kCW - kNA) * 32) {
          const int rh = tt / N2, t = tt % N2;
          double2 sacc = czero();
          for (int w = 0; w < kCW - kNA; ++w) sacc = cadd(sacc, part[rh * PS + w * N2 + t]);
          out[rh * ostr + t] = subtract ? csub(out[rh * ostr + t], sacc) : sacc;
        }
        asm volatile("bar.sync 3, %0;" ::"r"((kCW - kNA) * 32) : "memory");
      };
      // alpha_{k-1}, beta_k = (rows of R) tau
      cgemv(P.pfx[NP], 2 * B, tau, TS, ab, N2, false);
      stamp(ti, 44);
      if (G > 1) {
        // ---- second level (two-level partition, k_level2): post c_s / d_s,
        // the segment's first CTA solves for (P_s, Q_s) once every segment
        // has posted and hands them to the cluster, every CTA corrects
        // (alpha, beta) -= Pk P_s + Qk Q_s
        const int r_l2 = P.pfx[NP] + 2 * B;
        unsigned* fl = a.xflag + (size_t)front * 2 * kMaxG;
        double2* xb = a.xbuf + ((size_t)front * 2 + par) * kMaxG * 2 * TM;   // + rh * a.xs
        const unsigned want = a.xbase[front] + (unsigned)ti + 1u;
        const int wb = warp - kNA;
        if (P.ct && wb == 0) {
          const Item it = acquire(ti, r_l2);
          const bool isc = rank == B;   // c_s (last chunk) or d_s (first chunk)
          double2 acc[NR];
          mvxn<TM, HW, NR>(it.m0, isc ? ab : ab + TM, nullptr, nullptr, N2, lane, acc);
          release(it, true);
          if (lane < TM) {
#pragma unroll
            for (int rh = 0; rh < NR; ++rh) {
              const double2 gv = isc ? tau[rh * TS + 2 * B * TM + lane]
                                     : Yv[rh * FS + lane];   // g[last] / g[first]
              __stcg(&xb[rh * a.xs + (seg * 2 + (isc ? 0 : 1)) * TM + lane], csub(gv, acc[rh]));
            }
          }
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(&fl[(isc ? 0 : 1) * kMaxG + seg], 1u);
          stamp(ti, 45);
        }
        if (rank == 0) {
          const int nz = 2 * (G - 1);
          if (wb == 0 && lane < nz) {   // c_0 .. c_{G-2} (lanes < G-1), d_1 .. d_{G-1}
            const int isd = lane >= G - 1;
            const unsigned* f = fl + isd * kMaxG + (isd ? lane - (G - 1) + 1 : lane);
            while ((int)(ld_acquire_gpu(f) - want) < 0) {
            }
          }
          asm volatile("bar.sync 3, %0;" ::"r"((kCW - kNA) * 32) : "memory");
          // level-2 right-hand side in k_reduced order: block 2b = c_b, 2b + 1 = d_{b+1}
          for (int ii = threadIdx.x - kNA * 32; ii < NR * nz * TM; ii += (kCW - kNA) * 32) {
            const int rh = NR == 1 ? 0 : ii / (nz * TM), i = ii - rh * nz * TM;
            const int blk = i / TM, e = i % TM, b2 = blk / 2;
            const int sg = (blk & 1) ? b2 + 1 : b2;
            t2v[rh * T2S + i] = __ldcg(&xb[rh * a.xs + (sg * 2 + (blk & 1)) * TM + e]);
          }
          asm volatile("bar.sync 3, %0;" ::"r"((kCW - kNA) * 32) : "memory");
          double2* pql = part + PS - N2;   // (the slot after group B's partials)
          stamp(ti, 46);
          cgemv(r_l2 + P.ct, nz, t2v, T2S, pql, PS, false);
          if (wb == 0) {   // (P_s, Q_s) to every CTA of the cluster
            for (int ee = lane; ee < NR * N2; ee += 32) {
              const int rh = ee / N2, e = ee % N2;
              const double2 v = pql[rh * PS + e];
              for (int d = 0; d < C; ++d)
                st_async_c(map_rank(&pqv[(par * NR + rh) * N2 + e], d), v,
                           map_rank(&xbar[4 + par], d));
            }
          }
        }
        mbar_wait_cluster(&xbar[4 + par], (uint32_t)(ti >> 1) & 1);
        stamp(ti, 47);
        const double2* pqs = pqv + par * NR * N2;
        cgemv(r_l2 + P.ct + P.zq, 2, pqs, N2, ab, N2, true);
        for (int ee = threadIdx.x - kNA * 32; ee < NR * TM; ee += NR == 1 ? 1 << 20 : (kCW - kNA) * 32) {
          const int rh = ee / TM, e = ee % TM;
          const int nb = (((ti + 1) & 1) * NR + rh) * HS;   // next task's halo: edge values across segments
          if (rank == 0 && seg > 0) {
            ab[rh * N2 + e] = pqs[rh * N2 + e];
            halo2[nb + e] = pqs[rh * N2 + e];
          }
          if (rank == B && seg < G - 1) {
            ab[rh * N2 + TM + e] = pqs[rh * N2 + TM + e];
            halo2[nb + TM + e] = pqs[rh * N2 + TM + e];
          }
        }
      }
      stamp(ti, 41);
    }
    if (B > 0) {
      csync();   // back substitution and alpha, beta both done
      // ---- x_y = g_y - W_y alpha_{k-1} - V_y beta_k
      for (int jp = warp * HW; jp < m; jp += kCW * HW) {
        const int j = jp + sub;
        const bool has = j < m;
        const int r = P.pfx[NP + 1] + j;
        Item it{};
        if (has) {
          it = acquire(ti, r);   // W_j, V_j
          double2 acc[NR];
          if (g.nr) {                       // only the rows read later
            mvrn<TM, NR>(it.m0, rank > 0 || seg > 0 ? ab : nullptr,
                         rank < B || seg < G - 1 ? ab + TM : nullptr, N2, lane, acc);
            if (lane < kNR) {
#pragma unroll
              for (int rh = 0; rh < NR; ++rh)
                Yv[rh * FS + j * TM + rr[lane]] = csub(Yv[rh * FS + j * TM + rr[lane]], acc[rh]);
            }
          } else {
            const bool wl = rank > 0 || seg > 0, wr2 = rank < B || seg < G - 1;
            mvxn<TM, HW, NR>(wl ? it.m0 : nullptr, wl ? ab : nullptr,
                             wr2 ? it.m1 : nullptr, wr2 ? ab + TM : nullptr, N2, lane, acc);
            if (wr) {
#pragma unroll
              for (int rh = 0; rh < NR; ++rh)
                Yv[rh * FS + j * TM + x] = csub(Yv[rh * FS + j * TM + x], acc[rh]);
            }
          }
        }
        release(it, has);
      }
      stamp(ti, 42);
      csync();
    }
    // ---- edge blocks of x to the neighbours (next task's transmission halo)
    if (ti + 1 < fcount && lane < TM) {
#pragma unroll
      for (int rh = 0; rh < NR; ++rh) {
        const int nb = (((ti + 1) & 1) * NR + rh) * HS;
        if (warp == 0 && rank > 0)
          st_async_c(map_rank(&halo2[nb + TM + lane], rank - 1), Yv[rh * FS + lane],
                     map_rank(&xbar[2 + ((ti + 1) & 1)], rank - 1));
        if (warp == 1 && rank < B)
          st_async_c(map_rank(&halo2[nb + lane], rank + 1), Yv[rh * FS + (m - 1) * TM + lane],
                     map_rank(&xbar[2 + ((ti + 1) & 1)], rank + 1));
      }
    }
    // ---- outputs: solution rows into u (one producer per row and pass), traces
    const int ur0 = t.ta + 1 - t.lo, ur1 = t.tb + 1 - t.lo;
    for (int yl = warp * YPW + hh; yl < m; yl += kCW * YPW) {
      const int y = Y0 + yl;
#pragma unroll
      for (int rh = 0; rh < NR; ++rh) {
        const double2 xv = Yv[rh * FS + yl * TM + x];
        if (x >= ur0 && x < ur1)
          a.u[t.dst][rh * a.vs_u[t.dst] + (int64_t)(x + t.lo - 1) * M + y] = xv;
        if (t.out2 >= 0 && (x == t.orow2 || x == t.orow2 + 1))
          a.trace[rh * a.ts + ((int64_t)t.out2 * 2 + (x - t.orow2)) * M + y] = xv;
        if (t.out4 >= 0 && (x == t.orow4 || x == t.orow4 + 1))
          a.trace[rh * a.ts + ((int64_t)t.out4 * 2 + (x - t.orow4)) * M + y] = xv;
      }
    }
    stamp(ti, 43);
    prev = t;
    stamp(ti, 63);
  }
  cl.sync();   // no CTA leaves while a peer may still write its shared memory
  if (a.dbg && threadIdx.x == 0 && blockIdx.x < 16)
    for (int k = 0; k < 128; ++k) {
      a.dbg[blockIdx.x * 1024 + k] = tsm[k];
    }
}

__global__ void k_combine(double2* __restrict__ u, const double2* __restrict__ u2, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[i] = cadd(u[i], __ldg(u2 + i));
}

cudaLaunchConfig_t solve_config(int C, int nfront, int smem, cudaStream_t st,
                                cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nfront * C, 1, 1);
  cfg.blockDim = dim3(kWarps * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

template <int TM, int NR>
cudaError_t prepare_solve_nr(int C, int mmax, int* max_clusters) {
  cudaError_t e = cudaFuncSetAttribute(k_part_solve<TM, NR>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  const int smem = Ring<TM>::smem(mmax, C, NR);
  e = cudaFuncSetAttribute(k_part_solve<TM, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = solve_config(C, 1, smem, nullptr, attr);
  return cudaOccupancyMaxActiveClusters(max_clusters, k_part_solve<TM, NR>, &cfg);
}
// every right-hand-side width of the kernel (kSolveWidths); *max_clusters: the
// smallest co-residency over the widths (the fronts' clusters wait on each other)
template <int TM>
cudaError_t prepare_solve(int C, int mmax, int* max_clusters, int* max_nr = nullptr) {
  cudaError_t e = prepare_solve_nr<TM, 1>(C, mmax, max_clusters);
  if (e != cudaSuccess || !max_nr) return e;
  // wider kernels are optional: available when their vectors leave room for
  // a ring of >= 5 chunks (C3's 34-point chunks with 3 slots: 4 right-hand
  // sides per chain measured slower than 2) and as many clusters co-reside
  *max_nr = 1;
  int mc = 0;
  if (Ring<TM>::fixed(mmax, C, 2) + 5 * (Ring<TM>::CHUNK * 16 + 16) <= 225 * 1024 &&
      prepare_solve_nr<TM, 2>(C, mmax, &mc) == cudaSuccess && mc >= *max_clusters) {
    *max_nr = 2;
    if (Ring<TM>::fixed(mmax, C, 4) + 5 * (Ring<TM>::CHUNK * 16 + 16) <= 225 * 1024 &&
        prepare_solve_nr<TM, 4>(C, mmax, &mc) == cudaSuccess && mc >= *max_clusters)
      *max_nr = 4;
  }
  cudaGetLastError();
  return cudaSuccess;
}
// launch the slab-solve kernel for nr (1, 2 or 4) right-hand sides
static cudaError_t launch_solve(int tm, int nr, int C, int nclusters, int mmax, cudaStream_t st,
                                SolveArgs& a) {
  const int smem = tm == 16 ? Ring<16>::smem(mmax, C, nr) : Ring<32>::smem(mmax, C, nr);
  a.nchunk = tm == 16 ? Ring<16>::nchunk(mmax, C, nr) : Ring<32>::nchunk(mmax, C, nr);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = solve_config(C, nclusters, smem, st, attr);
  if (tm == 16) {
    switch (nr) {
      case 1: return cudaLaunchKernelEx(&cfg, k_part_solve<16, 1>, a);
      case 2: return cudaLaunchKernelEx(&cfg, k_part_solve<16, 2>, a);
      case 4: return cudaLaunchKernelEx(&cfg, k_part_solve<16, 4>, a);
    }
  } else {
    switch (nr) {
      case 1: return cudaLaunchKernelEx(&cfg, k_part_solve<32, 1>, a);
      case 2: return cudaLaunchKernelEx(&cfg, k_part_solve<32, 2>, a);
      case 4: return cudaLaunchKernelEx(&cfg, k_part_solve<32, 4>, a);
    }
  }
  return cudaErrorInvalidValue;
}

template <int TM, int Q>
cudaError_t launch_dense_top_q(Ctx* c, const Chunks& g, int J, const double2* D, const double2* Lc,
                               const double2* Uc, double2* qd, unsigned long long* err) {
  constexpr int N = Q * TM;
  const int smem = 2 * N * (N + 1) * (int)sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(k_dense_top<TM, Q>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_dense_top<TM, Q><<<J * g.nch(), 1024, smem, c->stream>>>(g, D, Lc, Uc, qd, err);
  c->launches++;
  return cudaGetLastError();
}

template <int TM>
cudaError_t launch_dense_top(Ctx* c, const Chunks& g, int J, const double2* D, const double2* Lc,
                             const double2* Uc, double2* qd, unsigned long long* err) {
  if constexpr (TM == 16) {
    switch (g.q) {
      case 1: return launch_dense_top_q<16, 1>(c, g, J, D, Lc, Uc, qd, err);
      case 2: return launch_dense_top_q<16, 2>(c, g, J, D, Lc, Uc, qd, err);
      case 3: return launch_dense_top_q<16, 3>(c, g, J, D, Lc, Uc, qd, err);
      case 4: return launch_dense_top_q<16, 4>(c, g, J, D, Lc, Uc, qd, err);
      case 5: return launch_dense_top_q<16, 5>(c, g, J, D, Lc, Uc, qd, err);
    }
  } else {
    switch (g.q) {
      case 1: return launch_dense_top_q<32, 1>(c, g, J, D, Lc, Uc, qd, err);
      case 2: return launch_dense_top_q<32, 2>(c, g, J, D, Lc, Uc, qd, err);
    }
  }
  return cudaErrorInvalidValue;
}

template <int TM>
int factorize(Ctx* c, Sweep* s, const std::vector<SlabInfo>& info, const Chunks& g) {
  constexpr int TM2 = Geo<TM>::TM2;
  const int J = s->J, M = s->M, L = s->L, C = s->C, B = C - 1, G = s->G, NCH = C * G;
  const size_t wbytes = (size_t)J * M * TM2 * sizeof(double2);
  const size_t ebytes = (size_t)J * NCH * TM2 * sizeof(double2);
  double2 *D = nullptr, *Lc = nullptr, *Uc = nullptr, *EL = nullptr, *EU = nullptr;
  double2 *Hw = nullptr, *Zw = nullptr, *tips = nullptr, *Gw = nullptr, *Zr = nullptr;
  double2 *tips2 = nullptr, *rk2 = nullptr, *Gw2 = nullptr, *Zr2 = nullptr;
  SlabInfo* d_info = nullptr;
  unsigned long long* d_err = nullptr;
  int rc = HS_OK;
  auto cleanup = [&]() {
    cudaFree(D); cudaFree(Lc); cudaFree(Uc); cudaFree(EL); cudaFree(EU); cudaFree(Hw);
    cudaFree(Zw); cudaFree(tips); cudaFree(Gw); cudaFree(Zr); cudaFree(d_info); cudaFree(d_err);
    cudaFree(tips2); cudaFree(rk2); cudaFree(Gw2); cudaFree(Zr2);
    Gw = Zr = tips2 = rk2 = Gw2 = Zr2 = nullptr;
  };
#define HS_TRYF(call, what)                                            \
  do {                                                                 \
    cudaError_t _e = (call);                                           \
    if (_e != cudaSuccess) { rc = check_cuda(c, _e, what); cleanup(); return rc; } \
  } while (0)
  HS_TRYF(cudaMalloc((void**)&D, wbytes), "bcr work alloc");
  HS_TRYF(cudaMalloc((void**)&Lc, wbytes), "bcr work alloc");
  HS_TRYF(cudaMalloc((void**)&Uc, wbytes), "bcr work alloc");
  HS_TRYF(cudaMalloc((void**)&EL, ebytes), "alloc");
  HS_TRYF(cudaMalloc((void**)&EU, ebytes), "alloc");
  HS_TRYF(cudaMalloc((void**)&tips, 4 * ebytes), "alloc");
  HS_TRYF(cudaMalloc((void**)&d_info, J * sizeof(SlabInfo)), "alloc");
  HS_TRYF(cudaMalloc((void**)&d_err, sizeof(unsigned long long)), "alloc");
  HS_TRYF(cudaMemcpyAsync(d_info, info.data(), J * sizeof(SlabInfo), cudaMemcpyHostToDevice,
                          c->stream), "upload");
  HS_TRYF(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), c->stream), "memset");
  HS_TRYF(cudaMemsetAsync(EL, 0, ebytes, c->stream), "memset");
  HS_TRYF(cudaMemsetAsync(EU, 0, ebytes, c->stream), "memset");
  HS_TRYF(cudaMemsetAsync(s->eb, 0, 2 * wbytes, c->stream), "memset");
  HS_TRYF(cudaMemsetAsync(s->kr, 0, (size_t)J * NCH * g.kstride * 2 * TM2 * sizeof(double2),
                          c->stream), "memset");
  const int smem3 = 3 * TM * (TM + 1) * (int)sizeof(double2);
  const int smem4 = 4 * TM * (TM + 1) * (int)sizeof(double2);
  const int smem7 = 7 * TM * (TM + 1) * (int)sizeof(double2);
  HS_TRYF(cudaFuncSetAttribute(k_bcr_elim<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem3), "attr");
  HS_TRYF(cudaFuncSetAttribute(k_bcr_keep<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem4), "attr");
  HS_TRYF(cudaFuncSetAttribute(k_spikes<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem7), "attr");
  k_bcr_init<TM><<<dim3(M, J), TM * TM, 0, c->stream>>>(d_info, g, D, Lc, Uc, EL, EU);
  c->launches++;
  HS_TRYF(cudaGetLastError(), "bcr init");
  if (s->cpl0) {
    k_cpl0<TM><<<dim3(M, J), 256, 0, c->stream>>>(d_info, M, s->cpl);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "level-0 couplings");
  }
  if (B > 0) {   // spikes from the pristine chunk operators
    HS_TRYF(cudaMalloc((void**)&Hw, wbytes), "spike work alloc");
    HS_TRYF(cudaMalloc((void**)&Zw, wbytes), "spike work alloc");
    k_spikes<TM><<<J * NCH, TM * TM, smem7, c->stream>>>(g, D, Lc, Uc, EL, EU, Hw, Zw, s->sp,
                                                         tips, d_err);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "spikes");
    constexpr int N = 2 * TM;
    const int NR = B * N;
    HS_TRYF(cudaMalloc((void**)&Gw, (size_t)J * G * B * N * N * sizeof(double2)), "alloc");
    HS_TRYF(cudaMalloc((void**)&Zr, (size_t)J * G * NR * NR * sizeof(double2)), "alloc");
    const int smemr = 2 * N * (N + 1) * (int)sizeof(double2);
    HS_TRYF(cudaFuncSetAttribute(k_reduced<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smemr), "attr");
    // level 1: each segment's C chunks
    k_reduced<TM><<<J * G, 1024, smemr, c->stream>>>(C, G, tips, Gw, Zr, s->rk, d_err);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "reduced system");
    if (G > 1) {
      // level 2: segment tips from the level-1 inverse rows, then the
      // G-segment interface inverse; its rows go to each segment's first chunk
      const int xs = g.xstride(), B2 = G - 1, NR2 = B2 * N;
      HS_TRYF(cudaMalloc((void**)&tips2, (size_t)J * G * 4 * TM2 * sizeof(double2)), "alloc");
      HS_TRYF(cudaMalloc((void**)&rk2, (size_t)J * G * 2 * B2 * 2 * TM2 * sizeof(double2)), "alloc");
      HS_TRYF(cudaMalloc((void**)&s->x2, (size_t)J * NCH * xs * TM2 * sizeof(double2)), "alloc");
      HS_TRYF(cudaMalloc((void**)&Gw2, (size_t)J * B2 * N * N * sizeof(double2)), "alloc");
      HS_TRYF(cudaMalloc((void**)&Zr2, (size_t)J * NR2 * NR2 * sizeof(double2)), "alloc");
      HS_TRYF(cudaMemsetAsync(s->x2, 0, (size_t)J * NCH * xs * TM2 * sizeof(double2), c->stream),
              "memset");
      const int smeml = 4 * TM * (TM + 1) * (int)sizeof(double2);
      HS_TRYF(cudaFuncSetAttribute(k_level2<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smeml), "attr");
      k_level2<TM><<<J * G, TM * TM, smeml, c->stream>>>(g, tips, s->rk, tips2, s->x2);
      c->launches++;
      HS_TRYF(cudaGetLastError(), "level-2 tips");
      k_reduced<TM><<<J, 1024, smemr, c->stream>>>(G, 1, tips2, Gw2, Zr2, rk2, d_err);
      c->launches++;
      HS_TRYF(cudaGetLastError(), "level-2 reduced system");
      // rows of segment s -> blocks 1 .. 4(G-1) of chunk s*C
      HS_TRYF(cudaMemcpy2DAsync(s->x2 + TM2, (size_t)C * xs * TM2 * sizeof(double2), rk2,
                                (size_t)4 * B2 * TM2 * sizeof(double2),
                                (size_t)4 * B2 * TM2 * sizeof(double2), (size_t)J * G,
                                cudaMemcpyDeviceToDevice, c->stream), "level-2 rows");
    }
  }
  const int mmax = s->mmax;
  for (int l = 0; l < L; ++l) {
    const int sl = 1 << l;
    const int nel = mmax - 1 >= sl ? (mmax - 1 - sl) / (2 * sl) + 1 : 0;
    const int nkeep = (mmax - 1) / (2 * sl) + 1;
    if (nel) {
      k_bcr_elim<TM><<<dim3(nel, J * NCH), TM * TM, smem3, c->stream>>>(l, g, 0, D, Lc, Uc,
                                                                        s->ef, s->eb, d_err);
      c->launches++;
      HS_TRYF(cudaGetLastError(), "bcr elim");
    }
    k_bcr_keep<TM><<<dim3(nkeep, J * NCH), TM * TM, smem4, c->stream>>>(l, g, D, Lc, Uc, s->kr);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "bcr keep");
  }
  HS_TRYF(launch_dense_top<TM>(c, g, J, D, Lc, Uc, s->qd, d_err), "dense top");
  if (g.nr) {   // restricted level-0 / spike updates
    HS_TRYF(cudaMalloc((void**)&s->ebr, (size_t)J * M * TM2 * sizeof(double2)), "alloc");
    HS_TRYF(cudaMalloc((void**)&s->spr, (size_t)J * M * TM2 * sizeof(double2)), "alloc");
    k_rows<TM><<<dim3(M, J), 256, 0, c->stream>>>(g, s->rows, s->eb, s->sp, s->ebr, s->spr);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "rows");
  }
  // repack into per-(slab, chunk) streams in the solve kernel's item order
  long long nbs = 1;
  for (int k = 0; k < NCH; ++k) nbs = std::max<long long>(nbs, stream_blocks<TM>(g, k));
  s->nbs = nbs;
  HS_TRYF(cudaMalloc((void**)&s->stream, (size_t)J * NCH * nbs * TM2 * sizeof(double2)),
          "stream alloc");
  k_pack<TM><<<J * NCH, 256, 0, c->stream>>>(
      g, FactorArrays{s->ef, s->eb, s->kr, s->rk, s->sp, s->qd, s->ebr, s->spr, s->x2, s->cpl},
      s->stream,
      (int)nbs);
  c->launches++;
  HS_TRYF(cudaGetLastError(), "pack");
  unsigned long long err = 0;
  HS_TRYF(cudaMemcpyAsync(&err, d_err, sizeof err, cudaMemcpyDeviceToHost, c->stream), "err");
  HS_TRYF(cudaStreamSynchronize(c->stream), "factor sync");
#undef HS_TRYF
  cleanup();
  for (double2** p : {&s->ef, &s->eb, &s->kr, &s->sp, &s->rk, &s->qd, &s->ebr, &s->spr, &s->x2,
                      &s->cpl}) {
    cudaFree(*p);
    *p = nullptr;
  }
  s->factor_bytes = (long long)J * NCH * nbs * TM2 * (long long)sizeof(double2);
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

Chunks make_chunks(const Sweep* s) {
  Chunks g{};
  g.M = s->M;
  g.C = s->C;
  g.G = s->G;
  g.L = s->L;
  g.q = s->q;
  g.nr = s->nr;
  g.cpl0 = s->cpl0;
  for (int k = 0; k <= s->C * s->G; ++k) g.y0s[k] = s->y0s[k];
  g.mmax = s->mmax;
  int acc = 0;
  for (int l = 0; l < s->L; ++l) {
    g.koff[l] = acc;
    acc += (s->mmax - 1) / (2 << l) + 1;
  }
  g.kstride = std::max(1, acc);
  return g;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

// Task lists and launch plans of the sweep schedules (prec_ud / prec_x /
// prec_nx, sweepdd.py:312-437), shared by the 2-D and 3-D sweeps.  A front
// is a chain of slab solves run in order by one cluster (2-D) with the
// traces of consecutive tasks handed over on chip; fronts of one launch are
// independent.  A trace consumed by two fronts comes from a task placed at
// the head of both (computed twice, identical results).
namespace {
struct SchedBuilder {
  Sweep* s;
  int J;
  const int64_t *beta, *bt, *lo, *hi;
  int ntin = 0;   // trace buffers handed out

  SweepTask mk(int j, int a_, int b_) const {
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
  }
  int want1(SweepTask& t) {   // tau1 (forward in), gated j > 1
    const int j = t.slab + 1;
    if (j <= 1) return -1;
    t.tin1 = ntin++;
    t.row1 = (int)beta[j - 1] - t.lo;
    return t.tin1;
  }
  int want3(SweepTask& t) {   // tau3 (backward in), gated j < J
    const int j = t.slab + 1;
    if (j >= J) return -1;
    t.tin3 = ntin++;
    t.row3 = (int)bt[j] - t.lo;
    return t.tin3;
  }
  void give2(SweepTask& t, int buf) const {   // tau2 (forward out), gated j < J
    const int j = t.slab + 1;
    if (j >= J || buf < 0) return;
    t.out2 = buf;
    t.orow2 = (int)beta[j] - t.lo;
  }
  void give4(SweepTask& t, int buf) const {   // tau4 (backward out), gated j > 1
    const int j = t.slab + 1;
    if (j <= 1 || buf < 0) return;
    t.out4 = buf;
    t.orow4 = (int)bt[j - 1] - t.lo;
  }
  SweepTask fwd_task(int j) const { return mk(j, (int)beta[j - 1], (int)beta[j]); }
  SweepTask bwd_task(int j) const { return mk(j, (int)bt[j - 1], (int)bt[j]); }
  SweepTask mid_in(int j) const { return mk(j, (int)beta[j - 1], (int)bt[j]); }    // midsolve_in
  SweepTask mid_out(int j) const { return mk(j, (int)bt[j - 1], (int)beta[j]); }   // midsolve_out
  // forward_sweep j0..j1 (out-of-range slabs skipped), chained through traces
  std::vector<SweepTask> fwd_chain(int j0, int j1) {
    std::vector<SweepTask> v;
    for (int j = j0; j <= j1; ++j) {
      if (j < 1 || j > J) continue;
      SweepTask t = fwd_task(j);
      const int in = want1(t);
      if (!v.empty()) give2(v.back(), in);
      v.push_back(t);
    }
    return v;
  }
  std::vector<SweepTask> bwd_chain(int j0, int j1) {
    std::vector<SweepTask> v;
    for (int j = j0; j >= j1; --j) {
      if (j < 1 || j > J) continue;
      SweepTask t = bwd_task(j);
      const int in = want3(t);
      if (!v.empty()) give4(v.back(), in);
      v.push_back(t);
    }
    return v;
  }
  // one solve launch per stage; a stage with more than kMaxFront fronts is
  // split into several launches (its fronts are independent)
  void emit(std::vector<SweepLaunch>& plan, int src,
            const std::vector<std::vector<std::vector<SweepTask>>>& stages) {
    std::vector<SweepTask>& T = s->tasks;
    for (const auto& st : stages) {
      SweepLaunch fl{};
      fl.kind = SweepLaunch::kSolve;
      fl.src = src;
      for (const auto& fr : st) {
        if (fr.empty()) continue;
        if (fl.nfront == std::min(kMaxFront, s->max_fronts)) {
          plan.push_back(fl);
          fl = SweepLaunch{};
          fl.kind = SweepLaunch::kSolve;
          fl.src = src;
        }
        fl.ffirst[fl.nfront] = (int)T.size();
        fl.fcount[fl.nfront] = (int)fr.size();
        fl.nfront++;
        for (SweepTask t : fr) {
          t.dst = src;
          T.push_back(t);
        }
      }
      if (fl.nfront) plan.push_back(fl);
    }
  }
};

std::vector<SweepTask> cat(const std::vector<SweepTask>& head, const std::vector<SweepTask>& v) {
  std::vector<SweepTask> r(head);
  r.insert(r.end(), v.begin(), v.end());
  return r;
}
}  // namespace

// UD and X plans; returns the number of trace buffers
static int build_schedule(Sweep* s, int J, const int64_t* beta, const int64_t* bt,
                          const int64_t* lo, const int64_t* hi) {
  s->hbeta.assign(beta, beta + J + 1);
  s->hbt.assign(bt, bt + J + 1);
  s->hlo.assign(lo, lo + J);
  s->hhi.assign(hi, hi + J);
  SchedBuilder b{s, J, beta, bt, lo, hi};
  // ---- UD: forward 1..J on f; g = f - A u; backward J..1 on g ----
  {
    std::vector<SweepLaunch>& plan = s->plan[HS_VARIANT_UD];
    b.emit(plan, 0, {{b.fwd_chain(1, J)}});
    plan.push_back(SweepLaunch{SweepLaunch::kResidual});
    b.emit(plan, 1, {{b.bwd_chain(J, 1)}});
    plan.push_back(SweepLaunch{SweepLaunch::kCombine});
  }
  // ---- X: simultaneous half sweeps meeting at jm = J/2 + 1 ----
  if (J % 2 == 0) {
    std::vector<SweepLaunch>& plan = s->plan[HS_VARIANT_X];
    const int jm = J / 2 + 1;
    std::vector<SweepTask> F = b.fwd_chain(1, jm - 1), Bk = b.bwd_chain(J, jm + 1);
    SweepTask mi = b.mid_in(jm);
    const int in1 = b.want1(mi), in3 = b.want3(mi);
    if (!F.empty()) b.give2(F.back(), in1);
    if (!Bk.empty()) b.give4(Bk.back(), in3);
    b.emit(plan, 0, {{F, Bk}, {{mi}}});
    plan.push_back(SweepLaunch{SweepLaunch::kResidual});
    SweepTask mo = b.mid_out(jm);
    std::vector<SweepTask> BB = b.bwd_chain(jm - 1, 1), FF = b.fwd_chain(jm + 1, J);
    if (!FF.empty()) b.give2(mo, FF.front().tin1);
    if (!BB.empty()) b.give4(mo, BB.front().tin3);
    // the middle solve opens both outward fronts (computed by both clusters,
    // identical results), so pass 2 is one launch with in-cluster handoffs
    b.emit(plan, 1, {{cat({mo}, BB), cat({mo}, FF)}});
    plan.push_back(SweepLaunch{SweepLaunch::kCombine});
  }
  return b.ntin;
}

// NX: ncell groups, each an X sweep over its cell; the group-boundary input
// solve of pass 2 runs once both of its traces exist (prec_nx's note,
// sweepdd.py:403-437).  Pass 1: every cell's forward and backward fronts in
// one launch -- the boundary output solve mid_out(jc[m]) heads both fronts
// that read its traces -- then the cells' meeting solves mid_in(jm[m]).
// Pass 2: mid_out(jm[m]) heads both outward fronts of cell m, then the
// boundary input solves mid_in(jc[m]).
static std::vector<SweepLaunch> build_nx(Sweep* s, int ncell, const int64_t* jc,
                                         const int64_t* jmid, int* ntin) {
  const int J = s->J;
  SchedBuilder b{s, J, s->hbeta.data(), s->hbt.data(), s->hlo.data(), s->hhi.data()};
  std::vector<SweepLaunch> plan;
  const int nc = ncell;
  // a chain's head task hands its trace to the chain's first task, or, for an
  // empty chain, to the solve after it (forward_sweep returns B unchanged)
  {   // ---- pass 1 ----
    std::vector<std::vector<SweepTask>> F(nc + 1), Bk(nc + 1);
    std::vector<SweepTask> MI(nc + 1), MO(nc + 1);
    for (int m = 1; m <= nc; ++m) {
      F[m] = b.fwd_chain((int)jc[m - 1] + 1, (int)jmid[m - 1] - 1);
      Bk[m] = b.bwd_chain((int)jc[m] - 1, (int)jmid[m - 1] + 1);
      MI[m] = b.mid_in((int)jmid[m - 1]);
      const int in1 = b.want1(MI[m]), in3 = b.want3(MI[m]);
      if (!F[m].empty()) b.give2(F[m].back(), in1);
      if (!Bk[m].empty()) b.give4(Bk[m].back(), in3);
    }
    for (int m = 1; m < nc; ++m) {   // mid_out(jc[m]) feeds F[m+1] and Bk[m]
      MO[m] = b.mid_out((int)jc[m]);
      b.give2(MO[m], F[m + 1].empty() ? MI[m + 1].tin1 : F[m + 1].front().tin1);
      b.give4(MO[m], Bk[m].empty() ? MI[m].tin3 : Bk[m].front().tin3);
    }
    std::vector<std::vector<SweepTask>> fronts, mids;
    for (int m = 1; m <= nc; ++m) {
      fronts.push_back(m > 1 && !F[m].empty() ? cat({MO[m - 1]}, F[m]) : F[m]);
      if (m < nc) {
        if (!Bk[m].empty()) fronts.push_back(cat({MO[m]}, Bk[m]));
        else if (F[m + 1].empty()) fronts.push_back({MO[m]});   // computed once
      } else {
        fronts.push_back(Bk[m]);
      }
      mids.push_back({MI[m]});
    }
    b.emit(plan, 0, {fronts, mids});
  }
  plan.push_back(SweepLaunch{SweepLaunch::kResidual});
  {   // ---- pass 2 ----
    std::vector<std::vector<SweepTask>> BB(nc + 1), FF(nc + 1);
    std::vector<SweepTask> MO(nc + 1), MI(nc + 1);
    for (int m = 1; m <= nc; ++m) {
      BB[m] = b.bwd_chain((int)jmid[m - 1] - 1, (int)jc[m - 1] + 1);
      FF[m] = b.fwd_chain((int)jmid[m - 1] + 1, (int)jc[m] - 1);
      MO[m] = b.mid_out((int)jmid[m - 1]);
    }
    for (int m = 2; m <= nc; ++m) {   // mid_in(jc[m-1]) after cells m-1 and m
      MI[m] = b.mid_in((int)jc[m - 1]);
      const int in1 = b.want1(MI[m]), in3 = b.want3(MI[m]);
      if (!FF[m - 1].empty()) b.give2(FF[m - 1].back(), in1);
      else b.give2(MO[m - 1], in1);
      if (!BB[m].empty()) b.give4(BB[m].back(), in3);
      else b.give4(MO[m], in3);
    }
    for (int m = 1; m <= nc; ++m) {
      if (!FF[m].empty()) b.give2(MO[m], FF[m].front().tin1);
      if (!BB[m].empty()) b.give4(MO[m], BB[m].front().tin3);
    }
    std::vector<std::vector<SweepTask>> fronts, mids;
    for (int m = 1; m <= nc; ++m) {
      if (BB[m].empty() && FF[m].empty()) {
        fronts.push_back({MO[m]});
      } else {
        if (!BB[m].empty()) fronts.push_back(cat({MO[m]}, BB[m]));
        if (!FF[m].empty()) fronts.push_back(cat({MO[m]}, FF[m]));
      }
      if (m > 1) mids.push_back({MI[m]});
    }
    b.emit(plan, 1, {fronts, mids});
  }
  plan.push_back(SweepLaunch{SweepLaunch::kCombine});
  *ntin = b.ntin;
  return plan;
}

// algorithmic HBM bytes of every solve launch of a plan (profiler), SURVEY
// 8(d): the no-pivot banded LU floor of each slab solved in the launch,
// (2 bw + 1) n 16 B with n = T * face unknowns and the sweep's bandwidth
// bw = T_max + 1 (2-D) / T_max n_y + T_max + 1 (3-D), thin axis fastest --
// the format-independent factor bytes a slab solve must read.  The bytes
// this build's own factor format streams are s->factor_bytes per pass.
static void plan_bytes(const Sweep* s, std::vector<SweepLaunch>& plan) {
  const double M = (double)s->M;
  int tmax = 1;
  for (const SweepTask& t : s->tasks) tmax = std::max(tmax, (int)t.T);
  const double ny = s->s3 ? (double)s->coarse->shape[1] : 1.0;
  const double bw = s->s3 ? tmax * ny + tmax + 1.0 : tmax + 1.0;
  for (auto& fl : plan) {
    if (fl.kind != SweepLaunch::kSolve) continue;
    fl.bytes = 0;
    for (int f = 0; f < fl.nfront; ++f)
      for (int i = fl.ffirst[f]; i < fl.ffirst[f] + fl.fcount[f]; ++i) {
        const SweepTask& t = s->tasks[i];
        const double n = (double)t.T * (s->s3 ? ny * (double)s->coarse->shape[2] : M);
        fl.bytes += (2.0 * bw + 1.0) * n * 16.0;
      }
  }
}

// level-2 exchange buffers of a work set (zeroed counters)
constexpr int64_t kXStride = (int64_t)kMaxFront * 2 * kMaxG * 2 * 32;   // per right-hand side
static cudaError_t alloc_exchange(SweepWork* w, int nrhs = 1) {
  const size_t nb = (size_t)nrhs * kXStride * sizeof(double2);
  const size_t nf = (size_t)kMaxFront * 2 * kMaxG * sizeof(unsigned);
  cudaError_t e = cudaMalloc((void**)&w->xbuf, nb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&w->xflag, nf);
  if (e == cudaSuccess) e = cudaMemset(w->xflag, 0, nf);
  for (auto& x : w->xcount) x = 0;
  return e;
}

int sweep_create(Ctx* c, const Stencil* coarse, int J, const int64_t* beta, const int64_t* bt,
                 const int64_t* lo, const int64_t* hi, const Stencil* const* slabs,
                 Sweep** out) {
  if (coarse->dim != 2 && coarse->dim != 3)
    return set_error(c, HS_E_SHAPE, "the device sweep needs a 2-D or 3-D level");
  if (J < 2) return set_error(c, HS_E_SHAPE, "the sweep needs at least 2 subdomains");
  if (J > kMaxTasks) return set_error(c, HS_E_SHAPE, "too many subdomains for the sweep");
  auto buffers = [&](Sweep* s, int ntin) -> int {   // traces, mid-sweep residual, pass-2 u
    cudaError_t e = cudaMalloc((void**)&s->trace, (size_t)std::max(1, ntin) * 2 * s->M * sizeof(double2));
    if (e == cudaSuccess) e = cudaMalloc((void**)&s->g, (size_t)s->n0 * s->M * sizeof(double2));
    if (e == cudaSuccess) e = cudaMalloc((void**)&s->u2, (size_t)s->n0 * s->M * sizeof(double2));
    s->own.trace = s->trace;   // the sweep's own work set (the default of sweep_apply)
    s->own.g = s->g;
    s->own.u2 = s->u2;
    return e == cudaSuccess ? HS_OK : check_cuda(c, e, "sweep buffers");
  };
  if (coarse->dim == 3) {   // block-LU slabs along face axis 1 (hs_sweep3.cu)
    Sweep* s = new Sweep();
    s->J = J;
    s->n0 = (int)coarse->shape[0];
    s->M = (int)(coarse->shape[1] * coarse->shape[2]);
    s->coarse = coarse;
    const int ntin = std::max(4, build_schedule(s, J, beta, bt, lo, hi));
    s->ntrace = ntin;
    int r = sweep3_create(c, s, coarse, slabs, lo, hi, nullptr);
    if (!r) r = buffers(s, ntin);
    if (!r)
      for (auto& plan : s->plan) plan_bytes(s, plan);
    if (r) {
      sweep_destroy(s);
      return r;
    }
    *out = s;
    return HS_OK;
  }
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
  // Layout: the face is cut into G segments per front (one cluster of C CTAs
  // each, one chunk of the face per CTA), coupled by the level-2 interface
  // system (two-level partition); both fronts' G clusters must co-reside
  // (2 G <= active clusters: they wait on each other).  Measured on B200
  // (DESIGN 5.1): the more CTAs the fronts use the faster the sweep, and
  // 9-CTA clusters (two per GPC) co-reside 14 at a time where 16-CTA
  // clusters fit 7 -- C = 9, G = 7 runs C3's sweep in 12.6 ms against 14.6
  // (C = 16, G = 3), C2's in 1.77 against 2.21 ms -- so the default is C = 9
  // with as many segments as co-reside, keeping chunks >= 8 face points;
  // short faces (M < 144) keep one segment of chunks of >= 16 points
  // (C = M / 16): many 4-point chunks or a level-2 system gain nothing there
  // and cost accuracy (the interface systems multiply: sweep error vs the
  // reference 1e-11 -> 2-4e-11 relative on a 39-point face).
  // One segment requested (sweep lanes: several fronts' sweeps side by side)
  // keeps the one-cluster layout with chunks of ~32 points, C <= 16.
  int C, G;
  if (c->sweep_segments == 1) {
    C = std::min(kMaxC, std::max(1, (M + 31) / 32));
    G = 1;
  } else {
    C = std::max(1, std::min(9, M / 16));
    G = M < 144 ? 1 : std::max(1, std::min(std::min(kMaxG, kMaxCh / C), M / (8 * C)));
    if (c->sweep_cluster > 1) C = std::max(2, std::min(std::min(kMaxC, c->sweep_cluster), M / 8));
    if (c->sweep_segments > 1) G = std::min(std::min(kMaxG, kMaxCh / C), c->sweep_segments);
  }
  if (const char* ev = getenv("HS_SWEEP_SEGMENTS")) G = std::max(1, std::min(kMaxG, atoi(ev)));
  if (const char* ev = getenv("HS_SWEEP_CPC")) C = std::max(1, std::min(kMaxC, atoi(ev)));
  G = std::max(1, std::min(G, kMaxCh / std::max(1, C)));
  if (C < 2) G = 1;
  int maxc = 0;
  for (;;) {
    const int mmax = (M + C * G - 1) / (C * G);
    cudaError_t e = TM == 16 ? prepare_solve<16>(C, mmax, &maxc) : prepare_solve<32>(C, mmax, &maxc);
    if (e == cudaSuccess && maxc >= 2 * G) break;
    cudaGetLastError();
    if (e == cudaSuccess && G > 1) {   // fewer segments (the fronts' clusters must co-reside)
      G = std::max(1, std::min(G - 1, maxc / 2));
      continue;
    }
    if (C == 1) {
      delete s;
      return set_error(c, HS_E_CUDA, "no schedulable cluster for the sweep kernel");
    }
    C = C > 8 ? 8 : C / 2;
    if (C < 2) G = 1;
  }
  const int NCH = C * G;
  s->C = C;
  s->G = G;
  s->mmax = (M + NCH - 1) / NCH;
  // cyclic reduction until at most qmax blocks per chunk are left, then a
  // dense inverse of that reduced system (qmax blocks fit the setup's smem)
  const int qmax = TM == 16 ? 5 : 2;
  s->L = 0;
  while ((s->mmax - 1) / (1 << s->L) + 1 > qmax) ++s->L;
  {
    // Chunk sizes m = 1 (mod S/2) for every chunk but the last, so each right
    // tip is final after the dense top or the first back-substitution level
    // and the interface solve overlaps the rest of the back substitution.
    const int S = 1 << s->L, h = std::max(1, S / 2), cap = S * qmax;
    std::vector<int> mk(NCH, 0);
    const double mean = (double)M / NCH;
    const int base = std::max(1, 1 + h * (int)std::lround((mean - 1.0) / h));
    int rem = M;
    for (int k = 0; k + 1 < NCH; ++k) { mk[k] = base; rem -= base; }
    for (int k = 0; k + 1 < NCH && rem > mean + h / 2.0; k = (k + 1) % (NCH - 1)) {
      if (mk[k] + h > cap) break;
      mk[k] += h; rem -= h;
    }
    for (int k = 0; k + 1 < NCH && rem < std::max(1.0, mean - h); k = (k + 1) % (NCH - 1)) {
      if (mk[k] - h < 1) break;
      mk[k] -= h; rem += h;
    }
    mk[NCH - 1] = rem;
    bool ok = true;
    for (int k = 0; k < NCH; ++k) ok = ok && mk[k] >= 1 && mk[k] <= cap;
    s->y0s[0] = 0;
    for (int k = 0; k < NCH; ++k)
      s->y0s[k + 1] = ok ? s->y0s[k] + mk[k] : (int)((int64_t)(k + 1) * M / NCH);
    s->mmax = 0;
    for (int k = 0; k < NCH; ++k) s->mmax = std::max(s->mmax, s->y0s[k + 1] - s->y0s[k]);
    while ((s->mmax - 1) / (1 << s->L) + 1 > qmax) ++s->L;   // (uniform fallback only)
    // the kernel's shared memory follows the final chunk length
    cudaError_t e0 = TM == 16 ? prepare_solve<16>(C, s->mmax, &maxc, &s->max_nr)
                              : prepare_solve<32>(C, s->mmax, &maxc, &s->max_nr);
    if (e0 != cudaSuccess || maxc < 2 * G) {
      cudaGetLastError();
      delete s;
      return set_error(c, HS_E_CUDA, "no schedulable cluster for the sweep kernel");
    }
    s->max_fronts = std::max(1, std::min(kMaxFront, maxc / G));
  }
  s->q = (s->mmax - 1) / (1 << s->L) + 1;
  {   // level-0 kept updates from the sparse couplings: opt-in (HS_SWEEP_CPL0=1).
      // 14% fewer streamed bytes at C3 but measured 2.5% slower (the extra
      // phase barrier and the coupling loads sit on the critical path), so
      // the streamed alpha / gamma blocks stay the default (DESIGN 5.1)
    int mmin = M;
    for (int k = 0; k < NCH; ++k) mmin = std::min(mmin, s->y0s[k + 1] - s->y0s[k]);
    const char* ev = getenv("HS_SWEEP_CPL0");
    s->cpl0 = s->L >= 1 && mmin >= 2 && ev && atoi(ev) == 1 ? 1 : 0;
  }
  if (s->L >= kMaxLevels || itab_len(s->mmax) > kMaxItems) {
    delete s;
    return set_error(c, HS_E_SHAPE, "face too long for the sweep's chunking");
  }
  Chunks g = make_chunks(s);
  s->kstride = g.kstride;
  const int B = C - 1;
  cudaError_t e = cudaSuccess;

  const int ntin = std::max(4, build_schedule(s, J, beta, bt, lo, hi));   // >= 4: sweep_solve_one
  s->ntrace = ntin;
  std::vector<SweepTask>& T = s->tasks;

  // ---- rows of each slab's solution the chain ever reads (outputs, traces):
  // the last back-substitution level and the spike correction only update
  // those (<= kNR rows; otherwise the slab keeps the full update)
  {
    std::vector<std::vector<int>> rows(J);
    for (const SweepTask& t : T) {
      auto& rs = rows[t.slab];
      for (int x = t.ta + 1 - t.lo; x < t.tb + 1 - t.lo; ++x) rs.push_back(x);
      if (t.out2 >= 0) { rs.push_back(t.orow2); rs.push_back(t.orow2 + 1); }
      if (t.out4 >= 0) { rs.push_back(t.orow4); rs.push_back(t.orow4 + 1); }
    }
    bool fits = TM == 16 && HS_SWEEP_HALF == 0;
    std::vector<int> rr((size_t)J * kNR, 0);
    for (int j = 0; j < J && fits; ++j) {
      auto& rs = rows[j];
      std::sort(rs.begin(), rs.end());
      rs.erase(std::unique(rs.begin(), rs.end()), rs.end());
      if (rs.empty()) rs.push_back(0);
      if ((int)rs.size() > kNR) fits = false;
      for (int i = 0; i < kNR; ++i) rr[(size_t)j * kNR + i] = rs[std::min(i, (int)rs.size() - 1)];
    }
    s->nr = fits ? kNR : 0;
    g.nr = s->nr;
    if (fits) s->hrows = rr;
    if (fits) {
      e = cudaMalloc((void**)&s->rows, rr.size() * sizeof(int));
      if (e == cudaSuccess)
        e = cudaMemcpy(s->rows, rr.data(), rr.size() * sizeof(int), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        sweep_destroy(s);
        return check_cuda(c, e, "row sets");
      }
    }
  }
  {   // algorithmic bytes of every solve launch (profiler): exactly the streamed blocks
    double rec_blocks = 0;
    for (int k = 0; k < NCH; ++k)
      rec_blocks += TM == 16 ? stream_blocks<16>(g, k) : stream_blocks<32>(g, k);
    // + the level-0 couplings read once per kept point (g.cpl0)
    const double rec_bytes = rec_blocks * TM2 * 16.0;
    s->rec_bytes = rec_bytes;
    for (auto& plan : s->plan) plan_bytes(s, plan);
  }

  const size_t efb = (size_t)J * M * TM2 * sizeof(double2);
  const size_t krb = (size_t)J * NCH * g.kstride * 2 * TM2 * sizeof(double2);
  const size_t rkb = (size_t)J * NCH * std::max(1, 2 * B) * 2 * TM2 * sizeof(double2);
  const size_t qdb = (size_t)J * NCH * s->q * s->q * TM2 * sizeof(double2);
  s->factor_bytes = (long long)(efb * 5 + krb + qdb + (B > 0 ? rkb : 0));
  if (s->cpl0) {   // level-0 couplings: 6 TM values per face point and slab
    const size_t cb = (size_t)J * M * TM2 * sizeof(double2);   // (packing only)
    e = cudaMalloc((void**)&s->cpl, cb);
    if (e == cudaSuccess) e = cudaMemset(s->cpl, 0, cb);
    if (e != cudaSuccess) {
      sweep_destroy(s);
      return check_cuda(c, e, "coupling alloc");
    }
    s->factor_bytes += (long long)cb;
  }
  e = cudaMalloc((void**)&s->ef, efb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->eb, 2 * efb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->kr, krb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->sp, 2 * efb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->rk, rkb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->qd, qdb);
  if (e != cudaSuccess) {
    sweep_destroy(s);
    return check_cuda(c, e, "factor alloc");
  }
  int r = TM == 16 ? factorize<16>(c, s, info, g) : factorize<32>(c, s, info, g);
  if (r) {
    sweep_destroy(s);
    return r;
  }
  {   // the solve kernel's per-rank item / chunk tables
    const int pw = plan_words(s->mmax);
    std::vector<uint32_t> hp((size_t)NCH * pw, 0u);
    for (int k = 0; k < NCH; ++k) {
      if (TM == 16) chunk_plan<16>(g, k, s->mmax, hp.data() + (size_t)k * pw);
      else chunk_plan<32>(g, k, s->mmax, hp.data() + (size_t)k * pw);
    }
    e = cudaMalloc((void**)&s->ptab, hp.size() * sizeof(uint32_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(s->ptab, hp.data(), hp.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      sweep_destroy(s);
      return check_cuda(c, e, "plan upload");
    }
  }

  const size_t tb = T.size() * sizeof(SweepTask);
  e = cudaMalloc((void**)&s->d_tasks, tb);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_tasks, T.data(), tb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMalloc((void**)&s->trace, (size_t)std::max(1, ntin) * 2 * M * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->g, (size_t)s->n0 * M * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->u2, (size_t)s->n0 * M * sizeof(double2));
  if (e == cudaSuccess) e = alloc_exchange(&s->own);
  if (e != cudaSuccess) {
    sweep_destroy(s);
    return check_cuda(c, e, "sweep buffers");
  }
  s->own.trace = s->trace;
  s->own.g = s->g;
  s->own.u2 = s->u2;
  *out = s;
  return HS_OK;
}

// Relay emulation of a sweep-axis shard layout:
// the X plan with every front cut where its slabs pass from one shard's
// range to the next (slab j on shard (j-1) G / J), one launch per shard
// step, the traces crossing a cut through the trace buffers -- the
// critical path of a relay whose shards own their slabs, without the P2P
// hop.  Same tasks, same results as the X plan.
static std::vector<SweepLaunch> build_relay(Sweep* s, int G, int* ntin) {
  const int J = s->J;
  SchedBuilder b{s, J, s->hbeta.data(), s->hbt.data(), s->hlo.data(), s->hhi.data()};
  auto shard = [&](const SweepTask& t) { return (int)((int64_t)t.slab * G / J); };
  auto runs = [&](const std::vector<SweepTask>& v) {
    std::vector<std::vector<SweepTask>> r;
    for (const SweepTask& t : v) {
      if (r.empty() || shard(r.back().back()) != shard(t)) r.emplace_back();
      r.back().push_back(t);
    }
    return r;
  };
  auto zip = [&](const std::vector<std::vector<SweepTask>>& a,
                 const std::vector<std::vector<SweepTask>>& c2) {
    std::vector<std::vector<std::vector<SweepTask>>> st;
    for (size_t k = 0; k < std::max(a.size(), c2.size()); ++k) {
      std::vector<std::vector<SweepTask>> fr;
      if (k < a.size()) fr.push_back(a[k]);
      if (k < c2.size()) fr.push_back(c2[k]);
      st.push_back(fr);
    }
    return st;
  };
  std::vector<SweepLaunch> plan;
  const int jm = J / 2 + 1;
  std::vector<SweepTask> F = b.fwd_chain(1, jm - 1), Bk = b.bwd_chain(J, jm + 1);
  SweepTask mi = b.mid_in(jm);
  const int in1 = b.want1(mi), in3 = b.want3(mi);
  if (!F.empty()) b.give2(F.back(), in1);
  if (!Bk.empty()) b.give4(Bk.back(), in3);
  auto st1 = zip(runs(F), runs(Bk));
  st1.push_back({{mi}});
  b.emit(plan, 0, st1);
  plan.push_back(SweepLaunch{SweepLaunch::kResidual});
  SweepTask mo = b.mid_out(jm);
  std::vector<SweepTask> BB = b.bwd_chain(jm - 1, 1), FF = b.fwd_chain(jm + 1, J);
  if (!FF.empty()) b.give2(mo, FF.front().tin1);
  if (!BB.empty()) b.give4(mo, BB.front().tin3);
  // the middle solve heads both outward fronts (as in the X plan): it joins
  // each front's first run, whichever shard the run's slabs are on
  auto headed = [&](const std::vector<SweepTask>& v) {
    std::vector<std::vector<SweepTask>> r = runs(v);
    if (r.empty()) r.emplace_back();
    r[0].insert(r[0].begin(), mo);
    return r;
  };
  b.emit(plan, 1, zip(headed(BB), headed(FF)));
  plan.push_back(SweepLaunch{SweepLaunch::kCombine});
  *ntin = b.ntin;
  return plan;
}

static int register_plan(Ctx* c, Sweep* s, std::vector<SweepLaunch>&& plan, size_t t0, int* variant) {
  plan_bytes(s, plan);
  if (!s->s3) {   // re-upload the task list (the plan indexes it)
    SweepTask* d = nullptr;
    const size_t tb = s->tasks.size() * sizeof(SweepTask);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = cudaMalloc((void**)&d, tb);
    if (e == cudaSuccess) e = cudaMemcpy(d, s->tasks.data(), tb, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(d);
      s->tasks.resize(t0);
      return check_cuda(c, e, "task upload");
    }
    cudaFree(s->d_tasks);
    s->d_tasks = d;
  }
  s->plan.push_back(std::move(plan));
  *variant = (int)s->plan.size() - 1;
  return HS_OK;
}

int sweep_plan_relay(Ctx* c, Sweep* s, int shards, int* variant) {
  if (s->J % 2) return set_error(c, HS_E_SHAPE, "X-sweep needs an even subdomain count");
  if (shards < 1 || shards > s->J) return set_error(c, HS_E_SHAPE, "shards must be in [1, J]");
  const size_t t0 = s->tasks.size();
  int ntin = 0;
  std::vector<SweepLaunch> plan = build_relay(s, shards, &ntin);
  if (ntin > std::max(1, s->ntrace) || s->tasks.size() > (size_t)kMaxTasks * 64) {
    s->tasks.resize(t0);
    return set_error(c, HS_E_SHAPE, "relay plan does not fit the sweep's buffers");
  }
  return register_plan(c, s, std::move(plan), t0, variant);
}

int sweep_plan_nx(Ctx* c, Sweep* s, int ncell, const int64_t* jc, const int64_t* jm,
                  int* variant) {
  const int J = s->J;
  // NxCells.validate (sweepdd.py:376-390)
  if (ncell < 1 || jc[0] != -1 || jc[ncell] != J + 1)
    return set_error(c, HS_E_SHAPE, "cell boundaries must start at -1 and end at J+1");
  for (int i = 0; i < ncell; ++i)
    if (jc[i] >= jc[i + 1]) return set_error(c, HS_E_SHAPE, "cell boundaries must be strictly increasing");
  for (int m = 1; m <= ncell; ++m) {
    const int64_t lo = std::max<int64_t>(1, jc[m - 1] + 1), hi = std::min<int64_t>(J, jc[m] - 1);
    if (jm[m - 1] < lo || jm[m - 1] > hi) {
      char buf[128];
      snprintf(buf, sizeof buf, "cell %d: meeting slab %lld outside [%lld,%lld]", m,
               (long long)jm[m - 1], (long long)lo, (long long)hi);
      return set_error(c, HS_E_SHAPE, buf);
    }
  }
  const size_t t0 = s->tasks.size();
  int ntin = 0;
  std::vector<SweepLaunch> plan = build_nx(s, ncell, jc, jm, &ntin);
  auto undo = [&](int rc) {
    s->tasks.resize(t0);
    return rc;
  };
  if (ntin > std::max(1, s->ntrace))
    return undo(set_error(c, HS_E_SHAPE, "NX cells need more trace buffers than the sweep has"));
  if (!s->s3 && s->nr) {   // every row the NX tasks read must be in the slab's restricted set
    for (size_t i = t0; i < s->tasks.size(); ++i) {
      const SweepTask& t = s->tasks[i];
      const int* rs = s->hrows.data() + (size_t)t.slab * kNR;
      auto has = [&](int x) { return std::find(rs, rs + kNR, x) != rs + kNR; };
      bool ok = true;
      for (int x = t.ta + 1 - t.lo; x < t.tb + 1 - t.lo; ++x) ok = ok && has(x);
      if (t.out2 >= 0) ok = ok && has(t.orow2) && has(t.orow2 + 1);
      if (t.out4 >= 0) ok = ok && has(t.orow4) && has(t.orow4 + 1);
      if (!ok) return undo(set_error(c, HS_E_SHAPE, "NX cells read slab rows outside the sweep's row sets"));
    }
  }
  if (s->tasks.size() > (size_t)kMaxTasks * 64)
    return undo(set_error(c, HS_E_SHAPE, "too many NX plans on one sweep"));
  return register_plan(c, s, std::move(plan), t0, variant);
}

void sweep_destroy(Sweep* s) {
  if (s) sweep3_destroy(s->s3);
  if (!s) return;
  delete s->view;
  cudaFree(s->cpl);
  cudaFree(s->ef);
  cudaFree(s->eb);
  cudaFree(s->kr);
  cudaFree(s->sp);
  cudaFree(s->rk);
  cudaFree(s->qd);
  cudaFree(s->stream);
  cudaFree(s->ptab);
  cudaFree(s->rows);
  cudaFree(s->ebr);
  cudaFree(s->spr);
  cudaFree(s->trace);
  cudaFree(s->g);
  cudaFree(s->u2);
  cudaFree(s->d_tasks);
  cudaFree(s->x2);
  cudaFree(s->own.xbuf);
  cudaFree(s->own.xflag);
  if (s->batch.trace) sweep_work_destroy(&s->batch);
  delete s;
}

__global__ void k_add_rows(double2* __restrict__ u, const double2* __restrict__ v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[i] = cadd(u[i], __ldg(v + i));
}

// One slab solve outside a schedule (subdom_solve, sweepdd.py:236-268):
// right-hand side rows [a, b) of f plus the transmission of the given input
// traces, solution rows [ta, tb) ADDED into u, outgoing traces on request.
int sweep_solve_one(Ctx* c, Sweep* s, int j, int64_t a, int64_t b, int64_t ta, int64_t tb,
                    const double2* B1, const double2* B3, double2* out2, double2* out4,
                    const double2* f, double2* u) {
  const int J = s->J, M = s->M;
  if (j < 1 || j > J) return set_error(c, HS_E_SHAPE, "slab index out of range");
  const int64_t lo = s->hlo[j - 1], hi = s->hhi[j - 1];
  // rows must lie inside the slab's layers lo..hi (1-based points -> rows lo-1..hi-1)
  if (a < lo - 1 || b > hi || a > b || ta < lo - 1 || tb > hi || ta > tb)
    return set_error(c, HS_E_SHAPE, "rows outside the slab");
  SweepTask t{};
  t.slab = j - 1;
  t.lo = (int)lo;
  t.T = (int)(hi - lo + 1);
  t.a = (int)a;
  t.b = (int)b;
  t.ta = (int)ta;
  t.tb = (int)tb;
  t.tin1 = t.tin3 = t.out2 = t.out4 = -1;
  t.row1 = t.row3 = t.orow2 = t.orow4 = -1;
  t.dst = 1;
  const size_t tr = (size_t)2 * M * sizeof(double2);
  if (B1 && j > 1) {
    t.tin1 = 0;
    t.row1 = (int)s->hbeta[j - 1] - t.lo;
    HS_CUDA(c, cudaMemcpyAsync(s->trace, B1, tr, cudaMemcpyDeviceToDevice, c->stream), "trace in");
  }
  if (B3 && j < J) {
    t.tin3 = 1;
    t.row3 = (int)s->hbt[j] - t.lo;
    HS_CUDA(c, cudaMemcpyAsync(s->trace + 2 * M, B3, tr, cudaMemcpyDeviceToDevice, c->stream),
            "trace in");
  }
  if (out2 && j < J) {
    t.out2 = 2;
    t.orow2 = (int)s->hbeta[j] - t.lo;
  }
  if (out4 && j > 1) {
    t.out4 = 3;
    t.orow4 = (int)s->hbt[j - 1] - t.lo;
  }
  if (!s->s3 && s->nr) {   // the restricted updates compute the chain's rows only
    const int* rs = s->hrows.data() + (size_t)t.slab * kNR;
    auto has = [&](int x) { return std::find(rs, rs + kNR, x) != rs + kNR; };
    bool ok = true;
    for (int x = t.ta + 1 - t.lo; x < t.tb + 1 - t.lo; ++x) ok = ok && has(x);
    if (t.out2 >= 0) ok = ok && has(t.orow2) && has(t.orow2 + 1);
    if (t.out4 >= 0) ok = ok && has(t.orow4) && has(t.orow4 + 1);
    if (!ok)
      return set_error(c, HS_E_SHAPE,
                       "solution rows outside the sweep's row sets (the device slab solve "
                       "computes the rows its schedules read)");
  }
  if (s->s3) {
    const SweepTask* ts[1] = {&t};
    double2* us[2] = {s->u2, s->u2};
    if (int r = sweep3_tasks(c, s, ts, 1, f, us, s->coarse->d.coeffs, s->coarse->d.n)) return r;
  } else {
    SweepTask* dt = (SweepTask*)scratch(c, sizeof(SweepTask), 3);
    if (!dt) return set_error(c, HS_E_CUDA, "scratch allocation failed");
    HS_CUDA(c, cudaMemcpyAsync(dt, &t, sizeof(SweepTask), cudaMemcpyHostToDevice, c->stream),
            "task upload");
    SolveArgs g{};
    g.tasks = dt;
    g.ffirst[0] = 0;
    g.fcount[0] = 1;
    g.g = make_chunks(s);
    g.stream = s->stream;
    g.nbs = s->nbs;
    g.plan = s->ptab;
    g.rows = s->rows;
    g.cpl = s->cpl;
    g.src = f;
    g.coarse = s->coarse->d.coeffs;
    g.ncoarse = s->coarse->d.n;
    if (int r = slot_table(s->coarse, g.cslot, c)) return r;
    g.trace = s->trace;
    g.u[0] = s->u2;
    g.u[1] = s->u2;
    g.xbuf = s->own.xbuf;
    g.xflag = s->own.xflag;
    for (int i = 0; i < kMaxFront; ++i) g.xbase[i] = s->own.xcount[i];
    ProfScope ps(c, K_SWEEP_FRONT, s->rec_bytes);
    cudaError_t e = launch_solve(s->tm, 1, s->C, s->G, s->mmax, c->stream, g);
    if (e != cudaSuccess) return check_cuda(c, e, "slab solve launch");
    s->own.xcount[0] += 1;
    HS_LAUNCH_CHECK(c, "slab solve kernel");
  }
  const int64_t n = (tb - ta) * (int64_t)M;
  if (n > 0) {
    k_add_rows<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(u + ta * M, s->u2 + ta * M, n);
    HS_LAUNCH_CHECK(c, "row scatter");
  }
  if (t.out2 >= 0)
    HS_CUDA(c, cudaMemcpyAsync(out2, s->trace + 4 * M, tr, cudaMemcpyDeviceToDevice, c->stream),
            "trace out");
  if (t.out4 >= 0)
    HS_CUDA(c, cudaMemcpyAsync(out4, s->trace + 6 * M, tr, cudaMemcpyDeviceToDevice, c->stream),
            "trace out");
  return HS_OK;
}

int sweep_work_create(Ctx* c, const Sweep* s, SweepWork* w, int nrhs, bool batch) {
  // (3-D levels: a batch's work set only -- their solve uses every SM, so no lanes)
  if (s->s3 && !batch)
    return set_error(c, HS_E_ARG, "sweep lanes need a 2-D level (the 3-D solve uses every SM)");
  if (nrhs < 1) return set_error(c, HS_E_ARG, "a work set holds at least one right-hand side");
  *w = SweepWork{};
  w->nrhs = nrhs;
  const size_t nf = (size_t)nrhs * s->n0 * s->M * sizeof(double2);
  cudaError_t e = cudaMalloc((void**)&w->trace,
                             (size_t)nrhs * std::max(1, s->ntrace) * 2 * s->M * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&w->g, nf);
  if (e == cudaSuccess) e = cudaMalloc((void**)&w->u2, nf);
  if (e == cudaSuccess) e = alloc_exchange(w, nrhs);
  if (e != cudaSuccess) {
    sweep_work_destroy(w);
    return check_cuda(c, e, "sweep work buffers");
  }
  return HS_OK;
}

void sweep_work_destroy(SweepWork* w) {
  cudaFree(w->trace);
  cudaFree(w->g);
  cudaFree(w->u2);
  cudaFree(w->xbuf);
  cudaFree(w->xflag);
  *w = SweepWork{};
}

// nr right-hand sides (f + r * stride -> u + r * stride) through the plan's
// launches; nr > 1 needs a work set of at least nr and a 2-D level
static int sweep_apply_nr(Ctx* c, Sweep* s, int variant, const double2* f, double2* u,
                          const SweepWork* w, int first, int last, int nr, int64_t stride);

int sweep_apply(Ctx* c, Sweep* s, int variant, const double2* f, double2* u,
                const SweepWork* w, int first, int last) {
  return sweep_apply_nr(c, s, variant, f, u, w, first, last, 1, 0);
}

int sweep_apply_many(Ctx* c, Sweep* s, int variant, int nrhs, const double2* f, double2* u,
                     int64_t stride, const SweepWork* w) {
  if (nrhs < 1) return set_error(c, HS_E_ARG, "nrhs must be at least 1");
  if (nrhs > 1 && stride < (int64_t)s->n0 * s->M)
    return set_error(c, HS_E_ARG, "right-hand-side stride shorter than a vector");
  int width = s->max_nr;
  if (w) {   // a lane's work set: as wide as it was created
    width = std::min(width, w->nrhs);
  } else if (width > 1 && nrhs > 1) {
    if (s->batch.nrhs < width || !s->batch.trace) {
      if (s->batch.trace) sweep_work_destroy(&s->batch);
      if (int r = sweep_work_create(c, s, &s->batch, width, true)) return r;
    }
    w = &s->batch;
  }
  for (int done = 0; done < nrhs;) {
    int nr = 1;
    while (nr * 2 <= width && done + nr * 2 <= nrhs) nr *= 2;
    // (a single right-hand side of the sweep's own stream: its own work set)
    if (int r = sweep_apply_nr(c, s, variant, f + done * stride, u + done * stride,
                               nr > 1 || (w && w != &s->batch) ? w : nullptr, 0, -1, nr, stride))
      return r;
    done += nr;
  }
  return HS_OK;
}

static int sweep_apply_nr(Ctx* c, Sweep* s, int variant, const double2* f, double2* u,
                          const SweepWork* w, int first, int last, int nr, int64_t stride) {
  if (!w) w = &s->own;
  if (nr > 1 && (w->nrhs < nr || nr > s->max_nr))
    return set_error(c, HS_E_ARG, "multi-right-hand-side sweep: unsupported level or work set");
  const int64_t nlev = (int64_t)s->n0 * s->M;   // stride of the work set's g / u2
  if (!s->has_plan(variant))
    return set_error(c, HS_E_ARG,
                     variant == HS_VARIANT_X ? "X-sweep needs an even subdomain count"
                                             : "unknown sweep variant");
  const int M = s->M;
  const int np_ = (int)s->plan[variant].size();
  if (last < 0 || last > np_) last = np_;
  for (int li = std::max(0, first); li < last; ++li) {
    const SweepLaunch& Lh = s->plan[variant][li];
    switch (Lh.kind) {
      case SweepLaunch::kCombine: {
        // u = u_pass1 + u_pass2 (the order of the reference's u[ta:tb] += ud)
        const int64_t n = (int64_t)s->n0 * M;
        for (int rh = 0; rh < nr; ++rh) {
          ProfScope ps(c, K_SWEEP_GATHER, 48.0 * n);
          k_combine<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(u + rh * stride,
                                                                          w->u2 + rh * nlev, n);
          HS_LAUNCH_CHECK(c, "combine kernel");
        }
        break;
      }
      case SweepLaunch::kResidual: {
        for (int rh = 0; rh < nr; ++rh) {
          int r = stencil_apply(c, s->coarse, u + rh * stride, w->g + rh * nlev, 1, f + rh * stride);
          if (r) return r;
        }
        break;
      }
      case SweepLaunch::kSolve: {
        if (s->s3) {   // 3-D: the fronts' slab solves in order (host-driven block LU;
                       // sweep3_tasks attributes the GEMV and chain kernels itself)
          double2* us[2] = {u, w->u2};
          Sweep3Rhs mr{nr, Lh.src ? nlev : stride, {stride, nlev},
                       (int64_t)std::max(1, s->ntrace) * 2 * M, w->trace};
          // fronts zipped in pairs (two chains per launch); a task identical
          // to one already run in this launch (a solve heading two fronts)
          // is not repeated -- its outputs are already in place
          std::vector<const SweepTask*> done;
          auto ran = [&](const SweepTask* t, size_t upto) {
            for (size_t k = 0; k < upto; ++k)
              if (!memcmp(done[k], t, sizeof(SweepTask))) return true;
            return false;
          };
          for (int fr = 0; fr < Lh.nfront; fr += 2) {
            std::vector<const SweepTask*> q[2];
            for (int h = 0; h < 2 && fr + h < Lh.nfront; ++h)
              for (int i = Lh.ffirst[fr + h]; i < Lh.ffirst[fr + h] + Lh.fcount[fr + h]; ++i)
                q[h].push_back(&s->tasks[i]);
            size_t p0 = 0, p1 = 0;
            while (p0 < q[0].size() || p1 < q[1].size()) {
              const size_t before = done.size();
              const SweepTask* ts[2];
              int nt = 0;
              while (p0 < q[0].size() && ran(q[0][p0], before)) ++p0;
              while (p1 < q[1].size() && ran(q[1][p1], before)) ++p1;
              if (p0 < q[0].size()) ts[nt++] = q[0][p0++];
              if (p1 < q[1].size()) {
                // the same solve heading both fronts runs once; the second
                // front's next task depends on it, so it waits a launch
                if (nt && !memcmp(ts[0], q[1][p1], sizeof(SweepTask))) ++p1;
                else ts[nt++] = q[1][p1++];
              }
              for (int k = 0; k < nt; ++k) done.push_back(ts[k]);
              if (nt) {
                const int r2 = sweep3_tasks(c, s, ts, nt, Lh.src ? w->g : f, us,
                                            s->coarse->d.coeffs, s->coarse->d.n, &mr);
                if (r2) return r2;
              }
            }
          }
          break;
        }
        SolveArgs a{};
        a.tasks = s->d_tasks;
        for (int i = 0; i < kMaxFront; ++i) {
          a.ffirst[i] = i < Lh.nfront ? Lh.ffirst[i] : 0;
          a.fcount[i] = i < Lh.nfront ? Lh.fcount[i] : 0;
        }
        a.g = make_chunks(s);
        a.stream = s->stream;
        a.nbs = s->nbs;
        a.plan = s->ptab;
        a.rows = s->rows;
        a.cpl = s->cpl;
        a.src = Lh.src ? w->g : f;
        a.coarse = s->coarse->d.coeffs;
        a.ncoarse = s->coarse->d.n;
        if (int r = slot_table(s->coarse, a.cslot, c)) return r;
        a.trace = w->trace;
        a.u[0] = u;
        a.u[1] = w->u2;
        a.xbuf = w->xbuf;
        a.xflag = w->xflag;
        for (int i = 0; i < kMaxFront; ++i) a.xbase[i] = w->xcount[i];
        a.vs_src = Lh.src ? nlev : stride;
        a.vs_u[0] = stride;
        a.vs_u[1] = nlev;
        a.ts = (int64_t)std::max(1, s->ntrace) * 2 * M;
        a.xs = kXStride;
        static const char* trace_path = getenv("HS_SWEEP_TRACE");
        static bool traced = false;
        unsigned long long* dbg = nullptr;
        static const int trace_nr = getenv("HS_SWEEP_TRACE_NR") ? atoi(getenv("HS_SWEEP_TRACE_NR")) : 1;
        if (trace_path && !traced && Lh.nfront == 2 && nr == trace_nr) {
          cudaMalloc((void**)&dbg, 16 * 1024 * sizeof(unsigned long long));
          cudaMemsetAsync(dbg, 0, 16 * 1024 * sizeof(unsigned long long), c->stream);
        }
        a.dbg = dbg;
        // (profiler: SURVEY 8(d)'s bytes per slab solve x the slab solves of the
        // launch -- nr right-hand sides are nr solves of every slab)
        ProfScope ps(c, K_SWEEP_FRONT, Lh.bytes * nr);
        cudaError_t e = launch_solve(s->tm, nr, s->C, Lh.nfront * s->G, s->mmax, c->stream, a);
        if (e != cudaSuccess) return check_cuda(c, e, "sweep solve launch");
        for (int i = 0; i < Lh.nfront; ++i)   // level-2 counters advance by the fronts' tasks
          const_cast<SweepWork*>(w)->xcount[i] += (unsigned)Lh.fcount[i];
        HS_LAUNCH_CHECK(c, "sweep solve kernel");
        if (dbg) {
          std::vector<unsigned long long> h(16 * 1024);
          cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, c->stream);
          cudaStreamSynchronize(c->stream);
          cudaFree(dbg);
          traced = true;
          if (FILE* fp = fopen(trace_path, "w")) {
            // per CTA of cluster 0 (task 1): [0] start, [1] rhs, [2+p] local phase p,
            // [40] tips barrier, [41] interface solve, [63] end (ns after CTA 0 start)
            fprintf(fp, "# C=%d M=%d L=%d q=%d\n", s->C, M, s->L, s->q);
            const unsigned long long t0 = h[0];
            for (int b = 0; b < std::min(16, s->C); ++b) {
              for (int k = 0; k < 1024; ++k)
                fprintf(fp, "%lld ", h[b * 1024 + k] ? (long long)(h[b * 1024 + k] - t0) : -1LL);
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
