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
#ifndef HS_SWEEP_PREFETCH
#define HS_SWEEP_PREFETCH 0
#endif
#ifndef HS_SWEEP_HALF      // tm 16: one ring item per half warp
#define HS_SWEEP_HALF 0
#endif
#ifndef HS_SWEEP_L2NEXT    // producer prefetches each item of the next slab into L2
#define HS_SWEEP_L2NEXT 0
#endif
constexpr int kMaxC = 16;
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

// chunk geometry: chunk k covers face points [k M / C, (k+1) M / C)
struct Chunks {
  int M, C, L, kstride;
  int q;                   // dense top: blocks per chunk left after L levels
  int koff[kMaxLevels];
  __host__ __device__ int y0(int k) const { return (int)((int64_t)k * M / C); }
  __host__ __device__ int len(int k) const { return y0(k + 1) - y0(k); }
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
  const int k = (int)(((int64_t)(y + 1) * g.C - 1) / M);
  if (y == g.y0(k)) {
    EL[((int64_t)s * g.C + k) * TM2 + r * TM + c] = l;
    l = czero();
  }
  if (y == g.y0(k + 1) - 1) {
    EU[((int64_t)s * g.C + k) * TM2 + r * TM + c] = u;
    u = czero();
  }
  Lc[off] = l;
  Uc[off] = u;
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
  const int slab = blockIdx.y / g.C, k = blockIdx.y % g.C;
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
  const int slab = blockIdx.y / g.C, k = blockIdx.y % g.C;
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
  double2* kout = kr + (((int64_t)slab * g.C + k) * g.kstride + g.koff[level] + j) * 2 * TM2;
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
  const int slab = blockIdx.x / g.C, k = blockIdx.x % g.C, M = g.M;
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
  double2* out = qd + ((int64_t)slab * g.C + k) * Q * Q * TM2;
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
  const int slab = blockIdx.x / g.C, k = blockIdx.x % g.C, M = g.M;
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
  const double2* el = EL + ((int64_t)slab * g.C + k) * TM2;
  const double2* eu = EU + ((int64_t)slab * g.C + k) * TM2;
  double2* tp = tips + ((int64_t)slab * g.C + k) * 4 * TM2;
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

// Inverse of the interface system (one CTA per slab).  Unknowns per boundary
// b (between chunks b and b+1): xi_b = (alpha_b = x at the last point of chunk
// b, beta_b = x at the first point of chunk b+1); right-hand side
// tau_b = (g_b[last], g_{b+1}[first]):
//   alpha_b + Vb[last] beta_b + Wb[last] alpha_{b-1}            = g_b[last]
//   beta_b + W_{b+1}[first] alpha_b + V_{b+1}[first] beta_{b+1} = g_{b+1}[first]
// Block Thomas over b with identity right-hand sides gives R = S^{-1}; CTA k
// keeps rows alpha_{k-1} and beta_k, stored per column block q (tm columns) as
// 2tm x tm with the row index fastest.
template <int TM>
__global__ void __launch_bounds__(1024)
k_reduced(Chunks g, const double2* __restrict__ tips, double2* __restrict__ Gw,
          double2* __restrict__ Zr, double2* __restrict__ rk,
          unsigned long long* __restrict__ err) {
  constexpr int TM2 = Geo<TM>::TM2;
  constexpr int N = 2 * TM;
  const int slab = blockIdx.x, C = g.C, B = C - 1, NR = B * N;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2(*A)[N + 1] = reinterpret_cast<double2(*)[N + 1]>(smraw);
  double2(*Inv)[N + 1] = A + N;
  __shared__ int piv_row;
  __shared__ double piv_abs;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double2* tp = tips + (int64_t)slab * C * 4 * TM2;
  auto tip = [&](int k, int which, int r, int c) -> double2 {   // 0 Wf 1 Wl 2 Vf 3 Vl
    return tp[((int64_t)k * 4 + which) * TM2 + r * TM + c];
  };
  double2* G = Gw + (int64_t)slab * B * N * N;    // G_b = Dt_b^{-1} Up_b
  double2* Z = Zr + (int64_t)slab * NR * NR;      // block row b: rows b*N.., all NR columns
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
  // rows of CTA k: alpha_{k-1} (block k-1, rows 0..TM-1), beta_k (block k,
  // rows TM..2TM-1); column block q of tm columns
  for (int e = tid; e < C * N * NR; e += nt) {
    const int k = e / (N * NR), rem = e % (N * NR);
    const int r = rem / NR, col = rem % NR;
    double2 v = czero();
    if (r < TM && k > 0) v = Z[((int64_t)(k - 1) * N + r) * NR + col];
    if (r >= TM && k < B) v = Z[((int64_t)k * N + r) * NR + col];
    const int q = col / TM, cq = col % TM;
    rk[(((int64_t)slab * C + k) * (2 * B) + q) * (2 * TM2) + cq * N + r] = v;
  }
}

// ---------------------------------------------------------------------------
// apply

struct SolveArgs {
  const SweepTask* tasks;
  int ffirst[2], fcount[2];
  Chunks g;
  int nslot;
  const double2* ef;
  const double2* eb;
  const double2* kr;
  const double2* sp;
  const double2* rk;
  const double2* qd;
  const double2* src;      // right-hand side field (n0 x M)
  const double2* coarse;   // global coarse operator [S][n0*M] (transmission couplings)
  int64_t ncoarse;
  int cslot[3][3];
  double2* trace;          // [ntrace][2][M]
  double2* u[2];
  unsigned long long* dbg; // optional per-phase timestamps (HS_SWEEP_TRACE)
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
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  if (bytes)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// acc = A0 v0 + A1 v1 (either term may be absent); A lane-major in shared
// memory, v in shared memory; every lane returns row (lane % tm)
template <int TM>
__device__ __forceinline__ double2 mvs2(const double2* m0, const double2* v0, const double2* m1,
                                        const double2* v1, int lane) {
  constexpr int CPL = Geo<TM>::CPL;
  const int hh = lane / TM;
  double2 a0 = czero(), a1 = czero();
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
      a0 = cfma(m1[k * 32 + lane], v1[CPL * hh + k], a0);
      a1 = cfma(m1[(k + 1) * 32 + lane], v1[CPL * hh + k + 1], a1);
    }
  }
  double2 acc = cadd(a0, a1);
  if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
  return acc;
}

// items of one chunk solve: <= 3m + 2L local, 2(C-1) R blocks, m spike blocks
__host__ __device__ inline int itab_len(int mmax) { return 4 * mmax + 2 * kMaxLevels + 2 * kMaxC + 16; }

// Item copy descriptor: array (bits 29-31; 7 = none), double length (bit 28),
// offset in double2 from the array's slab base (bits 0-27).
enum ItemArray : uint32_t { kArrEf = 0, kArrEb = 1, kArrKr = 2, kArrRk = 3, kArrSp = 4, kArrQd = 5 };
__host__ __device__ constexpr uint32_t item_enc(uint32_t arr, int64_t off, bool dbl = false) {
  return (arr << 29) | (dbl ? (1u << 28) : 0u) | (uint32_t)off;
}
constexpr uint32_t kItemNone = 0xffffffffu;

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

template <int TM>
struct Ring {
  static constexpr int SLOT = 2 * Geo<TM>::TM2;   // double2 per slot (two blocks)
  // F, Yv vectors + tau + R partials + bookkeeping, then the ring
  static int fixed(int mmax) {
    return 2 * (mmax + 1) * TM * 16 + 4 * kMaxC * TM * 16 + 4 * TM * 16 + (kWarps + 1) * 2 * TM * 16 + 32 +
           (64 + kMaxTasks) * 4 + itab_len(mmax) * 8 + 384;
  }
  static int nslot(int mmax) {
    const int avail = 225 * 1024 - fixed(mmax);
    return std::max(2, std::min(48, avail / (SLOT * 16 + 16)));
  }
  static int smem(int mmax) { return fixed(mmax) + nslot(mmax) * (SLOT * 16 + 16); }
};

template <int TM>
__global__ void __launch_bounds__(kWarps * 32, 1) k_part_solve(SolveArgs a) {
  constexpr int TM2 = Geo<TM>::TM2;
  constexpr int SLOT = Ring<TM>::SLOT;
  constexpr int YPW = 32 / TM;   // face points per warp pass in row-wise loops
  constexpr int N2 = 2 * TM;     // interface unknowns per chunk (alpha, beta)
  cg::cluster_group cl = cg::this_cluster();
  const Chunks& g = a.g;
  const int C = g.C, M = g.M, L = g.L, B = C - 1;
  const int rank = (int)cl.block_rank();
  const int front = blockIdx.x / C;
  const int Y0 = g.y0(rank), Y1 = g.y0(rank + 1);
  const int m = Y1 - Y0;
  const int mmax = (M + C - 1) / C;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int x = lane % TM, hh = lane / TM;
  constexpr int HW = (TM == 16 && HS_SWEEP_HALF) ? 2 : 1;   // items per warp pass
  const int sub = HW == 2 ? hh : 0;      // this lane's item within the pass
  const bool wr = HW == 2 || hh == 0;    // lane owns the result row it computed
  const int NS = a.nslot;
  extern __shared__ __align__(128) double2 sm[];
  double2* F = sm;                                  // [mmax+1][TM] rhs / reduced rhs
  double2* Yv = F + (mmax + 1) * TM;                // [mmax+1][TM] Dinv f, then x
  double2* tau2 = Yv + (mmax + 1) * TM;             // [2][2 kMaxC][TM] interface rhs (by task parity)
  double2* halo2 = tau2 + 4 * kMaxC * TM;           // [2][2][TM] neighbours' edge blocks of x
  double2* part = halo2 + 4 * TM;                   // [kWarps][2TM] R partial sums
  double2* ab = part + kWarps * N2;                 // [2TM] alpha_{k-1}, beta_k
  uint64_t* xbar = (uint64_t*)(ab + N2);            // [4] tips (2), halo (2) arrival barriers
  uint64_t* bars = xbar + 4;                        // [NS]
  volatile int* seq = (volatile int*)(bars + NS);   // [NS] item issued into a slot
  volatile int* done = seq + NS;                    // [NS] item consumed from a slot
  int* pfx = (int*)(bars + NS) + 2 * NS;            // [2L+3] items before each phase
  int* slabs = pfx + 64;                            // [fcount]
  uint2* itab = (uint2*)(slabs + kMaxTasks);        // [ITEMS] copy descriptors
  double2* ring = (double2*)(((uintptr_t)(itab + itab_len(mmax)) + 127) & ~(uintptr_t)127);

  auto cc = [&](int o0, int o1, int row, int y) -> double2 {
    const int sl = a.cslot[o0 + 1][o1 + 1];
    if (sl < 0 || y + o1 < 0 || y + o1 >= M) return czero();
    return __ldg(a.coarse + (int64_t)sl * a.ncoarse + (int64_t)row * M + y);
  };
  // transmission source into slab row p-lo (which 0) / p+1-lo (which 1)
  auto trans = [&](int buf, int p, int sign, int which, int y) -> double2 {
    const double2* Bt = a.trace + (int64_t)buf * 2 * M + (which == 0 ? M : 0);
    const int o0 = which == 0 ? 1 : -1;
    const int row = which == 0 ? p - 1 : p;
    double2 cv[3], bv[3];
#pragma unroll
    for (int o = -1; o <= 1; ++o) {   // all six loads in flight together
      const bool ok = y + o >= 0 && y + o < M;
      cv[o + 1] = ok ? cc(o0, o, row, y) : czero();
      bv[o + 1] = ok ? Bt[y + o] : czero();
    }
    double2 acc = cmul(cv[0], bv[0]);
    acc = cfma(cv[1], bv[1], acc);
    acc = cfma(cv[2], bv[2], acc);
    return cscale(which == 0 ? (double)sign : (double)-sign, acc);
  };

  // Item streams of one slab solve of this CTA: local phases (p < L forward
  // cyclic-reduction level p; p == L the dense top, items (row r, column pair
  // cp) of the level-L inverse; p > L back substitution of level 2L-p), then
  // the 2B column blocks of R, then the m spike blocks.
  const int NP = 2 * L + 1;
  const int S = 1 << L;
  const int qk = (m - 1) / S + 1;            // dense-top blocks of this chunk
  const int QP = (qk + 1) / 2;               // their column pairs
  auto ph_level = [&](int p) { return p <= L ? p : 2 * L - p; };
  auto ph_first = [&](int p) -> int { return p > L ? (1 << ph_level(p)) : 0; };
  auto ph_step = [&](int p) { return (p < L ? 1 : 2) << ph_level(p); };
  // face point of item j of a cyclic-reduction phase (forward phases list the
  // eliminated points first, so neighbouring items share a branch)
  auto item_yl = [&](int p, int j) -> int {
    if (p > L) return ph_first(p) + j * ph_step(p);
    const int ne = (pfx[p + 1] - pfx[p]) / 2;
    return (j < ne ? 2 * j + 1 : 2 * (j - ne)) << p;
  };
  const int ffirst = front ? a.ffirst[1] : a.ffirst[0];
  const int fcount = front ? a.fcount[1] : a.fcount[0];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int p = 0; p < NP; ++p) {
      pfx[p] = acc;
      const int f = ph_first(p);
      if (p == L) acc += qk * QP;
      else if (f < m) acc += (m - 1 - f) / ph_step(p) + 1;
    }
    pfx[NP] = acc;                               // R column blocks
    pfx[NP + 1] = acc + (B > 0 ? 2 * B : 0);     // spikes
    pfx[NP + 2] = pfx[NP + 1] + (B > 0 ? m : 0);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&bars[i], 1);
      seq[i] = -1;
      done[i] = i - NS;   // slot i is free for item i
    }
    for (int i = 0; i < 4; ++i) mbar_init(&xbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < fcount; i += blockDim.x) slabs[i] = a.tasks[ffirst + i].slab;
  cl.sync();   // every CTA's barriers initialised before any remote arrival
  const int ITEMS = pfx[NP + 2];
  const int total = fcount * ITEMS;
  const int64_t kbase = (int64_t)rank * g.kstride;
  if (ITEMS > itab_len(mmax)) __trap();   // bound of the descriptor table (host-sized)

  // Copy descriptors of one chunk solve (the same for every slab; offsets
  // relative to the slab's base in each factor array), built once.
  for (int r = threadIdx.x; r < ITEMS; r += blockDim.x) {
    int p = 0;
    while (pfx[p + 1] <= r) ++p;
    const int j = r - pfx[p];
    uint2 e = make_uint2(kItemNone, kItemNone);
    if (p == L) {           // dense top: blocks (r, 2cp) and (r, 2cp + 1)
      const int r = j / QP, c0 = 2 * (j % QP);
      e.x = item_enc(kArrQd, (((int64_t)rank * g.q + r) * g.q + c0) * TM2, c0 + 1 < qk);
    } else if (p < NP) {
      const int l = ph_level(p), s = 1 << l;
      const int yl = item_yl(p, j);
      const int y = Y0 + yl;
      if (p < L) {
        if ((yl >> l) & 1) {
          e.x = item_enc(kArrEf, (int64_t)y * TM2);
        } else {
          const int64_t k2 = (kbase + g.koff[l] + (yl >> (l + 1))) * 2 * TM2;
          if (yl - s >= 0) e.x = item_enc(kArrKr, k2);
          if (yl + s < m) e.y = item_enc(kArrKr, k2 + TM2);
        }
      } else {
        const int64_t e2 = (int64_t)y * 2 * TM2;
        if (yl - s >= 0) e.x = item_enc(kArrEb, e2);
        if (yl + s < m) e.y = item_enc(kArrEb, e2 + TM2);
      }
    } else if (p == NP) {   // R column block j
      e.x = item_enc(kArrRk, ((int64_t)rank * (2 * B) + j) * (2 * TM2), true);
    } else {                // spikes of block j
      e.x = item_enc(kArrSp, (int64_t)(Y0 + j) * 2 * TM2, true);
    }
    itab[r] = e;
  }
  __syncthreads();

  // producer state: the current task's slab base of every factor array
  const double2* sbase[6];
  auto slab_bases = [&](int slab, const double2** sb) {
    sb[kArrEf] = a.ef + (int64_t)slab * M * TM2;
    sb[kArrEb] = a.eb + (int64_t)slab * M * 2 * TM2;
    sb[kArrKr] = a.kr + (int64_t)slab * C * g.kstride * 2 * TM2;
    sb[kArrRk] = a.rk + (int64_t)slab * C * (2 * B) * 2 * TM2;
    sb[kArrSp] = a.sp + (int64_t)slab * M * 2 * TM2;
    sb[kArrQd] = a.qd + (int64_t)slab * C * g.q * g.q * TM2;
  };
  auto set_slab = [&](int slab) { slab_bases(slab, sbase); };
  auto src_of = [&](uint32_t e) -> const double2* {
    const uint32_t arr = e >> 29;
    const double2* b = arr == kArrEf ? sbase[0]
                       : arr == kArrEb ? sbase[1]
                       : arr == kArrKr ? sbase[2]
                       : arr == kArrRk ? sbase[3]
                       : arr == kArrSp ? sbase[4]
                                       : sbase[5];
    return b + (e & 0x0fffffffu);
  };
  const double2* nbase[6];   // next task's slab bases (L2 prefetch)
  auto issue = [&](int r, int sl, bool pf) {   // one lane: item r of the current task into slot sl
    const uint2 e = itab[r];
    if (HS_SWEEP_L2NEXT && pf) {   // the same item of the next slab into L2
      auto nsrc = [&](uint32_t q) {
        const uint32_t arr = q >> 29;
        const double2* b = arr == kArrEf ? nbase[0] : arr == kArrEb ? nbase[1]
                         : arr == kArrKr ? nbase[2] : arr == kArrRk ? nbase[3]
                         : arr == kArrSp ? nbase[4] : nbase[5];
        return b + (q & 0x0fffffffu);
      };
      constexpr uint32_t mb1 = TM2 * 16;
      if (e.x != kItemNone) prefetch_l2(nsrc(e.x), (e.x >> 28 & 1) ? 2 * mb1 : mb1);
      if (e.y != kItemNone) prefetch_l2(nsrc(e.y), mb1);
    }
    double2* slot = ring + sl * SLOT;
    uint64_t* bar = &bars[sl];
    constexpr uint32_t mb = TM2 * 16;
    if (e.x != kItemNone && (e.x >> 28 & 1)) {
      mbar_expect_tx(bar, 2 * mb);
      bulk_g2s(slot, src_of(e.x), 2 * mb, bar);
    } else {
      mbar_expect_tx(bar, (e.x != kItemNone ? mb : 0) + (e.y != kItemNone ? mb : 0));
      if (e.x != kItemNone) bulk_g2s(slot, src_of(e.x), mb, bar);
      if (e.y != kItemNone) bulk_g2s(slot + TM2, src_of(e.y), mb, bar);
    }
  };
  // optional instrumentation: task 1 timestamps kept in shared memory, dumped at exit
  __shared__ unsigned long long tsm[128];
  __shared__ unsigned long long tprod[128];   // producer: [spin start, issued] of task 1's first 64 items
  auto stamp = [&](int ti, int k) {
    if (a.dbg && threadIdx.x == 0 && ti == 1 && k < 64) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tsm[k] = tt;
    }
  };
  if (a.dbg && threadIdx.x == 0)
    for (int k = 0; k < 128; ++k) tsm[k] = tprod[k] = 0;
  auto stamp2 = [&](int ti, int p, int j, int k) {
    if (a.dbg && threadIdx.x == 0 && ti == 1 && j == 0 && p < 12) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tsm[64 + p * 5 + k] = tt;
    }
  };

  // consume item i: wait until issued into its slot (a parity wait is valid
  // only once the slot's previous occupant completed), then for the data
  int dbg_ti = 0, dbg_p = 0, dbg_j = 0;
  auto acquire = [&](int i) -> const double2* {
    stamp2(dbg_ti, dbg_p, dbg_j, 0);
    while (seq[i % NS] != i) {
    }
    stamp2(dbg_ti, dbg_p, dbg_j, 1);
    mbar_wait(&bars[i % NS], (uint32_t)((i / NS) & 1));
    stamp2(dbg_ti, dbg_p, dbg_j, 2);
    return ring + (i % NS) * SLOT;
  };
  // The warp's reads of the slot have returned (their values are consumed
  // before the __syncwarp), so the producer's async-proxy refill cannot race.
  auto release = [&](int i, bool has) {   // whole consumer warp, after its last read of the slot
    __syncwarp();
    if (has && lane % (32 / HW) == 0) done[i % NS] = i;
  };
  auto csync = [&]() {   // consumer warps only (the producer never joins)
    asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
  };

  if (warp == kCW) {
    // ---- TMA producer warp: issues every item in consumption order as soon
    // as its slot is free, prefetches the next slab into L2, and takes part in
    // the cluster barriers (arriving early: it never holds data others read).
    const int BW = max(1, min(8, NS / 2));   // items issued per batch (one lane each)
    int sl = 0;
    for (int ti = 0; ti < fcount; ++ti) {
      set_slab(slabs[ti]);
      const bool pf = ti + 1 < fcount;
      if (pf) slab_bases(slabs[ti + 1], nbase);
      if (HS_SWEEP_PREFETCH && lane == 0 && ti + 1 < fcount) {   // next slab's matrices into L2
        const int ns = slabs[ti + 1];
        prefetch_l2(a.ef + ((int64_t)ns * M + Y0) * TM2, (uint32_t)m * TM2 * 16);
        prefetch_l2(a.eb + ((int64_t)ns * M + Y0) * 2 * TM2, (uint32_t)m * 2 * TM2 * 16);
        prefetch_l2(a.kr + (((int64_t)ns * C) * g.kstride + kbase) * 2 * TM2,
                    (uint32_t)g.kstride * 2 * TM2 * 16);
        if (B > 0) {
          prefetch_l2(a.sp + ((int64_t)ns * M + Y0) * 2 * TM2, (uint32_t)m * 2 * TM2 * 16);
          prefetch_l2(a.rk + (((int64_t)ns * C + rank) * (2 * B)) * (2 * TM2),
                      (uint32_t)(2 * B) * 2 * TM2 * 16);
        }
      }
      // batches of up to BW items, one lane each
      const int base = ti * ITEMS;
      for (int r0 = 0; r0 < ITEMS;) {
        const int i0 = base + r0;
        const int cnt = min(BW, ITEMS - r0);
        if (lane < cnt) {
          const int i = i0 + lane;
          int sl_l = sl + lane;
          if (sl_l >= NS) sl_l -= NS;
          const int k = i - ITEMS;
          unsigned long long t0 = 0, t1 = 0;
          if (a.dbg && k >= 0 && k < 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          while (done[sl_l] != i - NS) {
          }
          issue(r0 + lane, sl_l, pf);
          seq[sl_l] = i;
          if (a.dbg && k >= 0 && k < 64) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            tprod[2 * k] = t0;
            tprod[2 * k + 1] = t1;
          }
        }
        sl += cnt;
        if (sl >= NS) sl -= NS;
        r0 += cnt;
        __syncwarp();
      }
    }
    cl.sync();   // matches the consumers' exit barrier
    return;
  }

  // Transmission from the previous task of this front without a trip through
  // global memory: its solution x is still in Yv (own face points) and the
  // neighbours' edge blocks arrive in halo (st.async + mbarrier).
  auto trans_local = [&](const double2* halo, int prow, int p, int sign, int which, int y) {
    const int o0 = which == 0 ? 1 : -1;
    const int row = which == 0 ? p - 1 : p;
    const int xr = prow + (which == 0 ? 1 : 0);   // trace row 1 feeds which 0, row 0 which 1
    double2 acc = czero();
#pragma unroll
    for (int o = -1; o <= 1; ++o) {
      if (y + o < 0 || y + o >= M) continue;
      const int yl = y + o - Y0;
      const double2 bv = yl < 0 ? halo[xr] : yl >= m ? halo[TM + xr] : Yv[yl * TM + xr];
      acc = cfma(cc(o0, o, row, y), bv, acc);
    }
    return cscale(which == 0 ? (double)sign : (double)-sign, acc);
  };
  const uint32_t halo_bytes = (rank > 0 ? TM * 16 : 0) + (rank < B ? TM * 16 : 0);

  SweepTask prev{};
  for (int ti = 0; ti < fcount; ++ti) {
    const SweepTask t = a.tasks[ffirst + ti];
    const int base = ti * ITEMS;
    const int par = ti & 1;
    double2* tau = tau2 + par * 2 * kMaxC * TM;
    const double2* halo = halo2 + par * 2 * TM;
    // previous task's traces consumed here straight from shared memory
    const bool loc1 = ti > 0 && t.tin1 >= 0 && prev.out2 == t.tin1;
    const bool loc3 = ti > 0 && t.tin3 >= 0 && prev.out4 == t.tin3;
    if (threadIdx.x == 0) {
      if (ti > 0) mbar_expect_tx(&xbar[2 + par], halo_bytes);
      if (B > 0) mbar_expect_tx(&xbar[par], 2 * B * TM * 16);
    }
    stamp(ti, 0);
    // ---- right-hand side of the owned blocks (restriction + transmission)
    for (int yl = warp * YPW + hh; yl < m; yl += kCW * YPW) {
      const int y = Y0 + yl;
      double2 v = czero();
      const int gr = x + t.lo - 1;
      if (x < t.T && gr >= t.a && gr < t.b) v = __ldg(a.src + (int64_t)gr * M + y);
      if (!loc1 && t.tin1 >= 0 && (x == t.row1 || x == t.row1 + 1))
        v = cadd(v, trans(t.tin1, t.row1 + t.lo, 1, x - t.row1, y));
      if (!loc3 && t.tin3 >= 0 && (x == t.row3 || x == t.row3 + 1))
        v = cadd(v, trans(t.tin3, t.row3 + t.lo, -1, x - t.row3, y));
      F[yl * TM + x] = v;
    }
    if (loc1 || loc3) {
      mbar_wait_cluster(&xbar[2 + par], (uint32_t)((ti - 1) >> 1) & 1);
      for (int yl = warp * YPW + hh; yl < m; yl += kCW * YPW) {
        const int y = Y0 + yl;
        double2 v = czero();
        if (loc1 && (x == t.row1 || x == t.row1 + 1))
          v = cadd(v, trans_local(halo, prev.orow2, t.row1 + t.lo, 1, x - t.row1, y));
        if (loc3 && (x == t.row3 || x == t.row3 + 1))
          v = cadd(v, trans_local(halo, prev.orow4, t.row3 + t.lo, -1, x - t.row3, y));
        F[yl * TM + x] = cadd(F[yl * TM + x], v);
      }
    }
    csync();
    stamp(ti, 1);
    // ---- chunk-local solve: L cyclic-reduction levels, the dense top, back substitution
    for (int p = 0; p < NP; ++p) {
      const int l = ph_level(p), s = 1 << l;
      const int cnt = pfx[p + 1] - pfx[p];
      for (int jp = warp * HW; jp < cnt; jp += kCW * HW) {
        const int j = jp + sub;
        const bool has = j < cnt;
        const int yl = has && p != L ? item_yl(p, j) : 0;
        const int i = base + pfx[p] + j;
        dbg_ti = ti; dbg_p = p; dbg_j = j;
        const double2* m0 = has ? acquire(i) : nullptr;
        const double2* m1 = m0 + TM2;
        if (has) {
          if (p == L) {            // partial x_r += Q[r][c0] f_c0 + Q[r][c0+1] f_c0+1
            const int c0 = 2 * (j % QP);
            const bool two = c0 + 1 < qk;
            const double2 acc = mvx<TM, HW>(m0, F + c0 * S * TM, two ? m1 : nullptr,
                                            two ? F + (c0 + 1) * S * TM : nullptr, lane);
            if (wr) part[j * TM + x] = acc;
          } else if (p < L) {
            if ((yl >> l) & 1) {   // eliminated at this level: y = Dinv f
              const double2 r = mvx<TM, HW>(m0, F + yl * TM, nullptr, nullptr, lane);
              if (wr) Yv[yl * TM + x] = r;
            } else {               // kept: f -= alpha f_{y-s} + gamma f_{y+s}
              const bool hl = yl - s >= 0, hr = yl + s < m;
              const double2 acc = mvx<TM, HW>(hl ? m0 : nullptr, hl ? F + (yl - s) * TM : nullptr,
                                          hr ? m1 : nullptr, hr ? F + (yl + s) * TM : nullptr,
                                          lane);
              if (wr) F[yl * TM + x] = csub(F[yl * TM + x], acc);
            }
          } else {                 // x_y = Dinv f - (Dinv L) x_{y-s} - (Dinv U) x_{y+s}
            const bool hl = yl - s >= 0, hr = yl + s < m;
            const double2 acc = mvx<TM, HW>(hl ? m0 : nullptr, hl ? Yv + (yl - s) * TM : nullptr,
                                        hr ? m1 : nullptr, hr ? Yv + (yl + s) * TM : nullptr,
                                        lane);
            if (wr) Yv[yl * TM + x] = csub(Yv[yl * TM + x], acc);
          }
        }
        stamp2(ti, p, j, 3);
        release(i, has);
        stamp2(ti, p, j, 4);
      }
      csync();
      if (p == L) {   // x at the level-L points = sum of the column-pair partials
        for (int t = threadIdx.x; t < qk * TM; t += kCW * 32) {
          const int r = t / TM, xx = t % TM;
          double2 acc = czero();
          for (int cp = 0; cp < QP; ++cp) acc = cadd(acc, part[(r * QP + cp) * TM + xx]);
          Yv[r * S * TM + xx] = acc;
        }
        csync();
      }
      stamp(ti, 2 + p);
    }
    if (B > 0) {
      // ---- push this chunk's tips g[first], g[last] into every CTA's tau:
      // tau block b = (g_b[last], g_{b+1}[first]) -> tm-slots 2b, 2b+1
      for (int d = warp; d < C && lane < TM; d += kCW) {
        const uint32_t bar = map_rank(&xbar[par], d);
        if (rank > 0) st_async_c(map_rank(&tau[(2 * (rank - 1) + 1) * TM + lane], d), Yv[lane], bar);
        if (rank < B) st_async_c(map_rank(&tau[(2 * rank) * TM + lane], d), Yv[(m - 1) * TM + lane], bar);
      }
      mbar_wait_cluster(&xbar[par], (uint32_t)(ti >> 1) & 1);
      stamp(ti, 40);
      // ---- alpha_{k-1}, beta_k = (rows of R) tau: 2B column blocks over warps
      // rows r0 = lane (tm 32) or x (tm 16, per half) and r0 + 32 / r0 + 16
      double2 acc0 = czero(), acc1 = czero();
      const int nq = 2 * B;
      const int r0 = HW == 1 ? lane : x, r1 = r0 + (HW == 1 ? 32 : 16);   // r1 unused: tm 16, HW 1
      for (int jp = warp * HW; jp < nq; jp += kCW * HW) {
        const int j = jp + sub;
        const bool has = j < nq;
        const int i = base + pfx[NP] + j;
        if (has) {
          const double2* mq = acquire(i);   // 2tm x tm, row index fastest
          const double2* tq = tau + j * TM;
#pragma unroll 4
          for (int c = 0; c < TM; ++c) {
            const double2 tv = tq[c];
            acc0 = cfma(mq[c * N2 + r0], tv, acc0);
            if (HW == 2 || TM == 32) acc1 = cfma(mq[c * N2 + r1], tv, acc1);
          }
        }
        release(i, has);
      }
      if (HW == 2) {   // both halves' items hold rows x and x + 16
        acc0 = cadd(acc0, shfl_xor_c(acc0, 16));
        acc1 = cadd(acc1, shfl_xor_c(acc1, 16));
      }
      if (lane < 32 / HW) {
        part[warp * N2 + r0] = acc0;
        if (HW == 2 || TM == 32) part[warp * N2 + r1] = acc1;
      }
      csync();
      if (threadIdx.x < N2) {
        double2 sacc = czero();
        for (int w = 0; w < kCW; ++w) sacc = cadd(sacc, part[w * N2 + threadIdx.x]);
        ab[threadIdx.x] = sacc;
      }
      csync();
      stamp(ti, 41);
      // ---- x_y = g_y - W_y alpha_{k-1} - V_y beta_k
      for (int jp = warp * HW; jp < m; jp += kCW * HW) {
        const int j = jp + sub;
        const bool has = j < m;
        const int i = base + pfx[NP + 1] + j;
        if (has) {
          const double2* ms = acquire(i);
          const double2 acc = mvx<TM, HW>(rank > 0 ? ms : nullptr, rank > 0 ? ab : nullptr,
                                      rank < B ? ms + TM2 : nullptr, rank < B ? ab + TM : nullptr,
                                      lane);
          if (wr) Yv[j * TM + x] = csub(Yv[j * TM + x], acc);
        }
        release(i, has);
      }
      stamp(ti, 42);
      csync();
    }
    // ---- edge blocks of x to the neighbours (next task's transmission halo)
    if (ti + 1 < fcount && lane < TM) {
      const int nb = ((ti + 1) & 1) * 2 * TM;
      if (warp == 0 && rank > 0)
        st_async_c(map_rank(&halo2[nb + TM + lane], rank - 1), Yv[lane],
                   map_rank(&xbar[2 + ((ti + 1) & 1)], rank - 1));
      if (warp == 1 && rank < B)
        st_async_c(map_rank(&halo2[nb + lane], rank + 1), Yv[(m - 1) * TM + lane],
                   map_rank(&xbar[2 + ((ti + 1) & 1)], rank + 1));
    }
    // ---- outputs: solution rows into u (one producer per row and pass), traces
    const int ur0 = t.ta + 1 - t.lo, ur1 = t.tb + 1 - t.lo;
    for (int yl = warp * YPW + hh; yl < m; yl += kCW * YPW) {
      const int y = Y0 + yl;
      const double2 xv = Yv[yl * TM + x];
      if (x >= ur0 && x < ur1) a.u[t.dst][(int64_t)(x + t.lo - 1) * M + y] = xv;
      if (t.out2 >= 0 && (x == t.orow2 || x == t.orow2 + 1))
        a.trace[((int64_t)t.out2 * 2 + (x - t.orow2)) * M + y] = xv;
      if (t.out4 >= 0 && (x == t.orow4 || x == t.orow4 + 1))
        a.trace[((int64_t)t.out4 * 2 + (x - t.orow4)) * M + y] = xv;
    }
    stamp(ti, 43);
    prev = t;
    stamp(ti, 63);
  }
  cl.sync();   // no CTA leaves while a peer may still write its shared memory
  if (a.dbg && threadIdx.x == 0 && blockIdx.x < 16)
    for (int k = 0; k < 128; ++k) {
      a.dbg[blockIdx.x * 256 + k] = tsm[k];
      a.dbg[blockIdx.x * 256 + 128 + k] = tprod[k];
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

template <int TM>
cudaError_t prepare_solve(int C, int mmax, int* max_clusters) {
  cudaError_t e = cudaFuncSetAttribute(k_part_solve<TM>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  const int smem = Ring<TM>::smem(mmax);
  e = cudaFuncSetAttribute(k_part_solve<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = solve_config(C, 1, smem, nullptr, attr);
  return cudaOccupancyMaxActiveClusters(max_clusters, k_part_solve<TM>, &cfg);
}

template <int TM, int Q>
cudaError_t launch_dense_top_q(Ctx* c, const Chunks& g, int J, const double2* D, const double2* Lc,
                               const double2* Uc, double2* qd, unsigned long long* err) {
  constexpr int N = Q * TM;
  const int smem = 2 * N * (N + 1) * (int)sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(k_dense_top<TM, Q>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_dense_top<TM, Q><<<J * g.C, 1024, smem, c->stream>>>(g, D, Lc, Uc, qd, err);
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
  const int J = s->J, M = s->M, L = s->L, C = s->C, B = C - 1;
  const size_t wbytes = (size_t)J * M * TM2 * sizeof(double2);
  const size_t ebytes = (size_t)J * C * TM2 * sizeof(double2);
  double2 *D = nullptr, *Lc = nullptr, *Uc = nullptr, *EL = nullptr, *EU = nullptr;
  double2 *Hw = nullptr, *Zw = nullptr, *tips = nullptr, *Gw = nullptr, *Zr = nullptr;
  SlabInfo* d_info = nullptr;
  unsigned long long* d_err = nullptr;
  int rc = HS_OK;
  auto cleanup = [&]() {
    cudaFree(D); cudaFree(Lc); cudaFree(Uc); cudaFree(EL); cudaFree(EU); cudaFree(Hw);
    cudaFree(Zw); cudaFree(tips); cudaFree(Gw); cudaFree(Zr); cudaFree(d_info); cudaFree(d_err);
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
  HS_TRYF(cudaMemsetAsync(s->kr, 0, (size_t)J * C * g.kstride * 2 * TM2 * sizeof(double2),
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
  if (B > 0) {   // spikes from the pristine chunk operators
    HS_TRYF(cudaMalloc((void**)&Hw, wbytes), "spike work alloc");
    HS_TRYF(cudaMalloc((void**)&Zw, wbytes), "spike work alloc");
    k_spikes<TM><<<J * C, TM * TM, smem7, c->stream>>>(g, D, Lc, Uc, EL, EU, Hw, Zw, s->sp,
                                                       tips, d_err);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "spikes");
    constexpr int N = 2 * TM;
    const int NR = B * N;
    HS_TRYF(cudaMalloc((void**)&Gw, (size_t)J * B * N * N * sizeof(double2)), "alloc");
    HS_TRYF(cudaMalloc((void**)&Zr, (size_t)J * NR * NR * sizeof(double2)), "alloc");
    const int smemr = 2 * N * (N + 1) * (int)sizeof(double2);
    HS_TRYF(cudaFuncSetAttribute(k_reduced<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smemr), "attr");
    k_reduced<TM><<<J, 1024, smemr, c->stream>>>(g, tips, Gw, Zr, s->rk, d_err);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "reduced system");
  }
  const int mmax = s->mmax;
  for (int l = 0; l < L; ++l) {
    const int sl = 1 << l;
    const int nel = mmax - 1 >= sl ? (mmax - 1 - sl) / (2 * sl) + 1 : 0;
    const int nkeep = (mmax - 1) / (2 * sl) + 1;
    if (nel) {
      k_bcr_elim<TM><<<dim3(nel, J * C), TM * TM, smem3, c->stream>>>(l, g, 0, D, Lc, Uc,
                                                                      s->ef, s->eb, d_err);
      c->launches++;
      HS_TRYF(cudaGetLastError(), "bcr elim");
    }
    k_bcr_keep<TM><<<dim3(nkeep, J * C), TM * TM, smem4, c->stream>>>(l, g, D, Lc, Uc, s->kr);
    c->launches++;
    HS_TRYF(cudaGetLastError(), "bcr keep");
  }
  HS_TRYF(launch_dense_top<TM>(c, g, J, D, Lc, Uc, s->qd, d_err), "dense top");
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

Chunks make_chunks(const Sweep* s) {
  Chunks g{};
  g.M = s->M;
  g.C = s->C;
  g.L = s->L;
  g.q = s->q;
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

int sweep_create(Ctx* c, const Stencil* coarse, int J, const int64_t* beta, const int64_t* bt,
                 const int64_t* lo, const int64_t* hi, const Stencil* const* slabs,
                 Sweep** out) {
  if (coarse->dim != 2)
    return set_error(c, HS_E_SHAPE, "the device sweep supports 2-D levels (3-D: not yet)");
  if (J < 2) return set_error(c, HS_E_SHAPE, "the sweep needs at least 2 subdomains");
  if (J > kMaxTasks) return set_error(c, HS_E_SHAPE, "too many subdomains for the sweep");
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
  // chunks: ~32 face points per CTA, at most 16 CTAs, cluster schedulable twice
  int C = std::min(kMaxC, std::max(1, (M + 31) / 32));
  for (;;) {
    const int mmax = (M + C - 1) / C;
    int maxc = 0;
    cudaError_t e = TM == 16 ? prepare_solve<16>(C, mmax, &maxc) : prepare_solve<32>(C, mmax, &maxc);
    if (e == cudaSuccess && maxc >= 2) break;
    cudaGetLastError();
    if (C == 1) {
      delete s;
      return set_error(c, HS_E_CUDA, "no schedulable cluster for the sweep kernel");
    }
    C = C > 8 ? 8 : C / 2;
  }
  s->C = C;
  s->mmax = (M + C - 1) / C;
  // cyclic reduction until at most qmax blocks per chunk are left, then a
  // dense inverse of that reduced system (qmax blocks fit the setup's smem)
  const int qmax = TM == 16 ? 5 : 2;
  s->L = 0;
  while ((s->mmax - 1) / (1 << s->L) + 1 > qmax) ++s->L;
  s->q = (s->mmax - 1) / (1 << s->L) + 1;
  if (s->L >= kMaxLevels) { delete s; return set_error(c, HS_E_SHAPE, "face too long"); }
  const Chunks g = make_chunks(s);
  s->kstride = g.kstride;
  const int B = C - 1;

  const size_t efb = (size_t)J * M * TM2 * sizeof(double2);
  const size_t krb = (size_t)J * C * g.kstride * 2 * TM2 * sizeof(double2);
  const size_t rkb = (size_t)J * C * std::max(1, 2 * B) * 2 * TM2 * sizeof(double2);
  const size_t qdb = (size_t)J * C * s->q * s->q * TM2 * sizeof(double2);
  s->factor_bytes = (long long)(efb * 5 + krb + qdb + (B > 0 ? rkb : 0));
  cudaError_t e = cudaMalloc((void**)&s->ef, efb);
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
  // factor blocks streamed per slab solve (exactly the items of k_part_solve)
  double rec_blocks = 0;
  for (int k = 0; k < C; ++k) {
    const int m = g.len(k), L = s->L;
    for (int l = 0; l < L; ++l) {
      const int sl = 1 << l;
      for (int yl = 0; yl < m; yl += sl) {
        if ((yl >> l) & 1) rec_blocks += 1 + 1 + (yl + sl < m);   // Dinv; back: Dinv L (+ Dinv U)
        else rec_blocks += (yl > 0) + (yl + sl < m);              // alpha, gamma
      }
    }
    const int qk = (m - 1) / (1 << L) + 1;
    rec_blocks += (double)qk * qk;
    if (B > 0) rec_blocks += 4.0 * B + 2.0 * m;                   // R rows, spikes
  }
  const double rec_bytes = rec_blocks * TM2 * 16.0;
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
    std::vector<SweepTask> F, Bk;
    fwd_chain(1, J, F);
    clear_placeholders(F);
    bwd_chain(J, 1, Bk);
    clear_placeholders(Bk);
    emit_pass(plan, 0, {{F}});
    plan.push_back(SweepLaunch{SweepLaunch::kResidual});
    emit_pass(plan, 1, {{Bk}});
    plan.push_back(SweepLaunch{SweepLaunch::kCombine});
    s->has_plan[HS_VARIANT_UD] = true;
  }
  // ---- X: simultaneous half sweeps meeting at jm = J/2 + 1 ----
  if (J % 2 == 0) {
    std::vector<SweepLaunch>& plan = s->plan[HS_VARIANT_X];
    const int jm = J / 2 + 1;
    std::vector<SweepTask> F, Bk, MI;
    fwd_chain(1, jm - 1, F);
    bwd_chain(J, jm + 1, Bk);
    SweepTask mi = mk(jm, (int)beta[jm - 1], (int)bt[jm]);
    want1(mi, jm);
    want3(mi, jm);
    if (!F.empty() && F.back().out2 == -2) give2(F.back(), jm - 1, mi.tin1);
    if (!Bk.empty() && Bk.back().out4 == -2) give4(Bk.back(), jm + 1, mi.tin3);
    clear_placeholders(F);
    clear_placeholders(Bk);
    MI.push_back(mi);
    emit_pass(plan, 0, {{F, Bk}, {MI}});
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
  cudaFree(s->sp);
  cudaFree(s->rk);
  cudaFree(s->qd);
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
        a.g = make_chunks(s);
        a.nslot = s->tm == 16 ? Ring<16>::nslot(s->mmax) : Ring<32>::nslot(s->mmax);
        a.ef = s->ef;
        a.eb = s->eb;
        a.kr = s->kr;
        a.sp = s->sp;
        a.rk = s->rk;
        a.qd = s->qd;
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
          cudaMalloc((void**)&dbg, 16 * 256 * sizeof(unsigned long long));
          cudaMemsetAsync(dbg, 0, 16 * 256 * sizeof(unsigned long long), c->stream);
        }
        a.dbg = dbg;
        const int smem = s->tm == 16 ? Ring<16>::smem(s->mmax) : Ring<32>::smem(s->mmax);
        cudaLaunchAttribute attr[1];
        cudaLaunchConfig_t cfg = solve_config(s->C, Lh.nfront, smem, c->stream, attr);
        ProfScope ps(c, K_SWEEP_FRONT, Lh.bytes);
        cudaError_t e = s->tm == 16 ? cudaLaunchKernelEx(&cfg, k_part_solve<16>, a)
                                    : cudaLaunchKernelEx(&cfg, k_part_solve<32>, a);
        if (e != cudaSuccess) return check_cuda(c, e, "sweep solve launch");
        HS_LAUNCH_CHECK(c, "sweep solve kernel");
        if (dbg) {
          std::vector<unsigned long long> h(16 * 256);
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
              for (int k = 0; k < 256; ++k)
                fprintf(fp, "%lld ", h[b * 256 + k] ? (long long)(h[b * 256 + k] - t0) : -1LL);
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
