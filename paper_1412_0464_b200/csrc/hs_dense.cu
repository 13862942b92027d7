// Batched dense complex128 linear algebra for the 3-D slab factorisation and
// the exact solver (hs_sweep3.cu): the block LU along a slab's planes needs,
// per plane and for every slab at once, a Schur update D' = D - L X, the
// inverse of D' (LU with partial pivoting inside the block) and the products
// Dinv U, Dinv L (sparselin.py:40-62 restated as dense block LU; SURVEY
// §8(a) A11).  Setup only -- the apply path reads the stored blocks.
//
// Kernels (all batched over independent matrices, one job per slab):
//   k_gemm      C = alpha op(A) op(B) + beta C, column-major, optional
//               transposed store; 64 x 64 complex tiles, 4 x 4 per thread,
//               FP64 FMA (no FP64 tensor-core path is needed at this size)
//   k_panel     unblocked LU with partial pivoting of a 32-column panel
//               (pivot = largest |re| + |im|, LAPACK's izamax), one CTA
//   k_swap_trsm the panel's row swaps on the other columns + U12 = L11^-1 A12
//   k_perm_eye  P^T I from the pivot sequence
//   k_trsm      the blocked triangular solves of the inverse (unit lower /
//               non-unit upper diagonal blocks)
//   k_transpose row-major copies of the results

#include "hs_common.cuh"
#include "hs_dense.cuh"

#include <algorithm>
#include <vector>

namespace hs {
namespace {

constexpr int kTile = 64;     // GEMM tile (complex entries per side)
constexpr int kKT = 8;        // GEMM k step
constexpr int kPanel = 32;    // LU panel width

__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm (no overflow for the magnitudes here)
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

struct GemmBatch {
  GemmJob j[kMaxDenseJobs];
};

__device__ __forceinline__ double2 ld_op(const double2* M, int ld, int op, int r, int c, int rows,
                                         int cols) {
  // element (r, c) of op(M), op(M) of size rows x cols
  if (r >= rows || c >= cols) return make_double2(0.0, 0.0);
  return op ? M[(int64_t)c + (int64_t)r * ld] : M[(int64_t)r + (int64_t)c * ld];
}

__global__ void __launch_bounds__(256) k_gemm(GemmBatch b) {
  const GemmJob& J = b.j[blockIdx.z];
  const int m0 = blockIdx.y * kTile, n0 = blockIdx.x * kTile;
  if (m0 >= J.m || n0 >= J.n) return;
  __shared__ double2 As[kKT][kTile + 1];
  __shared__ double2 Bs[kKT][kTile + 1];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < J.k; k0 += kKT) {
    for (int e = tid; e < kTile * kKT; e += 256) {
      // A tile: rows m0.., cols k0..; B tile: rows k0.., cols n0..
      const int ra = J.opA ? e / kKT : e % kTile, ka = J.opA ? e % kKT : e / kTile;
      As[ka][ra] = ld_op(J.A, J.lda, J.opA, m0 + ra, k0 + ka, J.m, J.k);
      const int kb = J.opB ? e / kTile : e % kKT, cb = J.opB ? e % kTile : e / kKT;
      Bs[kb][cb] = ld_op(J.B, J.ldb, J.opB, k0 + kb, n0 + cb, J.k, J.n);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKT; ++kk) {
      double2 a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tx + 16 * i];
#pragma unroll
      for (int q = 0; q < 4; ++q) bb[q] = Bs[kk][ty + 16 * q];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = cfma(a[i], bb[q], acc[i][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = m0 + tx + 16 * i, c = n0 + ty + 16 * q;
      if (r >= J.m || c >= J.n) continue;
      double2* dst = J.transC ? J.C + (int64_t)c + (int64_t)r * J.ldc : J.C + (int64_t)r + (int64_t)c * J.ldc;
      double2 v = cmul(J.alpha, acc[i][q]);
      if (J.beta.x != 0.0 || J.beta.y != 0.0) v = cfma(J.beta, *dst, v);
      *dst = v;
    }
}

struct LuBatch {
  LuJob j[kMaxDenseJobs];
};

// Unblocked LU with partial pivoting of the panel columns [k0, k0 + w) of
// an n x n column-major matrix (rows k0..n-1); the swaps touch the panel
// columns only (k_swap_trsm applies them elsewhere).  info: first zero pivot
// (1-based global row), kept if already set.
__global__ void __launch_bounds__(1024) k_panel(LuBatch b, int k0) {
  const LuJob& J = b.j[blockIdx.x];
  const int n = J.n, w = min(kPanel, n - k0);
  if (w <= 0) return;
  double2* A = J.A;
  const int ld = J.ld;
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int piv_s;
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32, nw = blockDim.x / 32;
  for (int jj = 0; jj < w; ++jj) {
    const int j = k0 + jj;
    // pivot: largest |re| + |im| in column j, rows j..n-1 (lowest index on ties)
    double best = -1.0;
    int bi = j;
    for (int i = j + tid; i < n; i += blockDim.x) {
      const double v = cabs1(A[i + (int64_t)j * ld]);
      if (v > best) { best = v; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { red_v[warp] = best; red_i[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = lane < nw ? red_v[lane] : -1.0;
      bi = lane < nw ? red_i[lane] : n;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) {
        piv_s = bi;
        J.piv[j] = bi;
        if (best == 0.0 && *J.info == 0) *J.info = j + 1;
      }
    }
    __syncthreads();
    const int p = piv_s;
    if (p != j)   // swap rows j, p across the panel columns
      for (int c = k0 + tid; c < k0 + w; c += blockDim.x) {
        double2* a = A + (int64_t)c * ld;
        const double2 t = a[j];
        a[j] = a[p];
        a[p] = t;
      }
    __syncthreads();
    const double2 d = A[j + (int64_t)j * ld];
    const bool zero = d.x == 0.0 && d.y == 0.0;
    // column j below the diagonal scaled; rank-1 update of the panel's later columns
    for (int i = j + 1 + tid; i < n; i += blockDim.x) {
      double2* aij = A + i + (int64_t)j * ld;
      const double2 l = zero ? make_double2(0.0, 0.0) : cdiv(*aij, d);
      *aij = l;
      for (int c = j + 1; c < k0 + w; ++c) {
        double2* aic = A + i + (int64_t)c * ld;
        *aic = csub(*aic, cmul(l, A[j + (int64_t)c * ld]));
      }
    }
    __syncthreads();
  }
}

// The panel's swaps on every column outside [k0, k0 + w), then for the
// columns right of the panel U12 = L11^{-1} A12 (unit lower 32 x 32).
// One thread per column.
__global__ void __launch_bounds__(256) k_swap_trsm(LuBatch b, int k0) {
  const LuJob& J = b.j[blockIdx.y];
  const int n = J.n, w = min(kPanel, n - k0);
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (w <= 0 || c >= n || (c >= k0 && c < k0 + w)) return;
  double2* a = J.A + (int64_t)c * J.ld;
  for (int jj = 0; jj < w; ++jj) {
    const int j = k0 + jj, p = J.piv[j];
    if (p != j) {
      const double2 t = a[j];
      a[j] = a[p];
      a[p] = t;
    }
  }
  if (c < k0) return;
  double2 x[kPanel];
#pragma unroll
  for (int r = 0; r < kPanel; ++r) x[r] = r < w ? a[k0 + r] : make_double2(0.0, 0.0);
#pragma unroll
  for (int r = 1; r < kPanel; ++r) {
    if (r >= w) break;
    double2 s = x[r];
    for (int q = 0; q < r; ++q) s = csub(s, cmul(J.A[k0 + r + (int64_t)(k0 + q) * J.ld], x[q]));
    x[r] = s;
  }
#pragma unroll
  for (int r = 0; r < kPanel; ++r)
    if (r < w) a[k0 + r] = x[r];
}

// X = P^T I: the pivot sequence applied to the identity (row i of X = e_q(i))
__global__ void __launch_bounds__(256) k_perm_eye(LuBatch b) {
  const LuJob& J = b.j[blockIdx.y];
  const int n = J.n;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;   // column of X
  if (c >= n) return;
  // position of unit c after the swaps: follow the swap sequence
  int pos = c;
  for (int j = 0; j < n; ++j) {
    const int p = J.piv[j];
    if (pos == j) pos = p;
    else if (pos == p) pos = j;
  }
  double2* x = J.X + (int64_t)c * J.ldx;
  for (int r = 0; r < n; ++r) x[r] = make_double2(r == pos ? 1.0 : 0.0, 0.0);
}

// Diagonal block of the blocked triangular solve L X = B (lower, unit) or
// U X = B (upper): rows [k0, k0 + w) of X for every column, in place.
__global__ void __launch_bounds__(256) k_trsm(LuBatch b, int k0, int upper) {
  const LuJob& J = b.j[blockIdx.y];
  const int n = J.n, w = min(kPanel, n - k0);
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (w <= 0 || c >= n) return;
  double2* x = J.X + (int64_t)c * J.ldx + k0;
  const double2* A = J.A;
  const int ld = J.ld;
  double2 v[kPanel];
#pragma unroll
  for (int r = 0; r < kPanel; ++r) v[r] = r < w ? x[r] : make_double2(0.0, 0.0);
  if (!upper) {
#pragma unroll
    for (int r = 1; r < kPanel; ++r) {
      if (r >= w) break;
      double2 s = v[r];
      for (int q = 0; q < r; ++q) s = csub(s, cmul(A[k0 + r + (int64_t)(k0 + q) * ld], v[q]));
      v[r] = s;
    }
  } else {
#pragma unroll
    for (int r = kPanel - 1; r >= 0; --r) {
      if (r >= w) continue;
      double2 s = v[r];
      for (int q = r + 1; q < w; ++q) s = csub(s, cmul(A[k0 + r + (int64_t)(k0 + q) * ld], v[q]));
      v[r] = cdiv(s, A[k0 + r + (int64_t)(k0 + r) * ld]);
    }
  }
#pragma unroll
  for (int r = 0; r < kPanel; ++r)
    if (r < w) x[r] = v[r];
}

struct TrBatch {
  TransposeJob j[kMaxDenseJobs];
};

// dst (row-major n x n, i.e. the column-major transpose) from src column-major
__global__ void __launch_bounds__(256) k_transpose(TrBatch b) {
  const TransposeJob& J = b.j[blockIdx.z];
  __shared__ double2 t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  if (c0 >= J.n || r0 >= J.n) return;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  for (int q = ty; q < 32; q += 8) {
    const int r = r0 + tx, c = c0 + q;
    if (r < J.n && c < J.n) t[q][tx] = J.src[r + (int64_t)c * J.lds];
  }
  __syncthreads();
  for (int q = ty; q < 32; q += 8) {
    const int c = c0 + tx, r = r0 + q;   // dst[r][c] row-major = src(r, c)
    if (r < J.n && c < J.n) J.dst[(int64_t)r * J.ldd + c] = t[tx][q];
  }
}

}  // namespace

int dense_gemm(Ctx* c, const GemmJob* jobs, int n) {
  for (int b0 = 0; b0 < n; b0 += kMaxDenseJobs) {
    GemmBatch b{};
    const int nb = std::min(kMaxDenseJobs, n - b0);
    int mt = 0, nt = 0;
    for (int i = 0; i < nb; ++i) {
      b.j[i] = jobs[b0 + i];
      mt = std::max(mt, (jobs[b0 + i].m + kTile - 1) / kTile);
      nt = std::max(nt, (jobs[b0 + i].n + kTile - 1) / kTile);
    }
    if (!mt || !nt) continue;
    k_gemm<<<dim3((unsigned)nt, (unsigned)mt, (unsigned)nb), 256, 0, c->stream>>>(b);
    HS_LAUNCH_CHECK(c, "dense GEMM");
  }
  return HS_OK;
}

// LU with partial pivoting of every job's A (n x n) and X = A^{-1}, batched.
int dense_lu_inverse(Ctx* c, const LuJob* jobs, int n) {
  for (int b0 = 0; b0 < n; b0 += kMaxDenseJobs) {
    LuBatch b{};
    const int nb = std::min(kMaxDenseJobs, n - b0);
    int nmax = 0;
    for (int i = 0; i < nb; ++i) {
      b.j[i] = jobs[b0 + i];
      nmax = std::max(nmax, jobs[b0 + i].n);
    }
    const unsigned cg = (unsigned)((nmax + 255) / 256);
    std::vector<GemmJob> g;
    // ---- LU: panels, swaps + U12, trailing update
    for (int k0 = 0; k0 < nmax; k0 += kPanel) {
      k_panel<<<(unsigned)nb, 1024, 0, c->stream>>>(b, k0);
      HS_LAUNCH_CHECK(c, "LU panel");
      k_swap_trsm<<<dim3(cg, (unsigned)nb), 256, 0, c->stream>>>(b, k0);
      HS_LAUNCH_CHECK(c, "LU swaps / U12");
      g.clear();
      for (int i = 0; i < nb; ++i) {
        const LuJob& J = b.j[i];
        const int r0 = k0 + kPanel, rest = J.n - r0;
        if (rest <= 0) continue;
        GemmJob q{};
        q.m = rest; q.n = rest; q.k = kPanel;
        q.A = J.A + r0 + (int64_t)k0 * J.ld; q.lda = J.ld;
        q.B = J.A + k0 + (int64_t)r0 * J.ld; q.ldb = J.ld;
        q.C = J.A + r0 + (int64_t)r0 * J.ld; q.ldc = J.ld;
        q.alpha = make_double2(-1.0, 0.0); q.beta = make_double2(1.0, 0.0);
        g.push_back(q);
      }
      if (int r = dense_gemm(c, g.data(), (int)g.size())) return r;
    }
    // ---- inverse: X = U^{-1} L^{-1} P^T I
    k_perm_eye<<<dim3(cg, (unsigned)nb), 256, 0, c->stream>>>(b);
    HS_LAUNCH_CHECK(c, "permuted identity");
    for (int k0 = 0; k0 < nmax; k0 += kPanel) {   // forward: unit lower
      k_trsm<<<dim3(cg, (unsigned)nb), 256, 0, c->stream>>>(b, k0, 0);
      HS_LAUNCH_CHECK(c, "lower solve");
      g.clear();
      for (int i = 0; i < nb; ++i) {
        const LuJob& J = b.j[i];
        const int r0 = k0 + kPanel, rest = J.n - r0;
        if (rest <= 0) continue;
        GemmJob q{};
        q.m = rest; q.n = J.n; q.k = kPanel;
        q.A = J.A + r0 + (int64_t)k0 * J.ld; q.lda = J.ld;
        q.B = J.X + k0; q.ldb = J.ldx;
        q.C = J.X + r0; q.ldc = J.ldx;
        q.alpha = make_double2(-1.0, 0.0); q.beta = make_double2(1.0, 0.0);
        g.push_back(q);
      }
      if (int r = dense_gemm(c, g.data(), (int)g.size())) return r;
    }
    for (int k0 = ((nmax - 1) / kPanel) * kPanel; k0 >= 0; k0 -= kPanel) {   // backward: upper
      k_trsm<<<dim3(cg, (unsigned)nb), 256, 0, c->stream>>>(b, k0, 1);
      HS_LAUNCH_CHECK(c, "upper solve");
      g.clear();
      for (int i = 0; i < nb; ++i) {
        const LuJob& J = b.j[i];
        if (k0 >= J.n || k0 == 0) continue;
        const int w = std::min(kPanel, J.n - k0);
        GemmJob q{};
        q.m = k0; q.n = J.n; q.k = w;
        q.A = J.A + (int64_t)k0 * J.ld; q.lda = J.ld;
        q.B = J.X + k0; q.ldb = J.ldx;
        q.C = J.X; q.ldc = J.ldx;
        q.alpha = make_double2(-1.0, 0.0); q.beta = make_double2(1.0, 0.0);
        g.push_back(q);
      }
      if (int r = dense_gemm(c, g.data(), (int)g.size())) return r;
    }
  }
  return HS_OK;
}

int dense_transpose(Ctx* c, const TransposeJob* jobs, int n) {
  for (int b0 = 0; b0 < n; b0 += kMaxDenseJobs) {
    TrBatch b{};
    const int nb = std::min(kMaxDenseJobs, n - b0);
    int nmax = 0;
    for (int i = 0; i < nb; ++i) {
      b.j[i] = jobs[b0 + i];
      nmax = std::max(nmax, jobs[b0 + i].n);
    }
    const unsigned t = (unsigned)((nmax + 31) / 32);
    k_transpose<<<dim3(t, t, (unsigned)nb), 256, 0, c->stream>>>(b);
    HS_LAUNCH_CHECK(c, "transpose");
  }
  return HS_OK;
}

}  // namespace hs
