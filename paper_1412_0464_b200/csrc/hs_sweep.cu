// Coarse-level sweeping preconditioner: batched slab factorisation (setup) and
// the sequential slab-solve chains of the UD / X schedules (apply).
//
// Reference: build_partition + Factorization (sweepdd.py:192-218,
// sparselin.py:40-68), subdom_solve (sweepdd.py:236-268), TransmissionMatrix
// (sweepdd.py:98-141), forward/backward/mid sweeps and prec_ud / prec_x
// (sweepdd.py:271-359).
//
// Slab systems.  A slab of T <= 16 layers along the sweep axis and M face
// points, ordered face-major (y slow, layer x fast), is block tridiagonal:
// block row y couples to y-1 (L_y), y (D_y) and y+1 (U_y), each 16x16 with
// tridiagonal structure in x.  Setup computes the block LU without inter-block
// pivoting (no-pivot LU is sound on these slabs, min pivot ratio
// 0.088) and stores per (slab, y):
//   forward record  Dinv_y = (D_y - L_y H_{y-1})^{-1}   (dense, Gauss-Jordan
//                   with partial pivoting inside the block) + L_y diagonals
//   backward record H_y = Dinv_y U_y (dense) + outgoing transmission coefs
// Apply: z_y = Dinv_y (fd_y - L_y z_{y-1}) ascending, x_y = z_y - H_y x_{y+1}
// descending.  One warp runs one chain; per step it multiplies a 16x16
// complex block, lanes (x, h) = (row, column half).  The records stream into
// a shared-memory ring with TMA bulk copies (cp.async.bulk + mbarrier
// complete_tx) NSLOT*G steps ahead of the dependency chain.
//
// Transmission (sweepdd.py:113-118): the producer of a trace turns it into
// the consumer's two source rows inside its own backward pass (coefficients
// of the global coarse operator on the interface rows ride in the backward
// record), so the consumer just streams them with its right-hand side.
//
// Dense blocks are stored with an XOR swizzle (element (r,c) at
// r*16 + (c ^ (r & 7))) so the half-row reads of 8 lanes hit 8 distinct
// 16-byte bank groups.

#include "hs_common.cuh"
#include "hs_sweep.cuh"

#include <algorithm>

namespace hs {

namespace {

// Per-block-size geometry.  TM = padded slab thickness (16 or 32 layers).
template <int TM>
struct Geo {
  static constexpr int FREC = TM * TM + 3 * TM;   // Dinv (swizzled) + 3 L diagonals
  static constexpr int BREC = TM * TM + 12;       // H (swizzled) + 12 transmission coefs
  static constexpr int G = TM == 16 ? 4 : 2;      // chain steps per ring slot
  static constexpr int NSLOT = 4;                 // ring depth in slots
  static constexpr int NH = 32 / TM;              // lanes sharing one row
  static constexpr int CPL = TM / NH;             // columns per lane
  static constexpr int SLOT_BYTES = G * (FREC * 16 + TM * 16 + 2 * 32);
  static constexpr int SMEM = NSLOT * SLOT_BYTES + 4 * TM * 16 + NSLOT * 8 + 64;
  static_assert(G * (BREC * 16 + TM * 16) <= SLOT_BYTES, "slot too small");
  static_assert(SMEM <= 227 * 1024, "ring does not fit shared memory");
};

// ---------------------------------------------------------------------------
// setup kernels

struct SlabInfo {
  const double2* coeffs;   // slab operator [S][T*M]
  int T;
  int slot[3][3];          // (o0+1, o1+1) -> coefficient slot or -1
};

template <int TM>
__device__ __forceinline__ int swz(int r, int c) { return r * TM + (c ^ (r & 7)); }

// One CTA (TM*TM threads, thread = (r, c)) factorises one slab sequentially in y.
template <int TM>
__global__ void __launch_bounds__(TM * TM)
k_slab_factor(const SlabInfo* __restrict__ slabs, int M, double2* __restrict__ fwd_rec,
              double2* __restrict__ bwd_rec, unsigned long long* __restrict__ err) {
  using Gm = Geo<TM>;
  const int s = blockIdx.x;
  const SlabInfo si = slabs[s];
  const int tid = threadIdx.x;
  const int r = tid / TM, c = tid % TM;
  const int T = si.T;
  const int64_t n = (int64_t)T * M;
  extern __shared__ __align__(16) unsigned char fsm[];
  double2(*A)[TM + 1] = reinterpret_cast<double2(*)[TM + 1]>(fsm);
  double2(*Inv)[TM + 1] = A + TM;
  double2(*Hs)[TM + 1] = Inv + TM;
  __shared__ int piv_row;
  __shared__ double piv_abs;

  auto coef = [&](int o0, int o1, int x, int y) -> double2 {
    // coupling (x, y) -> (x + o0, y + o1), zero outside the slab box
    const int sl = si.slot[o0 + 1][o1 + 1];
    if (sl < 0 || x < 0 || x >= T || x + o0 < 0 || x + o0 >= T || y + o1 < 0 || y + o1 >= M)
      return czero();
    return si.coeffs[(int64_t)sl * n + (int64_t)x * M + y];
  };

  Hs[r][c] = czero();
  __syncthreads();
  for (int y = 0; y < M; ++y) {
    // D~ = D_y - L_y H_{y-1}
    double2 d;
    if (r < T && c < T) {
      d = (c - r >= -1 && c - r <= 1) ? coef(c - r, 0, r, y) : czero();
      if (y > 0) {
        for (int k = r - 1; k <= r + 1; ++k) {
          if (k < 0 || k >= T) continue;
          d = csub(d, cmul(coef(k - r, -1, r, y), Hs[k][c]));
        }
      }
    } else {
      d = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
    A[r][c] = d;
    Inv[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    __syncthreads();
    // Gauss-Jordan inversion with partial pivoting inside the block
    for (int p = 0; p < TM; ++p) {
      if (tid < 32) {
        double v = (tid >= p && tid < TM) ? cabs2(A[tid][p]) : -1.0;
        int idx = tid;
        for (int m = 16; m > 0; m >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, m);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, m);
          if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
        if (tid == 0) { piv_row = idx; piv_abs = v; }
      }
      __syncthreads();
      const int pr = piv_row;
      if (piv_abs <= 0.0) {
        if (tid == 0) {
          const unsigned long long code =
              ((unsigned long long)s << 40) | ((unsigned long long)(p * M + y) & 0xffffffffffull);
          atomicMin(err, code);
        }
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
    double2* fr = fwd_rec + ((int64_t)s * M + y) * Gm::FREC;
    fr[swz<TM>(r, c)] = Inv[r][c];
    if (c < 3) fr[TM * TM + c * TM + r] = (r < T) ? coef(c - 1, -1, r, y) : czero();
    // H_y = Dinv_y U_y, U_y[k][c] = coupling (k, y) -> (c, y+1)
    double2 h = czero();
    if (c < T) {
      for (int k = c - 1; k <= c + 1; ++k) {
        if (k < 0 || k >= T) continue;
        h = cfma(Inv[r][k], coef(c - k, 1, k, y), h);
      }
    }
    __syncthreads();
    Hs[r][c] = h;
    bwd_rec[((int64_t)s * M + y) * Gm::BREC + swz<TM>(r, c)] = h;
    __syncthreads();
  }
}

struct ToutArgs {
  const double2* coarse;  // global coarse op coefficients [S][n0*M]
  int64_t n;              // n0 * M
  int slot[3][3];
  int J, M;
  const int* fwd_point;   // [J] beta_j   (1-based point) or -1
  const int* bwd_point;   // [J] beta~_{j-1}               or -1
};

// Outgoing transmission coefficients per (slab, y) into the backward records.
template <int TM>
__global__ void k_tout(ToutArgs a, double2* __restrict__ bwd_rec) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)a.J * a.M) return;
  const int s = (int)(idx / a.M), y = (int)(idx % a.M);
  double2* out = bwd_rec + idx * Geo<TM>::BREC + TM * TM;
  auto cc = [&](int o0, int o1, int row) -> double2 {
    const int sl = a.slot[o0 + 1][o1 + 1];
    if (sl < 0 || y + o1 < 0 || y + o1 >= a.M) return czero();
    return a.coarse[(int64_t)sl * a.n + (int64_t)row * a.M + y];
  };
  const int pf = a.fwd_point[s], pb = a.bwd_point[s];
  for (int o = -1; o <= 1; ++o) {
    out[0 + o + 1] = pf > 0 ? cc(1, o, pf - 1) : czero();   // A[b, b+1], b = p
    out[3 + o + 1] = pf > 0 ? cc(-1, o, pf) : czero();      // A[b+1, b]
    out[6 + o + 1] = pb > 0 ? cc(1, o, pb - 1) : czero();
    out[9 + o + 1] = pb > 0 ? cc(-1, o, pb) : czero();
  }
}

// ---------------------------------------------------------------------------
// apply kernels

template <int TM>
__global__ void k_gather(const SweepTask* __restrict__ tasks, int first, int M,
                         const double2* __restrict__ src, double2* __restrict__ fdpre) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)M * TM) return;
  const SweepTask t = tasks[first + blockIdx.y];
  const int y = (int)(idx / TM), x = (int)(idx % TM);
  double2 v = czero();
  const int g = x + t.lo - 1;  // global 0-based row
  if (x < t.T && g >= t.a && g < t.b) v = __ldg(src + (int64_t)g * M + y);
  fdpre[((int64_t)t.fdslot * M + y) * TM + x] = v;
}

__global__ void k_combine(double2* __restrict__ u, const double2* __restrict__ u2, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[i] = cadd(u[i], __ldg(u2 + i));
}

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
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async;" ::: "memory");
}

struct FrontArgs {
  const SweepTask* tasks;
  int ffirst[2], fcount[2];
  const double2* fwd_rec;
  const double2* bwd_rec;
  const double2* fdpre;
  double2* tin;
  double2* zs;
  double2* u[2];
  int M;
};

// One warp = one sequential chain of slab solves (a "front" of the sweep).
template <int TM>
__global__ void __launch_bounds__(32, 1) k_front(FrontArgs a) {
  using Gm = Geo<TM>;
  constexpr int FREC = Gm::FREC, BREC = Gm::BREC, G = Gm::G, NSLOT = Gm::NSLOT;
  constexpr int CPL = Gm::CPL, SLOT_BYTES = Gm::SLOT_BYTES;
  extern __shared__ __align__(128) unsigned char smem[];
  const int front = blockIdx.x;
  const int lane = threadIdx.x;
  const int x = lane % TM, hh = lane / TM;
  const int M = a.M;
  unsigned char* ring = smem;
  double2* zb = (double2*)(smem + NSLOT * SLOT_BYTES);   // [2][TM] chain vector (double buffer)
  double2* rb = zb + 2 * TM;                             // [TM] right-hand side broadcast
  uint64_t* bars = (uint64_t*)(rb + 2 * TM);
  if (lane == 0) {
    for (int i = 0; i < NSLOT; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  __syncwarp();
  uint32_t phase_bits = 0;      // parity per slot
  const int ffirst = front ? a.ffirst[1] : a.ffirst[0];
  const int fcount = front ? a.fcount[1] : a.fcount[0];
  double2* zs = a.zs + (int64_t)front * M * TM;
  // lanes that turn outgoing traces into the consumer's sources
  const int tl = lane - (TM == 16 ? 16 : 0);

  for (int ti = 0; ti < fcount; ++ti) {
    const SweepTask t = a.tasks[ffirst + ti];
    const double2* frec = a.fwd_rec + (int64_t)t.slab * M * FREC;
    const double2* brec = a.bwd_rec + (int64_t)t.slab * M * BREC;
    const double2* fdp = a.fdpre + (int64_t)t.fdslot * M * TM;
    const double2* tin1 = t.tin1 >= 0 ? a.tin + (int64_t)t.tin1 * M * 2 : nullptr;
    const double2* tin3 = t.tin3 >= 0 ? a.tin + (int64_t)t.tin3 * M * 2 : nullptr;
    const int ngroups = (M + G - 1) / G;

    // ---------------- forward: z_y = Dinv_y (fd_y - L_y z_{y-1}) ----------
    auto issue_f = [&](int g) {
      const int y0 = g * G;
      const int cnt = min(G, M - y0);
      unsigned char* slot = ring + (g % NSLOT) * SLOT_BYTES;
      uint64_t* bar = &bars[g % NSLOT];
      uint32_t bytes = cnt * (FREC * 16 + TM * 16);
      if (tin1) bytes += cnt * 32;
      if (tin3) bytes += cnt * 32;
      mbar_expect_tx(bar, bytes);
      bulk_g2s(slot, frec + (int64_t)y0 * FREC, cnt * FREC * 16, bar);
      bulk_g2s(slot + G * FREC * 16, fdp + (int64_t)y0 * TM, cnt * TM * 16, bar);
      if (tin1) bulk_g2s(slot + G * (FREC + TM) * 16, tin1 + (int64_t)y0 * 2, cnt * 32, bar);
      if (tin3)
        bulk_g2s(slot + G * (FREC + TM) * 16 + G * 32, tin3 + (int64_t)y0 * 2, cnt * 32, bar);
    };
    if (lane == 0)
      for (int g = 0; g < min(NSLOT, ngroups); ++g) issue_f(g);
    for (int i = lane; i < 2 * TM; i += 32) zb[i] = czero();
    __syncwarp();
    int cur = 0;
    for (int g = 0; g < ngroups; ++g) {
      const int sl = g % NSLOT;
      mbar_wait(&bars[sl], (phase_bits >> sl) & 1u);
      phase_bits ^= 1u << sl;
      const unsigned char* slot = ring + sl * SLOT_BYTES;
      const int cnt = min(G, M - g * G);
      for (int k = 0; k < cnt; ++k) {
        const int y = g * G + k;
        const double2* rec = (const double2*)slot + k * FREC;
        const double2* fdv = (const double2*)(slot + G * FREC * 16) + k * TM;
        double2 rv = fdv[x];
        if (tin1) {
          const double2* tv = (const double2*)(slot + G * (FREC + TM) * 16) + k * 2;
          if (x == t.row1) rv = cadd(rv, tv[0]);
          if (x == t.row1 + 1) rv = cadd(rv, tv[1]);
        }
        if (tin3) {
          const double2* tv = (const double2*)(slot + G * (FREC + TM) * 16 + G * 32) + k * 2;
          if (x == t.row3) rv = cadd(rv, tv[0]);
          if (x == t.row3 + 1) rv = cadd(rv, tv[1]);
        }
        const double2* zp = zb + (cur ^ 1) * TM;   // z_{y-1}
        const double2* L = rec + TM * TM;
        double2 lz = cmul(L[TM + x], zp[x]);
        if (x > 0) lz = cfma(L[x], zp[x - 1], lz);
        if (x < TM - 1) lz = cfma(L[2 * TM + x], zp[x + 1], lz);
        rv = csub(rv, lz);
        if (hh == 0) rb[x] = rv;
        __syncwarp();
        double2 acc0 = czero(), acc1 = czero();
#pragma unroll
        for (int q = 0; q < CPL; q += 2) {
          const int c0 = CPL * hh + q;
          acc0 = cfma(rec[swz<TM>(x, c0)], rb[c0], acc0);
          acc1 = cfma(rec[swz<TM>(x, c0 + 1)], rb[c0 + 1], acc1);
        }
        double2 acc = cadd(acc0, acc1);
        if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
        if (hh == 0) {
          zb[cur * TM + x] = acc;
          zs[(int64_t)y * TM + x] = acc;
        }
        cur ^= 1;
        __syncwarp();
      }
      __syncwarp();
      if (lane == 0 && g + NSLOT < ngroups) {
        fence_proxy_async();
        issue_f(g + NSLOT);
      }
    }
    fence_proxy_async();   // zs (generic stores) -> bulk reads below
    __syncwarp();

    // ---------------- backward: x_y = z_y - H_y x_{y+1} -------------------
    auto grp_lo = [&](int g) { return max(0, M - (g + 1) * G); };
    auto grp_cnt = [&](int g) { return (M - g * G) - grp_lo(g); };
    auto issue_b = [&](int g) {
      const int ylo = grp_lo(g), cnt = grp_cnt(g);
      unsigned char* slot = ring + (g % NSLOT) * SLOT_BYTES;
      uint64_t* bar = &bars[g % NSLOT];
      mbar_expect_tx(bar, cnt * (BREC * 16 + TM * 16));
      bulk_g2s(slot, brec + (int64_t)ylo * BREC, cnt * BREC * 16, bar);
      bulk_g2s(slot + G * BREC * 16, zs + (int64_t)ylo * TM, cnt * TM * 16, bar);
    };
    if (lane == 0)
      for (int g = 0; g < min(NSLOT, ngroups); ++g) issue_b(g);
    for (int i = lane; i < 2 * TM; i += 32) zb[i] = czero();
    __syncwarp();
    // transmission-out lanes: (coef block, trace row, sign, out buffer, component)
    int trow = -1, tsgn = 0, tcb = 0;
    double2* tout = nullptr;
    if (tl >= 0 && tl < 4) {
      const bool fwd = tl < 2;
      const int ob = fwd ? t.out2 : t.out4;
      const int orow = fwd ? t.orow2 : t.orow4;
      if (ob >= 0) {
        tout = a.tin + (int64_t)ob * M * 2 + (tl & 1);
        trow = (tl & 1) ? orow : orow + 1;            // src0 uses B[1], src1 uses B[0]
        const int sign = fwd ? 1 : -1;
        tsgn = (tl & 1) ? -sign : sign;
        tcb = tl * 3;
      }
    }
    double2 cprev[3] = {czero(), czero(), czero()};
    double2 w1 = czero(), w2 = czero();   // trace at y+1, y+2
    const int ur0 = t.ta + 1 - t.lo, ur1 = t.tb + 1 - t.lo;
    cur = 0;
    for (int g = 0; g < ngroups; ++g) {
      const int sl = g % NSLOT;
      mbar_wait(&bars[sl], (phase_bits >> sl) & 1u);
      phase_bits ^= 1u << sl;
      const unsigned char* slot = ring + sl * SLOT_BYTES;
      const int ylo = grp_lo(g), cnt = grp_cnt(g);
      for (int k = cnt - 1; k >= 0; --k) {
        const int y = ylo + k;
        const double2* rec = (const double2*)slot + k * BREC;
        const double2* zv = (const double2*)(slot + G * BREC * 16) + k * TM;
        const double2* xp = zb + (cur ^ 1) * TM;   // x_{y+1}
        double2 acc0 = czero(), acc1 = czero();
#pragma unroll
        for (int q = 0; q < CPL; q += 2) {
          const int c0 = CPL * hh + q;
          acc0 = cfma(rec[swz<TM>(x, c0)], xp[c0], acc0);
          acc1 = cfma(rec[swz<TM>(x, c0 + 1)], xp[c0 + 1], acc1);
        }
        double2 acc = cadd(acc0, acc1);
        if (TM == 16) acc = cadd(acc, shfl_xor_c(acc, 16));
        const double2 xv = csub(zv[x], acc);
        if (hh == 0) zb[cur * TM + x] = xv;
        __syncwarp();
        if (hh == 0 && x >= ur0 && x < ur1) {
          // each row of u is produced by exactly one task per pass: plain store
          a.u[t.dst][(int64_t)(x + t.lo - 1) * M + y] = xv;
        }
        if (tout) {
          const double2 tr = zb[cur * TM + trow];
          if (y + 1 < M) {
            double2 sacc = cmul(cprev[0], tr);
            sacc = cfma(cprev[1], w1, sacc);
            sacc = cfma(cprev[2], w2, sacc);
            tout[(int64_t)(y + 1) * 2] = cscale((double)tsgn, sacc);
          }
          w2 = w1;
          w1 = tr;
          const double2* tc = rec + TM * TM + tcb;
          cprev[0] = tc[0];
          cprev[1] = tc[1];
          cprev[2] = tc[2];
        }
        cur ^= 1;
      }
      __syncwarp();
      if (lane == 0 && g + NSLOT < ngroups) {
        fence_proxy_async();
        issue_b(g + NSLOT);
      }
    }
    if (tout) {
      double2 sacc = cmul(cprev[1], w1);
      sacc = cfma(cprev[2], w2, sacc);
      tout[0] = cscale((double)tsgn, sacc);
    }
    fence_proxy_async();   // tin / u generic stores before the next task's bulk reads
    __syncwarp();
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

static int slot_table(const Stencil* op, int slot[3][3], Ctx* c) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) slot[i][j] = -1;
  for (int s = 0; s < op->d.S; ++s) {
    const int o0 = op->d.off[s][1], o1 = op->d.off[s][2];
    if (op->d.off[s][0] != 0) return set_error(c, HS_E_SHAPE, "sweep needs 2-D operators");
    slot[o0 + 1][o1 + 1] = s;
  }
  return HS_OK;
}

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
  std::vector<int> fpt(J, -1), bpt(J, -1);
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
    if (j + 1 < J) fpt[j] = (int)beta[j + 1];   // out2 of slab j+1 (1-based) at beta_{j+1}
    if (j > 0) bpt[j] = (int)bt[j];             // out4 at beta~_{j}  (slab index j = (j+1)-1)
  }
  const int TM = s->tm;
  const int FREC = TM == 16 ? Geo<16>::FREC : Geo<32>::FREC;
  const int BREC = TM == 16 ? Geo<16>::BREC : Geo<32>::BREC;
  const size_t frec_bytes = (size_t)J * M * FREC * sizeof(double2);
  const size_t brec_bytes = (size_t)J * M * BREC * sizeof(double2);
  s->factor_bytes = (long long)(frec_bytes + brec_bytes);
  SlabInfo* d_info = nullptr;
  int* d_pts = nullptr;
  unsigned long long* d_err = nullptr;
  auto fail = [&](int code) {
    cudaFree(d_info);
    cudaFree(d_pts);
    cudaFree(d_err);
    sweep_destroy(s);
    return code;
  };
#define HS_TRY(call, what)                                   \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return fail(check_cuda(c, _e, what)); \
  } while (0)
  HS_TRY(cudaMalloc((void**)&s->fwd_rec, frec_bytes), "factor alloc");
  HS_TRY(cudaMalloc((void**)&s->bwd_rec, brec_bytes), "factor alloc");
  HS_TRY(cudaMalloc((void**)&d_info, J * sizeof(SlabInfo)), "slab info alloc");
  HS_TRY(cudaMalloc((void**)&d_pts, 2 * J * sizeof(int)), "alloc");
  HS_TRY(cudaMalloc((void**)&d_err, sizeof(unsigned long long)), "alloc");
  HS_TRY(cudaMemcpyAsync(d_info, info.data(), J * sizeof(SlabInfo), cudaMemcpyHostToDevice,
                         c->stream), "upload");
  HS_TRY(cudaMemcpyAsync(d_pts, fpt.data(), J * sizeof(int), cudaMemcpyHostToDevice, c->stream),
         "upload");
  HS_TRY(cudaMemcpyAsync(d_pts + J, bpt.data(), J * sizeof(int), cudaMemcpyHostToDevice,
                         c->stream), "upload");
  HS_TRY(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), c->stream), "memset");
  {
    const int fsmem = 3 * TM * (TM + 1) * (int)sizeof(double2);
    if (TM == 16) {
      k_slab_factor<16><<<J, 256, fsmem, c->stream>>>(d_info, M, s->fwd_rec, s->bwd_rec, d_err);
    } else {
      HS_TRY(cudaFuncSetAttribute(k_slab_factor<32>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem),
             "factor smem");
      k_slab_factor<32><<<J, 1024, fsmem, c->stream>>>(d_info, M, s->fwd_rec, s->bwd_rec,
                                                        d_err);
    }
  }
  c->launches++;
  HS_TRY(cudaGetLastError(), "slab factor kernel");
  ToutArgs ta{};
  ta.coarse = coarse->d.coeffs;
  ta.n = coarse->d.n;
  if (int r = slot_table(coarse, ta.slot, c)) return fail(r);
  ta.J = J;
  ta.M = M;
  ta.fwd_point = d_pts;
  ta.bwd_point = d_pts + J;
  const int64_t ntout = (int64_t)J * M;
  if (TM == 16)
    k_tout<16><<<(unsigned)((ntout + 255) / 256), 256, 0, c->stream>>>(ta, s->bwd_rec);
  else
    k_tout<32><<<(unsigned)((ntout + 255) / 256), 256, 0, c->stream>>>(ta, s->bwd_rec);
  c->launches++;
  HS_TRY(cudaGetLastError(), "tout kernel");
  unsigned long long err = 0;
  HS_TRY(cudaMemcpyAsync(&err, d_err, sizeof err, cudaMemcpyDeviceToHost, c->stream), "err");
  HS_TRY(cudaStreamSynchronize(c->stream), "factor sync");
  cudaFree(d_info);
  cudaFree(d_pts);
  cudaFree(d_err);
  d_info = nullptr;
  d_pts = nullptr;
  d_err = nullptr;
  if (err != ~0ull) {
    const int slab = (int)(err >> 40);
    const long long row = (long long)(err & 0xffffffffffull);
    char buf[128];
    snprintf(buf, sizeof buf, "zero pivot at row %lld (slab %d)", row, slab + 1);
    sweep_destroy(s);
    return set_error(c, HS_E_ZERO_PIVOT, buf, row);
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
  // consumer side: allocate an incoming buffer
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
  int max_pass = 0;
  // Forward chain j0..j1; the first consumer buffer may come from outside.
  // Returns [first, count); links producers to consumers inside the chain.
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

  // Helper to append a gather + front launches for one pass.
  auto emit_pass = [&](std::vector<SweepLaunch>& plan, int src,
                       std::vector<std::vector<std::vector<SweepTask>>> stages) {
    // stages: sequential launches; each stage = up to 2 fronts (chains)
    const int first = (int)T.size();
    int slot = 0;
    std::vector<std::vector<std::pair<int, int>>> ranges;
    for (auto& st : stages) {
      std::vector<std::pair<int, int>> rs;
      for (auto& fr : st) {
        const int f0 = (int)T.size();
        for (auto t : fr) {
          t.fdslot = slot++;
          t.dst = src;
          T.push_back(t);
        }
        rs.push_back({f0, (int)fr.size()});
      }
      ranges.push_back(rs);
    }
    max_pass = std::max(max_pass, slot);
    SweepLaunch gl{};
    gl.kind = SweepLaunch::kGather;
    gl.src = src;
    gl.first = first;
    gl.count = slot;
    gl.bytes = 2.0 * slot * M * TM * 16.0;
    if (slot) plan.push_back(gl);
    for (auto& rs : ranges) {
      SweepLaunch fl{};
      fl.kind = SweepLaunch::kFront;
      fl.nfront = 0;
      fl.bytes = 0.0;
      for (auto& r : rs) {
        if (r.second == 0) continue;
        fl.ffirst[fl.nfront] = r.first;
        fl.fcount[fl.nfront] = r.second;
        fl.nfront++;
        for (int i = r.first; i < r.first + r.second; ++i) {
          const SweepTask& t = T[i];
          // records + rhs + z round trip + transmission streams + u stores
          double b = (double)M * 16.0 * (FREC + BREC + 3 * TM);
          b += (double)M * 32.0 * ((t.tin1 >= 0) + (t.tin3 >= 0) + (t.out2 >= 0) + (t.out4 >= 0));
          b += (double)M * 16.0 * (t.tb - t.ta);
          fl.bytes += b;
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
#undef HS_TRY
  const size_t tb = T.size() * sizeof(SweepTask);
  cudaError_t e = cudaMalloc((void**)&s->d_tasks, tb);
  if (e == cudaSuccess)
    e = cudaMemcpy(s->d_tasks, T.data(), tb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMalloc((void**)&s->fdpre, (size_t)std::max(1, max_pass) * M * TM * sizeof(double2));
  if (e == cudaSuccess)
    e = cudaMalloc((void**)&s->tin, (size_t)std::max(1, ntin) * M * 2 * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->zs, (size_t)2 * M * TM * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->g, (size_t)s->n0 * M * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->u2, (size_t)s->n0 * M * sizeof(double2));
  if (e == cudaSuccess)
    e = TM == 16 ? cudaFuncSetAttribute(k_front<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Geo<16>::SMEM)
                 : cudaFuncSetAttribute(k_front<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Geo<32>::SMEM);
  if (e != cudaSuccess) {
    sweep_destroy(s);
    return check_cuda(c, e, "sweep buffers");
  }
  *out = s;
  return HS_OK;
}

void sweep_destroy(Sweep* s) {
  if (!s) return;
  cudaFree(s->fwd_rec);
  cudaFree(s->bwd_rec);
  cudaFree(s->fdpre);
  cudaFree(s->tin);
  cudaFree(s->zs);
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
  const int TM = s->tm;
  for (const SweepLaunch& L : s->plan[variant]) {
    switch (L.kind) {
      case SweepLaunch::kCombine: {
        // u = u_pass1 + u_pass2 (the order of the reference's u[ta:tb] += ud)
        const int64_t n = (int64_t)s->n0 * M;
        ProfScope ps(c, K_SWEEP_GATHER, 48.0 * n);
        k_combine<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(u, s->u2, n);
        HS_LAUNCH_CHECK(c, "combine kernel");
        break;
      }
      case SweepLaunch::kGather: {
        dim3 grid((unsigned)((M * TM + 255) / 256), (unsigned)L.count);
        ProfScope ps(c, K_SWEEP_GATHER, L.bytes);
        if (TM == 16)
          k_gather<16><<<grid, 256, 0, c->stream>>>(s->d_tasks, L.first, M, L.src ? s->g : f,
                                                    s->fdpre);
        else
          k_gather<32><<<grid, 256, 0, c->stream>>>(s->d_tasks, L.first, M, L.src ? s->g : f,
                                                    s->fdpre);
        HS_LAUNCH_CHECK(c, "gather kernel");
        break;
      }
      case SweepLaunch::kResidual: {
        int r = stencil_apply(c, s->coarse, u, s->g, 1, f);
        if (r) return r;
        break;
      }
      case SweepLaunch::kFront: {
        FrontArgs fa{};
        fa.tasks = s->d_tasks;
        for (int i = 0; i < 2; ++i) {
          fa.ffirst[i] = i < L.nfront ? L.ffirst[i] : 0;
          fa.fcount[i] = i < L.nfront ? L.fcount[i] : 0;
        }
        fa.fwd_rec = s->fwd_rec;
        fa.bwd_rec = s->bwd_rec;
        fa.fdpre = s->fdpre;
        fa.tin = s->tin;
        fa.zs = s->zs;
        fa.u[0] = u;
        fa.u[1] = s->u2;
        fa.M = M;
        ProfScope ps(c, K_SWEEP_FRONT, L.bytes);
        if (TM == 16)
          k_front<16><<<L.nfront, 32, Geo<16>::SMEM, c->stream>>>(fa);
        else
          k_front<32><<<L.nfront, 32, Geo<32>::SMEM, c->stream>>>(fa);
        HS_LAUNCH_CHECK(c, "front kernel");
        break;
      }
    }
  }
  return HS_OK;
}

}  // namespace hs
