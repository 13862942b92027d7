// GMRES vector kernels: batched dot products, block update, linear
// combination, norms.  Reference: _gmres_cycle (krylov.py:46-102) --
// vdot / axpy / norm on the Arnoldi basis, and the final basis combination.
//
// All are HBM-bound streams.  block_dot reads the k basis vectors and w once
// and produces k dots + ||w||^2 (a classical Gram-Schmidt pass) instead of
// k separate vdot passes; block_update subtracts the projection and emits the
// new norm in the same pass.  Reductions are two-stage (per-block partials,
// then one block in fixed order): bitwise reproducible run to run.

#include "hs_common.cuh"

namespace hs {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxK = 32;

// DGKS gate of the second Gram-Schmidt pass, evaluated on the device so the
// host never has to read the first pass before issuing the second:
// run = ||w_after||^2 < thresh * ||w_before||^2 (the host's test, same double ops).
struct Gate {
  const double2* after;    // null: always run
  const double2* before;
  double thresh;
};

__device__ __forceinline__ bool gate_open(const Gate& g) {
  return g.after == nullptr || g.after->x < g.thresh * g.before->x;
}

// per-block sums of acc[0..W) (fixed order: warp shuffles, then the block's
// warps in order) -> part[blockIdx.x * W + i]; one __syncthreads
template <int W>
__device__ __forceinline__ void block_sums(double2 (&acc)[W], double2* __restrict__ part) {
  __shared__ double2 sh[kThreads / 32][W];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    double2 v = acc[i];
    for (int m = 16; m > 0; m >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
    }
    if (l == 0) sh[w][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < W) {
    double2 s = czero();
    for (int q = 0; q < kThreads / 32; ++q) s = cadd(s, sh[q][threadIdx.x]);
    part[(int64_t)blockIdx.x * W + threadIdx.x] = s;
  }
}

template <int K>
__global__ void __launch_bounds__(kThreads)
k_block_dot(const double2* __restrict__ V, int64_t ldv, const double2* __restrict__ w,
            int64_t n, double2* __restrict__ part, Gate gate) {
  if (!gate_open(gate)) return;
  double2 acc[K + 1];
#pragma unroll
  for (int i = 0; i <= K; ++i) acc[i] = czero();
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads) {
    const double2 wj = __ldg(w + j);
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i] = cfma_conj(__ldg(V + i * ldv + j), wj, acc[i]);
    acc[K].x = fma(wj.x, wj.x, fma(wj.y, wj.y, acc[K].x));
  }
  block_sums<K + 1>(acc, part);
}

// First Gram-Schmidt update fused with the second pass's dots: w' = w - V h
// and, from the same reads of V, the partials of V^H w' and ||w'||^2.  Per
// element the arithmetic (and the grid-stride / reduction order) is that of
// k_block_update followed by k_block_dot: bitwise the same results.
template <int K>
__global__ void __launch_bounds__(kThreads)
k_block_update_dot(const double2* __restrict__ V, int64_t ldv, const double2* __restrict__ h,
                   double2* __restrict__ w, int64_t n, double2* __restrict__ part) {
  __shared__ double2 hv[K];   // broadcast reads (keeps the accumulators in registers)
  if (threadIdx.x < K) hv[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double2 acc[K + 1];
#pragma unroll
  for (int i = 0; i <= K; ++i) acc[i] = czero();
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads) {
    double2 wj = w[j];
#pragma unroll
    for (int i = 0; i < K; ++i) wj = csub(wj, cmul(hv[i], __ldg(V + i * ldv + j)));
    w[j] = wj;
#pragma unroll
    for (int i = 0; i < K; ++i)   // second read of V_ij: an L1 hit
      acc[i] = cfma_conj(__ldg(V + i * ldv + j), wj, acc[i]);
    acc[K].x = fma(wj.x, wj.x, fma(wj.y, wj.y, acc[K].x));
  }
  block_sums<K + 1>(acc, part);
}

template <int K>
__global__ void __launch_bounds__(kThreads)
k_block_update(const double2* __restrict__ V, int64_t ldv, const double2* __restrict__ h,
               double2* __restrict__ w, int64_t n, double2* __restrict__ part, Gate gate) {
  if (!gate_open(gate)) return;
  double2 hv[K > 0 ? K : 1];
#pragma unroll
  for (int i = 0; i < K; ++i) hv[i] = h[i];
  double nrm = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads) {
    double2 wj = w[j];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const double2 v = __ldg(V + i * ldv + j);
      wj = csub(wj, cmul(hv[i], v));
    }
    w[j] = wj;
    nrm = fma(wj.x, wj.x, fma(wj.y, wj.y, nrm));
  }
  double2 acc[1] = {make_double2(nrm, 0.0)};
  block_sums<1>(acc, part);
}

template <int K>
__global__ void __launch_bounds__(kThreads)
k_lincomb(const double2* __restrict__ V, int64_t ldv, const double2* __restrict__ y,
          double2* __restrict__ out, int64_t n) {
  double2 yv[K];
#pragma unroll
  for (int i = 0; i < K; ++i) yv[i] = y[i];
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads) {
    double2 acc = czero();
#pragma unroll
    for (int i = 0; i < K; ++i) acc = cfma(yv[i], __ldg(V + i * ldv + j), acc);
    out[j] = acc;
  }
}

// second stage: out[i] = sum_b part[b][i], fixed order.  A closed gate
// leaves `out` alone, or (pass_through) copies the gate's norm into out[0]
// so the caller always finds the final ||w||^2 in the same slot.
__global__ void k_reduce_parts(const double2* __restrict__ part, int nblk, int width,
                               double2* __restrict__ out, Gate gate, int pass_through) {
  if (!gate_open(gate)) {
    if (pass_through && threadIdx.x == 0) out[0] = *gate.after;
    return;
  }
  // one warp per output column, lanes over the blocks in fixed order; a
  // lane's loads are issued together (independent), then summed in order
  const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
  constexpr int kQ = 8;
  for (int i = wp; i < width; i += kThreads / 32) {
    double2 acc = czero();
    for (int b0 = l; b0 < nblk; b0 += 32 * kQ) {
      double2 v[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int b = b0 + 32 * q;
        v[q] = b < nblk ? __ldcg(part + (int64_t)b * width + i) : czero();
      }
#pragma unroll
      for (int q = 0; q < kQ; ++q) acc = cadd(acc, v[q]);
    }
    for (int m = 16; m > 0; m >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, m);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, m);
    }
    if (l == 0) out[i] = acc;
  }
}

__global__ void k_scale(double2* x, int64_t n, double2 a) {
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads)
    x[j] = cmul(a, x[j]);
}

// x *= 1 / sqrt(max(s.re, 0)): the Arnoldi normalisation with the norm read
// on the device (the host computes the same value for H[k+1,k]).
__global__ void k_scale_inv_sqrt(double2* x, int64_t n, const double2* __restrict__ s) {
  const double2 a = make_double2(1.0 / sqrt(fmax(s->x, 0.0)), 0.0);
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads)
    x[j] = cmul(a, x[j]);
}

__global__ void k_axpby(double2 a, const double2* __restrict__ x, double2 b, double2* y,
                        int64_t n) {
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads)
    y[j] = cfma(a, __ldg(x + j), cmul(b, y[j]));
}

__global__ void k_norm2(const double2* __restrict__ x, int64_t n, double2* part) {
  double s = 0.0, bad = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads) {
    const double2 v = __ldg(x + j);
    if (!isfinite(v.x) || !isfinite(v.y)) bad += 1.0;
    s = fma(v.x, v.x, fma(v.y, v.y, s));
  }
  double2 acc[1] = {make_double2(s, bad)};
  block_sums<1>(acc, part);
}

int grid_for(Ctx* c, int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)c->num_sms * 4;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace

int krylov_block_dot(Ctx* c, const double2* V, int64_t ldv, int k, const double2* w, int64_t n,
                     double2* h, const double2* g_after, const double2* g_before,
                     double thresh) {
  const Gate gate{g_after, g_before, thresh};
  if (k < 0 || k > kMaxK) return set_error(c, HS_E_ARG, "block_dot: k out of range");
  const int nb = grid_for(c, n);
  double2* part = (double2*)scratch(c, (size_t)nb * (k + 1) * sizeof(double2), 2);
  if (!part) return set_error(c, HS_E_CUDA, "scratch allocation failed");
  // (a gated launch usually exits at once -- the host cannot know: its bytes
  // are not counted, so the class's GB/s is that of the ungated passes)
  ProfScope ps(c, K_KRYLOV_DOT, g_after ? 0.0 : 16.0 * (k + 1) * (double)n);
  switch (k) {
#define HS_CASE(KK) \
  case KK: k_block_dot<KK><<<nb, kThreads, 0, c->stream>>>(V, ldv, w, n, part, gate); break;
    HS_CASE(0) HS_CASE(1) HS_CASE(2) HS_CASE(3) HS_CASE(4) HS_CASE(5) HS_CASE(6) HS_CASE(7)
    HS_CASE(8) HS_CASE(9) HS_CASE(10) HS_CASE(11) HS_CASE(12) HS_CASE(13) HS_CASE(14)
    HS_CASE(15) HS_CASE(16) HS_CASE(17) HS_CASE(18) HS_CASE(19) HS_CASE(20) HS_CASE(21)
    HS_CASE(22) HS_CASE(23) HS_CASE(24) HS_CASE(25) HS_CASE(26) HS_CASE(27) HS_CASE(28)
    HS_CASE(29) HS_CASE(30) HS_CASE(31) HS_CASE(32)
#undef HS_CASE
  }
  HS_LAUNCH_CHECK(c, "block_dot");
  k_reduce_parts<<<1, kThreads, 0, c->stream>>>(part, nb, k + 1, h, gate, 0);
  HS_LAUNCH_CHECK(c, "reduce");
  return HS_OK;
}

int krylov_block_update(Ctx* c, const double2* V, int64_t ldv, int k, const double2* h,
                        double2* w, int64_t n, double2* nrm2, const double2* g_after,
                        const double2* g_before, double thresh) {
  const Gate gate{g_after, g_before, thresh};
  if (k < 0 || k > kMaxK) return set_error(c, HS_E_ARG, "block_update: k out of range");
  const int nb = grid_for(c, n);
  double2* part = (double2*)scratch(c, (size_t)nb * sizeof(double2), 2);
  if (!part) return set_error(c, HS_E_CUDA, "scratch allocation failed");
  ProfScope ps(c, K_KRYLOV_UPDATE, g_after ? 0.0 : 16.0 * (k + 2) * (double)n);
  switch (k) {
#define HS_CASE(KK) \
  case KK: k_block_update<KK><<<nb, kThreads, 0, c->stream>>>(V, ldv, h, w, n, part, gate); \
    break;
    HS_CASE(0) HS_CASE(1) HS_CASE(2) HS_CASE(3) HS_CASE(4) HS_CASE(5) HS_CASE(6) HS_CASE(7)
    HS_CASE(8) HS_CASE(9) HS_CASE(10) HS_CASE(11) HS_CASE(12) HS_CASE(13) HS_CASE(14)
    HS_CASE(15) HS_CASE(16) HS_CASE(17) HS_CASE(18) HS_CASE(19) HS_CASE(20) HS_CASE(21)
    HS_CASE(22) HS_CASE(23) HS_CASE(24) HS_CASE(25) HS_CASE(26) HS_CASE(27) HS_CASE(28)
    HS_CASE(29) HS_CASE(30) HS_CASE(31) HS_CASE(32)
#undef HS_CASE
  }
  HS_LAUNCH_CHECK(c, "block_update");
  k_reduce_parts<<<1, kThreads, 0, c->stream>>>(part, nb, 1, nrm2, gate, 1);
  HS_LAUNCH_CHECK(c, "reduce");
  return HS_OK;
}

int krylov_block_update_dot(Ctx* c, const double2* V, int64_t ldv, int k, const double2* h,
                            double2* w, int64_t n, double2* nrm2, double2* h2) {
  if (k < 1 || k > kMaxK) return set_error(c, HS_E_ARG, "block_update_dot: k out of range");
  const int nb = grid_for(c, n);
  double2* part = (double2*)scratch(c, (size_t)nb * (k + 1) * sizeof(double2), 2);
  if (!part) return set_error(c, HS_E_CUDA, "scratch allocation failed");
  ProfScope ps(c, K_KRYLOV_UPDATE, 16.0 * (k + 2) * (double)n);
  switch (k) {
#define HS_CASE(KK) \
  case KK: k_block_update_dot<KK><<<nb, kThreads, 0, c->stream>>>(V, ldv, h, w, n, part); break;
    HS_CASE(1) HS_CASE(2) HS_CASE(3) HS_CASE(4) HS_CASE(5) HS_CASE(6) HS_CASE(7)
    HS_CASE(8) HS_CASE(9) HS_CASE(10) HS_CASE(11) HS_CASE(12) HS_CASE(13) HS_CASE(14)
    HS_CASE(15) HS_CASE(16) HS_CASE(17) HS_CASE(18) HS_CASE(19) HS_CASE(20) HS_CASE(21)
    HS_CASE(22) HS_CASE(23) HS_CASE(24) HS_CASE(25) HS_CASE(26) HS_CASE(27) HS_CASE(28)
    HS_CASE(29) HS_CASE(30) HS_CASE(31) HS_CASE(32)
#undef HS_CASE
  }
  HS_LAUNCH_CHECK(c, "block_update_dot");
  // second-pass dots (and ||w'||^2 at h2[k]), then ||w'||^2 into nrm2 as well
  k_reduce_parts<<<1, kThreads, 0, c->stream>>>(part, nb, k + 1, h2, Gate{nullptr, nullptr, 0.0}, 0);
  HS_LAUNCH_CHECK(c, "reduce");
  cudaMemcpyAsync(nrm2, h2 + k, sizeof(double2), cudaMemcpyDeviceToDevice, c->stream);
  return HS_OK;
}

int krylov_lincomb(Ctx* c, const double2* V, int64_t ldv, int k, const double2* y, double2* out,
                   int64_t n) {
  if (k < 1 || k > kMaxK) return set_error(c, HS_E_ARG, "lincomb: k out of range");
  const int nb = grid_for(c, n);
  ProfScope ps(c, K_KRYLOV_OTHER, 16.0 * (k + 1) * (double)n);
  switch (k) {
#define HS_CASE(KK) \
  case KK: k_lincomb<KK><<<nb, kThreads, 0, c->stream>>>(V, ldv, y, out, n); break;
    HS_CASE(1) HS_CASE(2) HS_CASE(3) HS_CASE(4) HS_CASE(5) HS_CASE(6) HS_CASE(7)
    HS_CASE(8) HS_CASE(9) HS_CASE(10) HS_CASE(11) HS_CASE(12) HS_CASE(13) HS_CASE(14)
    HS_CASE(15) HS_CASE(16) HS_CASE(17) HS_CASE(18) HS_CASE(19) HS_CASE(20) HS_CASE(21)
    HS_CASE(22) HS_CASE(23) HS_CASE(24) HS_CASE(25) HS_CASE(26) HS_CASE(27) HS_CASE(28)
    HS_CASE(29) HS_CASE(30) HS_CASE(31) HS_CASE(32)
#undef HS_CASE
  }
  HS_LAUNCH_CHECK(c, "lincomb");
  return HS_OK;
}

int krylov_scale(Ctx* c, double2* x, int64_t n, double2 a) {
  ProfScope ps(c, K_KRYLOV_OTHER, 32.0 * (double)n);
  k_scale<<<grid_for(c, n), kThreads, 0, c->stream>>>(x, n, a);
  HS_LAUNCH_CHECK(c, "scale");
  return HS_OK;
}

int krylov_scale_inv_sqrt(Ctx* c, double2* x, int64_t n, const double2* s) {
  ProfScope ps(c, K_KRYLOV_OTHER, 32.0 * (double)n);
  k_scale_inv_sqrt<<<grid_for(c, n), kThreads, 0, c->stream>>>(x, n, s);
  HS_LAUNCH_CHECK(c, "scale_inv_sqrt");
  return HS_OK;
}

int krylov_axpby(Ctx* c, double2 a, const double2* x, double2 b, double2* y, int64_t n) {
  ProfScope ps(c, K_KRYLOV_OTHER, 48.0 * (double)n);
  k_axpby<<<grid_for(c, n), kThreads, 0, c->stream>>>(a, x, b, y, n);
  HS_LAUNCH_CHECK(c, "axpby");
  return HS_OK;
}

int krylov_norm2(Ctx* c, const double2* x, int64_t n, double2* out) {
  const int nb = grid_for(c, n);
  double2* part = (double2*)scratch(c, (size_t)nb * sizeof(double2), 2);
  if (!part) return set_error(c, HS_E_CUDA, "scratch allocation failed");
  ProfScope ps(c, K_KRYLOV_OTHER, 16.0 * (double)n);
  k_norm2<<<nb, kThreads, 0, c->stream>>>(x, n, part);
  HS_LAUNCH_CHECK(c, "norm2");
  k_reduce_parts<<<1, kThreads, 0, c->stream>>>(part, nb, 1, out, Gate{nullptr, nullptr, 0.0}, 0);
  HS_LAUNCH_CHECK(c, "reduce");
  return HS_OK;
}

}  // namespace hs
