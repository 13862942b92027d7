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

__device__ __forceinline__ double2 block_sum(double2 v, double2* sh) {
  // sum over the block; result valid in thread 0
  for (int m = 16; m > 0; m >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double2 s = czero();
  if (threadIdx.x == 0)
    for (int i = 0; i < kThreads / 32; ++i) s = cadd(s, sh[i]);
  return s;
}

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
  __shared__ double2 sh[kThreads / 32];
#pragma unroll
  for (int i = 0; i <= K; ++i) {
    const double2 s = block_sum(acc[i], sh);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.x * (K + 1) + i] = s;
  }
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
  __shared__ double2 sh[kThreads / 32];
  const double2 s = block_sum(make_double2(nrm, 0.0), sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
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
  __shared__ double2 sh[kThreads / 32];
  for (int i = 0; i < width; ++i) {
    double2 acc = czero();
    for (int b = threadIdx.x; b < nblk; b += kThreads) acc = cadd(acc, part[(int64_t)b * width + i]);
    const double2 s = block_sum(acc, sh);
    if (threadIdx.x == 0) out[i] = s;
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
  __shared__ double2 sh[kThreads / 32];
  const double2 r = block_sum(make_double2(s, bad), sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
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
  ProfScope ps(c, K_KRYLOV_DOT, 16.0 * (k + 1) * (double)n);
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
  ProfScope ps(c, K_KRYLOV_UPDATE, 16.0 * (k + 2) * (double)n);
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
