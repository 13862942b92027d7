// Shared device/host helpers for libhsweep (sm_100a, complex128 = double2).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hsweep.h"

namespace hs {

// ---------------------------------------------------------------------------
// complex128 arithmetic on interleaved (re, im) doubles -- numpy's layout.

__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a * b
__host__ __device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a) * b
__host__ __device__ __forceinline__ double2 cfma_conj(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
__host__ __device__ __forceinline__ double2 cscale(double s, double2 a) {
  return make_double2(s * a.x, s * a.y);
}
__host__ __device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith-free straightforward division (b well scaled here: operator diagonals)
  double d = 1.0 / (b.x * b.x + b.y * b.y);
  return make_double2((a.x * b.x + a.y * b.y) * d, (a.y * b.x - a.x * b.y) * d);
}
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

__device__ __forceinline__ double2 shfl_xor_c(double2 v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  return v;
}

// ---------------------------------------------------------------------------
// Context: device, stream, last error, launch counter, scratch pool.

// Kernel classes for the built-in event profiler (hs_profile_*).
enum KernelClass : int {
  K_STENCIL = 0, K_RESIDUAL, K_JACOBI, K_JACOBI2Z, K_RESTRICT, K_PROLONG, K_SWEEP_GATHER,
  K_SWEEP_FRONT, K_KRYLOV_DOT, K_KRYLOV_UPDATE, K_KRYLOV_OTHER, K_SETUP, K_PRE_FUSED,
  K_POST_FUSED, K_NCLASS
};

struct ProfRec {
  int cls;
  double bytes;
  cudaEvent_t a, b;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string last_error;
  long long last_index = -1;
  long long launches = 0;
  int sweep_segments = 0;         // 2-D sweeps created next: face segments per front (0 = auto)
  int sweep_cluster = 0;          // ... and CTAs (face chunks) per segment's cluster (0 = auto)
  void* scratch[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t scratch_bytes[4] = {0, 0, 0, 0};
  // profiler: CUDA events bracketing every launch when enabled
  bool prof = false;
  std::vector<ProfRec> pending;
  std::vector<cudaEvent_t> pool;
  double prof_ms[K_NCLASS] = {};
  double prof_bytes[K_NCLASS] = {};
  long long prof_count[K_NCLASS] = {};
};

int set_error(Ctx* c, int code, const std::string& msg, long long index = -1);
int check_cuda(Ctx* c, cudaError_t e, const char* what);
void* scratch(Ctx* c, size_t bytes, int which = 0);
cudaEvent_t prof_event(Ctx* c);

// RAII scope: records an event pair around the launches inside it.
struct ProfScope {
  Ctx* c;
  int cls;
  double bytes;
  cudaEvent_t a = nullptr;
  ProfScope(Ctx* ctx, int k, double b) : c(ctx), cls(k), bytes(b) {
    if (c->prof) {
      a = prof_event(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~ProfScope() {
    if (c->prof && a) {
      cudaEvent_t b2 = prof_event(c);
      cudaEventRecord(b2, c->stream);
      c->pending.push_back(ProfRec{cls, bytes, a, b2});
    }
  }
};

#define HS_LAUNCH_CHECK(ctx, what)                                   \
  do {                                                               \
    (ctx)->launches++;                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::hs::check_cuda((ctx), _e, what); \
  } while (0)

#define HS_CUDA(ctx, call, what)                                     \
  do {                                                               \
    cudaError_t _e = (call);                                         \
    if (_e != cudaSuccess) return ::hs::check_cuda((ctx), _e, what); \
  } while (0)

// ---------------------------------------------------------------------------
// Stencil operator on device.  Shapes are canonicalised to 3 axes (n0, n1, n2)
// with the fastest axis last: 2-D (a, b) -> (1, a, b), 1-D (a) -> (1, 1, a).

constexpr int kMaxOffsets = 27;

struct StencilDesc {
  int64_t n0, n1, n2, n;
  int S;                          // stored offsets
  int diag;                       // slot of the (0,0,0) offset or -1
  int8_t off[kMaxOffsets][3];     // canonical offsets
  const double2* coeffs;          // [S][n]
  const double2* invd;            // [n] 1 / diagonal (smoother), or null
};

struct Stencil {
  int dim = 0;                    // user-facing dim (1, 2, 3)
  int64_t shape[3] = {1, 1, 1};   // user-facing shape
  StencilDesc d{};
  double2* coeffs = nullptr;      // owned device copy
  double2* invd = nullptr;        // owned 1 / diagonal
  int has_zero_diag = 0;
  long long zero_diag_node = -1;
};

// descriptor from shape / offsets (hs_abi.cu); coefficients untouched
int stencil_init_desc(Ctx* c, int dim, const int64_t* shape, int S, const int8_t* offsets,
                      Stencil* op);
// device-side completion of an operator whose coefficients were assembled on
// the device: 1/diagonal and the first zero-diagonal node (hs_assemble.cu)
int stencil_finish_device(Ctx* c, Stencil* op);

// kernels (hs_stencil.cu)
int stencil_apply(Ctx* c, const Stencil* op, const double2* x, double2* y, int nrhs,
                  const double2* f_minus /*if non-null: y = f - A x*/);
// fused 2-D V-cycle halves (nu = 2; hs_stencil.cu): pre = two Jacobi steps
// from zero + residual (-> u2, r); post = prolongation-correction + two
// Jacobi steps (u2, uc -> u)
struct Transfer;
bool fused2d_ok(const Stencil* op, const Transfer* t, int nu);
int stencil_pre2d(Ctx* c, const Stencil* op, const double2* f, double2* u2, double2* r,
                  double omega);
int stencil_post2d(Ctx* c, const Stencil* op, const Transfer* t, const double2* uc,
                   const double2* f, const double2* u2, double2* u, double omega);
int stencil_jacobi(Ctx* c, const Stencil* op, double2* u, const double2* f, double omega,
                   int steps, int u_is_zero, int nrhs);

}  // namespace hs

// opaque C-ABI handle types of the context and of stencil operators (the
// other handles are declared where their implementation lives)
struct hs_ctx : hs::Ctx {};
struct hs_stencil : hs::Stencil {};
