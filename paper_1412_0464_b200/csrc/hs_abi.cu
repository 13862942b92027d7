// extern "C" boundary of libhsweep (declarations and reference citations in
// include/hsweep.h).  Handles own their device memory; vectors are borrowed
// device pointers; all work is ordered on the context stream.

#include "hs_common.cuh"
#include <vector>
#include "hs_sweep.cuh"
#include "hs_transfer.cuh"

#include <algorithm>
#include <cmath>
#include <new>

namespace hs {

int set_error(Ctx* c, int code, const std::string& msg, long long index) {
  if (c) {
    c->last_error = msg;
    c->last_index = index;
  }
  return code;
}

int check_cuda(Ctx* c, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_error(c, HS_E_CUDA, m);
}

void* scratch(Ctx* c, size_t bytes, int which) {
  if (which < 0 || which > 3) return nullptr;
  if (c->scratch_bytes[which] >= bytes) return c->scratch[which];
  if (c->scratch[which]) {
    cudaStreamSynchronize(c->stream);
    cudaFree(c->scratch[which]);
    c->scratch[which] = nullptr;
    c->scratch_bytes[which] = 0;
  }
  const size_t want = std::max<size_t>(bytes, 1 << 20);
  if (cudaMalloc(&c->scratch[which], want) != cudaSuccess) return nullptr;
  c->scratch_bytes[which] = want;
  return c->scratch[which];
}

cudaEvent_t prof_event(Ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

static int prof_collect(Ctx* c) {
  if (c->pending.empty()) return HS_OK;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return check_cuda(c, e, "profile sync");
  for (const ProfRec& r : c->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    c->prof_ms[r.cls] += ms;
    c->prof_bytes[r.cls] += r.bytes;
    c->prof_count[r.cls] += 1;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->pending.clear();
  return HS_OK;
}

// declared in the kernel translation units
int krylov_block_dot(Ctx*, const double2*, int64_t, int, const double2*, int64_t, double2*,
                     const double2*, const double2*, double);
int krylov_block_update_dot(Ctx*, const double2*, int64_t, int, const double2*, double2*, int64_t,
                            double2*, double2*);
int krylov_block_update(Ctx*, const double2*, int64_t, int, const double2*, double2*, int64_t,
                        double2*, const double2*, const double2*, double);
int krylov_scale_inv_sqrt(Ctx*, double2*, int64_t, const double2*);
int krylov_lincomb(Ctx*, const double2*, int64_t, int, const double2*, double2*, int64_t);
int krylov_scale(Ctx*, double2*, int64_t, double2);
int krylov_axpby(Ctx*, double2, const double2*, double2, double2*, int64_t);
int krylov_norm2(Ctx*, const double2*, int64_t, double2*);

// Two-grid cycle (twogrid.py:119-164): fine smoother, transfers, sweep.
struct Cycle {
  const Stencil* fine = nullptr;
  const Transfer* t = nullptr;
  const Stencil* coarse = nullptr;
  Sweep* sweep = nullptr;
  double omega = 0.8;
  int nu = 2;
  double scale = 1.0;
  int variant = HS_VARIANT_X;
  double2* rc = nullptr;   // coarse right-hand side
  double2* uc = nullptr;   // coarse solution
  double2* r = nullptr;    // fine residual scratch
  double2* tmp = nullptr;  // fine M f for apply_a
  SweepWork work{};        // lane-private sweep scratch (null: the sweep's own)
  bool lane = false;
  bool fused = false;      // 2-D, nu = 2: fused pre / post kernels (u2 holds the pre-smoothed u)
  double2* u2 = nullptr;
  // scratch of vcycle_many (lazy): nb right-hand sides' rc, uc and (fused) u2
  int nb = 0;
  double2 *brc = nullptr, *buc = nullptr, *bu2 = nullptr;
};

static bool want_fused(const Stencil* fine, const Transfer* t, int nu) {
  static const bool off = getenv("HS_NO_FUSE") != nullptr;   // A/B switch
  return !off && fused2d_ok(fine, t, nu);
}

// First half of the cycle: pre-smoothing from zero, residual, restriction
// (everything before the coarse solve).
static int vcycle_begin(Ctx* c, Cycle* cy, const double2* f, double2* u) {
  const int64_t nf = cy->fine->d.n;
  int r;
  if (cy->fused) {   // u2 = S_pre(0), r = f - A u2 in one pass; then h^d P^T r
    if ((r = stencil_pre2d(c, cy->fine, f, cy->u2, cy->r, cy->omega))) return r;
    return transfer_restrict(c, cy->t, cy->r, cy->rc, cy->scale, 1);
  }
  if (cy->nu > 0) {
    r = stencil_jacobi(c, cy->fine, u, f, cy->omega, cy->nu, 1, 1);
  } else {
    cudaError_t e = cudaMemsetAsync(u, 0, nf * sizeof(double2), c->stream);
    r = e == cudaSuccess ? HS_OK : check_cuda(c, e, "memset");
  }
  if (r) return r;
  if ((r = stencil_apply(c, cy->fine, u, cy->r, 1, f))) return r;              // r = f - A u
  return transfer_restrict(c, cy->t, cy->r, cy->rc, cy->scale, 1);             // h^d P^T r
}

// Second half: coarse sweep (plan launches [sweep_first, end)), prolongation
// + correction, post-smoothing.
static int vcycle_end(Ctx* c, Cycle* cy, const double2* f, double2* u, int sweep_first = 0) {
  int r;
  if ((r = sweep_apply(c, cy->sweep, cy->variant, cy->rc, cy->uc,
                       cy->lane ? &cy->work : nullptr, sweep_first)))
    return r;                                                                    // coarse solve
  if (cy->fused)   // u = S_post(u2 + P uc) in one pass
    return stencil_post2d(c, cy->fine, cy->t, cy->uc, f, cy->u2, u, cy->omega);
  if ((r = transfer_prolong(c, cy->t, cy->uc, u, 1, 1))) return r;             // u += P uc
  if (cy->nu > 0) r = stencil_jacobi(c, cy->fine, u, f, cy->omega, cy->nu, 0, 1);
  return r;
}

static int vcycle(Ctx* c, Cycle* cy, const double2* f, double2* u) {
  int r = vcycle_begin(c, cy, f, u);
  return r ? r : vcycle_end(c, cy, f, u);
}

// nrhs cycles u_r = M f_r (vectors at f + r * stride, u + r * stride): the
// fine-level halves per right-hand side, the coarse sweeps of all of them
// through one chain of slab solves (sweep_apply_many).  Per right-hand side
// the kernels and their arithmetic are those of vcycle().
static int vcycle_many(Ctx* c, Cycle* cy, int nrhs, const double2* f, double2* u, int64_t stride) {
  if (nrhs == 1) return vcycle(c, cy, f, u);
  const int64_t nf = cy->fine->d.n, nc = cy->coarse->d.n;
  if (stride < nf) return set_error(c, HS_E_ARG, "right-hand-side stride shorter than a vector");
  if (cy->nb < nrhs) {
    cudaStreamSynchronize(c->stream);
    cudaFree(cy->brc); cudaFree(cy->buc); cudaFree(cy->bu2);
    cy->brc = cy->buc = cy->bu2 = nullptr;
    cy->nb = 0;
    cudaError_t e = cudaMalloc((void**)&cy->brc, (size_t)nrhs * nc * sizeof(double2));
    if (e == cudaSuccess) e = cudaMalloc((void**)&cy->buc, (size_t)nrhs * nc * sizeof(double2));
    if (e == cudaSuccess && cy->fused) e = cudaMalloc((void**)&cy->bu2, (size_t)nrhs * nf * sizeof(double2));
    if (e != cudaSuccess) return check_cuda(c, e, "multi-right-hand-side cycle buffers");
    cy->nb = nrhs;
  }
  int r;
  for (int k = 0; k < nrhs; ++k) {   // pre-smoothing from zero, residual, restriction
    const double2* fk = f + k * stride;
    double2* uk = u + k * stride;
    if (cy->fused) {
      if ((r = stencil_pre2d(c, cy->fine, fk, cy->bu2 + k * nf, cy->r, cy->omega))) return r;
    } else {
      if (cy->nu > 0) {
        r = stencil_jacobi(c, cy->fine, uk, fk, cy->omega, cy->nu, 1, 1);
      } else {
        cudaError_t e = cudaMemsetAsync(uk, 0, nf * sizeof(double2), c->stream);
        r = e == cudaSuccess ? HS_OK : check_cuda(c, e, "memset");
      }
      if (r) return r;
      if ((r = stencil_apply(c, cy->fine, uk, cy->r, 1, fk))) return r;
    }
    if ((r = transfer_restrict(c, cy->t, cy->r, cy->brc + k * nc, cy->scale, 1))) return r;
  }
  if ((r = sweep_apply_many(c, cy->sweep, cy->variant, nrhs, cy->brc, cy->buc, nc,
                            cy->lane ? &cy->work : nullptr)))
    return r;
  for (int k = 0; k < nrhs; ++k) {   // prolongation + correction, post-smoothing
    const double2* fk = f + k * stride;
    double2* uk = u + k * stride;
    if (cy->fused) {
      if ((r = stencil_post2d(c, cy->fine, cy->t, cy->buc + k * nc, fk, cy->bu2 + k * nf, uk, cy->omega)))
        return r;
    } else {
      if ((r = transfer_prolong(c, cy->t, cy->buc + k * nc, uk, 1, 1))) return r;
      if (cy->nu > 0 && (r = stencil_jacobi(c, cy->fine, uk, fk, cy->omega, cy->nu, 0, 1))) return r;
    }
  }
  return HS_OK;
}

// Stencil descriptor from (dim, shape, offsets); coefficients not touched.
int stencil_init_desc(Ctx* c, int dim, const int64_t* shape, int S, const int8_t* offsets,
                      Stencil* op) {
  if (dim < 1 || dim > 3) return set_error(c, HS_E_SHAPE, "stencil dim must be 1, 2 or 3");
  if (S < 1 || S > kMaxOffsets) return set_error(c, HS_E_SHAPE, "stencil needs 1..27 offsets");
  op->dim = dim;
  int64_t n = 1;
  for (int a = 0; a < dim; ++a) {
    if (shape[a] < 1) return set_error(c, HS_E_SHAPE, "empty stencil shape");
    op->shape[a] = shape[a];
    n *= shape[a];
  }
  int64_t cs[3] = {1, 1, 1};
  for (int a = 0; a < dim; ++a) cs[3 - dim + a] = shape[a];
  op->d.n0 = cs[0];
  op->d.n1 = cs[1];
  op->d.n2 = cs[2];
  op->d.n = n;
  op->d.S = S;
  op->d.diag = -1;
  for (int s = 0; s < S; ++s) {
    int8_t o[3] = {0, 0, 0};
    bool zero = true;
    for (int a = 0; a < dim; ++a) {
      const int8_t v = offsets[s * dim + a];
      if (v < -1 || v > 1) return set_error(c, HS_E_SHAPE, "offset breaks the compact-stencil contract");
      o[3 - dim + a] = v;
      zero = zero && v == 0;
    }
    for (int a = 0; a < 3; ++a) op->d.off[s][a] = o[a];
    if (zero) op->d.diag = s;
  }
  return HS_OK;
}

}  // namespace hs

using namespace hs;

struct hs_transfer : Transfer {};
struct hs_sweep : Sweep {};
struct hs_cycle : Cycle {};

extern "C" {

int hs_version(void) { return 1; }

int hs_ctx_create(int device, hs_ctx** out) {
  if (!out) return HS_E_ARG;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return HS_E_CUDA;
  hs_ctx* c = new (std::nothrow) hs_ctx();
  if (!c) return HS_E_ARG;
  c->device = device;
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess)
    c->num_sms = sms;
  *out = c;
  return HS_OK;
}

int hs_ctx_destroy(hs_ctx* c) {
  if (!c) return HS_OK;
  cudaStreamSynchronize(c->stream);
  for (int i = 0; i < 4; ++i)
    if (c->scratch[i]) cudaFree(c->scratch[i]);
  delete c;
  return HS_OK;
}

int hs_ctx_set_sweep_segments(hs_ctx* c, int segments) {
  if (!c || segments < 0) return HS_E_ARG;
  c->sweep_segments = segments;
  return HS_OK;
}

int hs_ctx_set_sweep_cluster(hs_ctx* c, int ctas) {
  if (!c || ctas < 0) return HS_E_ARG;
  c->sweep_cluster = ctas;
  return HS_OK;
}

int hs_ctx_set_stream(hs_ctx* c, void* stream) {
  if (!c) return HS_E_ARG;
  c->stream = (cudaStream_t)stream;
  return HS_OK;
}

const char* hs_last_error(hs_ctx* c) { return c ? c->last_error.c_str() : "null context"; }
long long hs_last_error_index(hs_ctx* c) { return c ? c->last_index : -1; }
long long hs_launch_count(hs_ctx* c) { return c ? c->launches : 0; }

int hs_profile_enable(hs_ctx* c, int on) {
  if (!c) return HS_E_ARG;
  if (!on) prof_collect(c);
  c->prof = on != 0;
  return HS_OK;
}

int hs_profile_reset(hs_ctx* c) {
  if (!c) return HS_E_ARG;
  int r = prof_collect(c);
  for (int i = 0; i < K_NCLASS; ++i) {
    c->prof_ms[i] = 0.0;
    c->prof_bytes[i] = 0.0;
    c->prof_count[i] = 0;
  }
  return r;
}

int hs_profile_read(hs_ctx* c, int nclass, double* ms, double* bytes, long long* counts) {
  if (!c || nclass < 0) return HS_E_ARG;
  int r = prof_collect(c);
  for (int i = 0; i < nclass && i < K_NCLASS; ++i) {
    if (ms) ms[i] = c->prof_ms[i];
    if (bytes) bytes[i] = c->prof_bytes[i];
    if (counts) counts[i] = c->prof_count[i];
  }
  return r;
}

int hs_synchronize(hs_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return check_cuda(c, e, "synchronize");
  return HS_OK;
}

// ---------------------------------------------------------------------------
int hs_stencil_create(hs_ctx* c, int dim, const int64_t* shape, int S, const int8_t* offsets,
                      const double* coeffs, hs_stencil** out) {
  if (!c || !out || !shape || !offsets || !coeffs) return HS_E_ARG;
  hs_stencil* op = new hs_stencil();
  if (int r = stencil_init_desc(c, dim, shape, S, offsets, op)) {
    delete op;
    return r;
  }
  const int64_t n = op->d.n;
  // zero-diagonal scan (jacobi_smooth's ZeroDivisionError, twogrid.py:43-46)
  if (op->d.diag >= 0) {
    const double* dg = coeffs + (size_t)2 * n * op->d.diag;
    for (int64_t i = 0; i < n; ++i) {
      if (dg[2 * i] == 0.0 && dg[2 * i + 1] == 0.0) {
        op->has_zero_diag = 1;
        op->zero_diag_node = i;
        break;
      }
    }
  }
  const size_t bytes = (size_t)S * n * sizeof(double2);
  cudaError_t e = cudaMalloc((void**)&op->coeffs, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(op->coeffs, coeffs, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(op->coeffs);
    delete op;
    return check_cuda(c, e, "stencil upload");
  }
  op->d.coeffs = op->coeffs;
  op->d.invd = nullptr;
  if (op->d.diag >= 0 && !op->has_zero_diag) {   // 1/diag for the smoother (products, no divisions)
    const double* dg = coeffs + (size_t)2 * n * op->d.diag;
    std::vector<double> inv((size_t)2 * n);
    for (int64_t i = 0; i < n; ++i) {
      const double re = dg[2 * i], im = dg[2 * i + 1], d = 1.0 / (re * re + im * im);
      inv[2 * i] = re * d;
      inv[2 * i + 1] = -im * d;
    }
    e = cudaMalloc((void**)&op->invd, (size_t)n * sizeof(double2));
    if (e == cudaSuccess)
      e = cudaMemcpy(op->invd, inv.data(), (size_t)n * sizeof(double2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(op->coeffs);
      cudaFree(op->invd);
      delete op;
      return check_cuda(c, e, "stencil upload");
    }
    op->d.invd = op->invd;
  }
  *out = op;
  return HS_OK;
}

int hs_stencil_download(hs_ctx* c, const hs_stencil* op, double* coeffs) {
  if (!c || !op || !coeffs) return HS_E_ARG;
  HS_CUDA(c, cudaStreamSynchronize(c->stream), "download sync");
  HS_CUDA(c, cudaMemcpy(coeffs, op->coeffs, (size_t)op->d.S * op->d.n * sizeof(double2),
                        cudaMemcpyDeviceToHost), "stencil download");
  return HS_OK;
}

int hs_stencil_destroy(hs_ctx* c, hs_stencil* op) {
  (void)c;
  if (!op) return HS_OK;
  cudaFree(op->coeffs);
  cudaFree(op->invd);
  delete op;
  return HS_OK;
}

int hs_stencil_apply(hs_ctx* c, const hs_stencil* op, const void* x, void* y, int nrhs) {
  if (!c || !op || !x || !y || nrhs < 1) return HS_E_ARG;
  return stencil_apply(c, op, (const double2*)x, (double2*)y, nrhs, nullptr);
}

int hs_stencil_residual(hs_ctx* c, const hs_stencil* op, const void* f, const void* u, void* r,
                        int nrhs) {
  if (!c || !op || !f || !u || !r || nrhs < 1) return HS_E_ARG;
  return stencil_apply(c, op, (const double2*)u, (double2*)r, nrhs, (const double2*)f);
}

int hs_jacobi(hs_ctx* c, const hs_stencil* op, void* u, const void* f, double omega, int steps,
              int u_is_zero, int nrhs) {
  if (!c || !op || !u || !f || nrhs < 1 || steps < 0) return HS_E_ARG;
  return stencil_jacobi(c, op, (double2*)u, (const double2*)f, omega, steps, u_is_zero, nrhs);
}

// ---------------------------------------------------------------------------
int hs_transfer_create(hs_ctx* c, int dim, const int64_t* fp_len, const int64_t* fp_concat,
                       const uint8_t* refined_concat, hs_transfer** out) {
  if (!c || !out || !fp_len || !fp_concat || !refined_concat) return HS_E_ARG;
  Transfer* t = nullptr;
  int r = transfer_create(c, dim, fp_len, fp_concat, refined_concat, &t);
  if (r) return r;
  hs_transfer* h = new hs_transfer();
  *(Transfer*)h = *t;
  delete t;
  *out = h;
  return HS_OK;
}

int hs_transfer_create_window(hs_ctx* c, int dim, const int64_t* fp_len,
                              const int64_t* fp_concat, const uint8_t* refined_concat,
                              const int64_t* window, hs_transfer** out) {
  if (!c || !out || !fp_len || !fp_concat || !refined_concat || !window) return HS_E_ARG;
  Transfer* t = nullptr;
  int r = transfer_create(c, dim, fp_len, fp_concat, refined_concat, &t, window);
  if (r) return r;
  hs_transfer* h = new hs_transfer();
  static_cast<Transfer&>(*h) = *t;
  delete t;
  *out = h;
  return HS_OK;
}

int hs_transfer_destroy(hs_ctx* c, hs_transfer* t) {
  (void)c;
  if (!t) return HS_OK;
  cudaFree(t->buf);
  delete t;
  return HS_OK;
}

int hs_restrict(hs_ctx* c, const hs_transfer* t, const void* r_fine, void* rc, double scale,
                int nrhs) {
  if (!c || !t || !r_fine || !rc || nrhs < 1) return HS_E_ARG;
  return transfer_restrict(c, t, (const double2*)r_fine, (double2*)rc, scale, nrhs);
}

int hs_restrict_residual(hs_ctx* c, const hs_transfer* t, const hs_stencil* op, const void* u,
                         const void* f, void* rc, double scale, int nrhs) {
  if (!c || !t || !op || !u || !f || !rc || nrhs < 1) return HS_E_ARG;
  double2* r = (double2*)scratch(c, (size_t)op->d.n * nrhs * sizeof(double2), 0);
  if (!r) return set_error(c, HS_E_CUDA, "scratch allocation failed");
  int e = stencil_apply(c, op, (const double2*)u, r, nrhs, (const double2*)f);
  if (e) return e;
  return transfer_restrict(c, t, r, (double2*)rc, scale, nrhs);
}

int hs_prolong_add(hs_ctx* c, const hs_transfer* t, const void* uc, void* u, int accumulate,
                   int nrhs) {
  if (!c || !t || !uc || !u || nrhs < 1) return HS_E_ARG;
  return transfer_prolong(c, t, (const double2*)uc, (double2*)u, accumulate, nrhs);
}

// ---------------------------------------------------------------------------
int hs_sweep_create(hs_ctx* c, const hs_stencil* coarse, int J, const int64_t* beta,
                    const int64_t* beta_tilde, const int64_t* slab_lo, const int64_t* slab_hi,
                    const hs_stencil* const* slab_ops, hs_sweep** out) {
  if (!c || !coarse || !beta || !beta_tilde || !slab_lo || !slab_hi || !slab_ops || !out)
    return HS_E_ARG;
  std::vector<const Stencil*> ops(J);
  for (int j = 0; j < J; ++j) ops[j] = slab_ops[j];
  Sweep* s = nullptr;
  int r = sweep_create(c, coarse, J, beta, beta_tilde, slab_lo, slab_hi, ops.data(), &s);
  if (r) return r;
  *out = reinterpret_cast<hs_sweep*>(s);
  return HS_OK;
}

int hs_sweep_solve_one(hs_ctx* c, hs_sweep* s, int j, int64_t a, int64_t b, int64_t ta,
                       int64_t tb, const void* B1, const void* B3, void* out2, void* out4,
                       const void* f, void* u) {
  if (!c || !s || !f || !u) return HS_E_ARG;
  return sweep_solve_one(c, s, j, a, b, ta, tb, (const double2*)B1, (const double2*)B3,
                         (double2*)out2, (double2*)out4, (const double2*)f, (double2*)u);
}

int hs_exact_create(hs_ctx* c, const hs_stencil* op, hs_sweep** out) {
  if (!c || !op || !out) return HS_E_ARG;
  Sweep* s = nullptr;
  int r = exact_create(c, op, &s);
  if (r) return r;
  *out = reinterpret_cast<hs_sweep*>(s);
  return HS_OK;
}

int hs_exact_create_csr(hs_ctx* c, int64_t n, int64_t nnz, const int64_t* indptr,
                        const int64_t* indices, const double* vals, int block, hs_sweep** out) {
  if (!c || !indptr || (nnz > 0 && (!indices || !vals)) || !out) return HS_E_ARG;
  Sweep* s = nullptr;
  int r = exact_create_csr(c, n, nnz, indptr, indices, (const double2*)vals, block, &s);
  if (r) return r;
  *out = reinterpret_cast<hs_sweep*>(s);
  return HS_OK;
}

int hs_sweep_destroy(hs_ctx* c, hs_sweep* s) {
  (void)c;
  sweep_destroy(s);
  return HS_OK;
}

int hs_sweep_apply(hs_ctx* c, hs_sweep* s, int variant, const void* f, void* u) {
  if (!c || !s || !f || !u) return HS_E_ARG;
  return sweep_apply(c, s, variant, (const double2*)f, (double2*)u);
}

int hs_sweep_apply_many(hs_ctx* c, hs_sweep* s, int variant, int nrhs, const void* f, void* u,
                        long long stride) {
  if (!c || !s || !f || !u) return HS_E_ARG;
  return sweep_apply_many(c, s, variant, nrhs, (const double2*)f, (double2*)u, stride);
}

int hs_sweep_rhs_width(hs_sweep* s) { return s ? s->max_nr : 1; }
int hs_sweep_max_fronts(hs_sweep* s) { return s && !s->s3 ? s->max_fronts : 0; }

int hs_sweep_plan_nx(hs_ctx* c, hs_sweep* s, int ncell, const int64_t* j_cell,
                     const int64_t* j_mid, int* variant) {
  if (!c || !s || !j_cell || !j_mid || !variant) return HS_E_ARG;
  return sweep_plan_nx(c, s, ncell, j_cell, j_mid, variant);
}

int hs_sweep_plan_relay(hs_ctx* c, hs_sweep* s, int shards, int* variant) {
  if (!c || !s || !variant) return HS_E_ARG;
  return sweep_plan_relay(c, s, shards, variant);
}

long long hs_sweep_factor_bytes(hs_sweep* s) { return s ? s->factor_bytes : 0; }

int hs_sweep_segments(hs_sweep* s) { return s && !s->s3 ? s->G : 1; }
int hs_sweep_chunks(hs_sweep* s) { return s && !s->s3 ? s->C : 0; }

int hs_sweep_plan_launches(hs_sweep* s, int variant) {
  if (!s || !s->has_plan(variant)) return 0;
  int n = 0;
  for (const auto& fl : s->plan[variant]) n += fl.kind == SweepLaunch::kSolve;
  return n;
}

// ---------------------------------------------------------------------------
int hs_cycle_create(hs_ctx* c, const hs_stencil* fine, const hs_transfer* t,
                    const hs_stencil* coarse, hs_sweep* sweep, double omega_jac, int nu,
                    double restrict_scale, int variant, hs_cycle** out) {
  if (!c || !fine || !t || !coarse || !sweep || !out || nu < 0) return HS_E_ARG;
  if (!sweep->has_plan(variant))
    return set_error(c, HS_E_ARG, variant == HS_VARIANT_X ? "X-sweep needs an even subdomain count"
                                                          : "unknown sweep variant");
  if (t->d.nf[0] * t->d.nf[1] * t->d.nf[2] != fine->d.n ||
      t->d.nc[0] * t->d.nc[1] * t->d.nc[2] != coarse->d.n)
    return set_error(c, HS_E_SHAPE, "coarsening map does not match the operators");
  if (nu > 0 && (fine->d.diag < 0 || fine->has_zero_diag)) {
    char buf[128];
    snprintf(buf, sizeof buf, "zero operator diagonal at node %lld", fine->zero_diag_node);
    return set_error(c, HS_E_ZERO_DIAG, buf, fine->zero_diag_node);
  }
  hs_cycle* cy = new hs_cycle();
  cy->fine = fine;
  cy->t = t;
  cy->coarse = coarse;
  cy->sweep = sweep;
  cy->omega = omega_jac;
  cy->nu = nu;
  cy->scale = restrict_scale;
  cy->variant = variant;
  cy->fused = want_fused(fine, t, nu);
  cudaError_t e = cudaMalloc((void**)&cy->rc, coarse->d.n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&cy->uc, coarse->d.n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&cy->r, fine->d.n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&cy->tmp, fine->d.n * sizeof(double2));
  if (e == cudaSuccess && cy->fused) e = cudaMalloc((void**)&cy->u2, fine->d.n * sizeof(double2));
  if (e != cudaSuccess) {
    cudaFree(cy->rc); cudaFree(cy->uc); cudaFree(cy->r); cudaFree(cy->tmp); cudaFree(cy->u2);
    delete cy;
    return check_cuda(c, e, "cycle buffers");
  }
  *out = cy;
  return HS_OK;
}

int hs_cycle_create_lane(hs_ctx* c, const hs_cycle* base, hs_cycle** out) {
  if (!c || !base || !out) return HS_E_ARG;
  hs_cycle* cy = new hs_cycle();
  cy->fine = base->fine;
  cy->t = base->t;
  cy->coarse = base->coarse;
  cy->sweep = base->sweep;
  cy->omega = base->omega;
  cy->nu = base->nu;
  cy->scale = base->scale;
  cy->variant = base->variant;
  cy->lane = true;
  // (as wide as the sweep's widest kernel: a lane can run hs_vcycle_many)
  if (int r = sweep_work_create(c, cy->sweep, &cy->work, std::max(1, cy->sweep->max_nr))) {
    delete cy;
    return r;
  }
  cy->fused = base->fused;
  cudaError_t e = cudaMalloc((void**)&cy->rc, cy->coarse->d.n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&cy->uc, cy->coarse->d.n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&cy->r, cy->fine->d.n * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc((void**)&cy->tmp, cy->fine->d.n * sizeof(double2));
  if (e == cudaSuccess && cy->fused) e = cudaMalloc((void**)&cy->u2, cy->fine->d.n * sizeof(double2));
  if (e != cudaSuccess) {
    cudaFree(cy->rc); cudaFree(cy->uc); cudaFree(cy->r); cudaFree(cy->tmp); cudaFree(cy->u2);
    sweep_work_destroy(&cy->work);
    delete cy;
    return check_cuda(c, e, "cycle lane buffers");
  }
  *out = cy;
  return HS_OK;
}

int hs_cycle_destroy(hs_ctx* c, hs_cycle* cy) {
  (void)c;
  if (!cy) return HS_OK;
  cudaFree(cy->rc); cudaFree(cy->uc); cudaFree(cy->r); cudaFree(cy->tmp); cudaFree(cy->u2);
  cudaFree(cy->brc); cudaFree(cy->buc); cudaFree(cy->bu2);
  if (cy->lane) sweep_work_destroy(&cy->work);
  delete cy;
  return HS_OK;
}

int hs_vcycle(hs_ctx* c, hs_cycle* cy, const void* f, void* u) {
  if (!c || !cy || !f || !u) return HS_E_ARG;
  return vcycle(c, cy, (const double2*)f, (double2*)u);
}

int hs_vcycle_many(hs_ctx* c, hs_cycle* cy, int nrhs, const void* f, void* u, long long stride) {
  if (!c || !cy || !f || !u || nrhs < 1) return HS_E_ARG;
  return vcycle_many(c, cy, nrhs, (const double2*)f, (double2*)u, stride);
}

int hs_vcycle_apply_a(hs_ctx* c, hs_cycle* cy, const void* f, void* w) {
  if (!c || !cy || !f || !w) return HS_E_ARG;
  int r = vcycle(c, cy, (const double2*)f, cy->tmp);
  if (r) return r;
  return stencil_apply(c, cy->fine, cy->tmp, (double2*)w, 1, nullptr);
}

int hs_vcycle_apply_a_begin(hs_ctx* c, hs_cycle* cy, const void* f) {
  if (!c || !cy || !f) return HS_E_ARG;
  return vcycle_begin(c, cy, (const double2*)f, cy->tmp);
}

int hs_vcycle_apply_a_part(hs_ctx* c, hs_cycle* cy, const void* f, void* w, int part) {
  if (!c || !cy || !f || (part == 2 && !w)) return HS_E_ARG;
  switch (part) {
    case 0:
      return vcycle_begin(c, cy, (const double2*)f, cy->tmp);
    case 1:   // the sweep's first launch (X: both pass-1 fronts)
      return sweep_apply(c, cy->sweep, cy->variant, cy->rc, cy->uc,
                         cy->lane ? &cy->work : nullptr, 0, 1);
    case 2: {
      int r = vcycle_end(c, cy, (const double2*)f, cy->tmp, 1);
      if (r) return r;
      return stencil_apply(c, cy->fine, cy->tmp, (double2*)w, 1, nullptr);
    }
    default:
      return set_error(c, HS_E_ARG, "apply_a part must be 0, 1 or 2");
  }
}

int hs_vcycle_apply_az_part(hs_ctx* c, hs_cycle* cy, const void* f, void* z, void* w, int part) {
  if (!c || !cy || !f || !z || (part != 1 && part != 0 && !w)) return HS_E_ARG;
  switch (part) {
    case 0:
      return vcycle_begin(c, cy, (const double2*)f, (double2*)z);
    case 1:
      return sweep_apply(c, cy->sweep, cy->variant, cy->rc, cy->uc,
                         cy->lane ? &cy->work : nullptr, 0, 1);
    case 2: {
      int r = vcycle_end(c, cy, (const double2*)f, (double2*)z, 1);
      if (r) return r;
      return stencil_apply(c, cy->fine, (const double2*)z, (double2*)w, 1, nullptr);
    }
    case 3: {   // the whole application: z = M f, w = A z
      int r = vcycle(c, cy, (const double2*)f, (double2*)z);
      if (r) return r;
      return stencil_apply(c, cy->fine, (const double2*)z, (double2*)w, 1, nullptr);
    }
    default:
      return set_error(c, HS_E_ARG, "apply_az part must be 0, 1, 2 or 3");
  }
}

int hs_vcycle_apply_a_end(hs_ctx* c, hs_cycle* cy, const void* f, void* w) {
  if (!c || !cy || !f || !w) return HS_E_ARG;
  int r = vcycle_end(c, cy, (const double2*)f, cy->tmp);
  if (r) return r;
  return stencil_apply(c, cy->fine, cy->tmp, (double2*)w, 1, nullptr);
}

// ---------------------------------------------------------------------------
int hs_block_dot(hs_ctx* c, const void* V, int64_t ldv, int k, const void* w, int64_t n,
                 void* h) {
  if (!c || (!V && k > 0) || !w || !h) return HS_E_ARG;
  return krylov_block_dot(c, (const double2*)V, ldv, k, (const double2*)w, n, (double2*)h,
                          nullptr, nullptr, 0.0);
}

int hs_block_update(hs_ctx* c, const void* V, int64_t ldv, int k, const void* h, void* w,
                    int64_t n, void* nrm2) {
  if (!c || (!V && k > 0) || !h || !w || !nrm2) return HS_E_ARG;
  return krylov_block_update(c, (const double2*)V, ldv, k, (const double2*)h, (double2*)w, n,
                             (double2*)nrm2, nullptr, nullptr, 0.0);
}

int hs_block_update_dot(hs_ctx* c, const void* V, int64_t ldv, int k, const void* h, void* w,
                        int64_t n, void* nrm2, void* h2) {
  if (!c || !V || !h || !w || !nrm2 || !h2) return HS_E_ARG;
  return krylov_block_update_dot(c, (const double2*)V, ldv, k, (const double2*)h, (double2*)w, n,
                                 (double2*)nrm2, (double2*)h2);
}

int hs_block_dot_gated(hs_ctx* c, const void* V, int64_t ldv, int k, const void* w, int64_t n,
                       void* h, const void* g_after, const void* g_before, double thresh) {
  if (!c || (!V && k > 0) || !w || !h || !g_after || !g_before) return HS_E_ARG;
  return krylov_block_dot(c, (const double2*)V, ldv, k, (const double2*)w, n, (double2*)h,
                          (const double2*)g_after, (const double2*)g_before, thresh);
}

int hs_block_update_gated(hs_ctx* c, const void* V, int64_t ldv, int k, const void* h, void* w,
                          int64_t n, void* nrm2, const void* g_after, const void* g_before,
                          double thresh) {
  if (!c || (!V && k > 0) || !h || !w || !nrm2 || !g_after || !g_before) return HS_E_ARG;
  return krylov_block_update(c, (const double2*)V, ldv, k, (const double2*)h, (double2*)w, n,
                             (double2*)nrm2, (const double2*)g_after,
                             (const double2*)g_before, thresh);
}

int hs_scale_inv_sqrt(hs_ctx* c, void* x, int64_t n, const void* s) {
  if (!c || !x || !s) return HS_E_ARG;
  return krylov_scale_inv_sqrt(c, (double2*)x, n, (const double2*)s);
}

int hs_lincomb(hs_ctx* c, const void* V, int64_t ldv, int k, const void* y, void* out,
               int64_t n) {
  if (!c || !V || !y || !out) return HS_E_ARG;
  return krylov_lincomb(c, (const double2*)V, ldv, k, (const double2*)y, (double2*)out, n);
}

int hs_scale(hs_ctx* c, void* x, int64_t n, double are, double aim) {
  if (!c || !x) return HS_E_ARG;
  return krylov_scale(c, (double2*)x, n, make_double2(are, aim));
}

int hs_axpby(hs_ctx* c, double are, double aim, const void* x, double bre, double bim, void* y,
             int64_t n) {
  if (!c || !x || !y) return HS_E_ARG;
  return krylov_axpby(c, make_double2(are, aim), (const double2*)x, make_double2(bre, bim),
                      (double2*)y, n);
}

int hs_norm2(hs_ctx* c, const void* x, int64_t n, void* out) {
  if (!c || !x || !out) return HS_E_ARG;
  return krylov_norm2(c, (const double2*)x, n, (double2*)out);
}

}  // extern "C"
