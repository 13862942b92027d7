// General sparse matrix-vector product on the device (CSR), for the
// reference's TwoGridCycle built from an explicit prolongation matrix
// (twogrid.py:119-159: rc = s P^T r, u += P uc with P any scipy matrix) --
// the BASELINE hierarchies use the tent tables of hs_transfer.cu instead.
// One thread per row (prolongation rows hold <= 2^d entries, restriction
// rows <= 3^d); fixed in-row order, so results are bitwise reproducible.

#include "hs_common.cuh"

#include <vector>

struct hs_csr {
  int64_t rows = 0, cols = 0, nnz = 0;
  int64_t* indptr = nullptr;
  int64_t* indices = nullptr;
  double2* vals = nullptr;
};

namespace hs {
namespace {

__global__ void k_csr_spmv(int64_t rows, const int64_t* __restrict__ indptr,
                           const int64_t* __restrict__ indices, const double2* __restrict__ vals,
                           const double2* __restrict__ x, double2* __restrict__ y, double2 alpha,
                           int accumulate) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double2 acc = czero();
  for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) acc = cfma(vals[e], __ldg(x + indices[e]), acc);
  acc = cmul(alpha, acc);
  y[i] = accumulate ? cadd(y[i], acc) : acc;
}

}  // namespace
}  // namespace hs

using namespace hs;

extern "C" {

int hs_csr_create(hs_ctx* c, int64_t rows, int64_t cols, int64_t nnz, const int64_t* indptr,
                  const int64_t* indices, const double* vals, hs_csr** out) {
  if (!c || !out || rows < 0 || cols < 0 || nnz < 0 || !indptr || (nnz && (!indices || !vals)))
    return HS_E_ARG;
  if (indptr[0] != 0 || indptr[rows] != nnz) return set_error(c, HS_E_SHAPE, "CSR row pointers do not match nnz");
  for (int64_t e = 0; e < nnz; ++e)
    if (indices[e] < 0 || indices[e] >= cols) return set_error(c, HS_E_SHAPE, "CSR column index out of range");
  hs_csr* m = new hs_csr();
  m->rows = rows;
  m->cols = cols;
  m->nnz = nnz;
  cudaError_t e = cudaMalloc((void**)&m->indptr, (rows + 1) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->indices, std::max<int64_t>(1, nnz) * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->vals, std::max<int64_t>(1, nnz) * sizeof(double2));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(m->indptr, indptr, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpyAsync(m->indices, indices, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpyAsync(m->vals, vals, nnz * sizeof(double2), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);   // host arrays may go away
  if (e != cudaSuccess) {
    cudaFree(m->indptr); cudaFree(m->indices); cudaFree(m->vals);
    delete m;
    return check_cuda(c, e, "CSR upload");
  }
  *out = m;
  return HS_OK;
}

int hs_csr_destroy(hs_ctx* c, hs_csr* m) {
  (void)c;
  if (!m) return HS_OK;
  cudaFree(m->indptr); cudaFree(m->indices); cudaFree(m->vals);
  delete m;
  return HS_OK;
}

int hs_csr_apply(hs_ctx* c, const hs_csr* m, const void* x, void* y, double alpha_re,
                 double alpha_im, int accumulate) {
  if (!c || !m || !x || !y) return HS_E_ARG;
  if (m->rows == 0) return HS_OK;
  k_csr_spmv<<<(unsigned)((m->rows + 255) / 256), 256, 0, c->stream>>>(
      m->rows, m->indptr, m->indices, m->vals, (const double2*)x, (double2*)y,
      make_double2(alpha_re, alpha_im), accumulate);
  HS_LAUNCH_CHECK(c, "CSR SpMV");
  return HS_OK;
}

}  // extern "C"
