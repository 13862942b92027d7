// Batched dense complex128 kernels for setup factorisations (hs_dense.cu).
#pragma once

#include "hs_common.cuh"

namespace hs {

constexpr int kMaxDenseJobs = 32;   // jobs per launch (passed by value)

// C = alpha op(A) op(B) + beta C (column-major; op = 1: transpose; transC:
// store the result transposed, i.e. C row-major)
struct GemmJob {
  int m = 0, n = 0, k = 0;
  const double2* A = nullptr;
  int lda = 0;
  const double2* B = nullptr;
  int ldb = 0;
  double2* C = nullptr;
  int ldc = 0;
  double2 alpha{1.0, 0.0}, beta{0.0, 0.0};
  int opA = 0, opB = 0, transC = 0;
};

// LU with partial pivoting of A (n x n, column-major, in place; piv [n]
// 0-based swap rows, info: first zero pivot, 1-based, 0 = none -- must be
// zero on entry) and X = A^{-1} (column-major, ldx)
struct LuJob {
  double2* A = nullptr;
  int ld = 0, n = 0;
  int* piv = nullptr;
  int* info = nullptr;
  double2* X = nullptr;
  int ldx = 0;
};

// dst (row-major, ldd) = src (column-major, lds), n x n
struct TransposeJob {
  const double2* src = nullptr;
  int lds = 0;
  double2* dst = nullptr;
  int ldd = 0, n = 0;
};

int dense_gemm(Ctx* c, const GemmJob* jobs, int n);
int dense_lu_inverse(Ctx* c, const LuJob* jobs, int n);
int dense_transpose(Ctx* c, const TransposeJob* jobs, int n);

}  // namespace hs
