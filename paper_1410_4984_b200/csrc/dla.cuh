// dla.cuh -- fp64 dense linear algebra on the device (dla.cu): the coordinator's M-sized algebra.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sgpx {
namespace dla {
// C = alpha op(A) op(B) + beta C (column-major; m x n result, inner dimension k).
int gemm(bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int64_t lda, const double* B,
         int64_t ldb, double beta, double* C, int64_t ldc, cudaStream_t st);
// Lower Cholesky of the m x m matrix a into L with the reference's escalation schedule:
// mode 0 = factor_gram (diag += f var, f from f0), mode 1 = factor_spd (diag += f max|a_ii|).
// out_scal[0] = log det, out_scal[1] = the factor used; info[0] = 0 ok / 1 failed.
int cholesky(const double* a, int m, double* L, int mode, double f0, double var, double* out_scal, int* info,
             cudaStream_t st);
// W = L^-1 for lower-triangular L.
int trinv(const double* L, int m, double* W, cudaStream_t st);
}  // namespace dla
}  // namespace sgpx
