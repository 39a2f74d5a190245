// Batched FP64 tensor-core GEMM (dgemm_batched.cu).
#pragma once

#include <cstdint>

#include "core.hpp"

namespace ldgmg_b200 {

/// D[b](m, n) = alpha * sum_k A[b](m, k) * B[b](n, k) + beta * D[b](m, n),
/// k contiguous in A and B, D column-major; batch b at the given strides.
struct GemmNT {
    const double* A;
    int64_t lda, sA;
    const double* B;
    int64_t ldb, sB;
    double* D;
    int64_t ldd, sD;
    int M, N, K;
    double alpha, beta;
};
void dgemm_nt_batched(Ctx& ctx, const GemmNT& g, int batch);

}  // namespace ldgmg_b200
