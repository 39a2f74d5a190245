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
    // optional further segments of the N index: rows n of B with
    // nsplit <= n < nsplit2 live at B2 + (n - nsplit) ldb (batch stride sB2),
    // those with n >= nsplit2 at B3 + (n - nsplit2) ldb (sB3); columns n >=
    // nsplit of D at D2 + (n - nsplit) ldd (sD2) -- one launch for the QR's
    // reflector Gram, the trailing columns of M and the right-hand sides W
    const double* B2 = nullptr;
    int64_t sB2 = 0;
    double* D2 = nullptr;
    int64_t sD2 = 0;
    int nsplit = 1 << 30;
    const double* B3 = nullptr;
    int64_t sB3 = 0;
    int nsplit2 = 1 << 30;
};
void dgemm_nt_batched(Ctx& ctx, const GemmNT& g, int batch);

}  // namespace ldgmg_b200
