// Batched FP64 GEMM on the tensor cores (DMMA, mma.sync m8n8k4.f64) for the
// SAI least-squares setup: the compact-WY trailing updates of the blocked
// Householder QR (C -= V (T^T (V^T C)), dense_lstsq blockla.hpp:278-309 ->
// LAPACK dgels), the Gram matrix of the wide panel's reflectors, and the
// small T^T Y product -- ~98 % of the setup flops.
//
//   D[b](m, n) = alpha * sum_k A[b](m, k) B[b](n, k) + beta * D[b](m, n)
//
// with the K index CONTIGUOUS in both operands (A(m,k) at A + m*lda + k,
// B(n,k) at B + n*ldb + k) and D column-major.  Every product of the QR
// update is of this form once the reflector block is also kept transposed
// (sai_build.cu).  tcgen05 has no FP64 kind, so the FP64 tensor-core path on
// sm_100a is the warp-level DMMA; one 64x64 tile per CTA (2x2 warps of
// 32x32 = 4x4 m8n8 accumulators each), K in steps of 16 through a 3-stage
// cp.async ring.  Shared rows are padded to 20 doubles: the fragment loads
// (row = lane / 4, k = lane % 4) of every quarter-warp hit 16 distinct banks.
#include <cuda_runtime.h>

#include <algorithm>

#include "core.hpp"
#include "dgemm.hpp"

namespace ldgmg_b200 {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, LDK = BK + 4, STAGES = 3, THREADS = 128;
constexpr size_t kSmemBytes = sizeof(double) * size_t(STAGES) * (BM + BN) * LDK;

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

/// One stage: rows [r0, r0+64) x k [k0, k0+16) of an operand into a padded
/// [row][k] tile; thread t copies 8 consecutive k of row t/2 (zero fill
/// outside the matrix).
__device__ __forceinline__ void load_tile(double* s, const double* G, int64_t ld, int rows, int K, int r0, int k0) {
    const int t = threadIdx.x;
    const int r = t >> 1, kb = (t & 1) * 8;
    const bool rv = r0 + r < rows;
    const double* src = G + (rv ? int64_t(r0 + r) * ld : 0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int k = k0 + kb + q;
        const bool v = rv && k < K;
        cp_async8(s + r * LDK + kb + q, v ? src + k : G, v);
    }
}

__global__ void __launch_bounds__(THREADS) dgemm_nt_kernel(const GemmNT g) {
    extern __shared__ __align__(16) double sm[];
    double* sA = sm;
    double* sB = sm + STAGES * BM * LDK;
    const int b = blockIdx.z;
    const double* A = g.A + int64_t(b) * g.sA;
    const double* B = g.B + int64_t(b) * g.sB;
    double* D = g.D + int64_t(b) * g.sD;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int nk = (g.K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) {
            load_tile(sA + s * BM * LDK, A, g.lda, g.M, g.K, m0, s * BK);
            load_tile(sB + s * BN * LDK, B, g.ldb, g.N, g.K, n0, s * BK);
        }
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        // refill the stage consumed STAGES-1 steps ago (everyone is past it)
        const int nxt = kt + STAGES - 1;
        if (nxt < nk) {
            const int s = nxt % STAGES;
            load_tile(sA + s * BM * LDK, A, g.lda, g.M, g.K, m0, nxt * BK);
            load_tile(sB + s * BN * LDK, B, g.ldb, g.N, g.K, n0, nxt * BK);
        }
        cp_async_commit();
        const double* tA = sA + (kt % STAGES) * BM * LDK + (wm + fr) * LDK + fk;
        const double* tB = sB + (kt % STAGES) * BN * LDK + (wn + fr) * LDK + fk;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = tA[i * 8 * LDK + kk];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = tB[j * 8 * LDK + kk];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
        }
    }
    cp_async_wait<0>();
    // accumulator (i, j): row wm + 8i + lane/4, columns wn + 8j + 2(lane%4) + {0, 1}
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + wm + i * 8 + fr;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = n0 + wn + j * 8 + fk * 2 + h;
                if (n >= g.N) continue;
                double* d = D + m + int64_t(n) * g.ldd;
                const double v = g.alpha * acc[i][j][h];
                *d = g.beta == 0.0 ? v : v + g.beta * *d;
            }
    }
}

}  // namespace

void dgemm_nt_batched(Ctx& ctx, const GemmNT& g, int batch) {
    if (batch <= 0 || g.M <= 0 || g.N <= 0) return;
    static bool once = (LDGMG_CUDA(cudaFuncSetAttribute(dgemm_nt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        int(kSmemBytes))),
                        true);
    (void)once;
    require(batch <= 65535, "dgemm_nt_batched: batch above 65535");
    const dim3 grid(div_up(g.N, BN), div_up(g.M, BM), batch);
    dgemm_nt_kernel<<<grid, THREADS, kSmemBytes, ctx.stream>>>(g);
    after_launch("dgemm_nt_kernel");
}

}  // namespace ldgmg_b200
