// Batched FP64 GEMM on the tensor cores (DMMA, mma.sync m8n8k4.f64) for the
// SAI least-squares setup: the compact-WY trailing updates of the blocked
// Householder QR (C -= V (T^T (V^T C)), dense_lstsq blockla.hpp:278-309 ->
// LAPACK dgels), the Gram matrix of the wide panel's reflectors, and the
// small T^T Y product -- ~94 % of the setup flops.
//
//   D[b](m, n) = alpha * sum_k A[b](m, k) B[b](n, k) + beta * D[b](m, n)
//
// with the K index CONTIGUOUS in both operands (A(m,k) at A + m*lda + k,
// B(n,k) at B + n*ldb + k) and D column-major.  Every product of the QR
// update is of this form once the reflector block is also kept row-major
// (sai_build.cu).  tcgen05 has no FP64 kind, so the FP64 tensor-core path on
// sm_100a is the warp-level DMMA: a BM x BN tile per CTA split over
// WM x WN warps (each an array of m8n8 accumulators), K in steps of BK
// through a STAGES-deep cp.async ring (16-byte copies when every operand row
// is 16-byte aligned, 8-byte otherwise).  Shared rows are padded to
// BK + 4 doubles (= 4 mod 16): the fragment loads (row = lane / 4,
// k = lane % 4) of every quarter warp hit 16 distinct banks.  With beta != 0
// the D tile is loaded into registers before the main loop, so its latency
// hides under the K loop (the C -= V Z update has K = 64 only).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "core.hpp"
#include "dgemm.hpp"

namespace ldgmg_b200 {

namespace {

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
struct Cfg {
    static constexpr int THREADS = WM * WN * 32;
    static constexpr int LDK = BK + 4;
    static constexpr int TM = BM / WM / 8, TN = BN / WN / 8;  // m8n8 tiles per warp
    static constexpr size_t SMEM = sizeof(double) * size_t(STAGES) * (BM + BN) * LDK;
    static_assert(BM % (WM * 8) == 0 && BN % (WN * 8) == 0, "tile shape");
    static_assert(LDK % 16 == 4, "padding keeps the fragment loads conflict-free");
};

/// rows [r0, r0+ROWS) x k [k0, k0+BK) of an operand into a padded [row][k]
/// tile; zero fill outside the matrix.
template <int ROWS, int BK, int LDK, int THREADS, bool VEC>
__device__ __forceinline__ void load_tile(double* s, const double* G, int64_t ld, int rows, int K, int r0, int k0,
                                          const double* G2 = nullptr, int split = 1 << 30,
                                          const double* G3 = nullptr, int split2 = 1 << 30) {
    constexpr int PER = VEC ? 2 : 1;                 // doubles per copy
    constexpr int COPIES = ROWS * BK / PER;          // copies per tile
    static_assert(COPIES % THREADS == 0, "tile copies divide over the threads");
    constexpr int CPR = BK / PER;                    // copies per row
#pragma unroll
    for (int c = 0; c < COPIES / THREADS; ++c) {
        const int id = c * THREADS + threadIdx.x;
        const int r = id / CPR, kk = (id - r * CPR) * PER;
        const int k = k0 + kk;
        const bool rv = r0 + r < rows;
        // rows past `split` / `split2` come from the second / third segment (pre-offset)
        const double* base = r0 + r < split ? G : r0 + r < split2 ? G2 : G3;
        const double* src = rv ? base + int64_t(r0 + r) * ld + (k < K ? k : 0) : G;
        if constexpr (VEC) {
            const int bytes = (rv && k < K) ? (k + 1 < K ? 16 : 8) : 0;
            cp_async16(s + r * LDK + kk, src, bytes);
        } else {
            cp_async8(s + r * LDK + kk, src, rv && k < K);
        }
    }
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES, bool VEC, bool BETA>
__global__ void __launch_bounds__(Cfg<BM, BN, WM, WN, BK, STAGES>::THREADS)
    dgemm_nt_kernel(const GemmNT g) {
    using CF = Cfg<BM, BN, WM, WN, BK, STAGES>;
    constexpr int LDK = CF::LDK, TM = CF::TM, TN = CF::TN, THREADS = CF::THREADS;
    extern __shared__ __align__(16) double sm[];
    double* sA = sm;
    double* sB = sm + STAGES * BM * LDK;
    const int b = blockIdx.z;
    const double* A = g.A + int64_t(b) * g.sA;
    const double* B = g.B + int64_t(b) * g.sB;
    double* D = g.D + int64_t(b) * g.sD;
    // second / third N segments, offset so that row / column n indexes them directly
    const double* B2 = g.B2 ? g.B2 + int64_t(b) * g.sB2 - int64_t(g.nsplit) * g.ldb : B;
    double* D2 = g.D2 ? g.D2 + int64_t(b) * g.sD2 - int64_t(g.nsplit) * g.ldd : D;
    const double* B3 = g.B3 ? g.B3 + int64_t(b) * g.sB3 - int64_t(g.nsplit2) * g.ldb : B2;
    const int bsplit = g.B2 ? g.nsplit : 1 << 30, bsplit2 = g.B3 ? g.nsplit2 : 1 << 30;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp / WN) * (TM * 8), wn = (warp % WN) * (TN * 8);
    const int fr = lane >> 2, fk = lane & 3;
    const int nk = (g.K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) {
            load_tile<BM, BK, LDK, THREADS, VEC>(sA + s * BM * LDK, A, g.lda, g.M, g.K, m0, s * BK);
            load_tile<BN, BK, LDK, THREADS, VEC>(sB + s * BN * LDK, B, g.ldb, g.N, g.K, n0, s * BK, B2, bsplit, B3, bsplit2);
        }
        cp_async_commit();
    }
    // D prefetch (beta != 0): in flight during the whole K loop
    double dold[BETA ? TM : 1][BETA ? TN : 1][2];
    if constexpr (BETA)
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = m0 + wm + i * 8 + fr, n = n0 + wn + j * 8 + fk * 2 + h;
                const double* Dn = n < g.nsplit ? D : D2;
                dold[i][j][h] = (m < g.M && n < g.N) ? Dn[m + int64_t(n) * g.ldd] : 0.0;
            }
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kt + STAGES - 1;  // refill the stage consumed last iteration
        if (nxt < nk) {
            const int s = nxt % STAGES;
            load_tile<BM, BK, LDK, THREADS, VEC>(sA + s * BM * LDK, A, g.lda, g.M, g.K, m0, nxt * BK);
            load_tile<BN, BK, LDK, THREADS, VEC>(sB + s * BN * LDK, B, g.ldb, g.N, g.K, n0, nxt * BK, B2, bsplit, B3, bsplit2);
        }
        cp_async_commit();
        const double* tA = sA + (kt % STAGES) * BM * LDK + (wm + fr) * LDK + fk;
        const double* tB = sB + (kt % STAGES) * BN * LDK + (wn + fr) * LDK + fk;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[TM], bb[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = tA[i * 8 * LDK + kk];
#pragma unroll
            for (int j = 0; j < TN; ++j) bb[j] = tB[j * 8 * LDK + kk];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
        }
    }
    cp_async_wait<0>();
    // accumulator (i, j): row wm + 8i + lane/4, columns wn + 8j + 2(lane%4) + {0, 1}
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int m = m0 + wm + i * 8 + fr;
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = n0 + wn + j * 8 + fk * 2 + h;
                double* Dn = n < g.nsplit ? D : D2;
                if (m < g.M && n < g.N) {
                    double v = g.alpha * acc[i][j][h];
                    if constexpr (BETA) v += g.beta * dold[i][j][h];
                    Dn[m + int64_t(n) * g.ldd] = v;
                }
            }
    }
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
void launch(Ctx& ctx, const GemmNT& g, int batch, bool vec) {
    using CF = Cfg<BM, BN, WM, WN, BK, STAGES>;
    const bool beta = g.beta != 0.0;
    auto kern = vec ? (beta ? dgemm_nt_kernel<BM, BN, WM, WN, BK, STAGES, true, true>
                            : dgemm_nt_kernel<BM, BN, WM, WN, BK, STAGES, true, false>)
                    : (beta ? dgemm_nt_kernel<BM, BN, WM, WN, BK, STAGES, false, true>
                            : dgemm_nt_kernel<BM, BN, WM, WN, BK, STAGES, false, false>);
    ensure_dyn_smem(kern, CF::SMEM);
    const dim3 grid(div_up(g.N, BN), div_up(g.M, BM), batch);
    kern<<<grid, CF::THREADS, CF::SMEM, ctx.stream>>>(g);
    after_launch("dgemm_nt_kernel");
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

void dgemm_nt_batched(Ctx& ctx, const GemmNT& g, int batch) {
    if (batch <= 0 || g.M <= 0 || g.N <= 0) return;
    require(batch <= 65535, "dgemm_nt_batched: batch above 65535");
    // 16-byte copies need every operand row to start 16-byte aligned
    const bool vec = aligned16(g.A) && aligned16(g.B) && !(g.lda & 1) && !(g.ldb & 1) && !(g.sA & 1) &&
                     !(g.sB & 1) && (!g.B2 || (aligned16(g.B2) && !(g.sB2 & 1))) &&
                     (!g.B3 || (aligned16(g.B3) && !(g.sB3 & 1)));
    static int variant = -1;
    if (variant < 0) {
        const char* e = std::getenv("LDGMG_DGEMM_VARIANT");  // measurement only (tools/dgemm_bench.py)
        variant = e ? std::atoi(e) : 0;
    }
    switch (variant) {
        case 1: launch<64, 64, 2, 2, 16, 3>(ctx, g, batch, vec); return;
        case 2: launch<128, 64, 4, 2, 16, 3>(ctx, g, batch, vec); return;
        case 3: launch<64, 64, 2, 2, 32, 3>(ctx, g, batch, vec); return;
        case 4: launch<128, 128, 4, 2, 16, 3>(ctx, g, batch, vec); return;
        case 5: launch<64, 128, 2, 4, 16, 3>(ctx, g, batch, vec); return;
        default: break;
    }
    // default: 64 x 64 tiles, 4 warps, 3 stages -- measured best on every
    // product of the C5 QR (tools/dgemm_bench.py, B200: V^T C 30.7, Gram
    // 20.9, T^T Y 21.7, C -= V Z 20.1 TF/s; 128-row tiles 15-19 TF/s).  The
    // K = 64 update is bound by its per-tile pipeline fill and barriers, not
    // by the 194 registers of the D prefetch: the accumulators seeded with D
    // (128 registers, 3 CTAs per SM) measured 6 % slower, D staged in shared
    // memory by bulk copies (2 stages) 11 % slower
    launch<64, 64, 2, 2, 16, 3>(ctx, g, batch, vec);
}

}  // namespace ldgmg_b200
