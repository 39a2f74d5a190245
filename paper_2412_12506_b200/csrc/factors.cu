// GPU diagonal-factor setup: factor_diagonal (smoothers.hpp:464-494) for
// every element in one launch -- power-of-two equilibration of the diagonal
// block, symmetry check, and the symmetric eigendecomposition of s D s by a
// parallel cyclic Jacobi method (one CTA per element, matrix and
// eigenvectors in shared memory, round-robin rotation sets so the n/2
// rotations of a step touch disjoint rows/columns).  Output goes straight
// into the DiagFactors device layout read by the relax row pass.
//
// The reference solves each block with Eigen's SelfAdjointEigenSolver
// (tridiagonalisation + implicit QL); Jacobi converges to the same
// eigenpairs to rounding (eigenvector signs / bases of repeated eigenvalues
// may differ, which the pseudoinverse V diag(1/lambda) V^T does not see).
// Parity is therefore to tolerance, like every other setup path here
// (tests/test_gpu_factors.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "core.hpp"
#include "mg.hpp"

namespace ldgmg_b200 {

namespace {

constexpr int kFactorThreads = 128;
constexpr int kMaxSweeps = 30;

__device__ __forceinline__ double cta_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
    __syncthreads();
    return s;
}

/// One element per CTA.  smem: A (n x ldA), V (n x ldA), cos/sin/pairs.
__global__ void __launch_bounds__(kFactorThreads) diag_factor_kernel(
    const double* __restrict__ val, int blk_stride, const int* __restrict__ dk, int n, int ld, int vstride,
    double* __restrict__ Vout, double* __restrict__ lam_out, double* __restrict__ s_out,
    double* __restrict__ lmax_out, int* __restrict__ bad) {
    extern __shared__ __align__(16) double sm[];
    const int ldA = n | 1;  // odd leading dimension: conflict-free row and column walks
    const int m = (n + 1) & ~1;
    double* A = sm;
    double* V = A + size_t(n) * ldA;
    double* cs = V + size_t(n) * ldA;
    double* sn = cs + m / 2;
    double* sc = sn + m / 2;
    double* lam = sc + n;
    double* red = lam + n;  // 32 doubles
    int* pp = reinterpret_cast<int*>(red + 32);
    int* qq = pp + m / 2;
    int* rank = qq + m / 2;
    const int e = blockIdx.x, tid = threadIdx.x, NT = blockDim.x;
    const double* D = val + size_t(__ldg(dk + e)) * blk_stride;  // column-major: (r,c) at c*n + r

    // power-of-two equilibration s_i = 2^-(ex/2), ex = frexp exponent of |D_ii|
    for (int i = tid; i < n; i += NT) {
        const double d = fabs(D[size_t(i) * n + i]);
        double s = 1.0;
        if (d > 0.0) {
            int ex;
            frexp(d, &ex);
            s = ldexp(1.0, -(ex / 2));
        }
        sc[i] = s;
    }
    __syncthreads();
    double nrm = 0.0, asym = 0.0;
    for (int t = tid; t < n * n; t += NT) {
        const int j = t / n, i = t - j * n;  // column j, row i
        const double a = (sc[i] * D[size_t(j) * n + i]) * sc[j];
        const double b = (sc[j] * D[size_t(i) * n + j]) * sc[i];
        nrm += a * a;
        asym += (a - b) * (a - b);
        // the lower triangle defines the matrix (Eigen's SelfAdjointEigenSolver)
        A[size_t(j) * ldA + i] = i >= j ? a : b;
        V[size_t(j) * ldA + i] = i == j ? 1.0 : 0.0;
    }
    nrm = cta_sum(nrm, red);
    asym = cta_sum(asym, red);
    if (sqrt(asym) > 1e-13 * fmax(1e-300, sqrt(nrm))) {
        if (tid == 0) bad[e] = 1;
        return;
    }
    // parallel cyclic Jacobi, round-robin pairs (player m-1 fixed)
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        double off = 0.0;
        for (int t = tid; t < n * n; t += NT) {
            const int j = t / n, i = t - j * n;
            if (i != j) off += A[size_t(j) * ldA + i] * A[size_t(j) * ldA + i];
        }
        off = cta_sum(off, red);
        if (off <= 1e-34 * nrm || off == 0.0) break;
        for (int step = 0; step < m - 1; ++step) {
            for (int k = tid; k < m / 2; k += NT) {
                int p, q;
                if (k == 0) {
                    p = step;
                    q = m - 1;
                } else {
                    p = (step + k) % (m - 1);
                    q = (step - k + m - 1) % (m - 1);
                }
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                double c = 1.0, s = 0.0;
                if (q < n) {
                    const double apq = A[size_t(q) * ldA + p];
                    if (apq != 0.0) {
                        const double app = A[size_t(p) * ldA + p], aqq = A[size_t(q) * ldA + q];
                        const double theta = (aqq - app) / (2.0 * apq);
                        const double at = fabs(theta);
                        double t = at > 1e150 ? 0.5 / at : 1.0 / (at + sqrt(at * at + 1.0));
                        if (theta < 0.0) t = -t;
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                } else {
                    q = -1;  // padding player: no rotation
                }
                pp[k] = p;
                qq[k] = q;
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            // rows: A <- P^T A
            for (int t = tid; t < (m / 2) * n; t += NT) {
                const int k = t / n, j = t - k * n;
                const int p = pp[k], q = qq[k];
                if (q < 0 || sn[k] == 0.0) continue;
                const double c = cs[k], s = sn[k];
                const double ap = A[size_t(j) * ldA + p], aq = A[size_t(j) * ldA + q];
                A[size_t(j) * ldA + p] = c * ap - s * aq;
                A[size_t(j) * ldA + q] = s * ap + c * aq;
            }
            __syncthreads();
            // columns: A <- A P, V <- V P
            for (int t = tid; t < (m / 2) * n * 2; t += NT) {
                const int w = t / ((m / 2) * n), u = t - w * ((m / 2) * n);
                const int k = u / n, i = u - k * n;
                const int p = pp[k], q = qq[k];
                if (q < 0 || sn[k] == 0.0) continue;
                const double c = cs[k], s = sn[k];
                double* X = w == 0 ? A : V;
                const double xp = X[size_t(p) * ldA + i], xq = X[size_t(q) * ldA + i];
                X[size_t(p) * ldA + i] = c * xp - s * xq;
                X[size_t(q) * ldA + i] = s * xp + c * xq;
            }
            __syncthreads();
        }
    }
    // ascending eigenvalues (ties by index), eigenvectors permuted alike
    for (int i = tid; i < n; i += NT) lam[i] = A[size_t(i) * ldA + i];
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
        int r = 0;
        const double li = lam[i];
        for (int j = 0; j < n; ++j) r += (lam[j] < li) || (lam[j] == li && j < i);
        rank[i] = r;
    }
    __syncthreads();
    double* Vo = Vout + size_t(e) * vstride;
    for (int t = tid; t < n * n; t += NT) {
        const int k = t / n, i = t - k * n;  // eigenvector k, row i
        Vo[size_t(rank[k]) * ld + i] = V[size_t(k) * ldA + i];
    }
    double mx = 0.0;
    for (int i = tid; i < n; i += NT) {
        lam_out[size_t(e) * n + rank[i]] = lam[i];
        s_out[size_t(e) * n + i] = sc[i];
        mx = fmax(mx, fabs(lam[i]));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
        double r = 0.0;
        for (int w = 0; w < NT / 32; ++w) r = fmax(r, red[w]);
        lmax_out[e] = r;
    }
}

}  // namespace

size_t diag_factor_smem(int n) {
    const int ldA = n | 1, m = (n + 1) & ~1;
    return sizeof(double) * (size_t(2) * n * ldA + m + 2 * n + 32) + sizeof(int) * (size_t(m) + n) + 16;
}

void compute_factors_gpu(Ctx& ctx, const Bsr& A, DiagFactors& F) {
    const int N = A.brows, bs = A.rbs;
    if (A.brows != A.bcols || A.rbs != A.cbs) fail(LDGMG_ERR_INVALID_ARGUMENT, "Smoother: operator must be block-square");
    std::vector<int> dk(N, -1);
    for (int e = 0; e < N; ++e) {
        for (int k = A.hptr[e]; k < A.hptr[e + 1]; ++k)
            if (A.hcol[k] == e) dk[e] = k;
        if (dk[e] < 0) fail(LDGMG_ERR_RUNTIME, "Smoother: missing diagonal block");
    }
    F.n = N;
    F.bs = bs;
    F.ld = bs | 1;
    F.vstride = even_up(int64_t(bs) * F.ld);
    F.V.alloc(sizeof(double) * std::max<size_t>(1, size_t(N) * F.vstride));
    F.lambda.alloc(sizeof(double) * std::max<size_t>(1, size_t(N) * bs));
    F.scale.alloc(sizeof(double) * std::max<size_t>(1, size_t(N) * bs));
    F.lmax.alloc(sizeof(double) * std::max(1, N));
    if (N == 0) return;
    LDGMG_CUDA(cudaMemsetAsync(F.V.p, 0, F.V.bytes, ctx.stream));
    DevBuf d_dk(sizeof(int) * N), d_bad(sizeof(int) * N);
    h2d(ctx, d_dk.p, dk.data(), sizeof(int) * N);
    LDGMG_CUDA(cudaMemsetAsync(d_bad.p, 0, d_bad.bytes, ctx.stream));
    const size_t smem = diag_factor_smem(bs);
    if (smem > 227 * 1024) fail(LDGMG_ERR_INVALID_ARGUMENT, "factor_diagonal: block too large for the GPU factor kernel");
    ensure_dyn_smem(diag_factor_kernel, size_t(smem));
    diag_factor_kernel<<<N, kFactorThreads, smem, ctx.stream>>>(
        A.val.as<double>(), A.blk_stride, d_dk.as<int>(), bs, F.ld, F.vstride, F.V.as<double>(),
        F.lambda.as<double>(), F.scale.as<double>(), F.lmax.as<double>(), d_bad.as<int>());
    after_launch("diag_factor_kernel");
    std::vector<int> bad(N);
    d2h(ctx, bad.data(), d_bad.p, sizeof(int) * N);
    for (int e = 0; e < N; ++e)
        if (bad[e]) fail(LDGMG_ERR_INVALID_ARGUMENT, "sym_eig: matrix is not symmetric");
}

}  // namespace ldgmg_b200
