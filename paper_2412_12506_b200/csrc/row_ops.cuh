// Device-side pieces shared by the row-pass kernels (bsr_kernels.cu) and the
// persistent coarse-level program (coarse_program.cu).  Every function keeps
// the reference's evaluation order (see bsr_kernels.cu header).
#pragma once

#include <cuda_runtime.h>

#include "core.hpp"

namespace ldgmg_b200 {

struct RowPassArgs {
    const int* ptr;
    const int* col;
    const double* val;
    int blk_stride;
    int rbs, cbs;
    int mode;
    const double* x;
    const double* b;
    const double* xe;
    double* y;
    const int* rows;
    int nrows;
    const double* V;
    const double* lam;
    const double* scal;
    const double* lmax;
    int ld, vstride;
    double omega, kernel_tol;
    int nstages, stage_doubles, xslot_doubles;
    // transpose view (bsr_transpose_view): block q of this operator is block
    // perm[q] of the base matrix, read transposed (lane r sums along a stored
    // column of the base block)
    const int* perm;
    int tview;
    // relax: CSR position of each row's diagonal block (-1 if none); the
    // streaming kernel skips it without reading col
    const int* dpos;
    // processor-block GS (smoothers.hpp:426-436): neighbour j of row e is read
    // from x when part[j] == part[e], else from x_alt (the sweep's snapshot)
    const int* part;
    const double* x_alt;
};

__device__ __forceinline__ const double* x_source(const RowPassArgs& a, int row, int j) {
    return (a.part && __ldg(a.part + j) != __ldg(a.part + row)) ? a.x_alt : a.x;
}

__device__ __forceinline__ int row_at(const RowPassArgs& a, int slot) {
    return a.rows ? __ldg(a.rows + slot) : slot;
}

/// One block row processed by a whole CTA (rbs, cbs <= 32): the row's blocks
/// spread over the warps (each computes s_k = 0 + b[r,0]x[0] + ... for its
/// blocks), warp 0 combines them in CSR order and runs the epilogue (relax:
/// the block-diagonal pseudoinverse with V read from global memory).
/// `ss` holds maxlen x 32 partial sums + 64 doubles.  All CTA threads call it.
__device__ __forceinline__ void split_row_task(const RowPassArgs& a, int row, int maxlen, double* ss) {
    double* ubuf = ss + size_t(maxlen) * 32;
    double* tbuf = ubuf + 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    const bool relax = a.mode == MODE_RELAX;
    const int k0 = __ldg(a.ptr + row), k1 = __ldg(a.ptr + row + 1);
    for (int k = k0 + warp; k < k1; k += W) {
        const int j = __ldg(a.col + k);
        if (relax && j == row) continue;
        if (lane < a.rbs) {
            const double* Bc = a.val + size_t(k) * a.blk_stride + lane;
            const double* xj = x_source(a, row, j) + size_t(j) * a.cbs;
            double s = 0.0;
#pragma unroll 9
            for (int c = 0; c < a.cbs; ++c) s = madd_rn(s, __ldg(Bc + size_t(c) * a.rbs), xj[c]);
            ss[size_t(k - k0) * 32 + lane] = s;
        }
    }
    __syncthreads();
    if (warp == 0) {
        const bool act = lane < a.rbs;
        const size_t o = size_t(row) * a.rbs + lane;
        double acc = 0.0;
        if (act) {
            if (relax) {
                acc = __ldg(a.b + o);
                for (int k = k0; k < k1; ++k)
                    if (__ldg(a.col + k) != row) acc = __dsub_rn(acc, ss[size_t(k - k0) * 32 + lane]);
            } else {
                for (int k = k0; k < k1; ++k) acc = __dadd_rn(acc, ss[size_t(k - k0) * 32 + lane]);
            }
        }
        if (relax) {
            const int bs = a.rbs, ld = a.ld;
            const double* Ve = a.V + size_t(row) * a.vstride;
            const double sc = act ? __ldg(a.scal + o) : 0.0;
            const double lam = act ? __ldg(a.lam + o) : 0.0;
            const double xe = act ? a.xe[o] : 0.0;
            if (act) ubuf[lane] = __dmul_rn(sc, acc);
            __syncwarp();
            if (act) {
                double tt = 0.0;
                const double* Vcol = Ve + size_t(lane) * ld;
                for (int kk = 0; kk < bs; ++kk) tt = madd_rn(tt, __ldg(Vcol + kk), ubuf[kk]);
                const double cut = a.kernel_tol * __ldg(a.lmax + row);
                tbuf[lane] = fabs(lam) <= cut ? 0.0 : tt / lam;
            }
            __syncwarp();
            if (act) {
                double w = 0.0;
                for (int kk = 0; kk < bs; ++kk) w = madd_rn(w, __ldg(Ve + size_t(kk) * ld + lane), tbuf[kk]);
                const double yv = __dmul_rn(sc, w);
                acc = __dadd_rn(__dmul_rn(1.0 - a.omega, xe), __dmul_rn(a.omega, yv));
            }
        }
        if (act) {
            double out;
            switch (a.mode) {
                case MODE_RESIDUAL: out = __dsub_rn(__ldg(a.b + o), acc); break;
                case MODE_ADD: out = __dadd_rn(a.xe[o], acc); break;
                default: out = acc; break;
            }
            a.y[o] = out;
        }
    }
    __syncthreads();
}

/// split_row_task with the row's operands staged in shared memory first:
/// the row's blocks (contiguous in CSR order) and, for relax, the element's
/// factor V arrive by TMA bulk copies on `bar`, while the threads gather the
/// x-blocks and the epilogue operands with all loads in flight at once.  A
/// row then costs ~3 dependent memory round trips (row pointers -> column
/// ids -> x) instead of one per 9-step chunk of every block product; the
/// arithmetic (and so the bits) is split_row_task's.
/// smem layout (doubles): blocks maxlen*blk_stride | V vstride | x maxlen*xs |
/// partial sums maxlen*32 | u 32 | t 32 | epilogue 4*32.  All threads call it.
/// The TMA part of split_row_task_tma: the row's blocks (and relax factor)
/// requested on `bar`.  Immutable data only, so it may run before the PDL
/// wait.  Thread 0 issues; all threads may call.
__device__ __forceinline__ void split_row_issue(const RowPassArgs& a, int row, int maxlen, double* sm,
                                                uint64_t* bar) {
    if (threadIdx.x != 0) return;
    const bool relax = a.mode == MODE_RELAX;
    double* sB = sm;
    double* sV = sB + size_t(maxlen) * a.blk_stride;
    const int k0 = __ldg(a.ptr + row), k1 = __ldg(a.ptr + row + 1), nk = k1 - k0;
    fence_proxy_async();  // the previous row's generic reads of sB/sV precede these async writes
    const uint32_t bb = uint32_t(nk) * uint32_t(a.blk_stride) * 8u;
    const uint32_t vb = relax ? uint32_t(a.vstride) * 8u : 0u;
    mbar_arrive_expect_tx(bar, bb + vb);
    if (bb) bulk_g2s(sB, a.val + size_t(k0) * a.blk_stride, bb, bar);
    if (vb) bulk_g2s(sV, a.V + size_t(row) * a.vstride, vb, bar);
}

/// Column index of this thread's first x-gather entry of `row` (immutable,
/// so it can be loaded before the PDL wait); -1 when the thread has none.
__device__ __forceinline__ int split_row_first_col(const RowPassArgs& a, int row) {
    const int k0 = __ldg(a.ptr + row), nk = __ldg(a.ptr + row + 1) - k0;
    const int t = threadIdx.x;
    if (t >= nk * a.cbs) return -1;
    return __ldg(a.col + k0 + t / a.cbs);
}

__device__ __forceinline__ void split_row_task_tma(const RowPassArgs& a, int row, int maxlen, double* sm,
                                                   uint64_t* bar, uint32_t& phase, bool issued = false,
                                                   int jfirst = -1) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, tid = threadIdx.x;
    const bool relax = a.mode == MODE_RELAX;
    const int xs = (a.cbs + 1) & ~1;
    double* sB = sm;
    double* sV = sB + size_t(maxlen) * a.blk_stride;
    double* sX = sV + (relax ? a.vstride : 0);
    double* ss = sX + size_t(maxlen) * xs;
    double* ubuf = ss + size_t(maxlen) * 32;
    double* tbuf = ubuf + 32;
    double* ep = tbuf + 32;  // b, xe, scal, lam
    const int k0 = __ldg(a.ptr + row), k1 = __ldg(a.ptr + row + 1), nk = k1 - k0;
    if (!issued) split_row_issue(a, row, maxlen, sm, bar);
    // x-blocks: thread t -> (block q, entry c), every load issued before use
    for (int t = tid; t < nk * a.cbs; t += blockDim.x) {
        const int q = t / a.cbs, c = t - q * a.cbs;
        const int j = (t == tid && jfirst >= 0) ? jfirst : __ldg(a.col + k0 + q);
        sX[size_t(q) * xs + c] = x_source(a, row, j)[size_t(j) * a.cbs + c];
    }
    if (tid < a.rbs) {
        const size_t o = size_t(row) * a.rbs + tid;
        if (a.mode == MODE_RESIDUAL || relax) ep[tid] = __ldg(a.b + o);
        if (relax || a.mode == MODE_ADD) ep[32 + tid] = a.xe[o];
        if (relax) {
            ep[64 + tid] = __ldg(a.scal + o);
            ep[96 + tid] = __ldg(a.lam + o);
        }
    }
    __syncthreads();
    mbar_wait(bar, phase);
    phase ^= 1u;
    for (int q = warp; q < nk; q += W) {
        if (relax && __ldg(a.col + k0 + q) == row) continue;
        if (lane < a.rbs) {
            const double* Bc = sB + size_t(q) * a.blk_stride + lane;
            const double* xq = sX + size_t(q) * xs;
            double s = 0.0;
#pragma unroll 9
            for (int c = 0; c < a.cbs; ++c) s = madd_rn(s, Bc[size_t(c) * a.rbs], xq[c]);
            ss[size_t(q) * 32 + lane] = s;
        }
    }
    __syncthreads();
    if (warp == 0) {
        const bool act = lane < a.rbs;
        const size_t o = size_t(row) * a.rbs + lane;
        double acc = 0.0;
        if (act) {
            if (relax) {
                acc = ep[lane];
                for (int q = 0; q < nk; ++q)
                    if (__ldg(a.col + k0 + q) != row) acc = __dsub_rn(acc, ss[size_t(q) * 32 + lane]);
            } else {
                for (int q = 0; q < nk; ++q) acc = __dadd_rn(acc, ss[size_t(q) * 32 + lane]);
            }
        }
        if (relax) {
            const int bs = a.rbs, ld = a.ld;
            const double sc = act ? ep[64 + lane] : 0.0;
            const double lam = act ? ep[96 + lane] : 0.0;
            const double xe = act ? ep[32 + lane] : 0.0;
            if (act) ubuf[lane] = __dmul_rn(sc, acc);
            __syncwarp();
            if (act) {
                double tt = 0.0;
                const double* Vcol = sV + size_t(lane) * ld;
                for (int kk = 0; kk < bs; ++kk) tt = madd_rn(tt, Vcol[kk], ubuf[kk]);
                const double cut = a.kernel_tol * __ldg(a.lmax + row);
                tbuf[lane] = fabs(lam) <= cut ? 0.0 : tt / lam;
            }
            __syncwarp();
            if (act) {
                double w = 0.0;
                for (int kk = 0; kk < bs; ++kk) w = madd_rn(w, sV[size_t(kk) * ld + lane], tbuf[kk]);
                const double yv = __dmul_rn(sc, w);
                acc = __dadd_rn(__dmul_rn(1.0 - a.omega, xe), __dmul_rn(a.omega, yv));
            }
        }
        if (act) {
            double out;
            switch (a.mode) {
                case MODE_RESIDUAL: out = __dsub_rn(ep[lane], acc); break;
                case MODE_ADD: out = __dadd_rn(ep[32 + lane], acc); break;
                default: out = acc; break;
            }
            a.y[o] = out;
        }
    }
    __syncthreads();
}

/// shared-memory doubles split_row_task_tma needs
__host__ __device__ inline size_t split_row_tma_doubles(int maxlen, int blk_stride, int vstride, int cbs) {
    return size_t(maxlen) * blk_stride + size_t(vstride) + size_t(maxlen) * ((cbs + 1) & ~1) + size_t(maxlen) * 32 +
           64 + 128;
}

/// Restriction of coarse element p (multigrid.hpp:127-149 order); `sh` holds
/// the children's blocks (<= 64 children x BS).  All CTA threads call it.
__device__ __forceinline__ void restrict_parent_task(const int* __restrict__ child_ptr, const int* __restrict__ child,
                                                     const int* __restrict__ orth, const double* __restrict__ K,
                                                     const double* __restrict__ rf, double* __restrict__ rc, int p,
                                                     int bss, int ncomp, double* sh, int* sch, int* sor) {
    const int BS = bss * ncomp;
    const int q0 = child_ptr[p], nch = child_ptr[p + 1] - q0;
    for (int q = threadIdx.x; q < nch; q += blockDim.x) {
        sch[q] = child[q0 + q];
        sor[q] = orth[sch[q]];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nch * BS; t += blockDim.x) {
        const int q = t / BS, e = t - q * BS;
        sh[t] = rf[size_t(sch[q]) * BS + e];
    }
    __syncthreads();
    for (int o = threadIdx.x; o < BS; o += blockDim.x) {
        const int c = o / bss, j = o - c * bss;
        double acc = 0.0;
        for (int q = 0; q < nch; ++q) {
            const double* src = sh + q * BS;
            const int ot = sor[q];
            if (ot < 0) {
                acc = __dadd_rn(acc, src[o]);
                continue;
            }
            const double* Ko = K + size_t(ot) * bss * bss + j;
            double s = 0.0;
#pragma unroll 9
            for (int i = 0; i < bss; ++i) s = madd_rn(s, __ldg(Ko + size_t(i) * bss), src[c * bss + i]);
            acc = __dadd_rn(acc, s);
        }
        rc[size_t(p) * BS + o] = acc;
    }
    __syncthreads();
}

/// Prolongation onto the children of coarse element p (multigrid.hpp:104-123).
__device__ __forceinline__ void prolong_parent_task(const int* __restrict__ child_ptr, const int* __restrict__ child,
                                                    const int* __restrict__ orth, const double* __restrict__ K,
                                                    const double* __restrict__ xc, double* __restrict__ xf, int p,
                                                    int bss, int ncomp, double* sx) {
    const int BS = bss * ncomp;
    for (int t = threadIdx.x; t < BS; t += blockDim.x) sx[t] = xc[size_t(p) * BS + t];
    __syncthreads();
    const int q0 = child_ptr[p], nch = child_ptr[p + 1] - q0;
    for (int t = threadIdx.x; t < nch * BS; t += blockDim.x) {
        const int q = t / BS, ii = t - q * BS;
        const int f = child[q0 + q], ot = orth[f];
        double* dst = xf + size_t(f) * BS + ii;
        if (ot < 0) {
            *dst = __dadd_rn(*dst, sx[ii]);
            continue;
        }
        const int c = ii / bss, i = ii - c * bss;
        const double* Ko = K + size_t(ot) * bss * bss + size_t(i) * bss;
        double s = 0.0;
#pragma unroll 9
        for (int j = 0; j < bss; ++j) s = madd_rn(s, __ldg(Ko + j), sx[c * bss + j]);
        *dst = __dadd_rn(*dst, s);
    }
    __syncthreads();
}

}  // namespace ldgmg_b200
