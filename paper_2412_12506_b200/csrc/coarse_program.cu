// Persistent cooperative kernel for the coarse levels of the V-cycle.
//
// Below a few thousand elements a level's operator passes are latency- and
// launch-bound (one CUDA-graph node per pass, 13-15 passes per level, 2x for
// coloured GS).  The whole V-cycle from the first small level down (smoother
// passes, residual, restriction, zeroing, the bottom pseudoinverse,
// prolongation, post-smoothing) is recorded once at setup as a straight-line
// program of ops and executed by ONE cooperative kernel that walks the
// program with a grid-wide barrier between ops.  Each op reuses the exact
// per-row / per-parent device code of the standalone kernels (row_ops.cuh),
// so the results are bit-identical to the launch-per-pass path
// (tests/test_gpu_coarse_program.py).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <functional>
#include <map>
#include <vector>

#include "core.hpp"
#include "mg.hpp"
#include "row_ops.cuh"

namespace cg = cooperative_groups;

namespace ldgmg_b200 {

enum CoarseOpType { OP_ROWS = 0, OP_COPY = 1, OP_ZERO = 2, OP_RESTRICT = 3, OP_PROLONG = 4, OP_PINV_T = 5, OP_PINV_X = 6 };

struct CoarseOp {
    int type;
    RowPassArgs rows;
    const int* child_ptr;
    const int* child;
    const int* orth;
    const double* K;
    int bss, ncomp, n_parents;
    const double* src;
    double* dst;
    int64_t count;
    const double* Vm;
    const double* lam;
    double cut;
    int n;
    // cluster tail, row ops: per-CTA wave plans precomputed on the host
    // (plan[cta] = offset of that CTA's plan within plan_base)
    const int* plan;
    const int* plan_base;
};

namespace {

__global__ void __launch_bounds__(256) coarse_program_kernel(const CoarseOp* __restrict__ ops, int nops, int maxlen) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int sch[64], sor[64];
    __shared__ CoarseOp sop;
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t nth = int64_t(gridDim.x) * blockDim.x;
    for (int i = 0; i < nops; ++i) {
        // stage the op descriptor once per CTA (one coalesced read, then smem)
        {
            const int nw = int(sizeof(CoarseOp) / sizeof(int));
            const int* src = reinterpret_cast<const int*>(ops + i);
            int* dst = reinterpret_cast<int*>(&sop);
            for (int w = threadIdx.x; w < nw; w += blockDim.x) dst[w] = src[w];
            __syncthreads();
        }
        const CoarseOp& op = sop;
        switch (op.type) {
            case OP_ROWS:
                for (int slot = blockIdx.x; slot < op.rows.nrows; slot += gridDim.x)
                    split_row_task(op.rows, row_at(op.rows, slot), maxlen, sm);
                break;
            case OP_COPY:
                for (int64_t t = tid; t < op.count; t += nth) op.dst[t] = op.src[t];
                break;
            case OP_ZERO:
                for (int64_t t = tid; t < op.count; t += nth) op.dst[t] = 0.0;
                break;
            case OP_RESTRICT:
                for (int p = blockIdx.x; p < op.n_parents; p += gridDim.x)
                    restrict_parent_task(op.child_ptr, op.child, op.orth, op.K, op.src, op.dst, p, op.bss, op.ncomp,
                                         sm, sch, sor);
                break;
            case OP_PROLONG:
                for (int p = blockIdx.x; p < op.n_parents; p += gridDim.x)
                    prolong_parent_task(op.child_ptr, op.child, op.orth, op.K, op.src, op.dst, p, op.bss, op.ncomp,
                                        sm);
                break;
            case OP_PINV_T:  // t_i = cut(sum_k V(k,i) b_k) / lambda_i, Vm row-major
                for (int64_t t = tid; t < op.n; t += nth) {
                    double s = 0.0;
#pragma unroll 8
                    for (int k = 0; k < op.n; ++k) s = madd_rn(s, __ldg(op.Vm + size_t(k) * op.n + t), op.src[k]);
                    const double l = op.lam[t];
                    op.dst[t] = fabs(l) <= op.cut ? 0.0 : s / l;
                }
                break;
            case OP_PINV_X:  // x_i = sum_k V(i,k) t_k, Vm column-major
                for (int64_t t = tid; t < op.n; t += nth) {
                    double s = 0.0;
#pragma unroll 8
                    for (int k = 0; k < op.n; ++k) s = madd_rn(s, __ldg(op.Vm + size_t(k) * op.n + t), op.src[k]);
                    op.dst[t] = s;
                }
                break;
        }
        grid.sync();  // also orders the next descriptor load after this op's smem reads
    }
}

// ------------------------------------------------------------------------
// Cluster tail: the same program run by ONE thread-block cluster (up to 16
// CTAs on 16 SMs of one GPC) with hardware cluster barriers between ops
// instead of grid-wide ones.  Used for the tail of the hierarchy whose level
// operators are only a few MB (C2 from 4^3, C1 from 16^2), where every
// graph-launched pass costs ~4-7 us of launch and dependency latency for
// ~1 us of work.  Every op keeps the reference order of the standalone
// kernels (bit-identical).  Data written inside the kernel (iterates,
// residuals, right-hand sides) is read with ld.global.cg (L2, never a stale
// L1 line) after the release/acquire cluster barrier; immutable operands
// (blocks, factors, K, bottom V) use TMA bulk copies / the read-only path.

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int kTailThreads = 512;

/// dst[t] = f(t) for t < n over the CTA, 4 loads in flight per thread (the
/// plain strided loop waits one memory latency per iteration)
template <class F>
__device__ __forceinline__ void tail_gather(double* dst, int n, F f) {
    const int B = blockDim.x;
    for (int t0 = threadIdx.x; t0 < n; t0 += 4 * B) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = (t0 + u * B < n) ? f(t0 + u * B) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (t0 + u * B < n) dst[t0 + u * B] = v[u];
    }
}

constexpr int kTailMaxRows = 64;     // rows per wave
constexpr int kTailMaxBlocks = 512;  // blocks per wave

/// One row op over the cluster: CTA `cta` of `ncta` takes rows cta, cta+ncta,
/// ... in waves that fit shared memory.  Per wave every step is flat over
/// the wave's blocks, not per row: the rows' contiguous blocks (and relax
/// factors V) arrive by TMA bulk copies, all x blocks and epilogue operands
/// are gathered in one pass (two dependent L2 round trips per wave), warps
/// compute s_k over all (row, block) items, then one warp per row combines
/// them in CSR order and runs the epilogue (split_row_task_tma's
/// arithmetic).  rbs, cbs <= 32.
__device__ void tail_rows(const RowPassArgs& a, const int* plan, int cta, double* sm, uint64_t* bar,
                          uint32_t& phase, int* srow, int* sk0, int* snk, int* soff, int* bk, int* bi,
                          long long* tprof) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, tid = threadIdx.x;
    const bool relax = a.mode == MODE_RELAX;
    const int xs = (a.cbs + 1) & ~1;
    const int nwaves = __ldg(plan);
    const int* wp = plan + 1;
    (void)cta;
    for (int wv = 0; wv < nwaves; ++wv) {
        if (tprof && tid == 0 && cta == 0) tprof[0] = clock64();
        // the wave's plan (rows, row pointers, per-block column / local row),
        // precomputed on the host: one coalesced copy
        const int nr = wp[0], nb = wp[1];
        {
            const int* rowv = wp + 2;
            const int* k0v = rowv + nr;
            const int* nkv = k0v + nr;
            const int* sov = nkv + nr;
            const int* bjv = sov + nr;
            const int* biv = bjv + nb;
            for (int t = tid; t < nr; t += blockDim.x) {
                srow[t] = __ldg(rowv + t);
                sk0[t] = __ldg(k0v + t);
                snk[t] = __ldg(nkv + t);
                soff[t] = __ldg(sov + t);
            }
            for (int t = tid; t < nb; t += blockDim.x) {
                bk[t] = __ldg(bjv + t);
                bi[t] = __ldg(biv + t);
            }
            wp = biv + nb;
        }
        __syncthreads();
        double* sB = sm;                                         // nb blocks
        double* sV = sB + size_t(nb) * a.blk_stride;             // nr factors
        double* sX = sV + (relax ? size_t(nr) * a.vstride : 0);  // nb x-blocks
        double* ss = sX + size_t(nb) * xs;                       // nb x 32 partial sums
        double* ep = ss + size_t(nb) * 32;                       // nr x (b, xe, scal, lam) x 32
        if (tid == 0) {
            fence_proxy_async();  // earlier generic reads of these stages precede the async writes
            const uint32_t bytes =
                uint32_t(nb) * uint32_t(a.blk_stride) * 8u + (relax ? uint32_t(nr * a.vstride) * 8u : 0u);
            mbar_arrive_expect_tx(bar, bytes);
            for (int i = 0; i < nr; ++i) {
                bulk_g2s(sB + size_t(soff[i]) * a.blk_stride, a.val + size_t(sk0[i]) * a.blk_stride,
                         uint32_t(snk[i]) * uint32_t(a.blk_stride) * 8u, bar);
                if (relax)
                    bulk_g2s(sV + size_t(i) * a.vstride, a.V + size_t(srow[i]) * a.vstride, uint32_t(a.vstride) * 8u,
                             bar);
            }
        }
        // every x block of the wave in one pass, then the epilogue operands
        {
            const int cbs = a.cbs;
            for (int t0 = tid; t0 < nb * cbs; t0 += 4 * int(blockDim.x)) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int t = t0 + u * int(blockDim.x);
                    if (t < nb * cbs) {
                        const int q = t / cbs, c = t - q * cbs;
                        v[u] = __ldcg(a.x + size_t(bk[q]) * cbs + c);  // bk = column index
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int t = t0 + u * int(blockDim.x);
                    if (t < nb * cbs) {
                        const int q = t / cbs, c = t - q * cbs;
                        sX[size_t(q) * xs + c] = v[u];
                    }
                }
            }
        }
        for (int t = tid; t < nr * 32; t += blockDim.x) {
            const int i = t >> 5, r = t & 31;
            if (r >= a.rbs) continue;
            const size_t o = size_t(srow[i]) * a.rbs + r;
            double* e = ep + size_t(i) * 128;
            if (a.mode == MODE_RESIDUAL || relax) e[r] = __ldcg(a.b + o);
            if (relax || a.mode == MODE_ADD) e[32 + r] = __ldcg(a.xe + o);
            if (relax) {
                e[64 + r] = __ldg(a.scal + o);
                e[96 + r] = __ldg(a.lam + o);
            }
        }
        if (tprof && tid == 0 && cta == 0) tprof[1] = clock64();
        __syncthreads();
        mbar_wait(bar, phase);
        phase ^= 1u;
        if (tprof && tid == 0 && cta == 0) tprof[2] = clock64();
        // s_k over all (row, block) items, one warp per item
        for (int q = warp; q < nb; q += 2 * W) {
            // two blocks per warp step, chains interleaved (each keeps its order)
            const int q2 = q + W;
            const bool d1 = !(relax && bk[q] == srow[bi[q]]);
            const bool d2 = q2 < nb && !(relax && bk[q2] == srow[bi[q2]]);
            if (lane < a.rbs) {
                const double* B1 = sB + size_t(q) * a.blk_stride + lane;
                const double* X1 = sX + size_t(q) * xs;
                const double* B2 = sB + size_t(q2 < nb ? q2 : q) * a.blk_stride + lane;
                const double* X2 = sX + size_t(q2 < nb ? q2 : q) * xs;
                double u = 0.0, v = 0.0;
#pragma unroll 9
                for (int c = 0; c < a.cbs; ++c) {
                    u = madd_rn(u, B1[size_t(c) * a.rbs], X1[c]);
                    v = madd_rn(v, B2[size_t(c) * a.rbs], X2[c]);
                }
                if (d1) ss[size_t(q) * 32 + lane] = u;
                if (d2) ss[size_t(q2) * 32 + lane] = v;
            }
        }
        __syncthreads();
        if (tprof && tid == 0 && cta == 0) tprof[3] = clock64();
        // epilogue, one warp per row
        for (int i = warp; i < nr; i += W) {
            const bool act = lane < a.rbs;
            const int row = srow[i];
            const double* e = ep + size_t(i) * 128;
            double acc = 0.0;
            if (act) {
                if (relax) {
                    acc = e[lane];
                    for (int q = 0; q < snk[i]; ++q)
                        if (__ldg(a.col + sk0[i] + q) != row) acc = __dsub_rn(acc, ss[size_t(soff[i] + q) * 32 + lane]);
                } else {
                    for (int q = 0; q < snk[i]; ++q) acc = __dadd_rn(acc, ss[size_t(soff[i] + q) * 32 + lane]);
                }
            }
            if (relax) {
                // reuse this row's x-block slots as the u / t scratch (consumed above)
                double* ubuf = sX + size_t(soff[i]) * xs;
                double* tbuf = ss + size_t(soff[i]) * 32;
                const int bs = a.rbs, ld = a.ld;
                const double* Vr = sV + size_t(i) * a.vstride;
                const double sc = act ? e[64 + lane] : 0.0;
                const double lam = act ? e[96 + lane] : 0.0;
                const double xe = act ? e[32 + lane] : 0.0;
                __syncwarp();
                if (act) ubuf[lane] = __dmul_rn(sc, acc);
                __syncwarp();
                double tv = 0.0;
                if (act) {
                    double tt = 0.0;
                    const double* Vcol = Vr + size_t(lane) * ld;
                    for (int kk = 0; kk < bs; ++kk) tt = madd_rn(tt, Vcol[kk], ubuf[kk]);
                    const double cut = a.kernel_tol * __ldg(a.lmax + row);
                    tv = fabs(lam) <= cut ? 0.0 : tt / lam;
                }
                __syncwarp();
                if (act) tbuf[lane] = tv;
                __syncwarp();
                if (act) {
                    double w = 0.0;
                    for (int kk = 0; kk < bs; ++kk) w = madd_rn(w, Vr[size_t(kk) * ld + lane], tbuf[kk]);
                    const double yv = __dmul_rn(sc, w);
                    acc = __dadd_rn(__dmul_rn(1.0 - a.omega, xe), __dmul_rn(a.omega, yv));
                }
            }
            if (act) {
                double out;
                switch (a.mode) {
                    case MODE_RESIDUAL: out = __dsub_rn(e[lane], acc); break;
                    case MODE_ADD: out = __dadd_rn(e[32 + lane], acc); break;
                    default: out = acc; break;
                }
                a.y[size_t(row) * a.rbs + lane] = out;
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kTailThreads) coarse_cluster_kernel(const CoarseOp* __restrict__ ops, int nops,
                                                                      int sm_doubles, long long* prof) {
    extern __shared__ __align__(128) double tsm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ int srow[kTailMaxRows], sk0[kTailMaxRows], snk[kTailMaxRows], soff[kTailMaxRows];
    __shared__ int bk[kTailMaxBlocks], bi[kTailMaxBlocks];
    __shared__ CoarseOp sop;
    const int cta = blockIdx.x, ncta = gridDim.x, tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    const int64_t gt = int64_t(cta) * blockDim.x + tid, nth = int64_t(ncta) * blockDim.x;
    for (int i = 0; i < nops; ++i) {
        if (prof && tid == 0) prof[size_t(cta) * (nops + 1) + i] = clock64();
        {
            const int nw = int(sizeof(CoarseOp) / sizeof(int));
            const int* src = reinterpret_cast<const int*>(ops + i);
            int* dst = reinterpret_cast<int*>(&sop);
            for (int w = tid; w < nw; w += blockDim.x) dst[w] = src[w];
            __syncthreads();
        }
        const CoarseOp& op = sop;
        switch (op.type) {
            case OP_ROWS:
                tail_rows(op.rows, op.plan_base + __ldg(op.plan + cta), cta, tsm, &bar, phase, srow, sk0, snk, soff,
                          bk, bi, prof ? prof + size_t(ncta) * (nops + 1) + size_t(i) * 4 : nullptr);
                break;
            case OP_COPY:
                for (int64_t t = gt; t < op.count; t += nth) op.dst[t] = __ldcg(op.src + t);
                break;
            case OP_ZERO:
                for (int64_t t = gt; t < op.count; t += nth) op.dst[t] = 0.0;
                break;
            case OP_RESTRICT:
            case OP_PROLONG: {
                // operands staged first (K, the parents' child blocks / coarse
                // blocks), then every chain runs from shared memory; restriction
                // sums s_q in child order (restrict_parent_task's bits),
                // prolongation adds per entry (prolong_parent_task's bits)
                const int BS = op.bss * op.ncomp, bb = op.bss * op.bss;
                const int nK = (op.child_ptr ? 0 : 0) + 8 * bb;  // up to 2^3 injection matrices
                double* sK = tsm;
                double* sx = sK + nK;       // child blocks (restrict) or the coarse block (prolong)
                double* ssum = sx + 64 * BS;
                tail_gather(sK, nK, [&](int t) { return __ldg(op.K + t); });
                for (int p = cta; p < op.n_parents; p += ncta) {
                    const int q0 = __ldg(op.child_ptr + p), nch = __ldg(op.child_ptr + p + 1) - q0;
                    if (op.type == OP_RESTRICT) {
                        tail_gather(sx, nch * BS, [&](int t) {
                            const int q = t / BS, e = t - q * BS;
                            return __ldcg(op.src + size_t(__ldg(op.child + q0 + q)) * BS + e);
                        });
                    } else {
                        for (int t = tid; t < BS; t += blockDim.x) sx[t] = __ldcg(op.src + size_t(p) * BS + t);
                    }
                    __syncthreads();
                    for (int t = tid; t < nch * BS; t += blockDim.x) {
                        const int q = t / BS, o = t - q * BS;
                        const int f = __ldg(op.child + q0 + q), ot = __ldg(op.orth + f);
                        const int c = o / op.bss, jj = o - c * op.bss;
                        if (op.type == OP_RESTRICT) {
                            const double* src = sx + q * BS;
                            double sq;
                            if (ot < 0) {
                                sq = src[o];
                            } else {
                                const double* Ko = sK + size_t(ot) * bb + jj;
                                sq = 0.0;
                                for (int ii = 0; ii < op.bss; ++ii)
                                    sq = madd_rn(sq, Ko[size_t(ii) * op.bss], src[c * op.bss + ii]);
                            }
                            ssum[t] = sq;
                        } else {
                            double* dst = op.dst + size_t(f) * BS + o;
                            const double old = __ldcg(dst);
                            if (ot < 0) {
                                *dst = __dadd_rn(old, sx[o]);
                            } else {
                                const double* Ko = sK + size_t(ot) * bb + size_t(jj) * op.bss;
                                double s = 0.0;
                                for (int j = 0; j < op.bss; ++j) s = madd_rn(s, Ko[j], sx[c * op.bss + j]);
                                *dst = __dadd_rn(old, s);
                            }
                        }
                    }
                    __syncthreads();
                    if (op.type == OP_RESTRICT) {
                        for (int o = tid; o < BS; o += blockDim.x) {
                            double acc = 0.0;
                            for (int q = 0; q < nch; ++q) acc = __dadd_rn(acc, ssum[q * BS + o]);
                            op.dst[size_t(p) * BS + o] = acc;
                        }
                        __syncthreads();
                    }
                }
                break;
            }
            case OP_PINV_T:
            case OP_PINV_X: {
                // src staged in every CTA's shared memory; CTA c owns a
                // contiguous chunk of outputs (coalesced V reads), every
                // output one k-ascending chain (pinv_apply order)
                double* sv = tsm;
                for (int k = tid; k < op.n; k += blockDim.x) sv[k] = __ldcg(op.src + k);
                const int chunk = (op.n + ncta - 1) / ncta;
                const int t0 = cta * chunk, t1 = min(op.n, t0 + chunk), w = t1 - t0;
                double* sVc = sv + ((op.n + 1) & ~1);  // this CTA's columns, [k][w]
                const bool staged = size_t(op.n) * w + size_t((op.n + 1) & ~1) <= size_t(sm_doubles);
                if (staged)
                    tail_gather(sVc, op.n * w, [&](int e) {
                        const int k = e / w, c = e - k * w;
                        return __ldg(op.Vm + size_t(k) * op.n + t0 + c);
                    });
                __syncthreads();
                for (int c = tid; c < w; c += blockDim.x) {
                    double s = 0.0;
                    if (staged)
                        for (int k = 0; k < op.n; ++k) s = madd_rn(s, sVc[size_t(k) * w + c], sv[k]);
                    else
                        for (int k = 0; k < op.n; ++k) s = madd_rn(s, __ldg(op.Vm + size_t(k) * op.n + t0 + c), sv[k]);
                    const int t = t0 + c;
                    if (op.type == OP_PINV_T) {
                        const double l = __ldg(op.lam + t);
                        op.dst[t] = fabs(l) <= op.cut ? 0.0 : s / l;
                    } else {
                        op.dst[t] = s;
                    }
                }
                break;
            }
        }
        cluster_sync_all();  // op results visible cluster-wide; descriptor reloaded after
    }
    if (prof && tid == 0) prof[size_t(cta) * (nops + 1) + nops] = clock64();
}

CoarseOp rows_op(const Bsr& A, int mode, const double* x, const double* b, const double* xe, double* y,
                 const int* rows, int nrows, const DiagFactors* F, double omega) {
    CoarseOp op{};
    op.type = OP_ROWS;
    RowPassArgs& a = op.rows;
    a.ptr = A.ptr.as<int>();
    a.col = A.col.as<int>();
    a.val = A.val.as<double>();
    a.blk_stride = A.blk_stride;
    a.rbs = A.rbs;
    a.cbs = A.cbs;
    a.mode = mode;
    a.x = x;
    a.b = b;
    a.xe = xe;
    a.y = y;
    a.rows = rows;
    a.nrows = nrows;
    a.omega = omega;
    a.kernel_tol = 1e-12;
    if (F) {
        a.V = F->V.as<double>();
        a.lam = F->lambda.as<double>();
        a.scal = F->scale.as<double>();
        a.lmax = F->lmax.as<double>();
        a.ld = F->ld;
        a.vstride = F->vstride;
    }
    return op;
}

}  // namespace

/// Record the V-cycle of levels >= lc (Mg::v_cycle order) as a program.
void Mg::build_coarse_program(Ctx& ctx) {
    coarse_level = -1;
    coarse_cluster = 0;
    int lc = -1;
    // LDGMG_COARSE_ROWS=n (> 0): grid-wide cooperative program for levels with
    // <= n elements.  LDGMG_TAIL=1: the cluster tail for the levels whose
    // operators are at most LDGMG_TAIL_BYTES (default 4 MB: ~256 KB per CTA
    // of a 16-CTA cluster).  Both are bit-identical to the graph-launched
    // passes and both measured slower on B200 (C2: 3.25 -> 3.62 ms grid-wide,
    // 3.20 -> 3.49 ms cluster: 18 dependent ops on one cluster take 350 us,
    // mostly cluster-barrier waits behind the busiest CTA's load round trips,
    // against ~85 us of graph nodes), so both are off by default.
    static int tail_env = -2;
    static long long tail_bytes = 0;
    if (tail_env == -2) {
        const char* e = getenv("LDGMG_TAIL");
        tail_env = e ? atoi(e) : 0;
        const char* tb = getenv("LDGMG_TAIL_BYTES");
        tail_bytes = tb ? atoll(tb) : (4ll << 20);
    }
    bool cluster = false;
    if (coarse_rows > 0) {
        for (int l = 1; l + 1 < depth; ++l)
            if (A[l]->brows <= coarse_rows) {
                lc = l;
                break;
            }
    } else if (tail_env) {
        for (int l = 1; l + 1 < depth; ++l)
            if (int64_t(A[l]->nnzb) * A[l]->blk_stride * 8 <= tail_bytes) {
                lc = l;
                break;
            }
        cluster = true;
    }
    if (lc < 0) return;
    int coop = 0;
    LDGMG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx.device));
    if (cluster) LDGMG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrClusterLaunch, ctx.device));
    if (!coop || bottom.n > 4096) return;
    int maxlen = 1;
    for (int l = lc; l < depth; ++l) {
        if (A[l]->rbs > 32) return;  // split-row ops need bs <= 32
        if (l + 1 < depth && sm[l]->cfg.kind == LDGMG_PROC_BLOCK_GS) return;  // not recorded
        maxlen = std::max(maxlen, A[l]->max_row);
        if (l + 1 < depth && T[l]->max_children > 64) return;
    }
    std::vector<CoarseOp> prog;
    auto smooth = [&](int l, double* x, const double* b, int sweep) {
        const Smoother& S = *sm[l];
        const int N = A[l]->brows;
        if (S.cfg.kind == LDGMG_JACOBI) {
            CoarseOp c{};
            c.type = OP_COPY;
            c.src = x;
            c.dst = S.snap.as<double>();
            c.count = int64_t(N) * bs;
            prog.push_back(c);
            prog.push_back(rows_op(*A[l], MODE_RELAX, S.snap.as<double>(), b, x, x, nullptr, N, &S.F, S.cfg.omega));
        } else if (S.cfg.kind == LDGMG_COLOURED_GS) {
            for (int ci = 0; ci < S.ncolours; ++ci) {
                const int c = sweep == LDGMG_SWEEP_FORWARD ? ci : S.ncolours - 1 - ci;
                prog.push_back(rows_op(*A[l], MODE_RELAX, x, b, x, x, S.colour_rows.as<int>() + S.colour_ptr[c],
                                       S.colour_ptr[c + 1] - S.colour_ptr[c], &S.F, 1.0));
            }
        } else {
            double* r = S.snap.as<double>();
            prog.push_back(rows_op(*A[l], MODE_RESIDUAL, x, b, nullptr, r, nullptr, N, nullptr, 1.0));
            const Bsr& Bm = sweep == LDGMG_SWEEP_FORWARD ? *S.B : bsr_transpose(ctx, *S.B);
            prog.push_back(rows_op(Bm, MODE_ADD, r, nullptr, x, x, nullptr, N, nullptr, 1.0));
        }
    };
    std::function<void(int, double*, const double*)> emit = [&](int l, double* x, const double* b) {
        if (l + 1 == depth) {
            CoarseOp t{};
            t.type = OP_PINV_T;
            t.Vm = bottom.Vr.as<double>();
            t.lam = bottom.lambda.as<double>();
            t.cut = cfg.bottom_tol * bottom.lmax;
            t.n = bottom.n;
            t.src = b;
            t.dst = bottom.t.as<double>();
            prog.push_back(t);
            CoarseOp u{};
            u.type = OP_PINV_X;
            u.Vm = bottom.Vc.as<double>();
            u.n = bottom.n;
            u.src = bottom.t.as<double>();
            u.dst = x;
            prog.push_back(u);
            return;
        }
        for (int i = 0; i < cfg.nu1; ++i) smooth(l, x, b, cfg.pre);
        prog.push_back(rows_op(*A[l], MODE_RESIDUAL, x, b, nullptr, r[l].as<double>(), nullptr, A[l]->brows, nullptr, 1.0));
        CoarseOp rs{};
        rs.type = OP_RESTRICT;
        rs.child_ptr = T[l]->child_ptr.as<int>();
        rs.child = T[l]->child_list.as<int>();
        rs.orth = T[l]->orth.as<int>();
        rs.K = T[l]->K.as<double>();
        rs.bss = T[l]->bss;
        rs.ncomp = T[l]->ncomp;
        rs.n_parents = T[l]->n_coarse;
        rs.src = r[l].as<double>();
        rs.dst = bl[l + 1].as<double>();
        prog.push_back(rs);
        CoarseOp z{};
        z.type = OP_ZERO;
        z.dst = xl[l + 1].as<double>();
        z.count = int64_t(A[l + 1]->brows) * bs;
        prog.push_back(z);
        emit(l + 1, xl[l + 1].as<double>(), bl[l + 1].as<double>());
        CoarseOp pr = rs;
        pr.type = OP_PROLONG;
        pr.src = xl[l + 1].as<double>();
        pr.dst = x;
        prog.push_back(pr);
        for (int i = 0; i < cfg.nu2; ++i) smooth(l, x, b, cfg.post);
    };
    emit(lc, xl[lc].as<double>(), bl[lc].as<double>());
    coarse_prog.alloc(sizeof(CoarseOp) * prog.size());
    h2d(ctx, coarse_prog.p, prog.data(), sizeof(CoarseOp) * prog.size());
    coarse_nops = int(prog.size());
    coarse_maxlen = maxlen;
    int maxbs = 0, maxch = 1;
    for (int l = lc; l < depth; ++l) {
        maxbs = std::max(maxbs, A[l]->rbs);
        if (l + 1 < depth) maxch = std::max(maxch, T[l]->max_children);
    }
    if (cluster) {
        // one cluster of up to 16 CTAs (non-portable size), ~200 KB of shared memory each
        const size_t sm_doubles = 200 * 1024 / 8;
        if (sm_doubles < size_t(maxch) * maxbs) return;
        int csize = 16;
        if (const char* e = getenv("LDGMG_TAIL_CTAS")) csize = std::max(1, std::min(16, atoi(e)));
        LDGMG_CUDA(cudaFuncSetAttribute(coarse_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        LDGMG_CUDA(cudaFuncSetAttribute(coarse_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(sm_doubles * 8)));
        for (; csize >= 1; csize /= 2) {
            cudaLaunchConfig_t lc_cfg{};
            lc_cfg.gridDim = dim3(csize);
            lc_cfg.blockDim = dim3(kTailThreads);
            lc_cfg.dynamicSmemBytes = sm_doubles * 8;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = csize;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc_cfg.attrs = at;
            lc_cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, coarse_cluster_kernel, &lc_cfg) == cudaSuccess &&
                nclusters >= 1)
                break;
            cudaGetLastError();
        }
        if (csize < 1) return;
        // per-CTA wave plans of every row op, precomputed here (the device
        // only copies them): rows, row pointers, shared-memory offsets, and
        // each block's column index and local row
        std::map<const int*, const Bsr*> byptr;
        for (int l = lc; l < depth; ++l) {
            byptr[A[l]->ptr.as<int>()] = A[l];
            if (l + 1 < depth && sm[l]->B) {
                const Bsr* Bm = sm[l]->B.get();
                byptr[Bm->ptr.as<int>()] = Bm;
                if (Bm->T) byptr[Bm->T->ptr.as<int>()] = Bm->T.get();
            }
        }
        std::vector<int> plan;
        std::vector<std::pair<size_t, size_t>> op_plan(prog.size(), {0, 0});  // (offsets index, -)
        for (size_t oi = 0; oi < prog.size(); ++oi) {
            CoarseOp& op = prog[oi];
            if (op.type != OP_ROWS) continue;
            const RowPassArgs& ra = op.rows;
            auto it = byptr.find(ra.ptr);
            if (it == byptr.end()) return;  // unknown operator: no cluster tail
            const Bsr& M = *it->second;
            std::vector<int> rows(ra.nrows);
            if (ra.rows) {
                d2h(ctx, rows.data(), ra.rows, sizeof(int) * ra.nrows);
            } else {
                for (int i = 0; i < ra.nrows; ++i) rows[i] = i;
            }
            const bool relax = ra.mode == MODE_RELAX;
            const size_t xs = size_t((ra.cbs + 1) & ~1);
            const size_t offs_at = plan.size();
            plan.resize(plan.size() + csize, 0);
            for (int c = 0; c < csize; ++c) {
                plan[offs_at + c] = int(plan.size());  // this CTA's plan: index within plan_base
                const size_t nw_at = plan.size();
                plan.push_back(0);
                std::vector<int> mine;
                for (int sl = c; sl < ra.nrows; sl += csize) mine.push_back(rows[sl]);
                for (size_t k = 0; k < mine.size();) {
                    std::vector<int> wr, wk0, wnk, wso, wbj, wbi;
                    size_t need = 0;
                    int nb = 0;
                    while (k < mine.size() && int(wr.size()) < kTailMaxRows) {
                        const int row = mine[k];
                        const int k0 = M.hptr[row], len = M.hptr[row + 1] - k0;
                        const size_t add = size_t(len) * (size_t(ra.blk_stride) + xs + 32) +
                                           (relax ? size_t(ra.vstride) : 0) + 128;
                        if (!wr.empty() && (need + add > sm_doubles || nb + len > kTailMaxBlocks)) break;
                        if (len > kTailMaxBlocks || add > sm_doubles) return;  // row does not fit a wave
                        wr.push_back(row);
                        wk0.push_back(k0);
                        wnk.push_back(len);
                        wso.push_back(nb);
                        for (int q = 0; q < len; ++q) {
                            wbj.push_back(M.hcol[k0 + q]);
                            wbi.push_back(int(wr.size()) - 1);
                        }
                        need += add;
                        nb += len;
                        ++k;
                    }
                    plan.push_back(int(wr.size()));
                    plan.push_back(nb);
                    for (auto* v : {&wr, &wk0, &wnk, &wso, &wbj, &wbi}) plan.insert(plan.end(), v->begin(), v->end());
                    ++plan[nw_at];
                }
            }
            op_plan[oi] = {offs_at, 0};
        }
        coarse_plan.alloc(sizeof(int) * std::max<size_t>(1, plan.size()));
        if (!plan.empty()) h2d(ctx, coarse_plan.p, plan.data(), sizeof(int) * plan.size());
        for (size_t oi = 0; oi < prog.size(); ++oi) {
            if (prog[oi].type != OP_ROWS) continue;
            prog[oi].plan = coarse_plan.as<int>() + op_plan[oi].first;  // [csize] offsets into plan_base
            prog[oi].plan_base = coarse_plan.as<int>();
        }
        h2d(ctx, coarse_prog.p, prog.data(), sizeof(CoarseOp) * prog.size());
        coarse_cluster = csize;
        coarse_smem = sm_doubles * 8;
        coarse_level = lc;
        return;
    }
    coarse_smem = sizeof(double) * std::max<size_t>(size_t(maxlen) * 32 + 64, size_t(maxch) * maxbs);
    int occ = 0;
    LDGMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, coarse_program_kernel, 256, coarse_smem));
    if (occ < 1) return;
    static int env_grid = -2;
    if (env_grid == -2) {
        const char* e = getenv("LDGMG_COARSE_CTAS_PER_SM");
        env_grid = e ? atoi(e) : -1;
    }
    coarse_grid = ctx.num_sms * std::max(1, std::min(occ, env_grid > 0 ? env_grid : 1));
    coarse_level = lc;
}

void Mg::launch_coarse_program(Ctx& ctx) {
    const CoarseOp* ops = coarse_prog.as<CoarseOp>();
    int nops = coarse_nops, maxlen = coarse_maxlen;
    if (coarse_cluster) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(coarse_cluster);
        cfg.blockDim = dim3(kTailThreads);
        cfg.dynamicSmemBytes = coarse_smem;
        cfg.stream = ctx.stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = coarse_cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int smd = int(coarse_smem / 8);
        // LDGMG_TAIL_PROFILE=1: per-op clock64 stamps of every CTA, printed once
        static const bool tprof = getenv("LDGMG_TAIL_PROFILE") && atoi(getenv("LDGMG_TAIL_PROFILE"));
        static int printed = 0;
        long long* prof = nullptr;
        if (tprof && printed < 2)
            LDGMG_CUDA(cudaMallocManaged(&prof, sizeof(long long) * (coarse_cluster * (nops + 1) + 4 * nops)));
        cuda_check(cudaLaunchKernelEx(&cfg, coarse_cluster_kernel, ops, nops, smd, prof), "coarse_cluster_kernel");
        after_launch("coarse_cluster_kernel");
        if (prof) {
            LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
            std::vector<CoarseOp> h(nops);
            LDGMG_CUDA(cudaMemcpy(h.data(), ops, sizeof(CoarseOp) * nops, cudaMemcpyDeviceToHost));
            fprintf(stderr, "[tail] %d ops, cluster %d:", nops, coarse_cluster);
            for (int i = 0; i < nops; ++i) {
                long long mx = 0;
                for (int c = 0; c < coarse_cluster; ++c) {
                    const long long* pc = prof + size_t(c) * (nops + 1);
                    mx = std::max(mx, pc[i + 1] - pc[i]);
                }
                fprintf(stderr, " %d:%lld", h[i].type, mx);
            }
            fprintf(stderr, "\n[tail] CTA0 row-op phases (plan->issued, issued->data, data->computed):");
            for (int i = 0; i < nops; ++i)
                if (h[i].type == 0) {
                    const long long* q = prof + size_t(coarse_cluster) * (nops + 1) + size_t(i) * 4;
                    fprintf(stderr, " [%lld %lld %lld]", q[1] - q[0], q[2] - q[1], q[3] - q[2]);
                }
            fprintf(stderr, "\n");
            cudaFree(prof);
            ++printed;
        }
        return;
    }
    void* args[] = {&ops, &nops, &maxlen};
    LDGMG_CUDA(cudaLaunchCooperativeKernel((const void*)coarse_program_kernel, dim3(coarse_grid), dim3(256), args,
                                           coarse_smem, ctx.stream));
    after_launch("coarse_program_kernel");
}

}  // namespace ldgmg_b200
