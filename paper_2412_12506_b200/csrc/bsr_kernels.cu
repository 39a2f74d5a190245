// BSR storage and the streaming row-pass kernel: the HBM-bound hot loop of
// every operator application in the V-cycle.
//
// One "row group" (= one CTA of G warps, lane r <-> output row r of the block
// row) walks a persistent, grid-strided list of block rows.  The matrix
// blocks of those rows are streamed into a ring of shared-memory stages with
// TMA 1-D bulk copies (cp.async.bulk + mbarrier complete_tx); the matching
// x-blocks are gathered into per-stage slots with cp.async whose completion
// is folded into the same mbarrier.  NS items are always in flight per group,
// so HBM sees long contiguous bulk reads while the FP64 pipe does the dot
// products out of conflict-free shared memory.
//
// Arithmetic order is the reference's, bit for bit (compiled without FMA
// contraction; every multiply-add here is an explicit __dmul_rn/__dadd_rn):
//   spmv:      y_i[r] = 0 + s_k1 + s_k2 + ...,  s_k = 0 + b[r,0]x[0] + b[r,1]x[1] + ...
//              (blockla.hpp:141-153), blocks in CSR (ascending column) order;
//   residual:  b - (A x)   (multigrid.hpp:256-258);
//   add:       x + (B r)   (smoothers.hpp:441-446, axpy with alpha = 1);
//   relax:     r = ((b - s_k1) - s_k2) - ... over off-diagonal blocks, then
//              y = s o V diag(1/lambda, cut) V^T (s o r), x = (1-w) x + w y
//              (smoothers.hpp:496-518 with pinv_apply blockla.hpp:330-339 and
//              the Eigen-shim product order, oracle/shim/Eigen/Dense).
#include <cuda_runtime.h>

#include <mutex>

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <vector>

#include "core.hpp"
#include "host_eig.hpp"
#include "row_ops.cuh"

namespace ldgmg_b200 {

namespace {

/// Row descriptors of a CTA's grid-strided row sequence, pipelined so that
/// the dependent index loads (row list -> row pointers / diagonal position)
/// of row m+1 and m+2 are in flight while row m is processed: no warp ever
/// waits on an index load at a row boundary.
struct RowPipe {
    int m;
    int row, k0, k1, dk;          // row m (row = -1: exhausted)
    int n_row, n_k0, n_k1, n_dk;  // row m+1
    int nn_row;                   // row m+2
};

__device__ __forceinline__ int rp_row(const RowPassArgs& a, int m, int g, int ng) {
    const int slot = g + m * ng;
    return slot < a.nrows ? row_at(a, slot) : -1;
}

__device__ __forceinline__ void rp_fetch(const RowPassArgs& a, int row, int& k0, int& k1, int& dk) {
    if (row < 0) return;
    k0 = __ldg(a.ptr + row);
    k1 = __ldg(a.ptr + row + 1);
    dk = a.dpos ? __ldg(a.dpos + row) : -1;
}

__device__ __forceinline__ void rp_init(const RowPassArgs& a, RowPipe& p, int g, int ng) {
    p.m = 0;
    p.row = rp_row(a, 0, g, ng);
    p.n_row = rp_row(a, 1, g, ng);
    p.nn_row = rp_row(a, 2, g, ng);
    p.k0 = p.k1 = p.n_k0 = p.n_k1 = 0;
    p.dk = p.n_dk = -1;
    rp_fetch(a, p.row, p.k0, p.k1, p.dk);
    rp_fetch(a, p.n_row, p.n_k0, p.n_k1, p.n_dk);
}

__device__ __forceinline__ void rp_advance(const RowPassArgs& a, RowPipe& p, int g, int ng) {
    ++p.m;
    p.row = p.n_row;
    p.k0 = p.n_k0;
    p.k1 = p.n_k1;
    p.dk = p.n_dk;
    p.n_row = p.nn_row;
    rp_fetch(a, p.n_row, p.n_k0, p.n_k1, p.n_dk);
    p.nn_row = rp_row(a, p.m + 2, g, ng);
}

/// Producer iterator over the items of the CTA's rows (identical on every
/// thread).  The column index of the next block is loaded one item ahead,
/// so issuing an item never waits on it.
struct ItemIt {
    RowPipe rp;
    int k;      // next block of the current row
    int vdone;
    int jk, jv;  // prefetched column index: col[jk] = jv
};

__device__ __forceinline__ void it_prefetch_col(const RowPassArgs& a, ItemIt& it) {
    int k = it.k;
    if (k == it.rp.dk) ++k;  // relax skips the diagonal block (dk = -1 otherwise)
    it.jk = k;
    if (k < it.rp.k1) it.jv = __ldg(a.col + k);
}

__device__ __forceinline__ void it_start(const RowPassArgs& a, ItemIt& it, int g, int ng) {
    rp_init(a, it.rp, g, ng);
    it.k = it.rp.k0;
    it.vdone = 0;
    it.jk = -1;
    if (it.rp.row >= 0) it_prefetch_col(a, it);
}

/// Next item of the group's stream: kind 0 = matrix block `idx` (column
/// `j`), kind 1 = diagonal factor V of element `idx`.
__device__ __forceinline__ bool it_next(const RowPassArgs& a, ItemIt& it, int g, int ng, int& kind, int& idx,
                                        int& j) {
    for (;;) {
        if (it.rp.row < 0) return false;
        if (it.k == it.rp.dk) ++it.k;
        if (it.k < it.rp.k1) {
            kind = 0;
            idx = it.k;
            j = it.jk == idx ? it.jv : __ldg(a.col + idx);
            ++it.k;
            it_prefetch_col(a, it);
            return true;
        }
        if (a.mode == MODE_RELAX && !it.vdone) {
            it.vdone = 1;
            kind = 1;
            idx = it.rp.row;
            j = -1;
            return true;
        }
        rp_advance(a, it.rp, g, ng);
        it.k = it.rp.k0;
        it.vdone = 0;
        if (it.rp.row >= 0) it_prefetch_col(a, it);
    }
}

template <int GT>
__device__ __forceinline__ void issue_item(const RowPassArgs& a, int kind, int idx, int j, int row, int st,
                                           double* stages, double* xslots, uint64_t* bars, int* xoffs) {
    const int t = threadIdx.x;
    double* xs = xslots + size_t(st) * a.xslot_doubles;
    // one elected thread issues the block and (kind 0) the 16-byte aligned
    // window around x_j as two bulk copies on the stage's mbarrier
    if (t == 0) {
        const double* src;
        uint32_t bytes;
        if (kind == 0) {
            const int64_t blk = a.perm ? int64_t(__ldg(a.perm + idx)) : int64_t(idx);
            src = a.val + size_t(blk) * a.blk_stride;
            bytes = uint32_t(a.blk_stride) * 8u;
            const double* xsrc = x_source(a, row, j) + size_t(j) * a.cbs;
            const uintptr_t xa = reinterpret_cast<uintptr_t>(xsrc) & ~uintptr_t(15);
            const int off = int((reinterpret_cast<uintptr_t>(xsrc) - xa) >> 3);
            const uint32_t xbytes = (uint32_t((off + a.cbs) * 8) + 15u) & ~15u;
            xoffs[st] = off;
            mbar_arrive_expect_tx(bars + st, bytes + xbytes);
            bulk_g2s(stages + size_t(st) * a.stage_doubles, src, bytes, bars + st);
            bulk_g2s(xs, reinterpret_cast<const void*>(xa), xbytes, bars + st);
        } else {
            src = a.V + size_t(idx) * a.vstride;
            bytes = uint32_t(a.vstride) * 8u;
            mbar_arrive_expect_tx(bars + st, bytes);
            bulk_g2s(stages + size_t(st) * a.stage_doubles, src, bytes, bars + st);
        }
    }
}

/// s = 0 + B[t,0] X[0] + B[t,1] X[1] + ... from a column-major stage (lane t
/// holds Bc = stage + t); BS compile-time for the common block sizes (fully
/// unrolled, immediate offsets), 0 = runtime (any rbs x cbs).
template <int BS>
__device__ __forceinline__ double bdot(const double* __restrict__ Bc, const double* __restrict__ X, int cbs,
                                       int rbs) {
    double s = 0.0;
    if constexpr (BS > 0) {
#pragma unroll
        for (int c = 0; c < BS; ++c) s = madd_rn(s, Bc[c * BS], X[c]);
    } else {
#pragma unroll 8
        for (int c = 0; c < cbs; ++c) s = madd_rn(s, Bc[size_t(c) * rbs], X[c]);
    }
    return s;
}

/// Two independent block dot products interleaved: the sequential FP64 add
/// chain of one block is what bounds a warp, two chains double its ILP while
/// every s_k keeps the reference's order.
template <int BS>
__device__ __forceinline__ void bdot2(const double* __restrict__ B1, const double* __restrict__ X1,
                                      const double* __restrict__ B2, const double* __restrict__ X2, int cbs, int rbs,
                                      double& s1, double& s2) {
    double u = 0.0, v = 0.0;
    if constexpr (BS > 0) {
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            u = madd_rn(u, B1[c * BS], X1[c]);
            v = madd_rn(v, B2[c * BS], X2[c]);
        }
    } else {
#pragma unroll 4
        for (int c = 0; c < cbs; ++c) {
            u = madd_rn(u, B1[size_t(c) * rbs], X1[c]);
            v = madd_rn(v, B2[size_t(c) * rbs], X2[c]);
        }
    }
    s1 = u;
    s2 = v;
}

/// Transposed-view dot products: lane t reads ROW t of the transposed block,
/// i.e. the stored column t of the base block, consecutive words Bt[0..cbs)
/// (Bt = stage + t*cbs).  Odd cbs: 8-byte loads, lane stride odd ->
/// conflict-free.  Even cbs: 16-byte loads (pairs), conflict-free when cbs/2
/// is odd, 2-way for cbs = 108.  Sum order c = 0, 1, ... as bdot.
template <int BS>
__device__ __forceinline__ double bdot_t(const double* __restrict__ Bt, const double* __restrict__ X, int cbs) {
    double s = 0.0;
    if constexpr (BS > 0 && (BS % 2) == 0) {
        const double2* B2 = reinterpret_cast<const double2*>(Bt);
#pragma unroll
        for (int c = 0; c < BS / 2; ++c) {
            const double2 v = B2[c];
            s = madd_rn(s, v.x, X[2 * c]);
            s = madd_rn(s, v.y, X[2 * c + 1]);
        }
    } else if constexpr (BS > 0) {
#pragma unroll
        for (int c = 0; c < BS; ++c) s = madd_rn(s, Bt[c], X[c]);
    } else {
#pragma unroll 8
        for (int c = 0; c < cbs; ++c) s = madd_rn(s, Bt[c], X[c]);
    }
    return s;
}

template <int BS>
__device__ __forceinline__ void bdot2_t(const double* __restrict__ B1, const double* __restrict__ X1,
                                        const double* __restrict__ B2, const double* __restrict__ X2, int cbs,
                                        double& s1, double& s2) {
    double u = 0.0, v = 0.0;
    if constexpr (BS > 0 && (BS % 2) == 0) {
        const double2* P1 = reinterpret_cast<const double2*>(B1);
        const double2* P2 = reinterpret_cast<const double2*>(B2);
#pragma unroll
        for (int c = 0; c < BS / 2; ++c) {
            const double2 a1 = P1[c], a2 = P2[c];
            u = madd_rn(u, a1.x, X1[2 * c]);
            v = madd_rn(v, a2.x, X2[2 * c]);
            u = madd_rn(u, a1.y, X1[2 * c + 1]);
            v = madd_rn(v, a2.y, X2[2 * c + 1]);
        }
    } else if constexpr (BS > 0) {
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            u = madd_rn(u, B1[c], X1[c]);
            v = madd_rn(v, B2[c], X2[c]);
        }
    } else {
#pragma unroll 4
        for (int c = 0; c < cbs; ++c) {
            u = madd_rn(u, B1[c], X1[c]);
            v = madd_rn(v, B2[c], X2[c]);
        }
    }
    s1 = u;
    s2 = v;
}

template <int GT, int BS>
__global__ void __launch_bounds__(GT) rowpass_kernel(const RowPassArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* stages = reinterpret_cast<double*>(smem_raw);
    double* xslots = stages + size_t(a.nstages) * a.stage_doubles;
    double* ubuf = xslots + size_t(a.nstages) * a.xslot_doubles;
    double* tbuf = ubuf + a.xslot_doubles;
    uint64_t* bars = reinterpret_cast<uint64_t*>(tbuf + a.xslot_doubles);
    int* xoffs = reinterpret_cast<int*>(bars + a.nstages);  // x-TMA: start of x_j within each stage's slot

    const int t = threadIdx.x;
    const int g = blockIdx.x, ng = gridDim.x;
    const int NS = a.nstages;
    const int rbs = BS > 0 ? BS : a.rbs, cbs = BS > 0 ? BS : a.cbs;

    if (t == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(bars + s, 1u);
        fence_mbar_init();
    }
    __syncthreads();

    // producer iterator: runs NS items ahead of the consumer (row lists and
    // row pointers are immutable: read before the PDL wait)
    ItemIt pit;
    it_start(a, pit, g, ng);
    RowPipe crp;  // the consumer's own row pipeline (same row sequence)
    rp_init(a, crp, g, ng);
    pdl_wait();
    pdl_trigger();
    int kind, idx, jcol;
    for (int s = 0; s < NS; ++s) {
        if (!it_next(a, pit, g, ng, kind, idx, jcol)) break;
        issue_item<GT>(a, kind, idx, jcol, pit.rp.row, s, stages, xslots, bars, xoffs);
    }

    uint32_t q = 0;  // items consumed
    const bool relax = a.mode == MODE_RELAX;
    const bool pairs = NS >= 3;
    for (;; rp_advance(a, crp, g, ng)) {
        const int row = crp.row;
        if (row < 0) break;
        const int k0 = crp.k0, k1 = crp.k1, dk = crp.dk;
        const bool act = t < rbs;
        // epilogue operands fetched early; their latency hides under the blocks
        double pre_b = 0.0, pre_x = 0.0, pre_s = 0.0, pre_l = 0.0;
        if (act) {
            const size_t o = size_t(row) * rbs + t;
            if (a.mode == MODE_RESIDUAL || relax) pre_b = __ldg(a.b + o);
            if (a.mode == MODE_ADD || relax) pre_x = a.xe[o];
            if (relax) {
                pre_s = __ldg(a.scal + o);
                pre_l = __ldg(a.lam + o);
            }
        }
        double acc = relax ? pre_b : 0.0;
        int k = k0;
        bool vdone = !relax;
        for (;;) {
            if (k == dk) ++k;  // relax skips the diagonal block (dk = -1 otherwise)
            int nblk = 0, k2 = k;
            if (k < k1) {
                nblk = 1;
                k2 = k + 1;
                if (k2 == dk) ++k2;
                if (pairs && k2 < k1) nblk = 2;
            } else if (vdone) {
                break;
            }
            const int st = int(q % uint32_t(NS));
            mbar_wait(bars + st, (q / uint32_t(NS)) & 1u);
            const double* S = stages + size_t(st) * a.stage_doubles;
            const double* X = xslots + size_t(st) * a.xslot_doubles + xoffs[st];
            int used = 1;
            if (nblk == 2) {
                const int st2 = int((q + 1) % uint32_t(NS));
                mbar_wait(bars + st2, ((q + 1) / uint32_t(NS)) & 1u);
                if constexpr (BS > 0 && 2 * BS <= 32) {
                    // small blocks: the pair's second block on the upper lanes
                    // (one chain per lane instead of two), s2 shuffled down to
                    // lane r; the row sum still adds s1 then s2
                    const bool hi = t >= BS;
                    const int r = hi ? t - BS : t;
                    const double* Sx = hi ? stages + size_t(st2) * a.stage_doubles : S;
                    const double* Xx = hi ? xslots + size_t(st2) * a.xslot_doubles + xoffs[st2] : X;
                    double s = 0.0;
                    if (t < 2 * BS)
                        s = a.tview ? bdot_t<BS>(Sx + size_t(r) * cbs, Xx, cbs) : bdot<BS>(Sx + r, Xx, cbs, rbs);
                    const double s2 = __shfl_down_sync(0xffffffffu, s, BS);
                    if (act) {
                        acc = relax ? __dsub_rn(acc, s) : __dadd_rn(acc, s);
                        acc = relax ? __dsub_rn(acc, s2) : __dadd_rn(acc, s2);
                    }
                } else if (act) {
                    double s1, s2;
                    if (a.tview)
                        bdot2_t<BS>(S + size_t(t) * cbs, X, stages + size_t(st2) * a.stage_doubles + size_t(t) * cbs,
                                    xslots + size_t(st2) * a.xslot_doubles + xoffs[st2], cbs, s1, s2);
                    else
                        bdot2<BS>(S + t, X, stages + size_t(st2) * a.stage_doubles + t,
                                  xslots + size_t(st2) * a.xslot_doubles + xoffs[st2], cbs, rbs, s1,
                                  s2);
                    acc = relax ? __dsub_rn(acc, s1) : __dadd_rn(acc, s1);
                    acc = relax ? __dsub_rn(acc, s2) : __dadd_rn(acc, s2);
                }
                k = k2 + 1;
                used = 2;
            } else if (nblk == 1) {
                if (act) {
                    const double s = a.tview ? bdot_t<BS>(S + size_t(t) * cbs, X, cbs) : bdot<BS>(S + t, X, cbs, rbs);
                    acc = relax ? __dsub_rn(acc, s) : __dadd_rn(acc, s);
                }
                k = k + 1;
            } else {
                // block-diagonal pseudoinverse solve with the staged factor V
                const int bs = rbs, ld = a.ld;
                if (act) ubuf[t] = __dmul_rn(pre_s, acc);
                group_sync(1, GT);
                if (act) {
                    double tt = 0.0;
                    const double* Vcol = S + size_t(t) * ld;  // V(:, t)
#pragma unroll 8
                    for (int kk = 0; kk < bs; ++kk) tt = madd_rn(tt, Vcol[kk], ubuf[kk]);
                    const double cut = a.kernel_tol * __ldg(a.lmax + row);
                    tbuf[t] = fabs(pre_l) <= cut ? 0.0 : tt / pre_l;
                }
                group_sync(1, GT);
                if (act) {
                    double w = 0.0;
#pragma unroll 8
                    for (int kk = 0; kk < bs; ++kk) w = madd_rn(w, S[size_t(kk) * ld + t], tbuf[kk]);
                    const double yv = __dmul_rn(pre_s, w);
                    const double om = a.omega;
                    double px = pre_x;
                    asm volatile("" : "+d"(px));  // keep (1 - w) x here, not at the row-start load
                    acc = __dadd_rn(__dmul_rn(1.0 - om, px), __dmul_rn(om, yv));
                }
                vdone = true;
            }
            group_sync(1, GT);  // every lane is done with these stages
            for (int u = 0; u < used; ++u) {
                const int su = int(q % uint32_t(NS));
                ++q;
                if (it_next(a, pit, g, ng, kind, idx, jcol)) {
                    if (t == 0) fence_proxy_async();
                    issue_item<GT>(a, kind, idx, jcol, pit.rp.row, su, stages, xslots, bars, xoffs);
                }
            }
        }
        if (act) {
            const size_t o = size_t(row) * rbs + t;
            double out;
            switch (a.mode) {
                case MODE_RESIDUAL: out = __dsub_rn(pre_b, acc); break;
                case MODE_ADD: out = __dadd_rn(pre_x, acc); break;
                default: out = acc; break;
            }
            a.y[o] = out;
        }
    }
    // drain: nothing outstanding (every issued item was consumed)
}

template <int GT, int BS>
int rowpass_occupancy(Ctx& ctx, size_t smem) {
    // host threads may drive several contexts at once (one per rank)
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    static int attr_set_device = -1;
    if (attr_set_device != ctx.device) {
        LDGMG_CUDA(cudaFuncSetAttribute(rowpass_kernel<GT, BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(ctx.smem_optin)));
        max_carveout(rowpass_kernel<GT, BS>);
        attr_set_device = ctx.device;
    }
    static std::vector<std::pair<size_t, int>> occ_cache;
    for (const auto& e : occ_cache)
        if (e.first == smem) return e.second;
    int occ = 0;
    LDGMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowpass_kernel<GT, BS>, GT, smem));
    occ_cache.push_back({smem, occ});
    return occ;
}

/// Ring depth and grid for one pass.  Large passes: 3 stages (block pairs in
/// compute + one in flight).  Passes with only a few rows per resident CTA
/// (C2 level 1: 4096 rows over 1628 CTAs): 2 stages -> more resident CTAs,
/// and the grid sized so every CTA gets the same number of rows (the pass
/// ends with the CTA holding the most rows).  Measured on B200, C2 level 1:
/// 33.5 us (3 stages, 1628 CTAs) -> 30.9 us (2 stages).  ns_env > 1 forces a
/// depth (measurement builds only; the library passes -1).
template <int GT, int BS>
void configure_and_launch(Ctx& ctx, RowPassArgs a, size_t stage_bytes, int ns_env) {
    auto smem_for = [&](int ns) {
        return size_t(ns) * stage_bytes + size_t(ns) * a.xslot_doubles * 8 + 2 * size_t(a.xslot_doubles) * 8 +
               size_t(ns) * 8 + size_t(ns) * 8;
    };
    int ns = ns_env > 1 ? ns_env : 3;
    while (ns > 2 && ns * stage_bytes > 200 * 1024) --ns;
    // (blocks of <= 16 rows keep 3: their pairs run on the two half-warps,
    // C1 at 64^2: 0.195 -> 0.189 ms per V-cycle)
    if (ns_env <= 1 && ns == 3 && 2 * a.rbs > 32) {
        const int occ3 = rowpass_occupancy<GT, BS>(ctx, smem_for(3));
        if (occ3 >= 1 && a.nrows < 4 * occ3 * ctx.num_sms) ns = 2;
    }
    const size_t smem = smem_for(ns);
    if (smem > ctx.smem_optin) fail(LDGMG_ERR_INVALID_ARGUMENT, "rowpass: block too large for shared memory");
    a.nstages = ns;
    const int occ = rowpass_occupancy<GT, BS>(ctx, smem);
    if (occ < 1) fail(LDGMG_ERR_CUDA, "rowpass: block does not fit on an SM");
    const int slots = occ * ctx.num_sms;
    int grid = std::max(1, std::min(a.nrows, slots));
    const int per = (a.nrows + slots - 1) / slots;  // rows of the busiest CTA
    if (per <= 8) grid = std::max(1, (a.nrows + per - 1) / per);
    launch_pdl(rowpass_kernel<GT, BS>, dim3(grid), dim3(GT), smem, ctx.stream, a);
    after_launch("rowpass_kernel");
}

__global__ void upload_permute_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                      int64_t nnzb, int rbs, int cbs, int stride) {
    // src: reference row-major blocks (r,c) at r*cbs+c; dst: column-major padded
    const int64_t total = nnzb * int64_t(rbs) * cbs;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = i / (int64_t(rbs) * cbs);
        const int e = int(i - k * int64_t(rbs) * cbs);
        const int r = e / cbs, c = e % cbs;
        dst[k * stride + int64_t(c) * rbs + r] = src[i];
    }
}

__global__ void download_permute_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                        int64_t nnzb, int rbs, int cbs, int stride) {
    const int64_t total = nnzb * int64_t(rbs) * cbs;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = i / (int64_t(rbs) * cbs);
        const int e = int(i - k * int64_t(rbs) * cbs);
        const int r = e / cbs, c = e % cbs;
        dst[i] = src[k * stride + int64_t(c) * rbs + r];
    }
}

/// B^T block q (= (B_ij)^T for source block k = perm[q]): element (c, r) of the
/// transposed block, column-major with leading dim cbs: r*cbs + c.
__global__ void transpose_blocks_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                        const int* __restrict__ perm, int64_t nnzb, int rbs,
                                        int cbs, int stride) {
    const int64_t total = nnzb * int64_t(rbs) * cbs;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = i / (int64_t(rbs) * cbs);
        const int e = int(i - q * int64_t(rbs) * cbs);
        const int r = e % rbs, c = e / rbs;  // source element (r, c)
        const int64_t k = perm[q];
        dst[q * stride + int64_t(r) * cbs + c] = src[k * stride + int64_t(c) * rbs + r];
    }
}

/// dst block q = src block idx[q] (stored layout, same stride), 16-byte words.
__global__ void gather_blocks_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                                     const int64_t* __restrict__ idx, int64_t nnzb, int words) {
    const int64_t total = nnzb * words;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = t / words;
        const int w = int(t - q * words);
        dst[t] = src[idx[q] * words + w];
    }
}

int grid_for(int64_t n, int threads, const Ctx& ctx) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, ctx.num_sms * 16)));
}

}  // namespace

void* pinned_alloc(size_t bytes) {
    // page-locking a multi-GB allocation cost ~0.5 s/GB on the box (C5 32^3:
    // +10.5 s assembly for -2.3 s upload), so setup buffers stay pageable
    constexpr bool kPinnedSetup = false;
    if (!kPinnedSetup) return nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return nullptr;
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

bool pinned_free(void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (at.type != cudaMemoryTypeHost) return false;
    cudaFreeHost(p);
    return true;
}

void h2d_staged(Ctx& ctx, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    {  // page-locked source: one direct DMA
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost) {
            LDGMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx.stream));
            LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
            return;
        }
        cudaGetLastError();
    }
    constexpr size_t kSlot = size_t(64) << 20;
    if (bytes < (size_t(8) << 20)) {
        h2d(ctx, dst, src, bytes);
        return;
    }
    if (!ctx.pin[0]) {
        for (int i = 0; i < 2; ++i) {
            LDGMG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx.pin[i]), kSlot));
            LDGMG_CUDA(cudaEventCreateWithFlags(&ctx.pin_ev[i], cudaEventDisableTiming));
            LDGMG_CUDA(cudaEventRecord(ctx.pin_ev[i], ctx.stream));
        }
        ctx.pin_bytes = kSlot;
    }
    const unsigned char* s = static_cast<const unsigned char*>(src);
    unsigned char* d = static_cast<unsigned char*>(dst);
    static const bool timing = getenv("LDGMG_SETUP_TIMING") && atoi(getenv("LDGMG_SETUP_TIMING"));
    const auto t0 = std::chrono::steady_clock::now();
    double t_copy = 0.0, t_wait = 0.0;
    int slot = 0;
    for (size_t off = 0; off < bytes; off += kSlot, slot ^= 1) {
        const size_t n = std::min(kSlot, bytes - off);
        auto ta = std::chrono::steady_clock::now();
        LDGMG_CUDA(cudaEventSynchronize(ctx.pin_ev[slot]));  // the slot's previous DMA is done
        auto tb = std::chrono::steady_clock::now();
        unsigned char* buf = ctx.pin[slot];
        const int parts = 8;
        parallel_for(parts, [&](int lo, int hi) {
            for (int q = lo; q < hi; ++q) {
                const size_t a = n * q / parts, b = n * (q + 1) / parts;
                std::memcpy(buf + a, s + off + a, b - a);
            }
        });
        auto tc = std::chrono::steady_clock::now();
        t_wait += std::chrono::duration<double>(tb - ta).count();
        t_copy += std::chrono::duration<double>(tc - tb).count();
        LDGMG_CUDA(cudaMemcpyAsync(d + off, buf, n, cudaMemcpyHostToDevice, ctx.stream));
        LDGMG_CUDA(cudaEventRecord(ctx.pin_ev[slot], ctx.stream));
    }
    LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    if (timing)
        fprintf(stderr, "[h2d_staged] %.1f MB in %.3f s (memcpy %.3f s, dma waits %.3f s)\n", bytes / 1e6,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(), t_copy, t_wait);
}

void ctx_release_staging(Ctx& ctx) {
    for (int i = 0; i < 2; ++i) {
        if (ctx.pin[i]) cudaFreeHost(ctx.pin[i]);
        if (ctx.pin_ev[i]) cudaEventDestroy(ctx.pin_ev[i]);
        ctx.pin[i] = nullptr;
        ctx.pin_ev[i] = nullptr;
    }
    ctx.pin_bytes = 0;
}

std::unique_ptr<Bsr> bsr_upload(Ctx& ctx, int brows, int bcols, int rbs, int cbs, const int* ptr,
                                const int* col, const double* val, bool require_sorted) {
    require(brows >= 0 && bcols >= 0 && rbs > 0 && cbs > 0, "bsr_upload: bad shape");
    require(rbs <= 256 && cbs <= 256, "bsr_upload: block size above 256 is not supported");
    auto A = std::make_unique<Bsr>();
    A->brows = brows;
    A->bcols = bcols;
    A->rbs = rbs;
    A->cbs = cbs;
    A->hptr.assign(ptr, ptr + brows + 1);
    require(A->hptr[0] == 0, "bsr_upload: ptr[0] must be 0");
    for (int i = 0; i < brows; ++i)
        require(A->hptr[i + 1] >= A->hptr[i], "bsr_upload: ptr must be nondecreasing");
    A->nnzb = A->hptr[brows];
    A->hcol.assign(col, col + A->nnzb);
    set_max_row(*A);
    for (int i = 0; i < brows; ++i)
        for (int k = A->hptr[i]; k < A->hptr[i + 1]; ++k) {
            require(A->hcol[k] >= 0 && A->hcol[k] < bcols, "bsr_upload: column out of range");
            if (require_sorted && k > A->hptr[i])
                require(A->hcol[k] > A->hcol[k - 1], "bsr_upload: columns must ascend");
        }
    A->blk_stride = even_up(int64_t(rbs) * cbs);
    A->ptr.alloc(sizeof(int) * (brows + 1));
    A->col.alloc(sizeof(int) * std::max<int64_t>(1, A->nnzb));
    A->val.alloc(sizeof(double) * std::max<int64_t>(1, A->nnzb * A->blk_stride));
    LDGMG_CUDA(cudaMemcpyAsync(A->ptr.p, ptr, sizeof(int) * (brows + 1), cudaMemcpyHostToDevice, ctx.stream));
    if (A->nnzb) {
        LDGMG_CUDA(cudaMemcpyAsync(A->col.p, col, sizeof(int) * A->nnzb, cudaMemcpyHostToDevice, ctx.stream));
        LDGMG_CUDA(cudaMemsetAsync(A->val.p, 0, A->val.bytes, ctx.stream));
        if (val) bsr_set_values(ctx, *A, 0, A->nnzb, val);  // null: zero blocks, filled later
    }
    LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    return A;
}

void bsr_set_values(Ctx& ctx, Bsr& A, int64_t k0, int64_t nb, const double* val) {
    require(!A.tbase && !A.vbase, "bsr_set_values: a view has no values of its own");
    require(k0 >= 0 && nb >= 0 && k0 + nb <= A.nnzb, "bsr_set_values: block range out of bounds");
    if (!nb) return;
    require(val != nullptr, "bsr_set_values: null values");
    // stage through a device buffer in chunks to bound the temporary
    const int64_t per_blk = int64_t(A.rbs) * A.cbs;
    const int64_t chunk_blocks = std::max<int64_t>(1, (int64_t(256) << 20) / (per_blk * 8));
    DevBuf tmp(sizeof(double) * std::min(nb, chunk_blocks) * per_blk);
    for (int64_t q0 = 0; q0 < nb; q0 += chunk_blocks) {
        const int64_t n = std::min(chunk_blocks, nb - q0);
        h2d_staged(ctx, tmp.p, val + q0 * per_blk, sizeof(double) * n * per_blk);
        upload_permute_kernel<<<grid_for(n * per_blk, 256, ctx), 256, 0, ctx.stream>>>(
            tmp.as<double>(), A.val.as<double>() + (k0 + q0) * A.blk_stride, n, A.rbs, A.cbs, A.blk_stride);
        after_launch("upload_permute_kernel");
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    }
}

std::unique_ptr<Bsr> bsr_gather(Ctx& ctx, const Bsr& src, int brows, int bcols, const int* ptr, const int* col,
                                const int64_t* src_blocks) {
    require(!src.tbase && !src.vbase, "bsr_gather: source is a view");
    require(brows >= 0 && bcols >= 0 && ptr && ptr[0] == 0, "bsr_gather: bad shape");
    auto A = std::make_unique<Bsr>();
    A->brows = brows;
    A->bcols = bcols;
    A->rbs = src.rbs;
    A->cbs = src.cbs;
    A->blk_stride = src.blk_stride;
    A->hptr.assign(ptr, ptr + brows + 1);
    for (int i = 0; i < brows; ++i) require(A->hptr[i + 1] >= A->hptr[i], "bsr_gather: ptr must be nondecreasing");
    A->nnzb = A->hptr[brows];
    A->hcol.assign(col, col + A->nnzb);
    for (int64_t q = 0; q < A->nnzb; ++q) {
        require(A->hcol[q] >= 0 && A->hcol[q] < bcols, "bsr_gather: column out of range");
        require(src_blocks[q] >= 0 && src_blocks[q] < src.nnzb, "bsr_gather: source block out of range");
    }
    set_max_row(*A);
    A->ptr.alloc(sizeof(int) * (brows + 1));
    A->col.alloc(sizeof(int) * std::max<int64_t>(1, A->nnzb));
    A->val.alloc(sizeof(double) * std::max<int64_t>(1, A->nnzb * A->blk_stride));
    h2d(ctx, A->ptr.p, A->hptr.data(), sizeof(int) * A->hptr.size());
    if (A->nnzb) {
        h2d(ctx, A->col.p, A->hcol.data(), sizeof(int) * A->nnzb);
        DevBuf d_idx(sizeof(int64_t) * A->nnzb);
        h2d(ctx, d_idx.p, src_blocks, d_idx.bytes);
        const int words = A->blk_stride / 2;  // blk_stride is even: 16-byte words
        gather_blocks_kernel<<<grid_for(A->nnzb * words, 256, ctx), 256, 0, ctx.stream>>>(
            reinterpret_cast<const double2*>(src.val.p), reinterpret_cast<double2*>(A->val.p), d_idx.as<int64_t>(),
            A->nnzb, words);
        after_launch("gather_blocks_kernel");
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    return A;
}

std::unique_ptr<Bsr> bsr_row_prefix_view(Ctx& ctx, const Bsr& base, int nrows) {
    require(!base.tbase && !base.vbase, "bsr_row_prefix_view: base is a view");
    require(nrows >= 0 && nrows <= base.brows, "bsr_row_prefix_view: row count out of range");
    auto V = std::make_unique<Bsr>();
    V->brows = nrows;
    V->bcols = base.bcols;
    V->rbs = base.rbs;
    V->cbs = base.cbs;
    V->blk_stride = base.blk_stride;
    V->vbase = &base;
    V->hptr.assign(base.hptr.begin(), base.hptr.begin() + nrows + 1);
    V->nnzb = V->hptr[nrows];
    V->hcol.assign(base.hcol.begin(), base.hcol.begin() + V->nnzb);
    set_max_row(*V);
    V->ptr.alloc(sizeof(int) * (nrows + 1));
    V->col.alloc(sizeof(int) * std::max<int64_t>(1, V->nnzb));
    h2d(ctx, V->ptr.p, V->hptr.data(), sizeof(int) * V->hptr.size());
    if (V->nnzb) h2d(ctx, V->col.p, V->hcol.data(), sizeof(int) * V->nnzb);
    return V;
}

const Bsr& bsr_materialize(Ctx& ctx, const Bsr& view) {
    if (!view.tbase) return view;  // stored layout already (own or prefix-view values)
    if (view.mat) return *view.mat;
    auto M = std::make_unique<Bsr>();
    M->brows = view.brows;
    M->bcols = view.bcols;
    M->rbs = view.rbs;
    M->cbs = view.cbs;
    M->nnzb = view.nnzb;
    M->blk_stride = view.blk_stride;
    M->hptr = view.hptr;
    M->hcol = view.hcol;
    M->max_row = view.max_row;
    M->ptr.alloc(sizeof(int) * (M->brows + 1));
    M->col.alloc(sizeof(int) * std::max<int64_t>(1, M->nnzb));
    M->val.alloc(sizeof(double) * std::max<int64_t>(1, M->nnzb * M->blk_stride));
    h2d(ctx, M->ptr.p, M->hptr.data(), sizeof(int) * M->hptr.size());
    if (M->nnzb) {
        h2d(ctx, M->col.p, M->hcol.data(), sizeof(int) * M->nnzb);
        LDGMG_CUDA(cudaMemsetAsync(M->val.p, 0, M->val.bytes, ctx.stream));
        const Bsr& B = *view.tbase;
        transpose_blocks_kernel<<<grid_for(M->nnzb * int64_t(B.rbs) * B.cbs, 256, ctx), 256, 0, ctx.stream>>>(
            B.val.as<double>(), M->val.as<double>(), view.tperm.as<int>(), M->nnzb, B.rbs, B.cbs, B.blk_stride);
        after_launch("transpose_blocks_kernel");
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    const_cast<Bsr&>(view).mat = std::move(M);
    return *view.mat;
}

std::unique_ptr<Bsr> bsr_transposed_view(Ctx& ctx, const Bsr& base, int brows, int bcols, const int* ptr,
                                         const int* col, const int* perm) {
    require(!base.tbase && !base.vbase, "bsr_transposed_view: base is a view");
    require(brows >= 0 && bcols >= 0 && ptr && ptr[0] == 0, "bsr_transposed_view: bad shape");
    auto T = std::make_unique<Bsr>();
    T->brows = brows;
    T->bcols = bcols;
    T->rbs = base.cbs;
    T->cbs = base.rbs;
    T->blk_stride = base.blk_stride;
    T->tbase = &base;
    T->hptr.assign(ptr, ptr + brows + 1);
    for (int i = 0; i < brows; ++i) require(T->hptr[i + 1] >= T->hptr[i], "bsr_transposed_view: ptr must be nondecreasing");
    T->nnzb = T->hptr[brows];
    T->hcol.assign(col, col + T->nnzb);
    for (int64_t q = 0; q < T->nnzb; ++q) {
        require(T->hcol[q] >= 0 && T->hcol[q] < bcols, "bsr_transposed_view: column out of range");
        require(perm[q] >= 0 && perm[q] < base.nnzb, "bsr_transposed_view: block index out of range");
    }
    set_max_row(*T);
    T->ptr.alloc(sizeof(int) * (brows + 1));
    T->col.alloc(sizeof(int) * std::max<int64_t>(1, T->nnzb));
    T->tperm.alloc(sizeof(int) * std::max<int64_t>(1, T->nnzb));
    h2d(ctx, T->ptr.p, T->hptr.data(), sizeof(int) * T->hptr.size());
    if (T->nnzb) {
        h2d(ctx, T->col.p, T->hcol.data(), sizeof(int) * T->nnzb);
        h2d(ctx, T->tperm.p, perm, sizeof(int) * T->nnzb);
    }
    return T;
}

void bsr_download(Ctx& ctx, const Bsr& A, int* ptr, int* col, double* val) {
    if (A.tbase && val) {
        bsr_download(ctx, bsr_materialize(ctx, A), ptr, col, val);
        return;
    }
    if (ptr) std::memcpy(ptr, A.hptr.data(), sizeof(int) * A.hptr.size());
    if (col) std::memcpy(col, A.hcol.data(), sizeof(int) * A.hcol.size());
    if (val && A.nnzb) {
        const int64_t per_blk = int64_t(A.rbs) * A.cbs;
        DevBuf tmp(sizeof(double) * A.nnzb * per_blk);
        download_permute_kernel<<<grid_for(A.nnzb * per_blk, 256, ctx), 256, 0, ctx.stream>>>(
            bsr_values(A), tmp.as<double>(), A.nnzb, A.rbs, A.cbs, A.blk_stride);
        after_launch("download_permute_kernel");
        LDGMG_CUDA(cudaMemcpyAsync(val, tmp.p, tmp.bytes, cudaMemcpyDeviceToHost, ctx.stream));
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    }
}

const Bsr& bsr_transpose(Ctx& ctx, const Bsr& A) {
    if (A.T) return *A.T;
    auto T = std::make_unique<Bsr>();
    T->brows = A.bcols;
    T->bcols = A.brows;
    T->rbs = A.cbs;
    T->cbs = A.rbs;
    T->nnzb = A.nnzb;
    T->blk_stride = A.blk_stride;
    // CSC of A = CSR of A^T; rows i ascend within each column by construction
    T->hptr.assign(A.bcols + 1, 0);
    for (int64_t k = 0; k < A.nnzb; ++k) ++T->hptr[A.hcol[k] + 1];
    for (int j = 0; j < A.bcols; ++j) T->hptr[j + 1] += T->hptr[j];
    T->hcol.resize(A.nnzb);
    std::vector<int> perm(std::max<int64_t>(1, A.nnzb)), fill(T->hptr.begin(), T->hptr.end() - 1);
    for (int i = 0; i < A.brows; ++i)
        for (int k = A.hptr[i]; k < A.hptr[i + 1]; ++k) {
            const int q = fill[A.hcol[k]]++;
            T->hcol[q] = i;
            perm[q] = k;
        }
    set_max_row(*T);
    T->ptr.alloc(sizeof(int) * (T->brows + 1));
    T->col.alloc(sizeof(int) * std::max<int64_t>(1, T->nnzb));
    T->val.alloc(sizeof(double) * std::max<int64_t>(1, T->nnzb * T->blk_stride));
    LDGMG_CUDA(cudaMemcpyAsync(T->ptr.p, T->hptr.data(), sizeof(int) * T->hptr.size(), cudaMemcpyHostToDevice, ctx.stream));
    if (T->nnzb) {
        LDGMG_CUDA(cudaMemcpyAsync(T->col.p, T->hcol.data(), sizeof(int) * T->nnzb, cudaMemcpyHostToDevice, ctx.stream));
        LDGMG_CUDA(cudaMemsetAsync(T->val.p, 0, T->val.bytes, ctx.stream));
        DevBuf dperm(sizeof(int) * perm.size());
        LDGMG_CUDA(cudaMemcpyAsync(dperm.p, perm.data(), dperm.bytes, cudaMemcpyHostToDevice, ctx.stream));
        const int64_t per_blk = int64_t(A.rbs) * A.cbs;
        transpose_blocks_kernel<<<grid_for(A.nnzb * per_blk, 256, ctx), 256, 0, ctx.stream>>>(
            A.val.as<double>(), T->val.as<double>(), dperm.as<int>(), A.nnzb, A.rbs, A.cbs,
            A.blk_stride);
        after_launch("transpose_blocks_kernel");
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    const_cast<Bsr&>(A).T = std::move(T);
    return *A.T;
}

namespace {
int split_threshold_rows(const Ctx& ctx);
}  // namespace

const Bsr& bsr_transpose_view(Ctx& ctx, const Bsr& A) {
    if (A.TV) return *A.TV;
    require(!A.tbase, "bsr_transpose_view: already a view");
    auto T = std::make_unique<Bsr>();
    T->brows = A.bcols;
    T->bcols = A.brows;
    T->rbs = A.cbs;
    T->cbs = A.rbs;
    T->nnzb = A.nnzb;
    T->blk_stride = A.blk_stride;
    T->tbase = &A;
    T->hptr.assign(A.bcols + 1, 0);
    for (int64_t k = 0; k < A.nnzb; ++k) ++T->hptr[A.hcol[k] + 1];
    for (int j = 0; j < A.bcols; ++j) T->hptr[j + 1] += T->hptr[j];
    T->hcol.resize(A.nnzb);
    std::vector<int> perm(std::max<int64_t>(1, A.nnzb)), fill(T->hptr.begin(), T->hptr.end() - 1);
    for (int i = 0; i < A.brows; ++i)
        for (int k = A.hptr[i]; k < A.hptr[i + 1]; ++k) {
            const int q = fill[A.hcol[k]]++;
            T->hcol[q] = i;
            perm[q] = k;
        }
    set_max_row(*T);
    T->ptr.alloc(sizeof(int) * (T->brows + 1));
    T->col.alloc(sizeof(int) * std::max<int64_t>(1, T->nnzb));
    T->tperm.alloc(sizeof(int) * perm.size());
    h2d(ctx, T->ptr.p, T->hptr.data(), sizeof(int) * T->hptr.size());
    if (T->nnzb) h2d(ctx, T->col.p, T->hcol.data(), sizeof(int) * T->nnzb);
    h2d(ctx, T->tperm.p, perm.data(), sizeof(int) * perm.size());
    const_cast<Bsr&>(A).TV = std::move(T);
    return *A.TV;
}

const Bsr& bsr_transpose_for_sweep(Ctx& ctx, const Bsr& A) {
    if (A.T) return *A.T;
    if (A.TV) return *A.TV;
    // LDGMG_TVIEW=1 always views, 0 always copies; default: copy while the
    // copy fits with a margin (measured 0.4 % (bs 27) to 5 % (bs 108) faster
    // than the view), view when it does not (C5 at 48^3 on one GPU)
    static int env = -2;
    if (env == -2) {
        const char* e = getenv("LDGMG_TVIEW");
        env = e ? atoi(e) : -1;
    }
    if (env < 0) {
        size_t free_b = 0, total_b = 0;
        LDGMG_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const size_t need = size_t(A.val.bytes) + std::max<size_t>(size_t(4) << 30, total_b / 20);
        if (free_b >= need) return bsr_transpose(ctx, A);
    }
    // transposed reads are conflict-free for odd sizes, and for even sizes
    // whose half is odd (pairs); 108 = 2*54 costs a 2-way conflict, still
    // well under the block's HBM time; 16/48 (8-way) keep the explicit copy
    const int s = A.rbs;
    int g = 1;
    if (s % 2 == 0) {
        int h = s / 2;
        g = 1;
        while (h % 2 == 0 && g < 8) {
            h /= 2;
            g *= 2;
        }
    }
    const bool ok = env != 0 && A.rbs == A.cbs && A.brows == A.bcols && g <= 2 && A.brows > split_threshold_rows(ctx);
    return ok ? bsr_transpose_view(ctx, A) : bsr_transpose(ctx, A);
}

namespace {

/// Split-row variant for SMALL levels (few rows per SM): one CTA per block
/// row, its blocks spread over the warps (each warp computes whole s_k dot
/// products for its blocks straight from L2/HBM), then warp 0 combines the
/// s_k in CSR order -- the same arithmetic, bit for bit, as rowpass_kernel,
/// with the per-row latency of one block instead of the whole row.
/// Requires rbs, cbs <= 32.
__global__ void __launch_bounds__(256) rowsplit_kernel(const RowPassArgs a, int maxlen) {
    extern __shared__ __align__(16) double ss[];  // maxlen x 32 partial sums, then u, t
    pdl_launch_dependents();
    pdl_wait();
    for (int slot = blockIdx.x; slot < a.nrows; slot += gridDim.x) split_row_task(a, row_at(a, slot), maxlen, ss);
}

/// rowsplit_kernel with TMA-staged rows (split_row_task_tma).
__global__ void __launch_bounds__(256) rowsplit_tma_kernel(const RowPassArgs a, int maxlen) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();
    // immutable prologue: the first row's blocks (and factor) are requested
    // before waiting on the predecessor
    int jfirst = -1;
    if (blockIdx.x < a.nrows) {
        const int row0 = row_at(a, blockIdx.x);
        split_row_issue(a, row0, maxlen, sm, &bar);
        jfirst = split_row_first_col(a, row0);  // the x gather's first column index, also immutable
    }
    pdl_wait();
    uint32_t phase = 0;
    bool issued = true;
    for (int slot = blockIdx.x; slot < a.nrows; slot += gridDim.x) {
        split_row_task_tma(a, row_at(a, slot), maxlen, sm, &bar, phase, issued, issued ? jfirst : -1);
        issued = false;
    }
}

int split_threshold_rows(const Ctx& ctx) {
    static int env = -2;
    if (env == -2) {
        const char* s = getenv("LDGMG_SPLIT_ROWS");
        env = s ? atoi(s) : -1;
    }
    // measured on B200 (C2 hierarchy): split-row wins at 512 rows (6.3 vs 9.2 us),
    // the TMA ring wins at 4096 rows (33 vs 43 us)
    return env >= 0 ? env : 8 * ctx.num_sms;
}

}  // namespace

void launch_rowpass(Ctx& ctx, const RowPass& p) {
    const Bsr& A = *p.A;
    if (p.nrows == 0) return;
    if (A.tbase) {
        require(p.mode != MODE_RELAX, "rowpass: a transpose view cannot be relaxed");
        // small levels: the split-row kernels read blocks in stored layout
        if (A.rbs <= 32 && A.cbs <= 32 && p.nrows <= split_threshold_rows(ctx)) {
            RowPass q = p;
            q.A = &bsr_materialize(ctx, A);
            launch_rowpass(ctx, q);
            return;
        }
    }
    if (A.rbs <= 32 && A.cbs <= 32 && p.nrows <= split_threshold_rows(ctx)) {
        RowPassArgs a{};
        a.ptr = A.ptr.as<int>();
        a.col = A.col.as<int>();
        a.val = bsr_values(A);
        a.blk_stride = A.blk_stride;
        a.rbs = A.rbs;
        a.cbs = A.cbs;
        a.mode = p.mode;
        a.x = p.x;
        a.part = p.part;
        a.x_alt = p.x_alt;
        a.b = p.b;
        a.xe = p.xe;
        a.y = p.y;
        a.rows = p.rows;
        a.nrows = p.nrows;
        a.omega = p.omega;
        a.kernel_tol = p.kernel_tol;
        if (p.mode == MODE_RELAX) {
            require(p.F != nullptr && A.rbs == A.cbs && p.F->bs == A.rbs, "relax: factor shape mismatch");
            a.V = p.F->V.as<double>();
            a.lam = p.F->lambda.as<double>();
            a.scal = p.F->scale.as<double>();
            a.lmax = p.F->lmax.as<double>();
            a.ld = p.F->ld;
            a.vstride = p.F->vstride;
        }
        const int maxlen = std::max(1, A.max_row);
        const int warps = std::min(8, maxlen);
        const size_t smem_tma =
            sizeof(double) * split_row_tma_doubles(maxlen, A.blk_stride, p.mode == MODE_RELAX ? p.F->vstride : 0, A.cbs);
        if (smem_tma <= 120 * 1024) {  // else: long rows, plain-load kernel
            ensure_dyn_smem(rowsplit_tma_kernel, smem_tma);
            const int grid = std::min(p.nrows, ctx.num_sms * 16);
            static bool once = (max_carveout(rowsplit_tma_kernel), true);
            (void)once;
            const int threads = std::max(warps * 32, std::min(256, ((maxlen * A.cbs + 31) / 32) * 32));
            launch_pdl_small(rowsplit_tma_kernel, dim3(grid), dim3(threads), smem_tma, ctx.stream, a, maxlen);
            after_launch("rowsplit_tma_kernel");
            return;
        }
        const size_t smem = sizeof(double) * (size_t(maxlen) * 32 + 64);
        ensure_dyn_smem(rowsplit_kernel, size_t(smem));
        const int grid = std::min(p.nrows, ctx.num_sms * 16);
        static bool once = (max_carveout(rowsplit_kernel), true);
        (void)once;
        launch_pdl_small(rowsplit_kernel, dim3(grid), dim3(warps * 32), smem, ctx.stream, a, maxlen);
        after_launch("rowsplit_kernel");
        return;
    }
    RowPassArgs a{};
    a.ptr = A.ptr.as<int>();
    a.col = A.col.as<int>();
    a.val = bsr_values(A);
    a.perm = A.tbase ? A.tperm.as<int>() : nullptr;
    a.tview = A.tbase ? 1 : 0;
    a.blk_stride = A.blk_stride;
    a.rbs = A.rbs;
    a.cbs = A.cbs;
    a.mode = p.mode;
    a.x = p.x;
    a.part = p.part;
    a.x_alt = p.x_alt;
    a.b = p.b;
    a.xe = p.xe;
    a.y = p.y;
    a.rows = p.rows;
    a.nrows = p.nrows;
    a.omega = p.omega;
    a.kernel_tol = p.kernel_tol;
    int stage = A.blk_stride;
    if (p.mode == MODE_RELAX) {
        require(p.F != nullptr && A.rbs == A.cbs && p.F->bs == A.rbs, "relax: factor shape mismatch");
        a.V = p.F->V.as<double>();
        a.lam = p.F->lambda.as<double>();
        a.scal = p.F->scale.as<double>();
        a.lmax = p.F->lmax.as<double>();
        a.ld = p.F->ld;
        a.vstride = p.F->vstride;
        stage = std::max(stage, p.F->vstride);
        if (!A.dpos.p) {  // diagonal positions, once per operator
            std::vector<int> d(std::max(1, A.brows), -1);
            for (int i = 0; i < A.brows; ++i)
                for (int k = A.hptr[i]; k < A.hptr[i + 1]; ++k)
                    if (A.hcol[k] == i) d[i] = k;
            Bsr& Am = const_cast<Bsr&>(A);
            Am.dpos.alloc(sizeof(int) * d.size());
            h2d(ctx, Am.dpos.p, d.data(), sizeof(int) * d.size());
        }
        a.dpos = A.dpos.as<int>();
    }
    a.stage_doubles = even_up(stage);
    // x slots hold a 16-byte aligned window around x_j (up to one extra
    // double in front and the tail rounded up to 16 bytes)
    a.xslot_doubles = even_up(std::max(A.cbs, A.rbs)) + 2;
    const int wide = std::max(A.rbs, A.cbs);
    const int GT = wide <= 32 ? 32 : wide <= 64 ? 64 : wide <= 128 ? 128 : 256;
    // ring depth: keep >= ~3 blocks in flight per group within a 200 KB budget
    const size_t stage_bytes = size_t(a.stage_doubles) * 8;
    constexpr int ns_env = -1;  // ring depth chosen per pass (configure_and_launch)
    const bool sq = A.rbs == A.cbs;
    if (sq && A.rbs == 16) configure_and_launch<32, 16>(ctx, a, stage_bytes, ns_env);
    else if (sq && A.rbs == 25) configure_and_launch<32, 25>(ctx, a, stage_bytes, ns_env);
    else if (sq && A.rbs == 27) configure_and_launch<32, 27>(ctx, a, stage_bytes, ns_env);
    else if (sq && A.rbs == 48) configure_and_launch<64, 48>(ctx, a, stage_bytes, ns_env);
    else if (sq && A.rbs == 108) configure_and_launch<128, 108>(ctx, a, stage_bytes, ns_env);
    else switch (GT) {
        case 32: configure_and_launch<32, 0>(ctx, a, stage_bytes, ns_env); break;
        case 64: configure_and_launch<64, 0>(ctx, a, stage_bytes, ns_env); break;
        case 128: configure_and_launch<128, 0>(ctx, a, stage_bytes, ns_env); break;
        default: configure_and_launch<256, 0>(ctx, a, stage_bytes, ns_env); break;
    }
}

}  // namespace ldgmg_b200
