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
#include <functional>
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
    int lc = -1;
    for (int l = 1; l + 1 < depth && coarse_rows > 0; ++l)
        if (A[l]->brows <= coarse_rows) {
            lc = l;
            break;
        }
    if (lc < 0) return;
    int coop = 0;
    LDGMG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx.device));
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
    void* args[] = {&ops, &nops, &maxlen};
    LDGMG_CUDA(cudaLaunchCooperativeKernel((const void*)coarse_program_kernel, dim3(coarse_grid), dim3(256), args,
                                           coarse_smem, ctx.stream));
    after_launch("coarse_program_kernel");
}

}  // namespace ldgmg_b200
