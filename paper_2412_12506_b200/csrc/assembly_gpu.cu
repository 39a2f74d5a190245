// Device assembly of the level operators from a LevelProgram (setup.hpp):
// the G_k^T D G_k products of accumulate_AtDB (ldg_core.hpp:547-586) plus the
// penalty blocks ("inner" blocks), then the Stokes saddle layout
// (ldg_stokes.hpp:149-191) composed from inner and stored blocks.  Every
// entry is evaluated in the host assembly's order with explicit
// __dmul_rn/__dadd_rn, so the operator is bit-identical to problem_build's
// (tests/test_gpu_assembly.py) -- and is never materialised on the host: only
// the gradient / penalty blocks (1/ncomp^2 of the operator for Stokes) cross
// PCIe.
#include <cuda_runtime.h>

#include <algorithm>

#include "core.hpp"
#include "setup.hpp"

namespace ldgmg_b200 {

namespace {

/// inner block id = CTA (grid-strided); thread per entry (i, j).  With
/// `direct` the block is the final operator block (scalar operators) and is
/// written straight into the device BSR layout (column-major, blk_stride).
__global__ void __launch_bounds__(256) inner_kernel(const double* __restrict__ blocks,
                                                    const int64_t* __restrict__ inner_ptr,
                                                    const int* __restrict__ b1, const int* __restrict__ b2,
                                                    const double* __restrict__ d, const int* __restrict__ add,
                                                    int64_t ninner, int bsv, double* __restrict__ out, int direct,
                                                    int blk_stride) {
    const int nb2 = bsv * bsv;
    for (int64_t id = blockIdx.x; id < ninner; id += gridDim.x) {
        const int64_t p0 = inner_ptr[id], p1 = inner_ptr[id + 1];
        const int ad = add[id];
        for (int t = threadIdx.x; t < nb2; t += blockDim.x) {
            const int i = t / bsv, j = t - i * bsv;
            double v = 0.0;
            for (int64_t p = p0; p < p1; ++p) {
                const double* B1 = blocks + size_t(b1[p]) * nb2 + i;
                const double* B2 = blocks + size_t(b2[p]) * nb2 + j;
                double s = 0.0;
                for (int k = 0; k < bsv; ++k) s = madd_rn(s, __ldg(B1 + size_t(k) * bsv), __ldg(B2 + size_t(k) * bsv));
                v = __dadd_rn(v, __dmul_rn(d[p], s));
            }
            if (ad >= 0) v = __dadd_rn(v, __dmul_rn(1.0, __ldg(blocks + size_t(ad) * nb2 + t)));
            if (direct)
                out[size_t(id) * blk_stride + size_t(j) * bsv + i] = v;
            else
                out[size_t(id) * nb2 + t] = v;
        }
    }
}

/// final block (cell) = CTA; thread per entry (i, j) of the BS x BS block.
__global__ void __launch_bounds__(256) final_kernel(const double* __restrict__ blocks,
                                                    const double* __restrict__ inner,
                                                    const int64_t* __restrict__ term_ptr,
                                                    const int* __restrict__ kind, const int* __restrict__ idx,
                                                    const double* __restrict__ scale, int64_t ncells, int bsv, int nc,
                                                    int blk_stride, double* __restrict__ val) {
    const int BS = bsv * nc, nb2 = bsv * bsv;
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        for (int t = threadIdx.x; t < BS * BS; t += blockDim.x) {
            const int i = t / BS, j = t - i * BS;
            const int ci = i / bsv, cj = j / bsv, ii = i - ci * bsv, jj = j - cj * bsv;
            const int64_t s = cell * nc * nc + ci * nc + cj;
            double acc = 0.0;
            for (int64_t q = term_ptr[s]; q < term_ptr[s + 1]; ++q) {
                const int x = idx[q];
                const double sc = scale[q];
                switch (kind[q]) {
                    case 0: acc = __dadd_rn(acc, __dmul_rn(sc, inner[size_t(x) * nb2 + ii * bsv + jj])); break;
                    case 1: acc = __dadd_rn(acc, __dmul_rn(sc, __ldg(blocks + size_t(x) * nb2 + ii * bsv + jj))); break;
                    case 2: acc = __dadd_rn(acc, __dmul_rn(sc, __ldg(blocks + size_t(x) * nb2 + jj * bsv + ii))); break;
                    case 3: acc = inner[size_t(x) * nb2 + ii * bsv + jj]; break;
                    default:
                        if (ii == jj) acc = __dadd_rn(acc, sc);
                        break;
                }
            }
            val[size_t(cell) * blk_stride + size_t(j) * BS + i] = acc;
        }
    }
}

template <class V>
DevBuf upload_vec(Ctx& ctx, const V& v) {
    using T = typename V::value_type;
    DevBuf d(sizeof(T) * std::max<size_t>(1, v.size()));
    if (!v.empty()) h2d_staged(ctx, d.p, v.data(), sizeof(T) * v.size());
    return d;
}

}  // namespace

std::unique_ptr<Bsr> assemble_on_device(Ctx& ctx, const LevelProgram& P) {
    auto A = std::make_unique<Bsr>();
    const int N = P.n, bs = P.bs;
    A->brows = A->bcols = N;
    A->rbs = A->cbs = bs;
    A->hptr = P.ptr;
    A->hcol = P.col;
    A->nnzb = P.ptr.empty() ? 0 : P.ptr[N];
    set_max_row(*A);
    A->blk_stride = even_up(int64_t(bs) * bs);
    A->ptr.alloc(sizeof(int) * (N + 1));
    A->col.alloc(sizeof(int) * std::max<int64_t>(1, A->nnzb));
    A->val.alloc(sizeof(double) * std::max<int64_t>(1, A->nnzb * A->blk_stride));
    h2d(ctx, A->ptr.p, P.ptr.data(), sizeof(int) * (N + 1));
    if (!A->nnzb) return A;
    h2d(ctx, A->col.p, P.col.data(), sizeof(int) * A->nnzb);
    LDGMG_CUDA(cudaMemsetAsync(A->val.p, 0, A->val.bytes, ctx.stream));
    DevBuf blocks = upload_vec(ctx, P.blocks), iptr = upload_vec(ctx, P.inner_ptr), b1 = upload_vec(ctx, P.prod_b1),
           b2 = upload_vec(ctx, P.prod_b2), d = upload_vec(ctx, P.prod_d), add = upload_vec(ctx, P.inner_add);
    const int64_t ninner = int64_t(P.inner_ptr.size()) - 1;
    const int grid_i = int(std::min<int64_t>(std::max<int64_t>(1, ninner), int64_t(ctx.num_sms) * 16));
    const bool direct = P.ncomp == 1;  // scalar: inner block i IS operator block i
    if (direct) {
        if (ninner != A->nnzb) fail(LDGMG_ERR_RUNTIME, "assembly: scalar program shape mismatch");
        inner_kernel<<<grid_i, 256, 0, ctx.stream>>>(blocks.as<double>(), iptr.as<int64_t>(), b1.as<int>(),
                                                    b2.as<int>(), d.as<double>(), add.as<int>(), ninner, P.bsv,
                                                    A->val.as<double>(), 1, A->blk_stride);
        after_launch("assembly_inner_kernel");
    } else {
        DevBuf inner(sizeof(double) * std::max<int64_t>(1, ninner) * P.bsv * P.bsv);
        if (ninner) {
            inner_kernel<<<grid_i, 256, 0, ctx.stream>>>(blocks.as<double>(), iptr.as<int64_t>(), b1.as<int>(),
                                                        b2.as<int>(), d.as<double>(), add.as<int>(), ninner, P.bsv,
                                                        inner.as<double>(), 0, 0);
            after_launch("assembly_inner_kernel");
        }
        DevBuf tptr = upload_vec(ctx, P.term_ptr), tk = upload_vec(ctx, P.term_kind), ti = upload_vec(ctx, P.term_idx),
               ts = upload_vec(ctx, P.term_scale);
        const int grid_f = int(std::min<int64_t>(A->nnzb, int64_t(ctx.num_sms) * 16));
        final_kernel<<<grid_f, 256, 0, ctx.stream>>>(blocks.as<double>(), inner.as<double>(), tptr.as<int64_t>(),
                                                    tk.as<int>(), ti.as<int>(), ts.as<double>(), A->nnzb, P.bsv,
                                                    P.ncomp, A->blk_stride, A->val.as<double>());
        after_launch("assembly_final_kernel");
    }
    LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    return A;
}

}  // namespace ldgmg_b200
