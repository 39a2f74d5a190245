// Inter-level transfers, the bottom pseudoinverse and the BLAS-1 pieces of
// the V-cycle.  All reference summation orders are kept (no FMA contraction):
//   restrict:  rc_p[c,j] = 0 + s_f1 + s_f2 + ...  over the children f of p in
//              ascending fine index, s_f = sum_i K_o[i,j] src_f[c,i]
//              (multigrid.hpp:127-149);
//   prolong:   xf[c,i] += sum_j K_o[i,j] xc_p[c,j]   (multigrid.hpp:104-123);
//   bottom:    t = V^T b (k ascending), cut |lambda| <= tol*max|lambda|,
//              x = V t (blockla.hpp:330-339, multigrid.hpp:249-253);
//   kernel projection: v -= (v.k) k with the dot taken over the mode-0
//              entries only (the kernel vectors vanish elsewhere,
//              ldg_core.hpp:64-78), multigrid.hpp:243-245.
#include <cuda_runtime.h>

#include <algorithm>

#include "core.hpp"

namespace ldgmg_b200 {

namespace {

__global__ void restrict_kernel(const int* __restrict__ child_ptr, const int* __restrict__ child,
                                const int* __restrict__ orth, const double* __restrict__ K,
                                const double* __restrict__ rf, double* __restrict__ rc,
                                int n_coarse, int bss, int ncomp) {
    const int BS = bss * ncomp;
    const int64_t total = int64_t(n_coarse) * BS;
    for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total;
         o += int64_t(gridDim.x) * blockDim.x) {
        const int p = int(o / BS);
        const int i = int(o - int64_t(p) * BS);  // = c*bss + j
        const int c = i / bss, j = i - c * bss;
        double acc = 0.0;
        for (int q = child_ptr[p]; q < child_ptr[p + 1]; ++q) {
            const int f = child[q];
            const int ot = orth[f];
            const double* src = rf + size_t(f) * BS;
            if (ot < 0) {
                acc = __dadd_rn(acc, src[i]);
                continue;
            }
            const double* Ko = K + size_t(ot) * bss * bss;
            double s = 0.0;
            for (int ii = 0; ii < bss; ++ii) s = madd_rn(s, __ldg(Ko + size_t(ii) * bss + j), src[c * bss + ii]);
            acc = __dadd_rn(acc, s);
        }
        rc[o] = acc;
    }
}

__global__ void prolong_kernel(const int* __restrict__ parent, const int* __restrict__ orth,
                               const double* __restrict__ K, const double* __restrict__ xc,
                               double* __restrict__ xf, int n_fine, int bss, int ncomp) {
    const int BS = bss * ncomp;
    const int64_t total = int64_t(n_fine) * BS;
    for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total;
         o += int64_t(gridDim.x) * blockDim.x) {
        const int f = int(o / BS);
        const int ii = int(o - int64_t(f) * BS);
        const int p = parent[f], ot = orth[f];
        const double* src = xc + size_t(p) * BS;
        if (ot < 0) {
            xf[o] = __dadd_rn(xf[o], src[ii]);
            continue;
        }
        const int c = ii / bss, i = ii - c * bss;
        const double* Ko = K + size_t(ot) * bss * bss + size_t(i) * bss;
        double s = 0.0;
        for (int j = 0; j < bss; ++j) s = madd_rn(s, __ldg(Ko + j), src[c * bss + j]);
        xf[o] = __dadd_rn(xf[o], s);
    }
}

/// Restriction, one CTA per coarse element p: the children's residual
/// blocks are staged in shared memory, thread (c, j) runs the reference's
/// sequential sums (children ascending, i ascending) with K read through the
/// read-only path.  Same bits as restrict_kernel, no dependent-load chains.
__global__ void restrict_cta_kernel(const int* __restrict__ child_ptr, const int* __restrict__ child,
                                    const int* __restrict__ orth, const double* __restrict__ K,
                                    const double* __restrict__ rf, double* __restrict__ rc, int n_coarse,
                                    int bss, int ncomp, int maxch) {
    extern __shared__ double sh[];  // maxch x BS
    __shared__ int sch[64], sor[64];
    const int BS = bss * ncomp;
    for (int p = blockIdx.x; p < n_coarse; p += gridDim.x) {
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
    (void)maxch;
}

/// Prolongation, one CTA per coarse element p: xc_p staged in shared memory,
/// every child f of p updated by thread (f, c, i) (reference order, j ascending).
__global__ void prolong_cta_kernel(const int* __restrict__ child_ptr, const int* __restrict__ child,
                                   const int* __restrict__ orth, const double* __restrict__ K,
                                   const double* __restrict__ xc, double* __restrict__ xf, int n_coarse,
                                   int bss, int ncomp) {
    extern __shared__ double sx[];  // BS
    const int BS = bss * ncomp;
    for (int p = blockIdx.x; p < n_coarse; p += gridDim.x) {
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
}

/// Bottom pseudoinverse in one CTA (n <= 4096): b and t in shared memory.
__global__ void __launch_bounds__(1024) pinv_cta_kernel(const double* __restrict__ Vr, const double* __restrict__ Vc,
                                                        const double* __restrict__ lam, const double* __restrict__ b,
                                                        double* __restrict__ x, int n, double cut) {
    extern __shared__ double sb[];  // b (n) then t (n)
    double* st = sb + n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sb[i] = b[i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0.0;
#pragma unroll 8
        for (int k = 0; k < n; ++k) s = madd_rn(s, __ldg(Vr + size_t(k) * n + i), sb[k]);
        const double l = lam[i];
        st[i] = fabs(l) <= cut ? 0.0 : s / l;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0.0;
#pragma unroll 8
        for (int k = 0; k < n; ++k) s = madd_rn(s, __ldg(Vc + size_t(k) * n + i), st[k]);
        x[i] = s;
    }
}

/// t_i = cut(sum_k V(k,i) b_k) / lambda_i ; Vr row-major: V(k,i) at k*n+i.
__global__ void pinv_t_kernel(const double* __restrict__ Vr, const double* __restrict__ lam,
                              const double* __restrict__ b, double* __restrict__ t, int n,
                              double cut) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int k = 0; k < n; ++k) s = madd_rn(s, Vr[size_t(k) * n + i], b[k]);
    const double l = lam[i];
    t[i] = fabs(l) <= cut ? 0.0 : s / l;
}

/// x_i = sum_k V(i,k) t_k ; Vc column-major: V(i,k) at k*n+i.
__global__ void pinv_x_kernel(const double* __restrict__ Vc, const double* __restrict__ t,
                              double* __restrict__ x, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int k = 0; k < n; ++k) s = madd_rn(s, Vc[size_t(k) * n + i], t[k]);
    x[i] = s;
}

/// Kernel projection, reference order: one thread per kernel component walks
/// the elements sequentially (bitwise equal to dot/axpy, blockla.hpp:60-68).
__global__ void project_strict_kernel(double* v, int N, int bs, const int* offs, int ncomp,
                                      double kval) {
    const int c = threadIdx.x;
    if (c >= ncomp) return;
    const int off = offs[c];
    double d = 0.0;
    for (int e = 0; e < N; ++e) d = madd_rn(d, v[size_t(e) * bs + off], kval);
    const double md = -d;
    for (int e = 0; e < N; ++e) {
        double& x = v[size_t(e) * bs + off];
        x = __dadd_rn(x, __dmul_rn(md, kval));
    }
}

/// Fast projection: fixed-shape two-level tree (per-thread strided partials,
/// warp tree, CTA tree), one CTA per kernel component, deterministic and
/// independent of the device count; then the axpy.
__global__ void project_fast_kernel(double* v, int N, int bs, const int* offs, int ncomp,
                                    double kval) {
    const int c = blockIdx.x;
    if (c >= ncomp) return;
    const int off = offs[c];
    __shared__ double red[32];
    double s = 0.0;
    for (int e = threadIdx.x; e < N; e += blockDim.x) s += v[size_t(e) * bs + off] * kval;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) red[0] = s;
    }
    __syncthreads();
    const double md = -red[0];
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        double& x = v[size_t(e) * bs + off];
        x = __dadd_rn(x, __dmul_rn(md, kval));
    }
}

__global__ void axpy_kernel(int64_t n, double alpha, const double* __restrict__ x,
                            double* __restrict__ y) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i]));
}

__global__ void fill_kernel(int64_t n, double v, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        y[i] = v;
}

constexpr int kDotBlocks = 296;  // fixed -> deterministic tree independent of launch config
__global__ void dot_partial_kernel(int64_t n, const double* __restrict__ a,
                                   const double* __restrict__ b, double* __restrict__ part) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        s += a[i] * b[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}
__global__ void dot_final_kernel(const double* __restrict__ part, int np, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < np; ++i) s += part[i];
        *out = s;
    }
}

__global__ void gather_blocks_kernel(const double* __restrict__ x, const int* __restrict__ idx, int n, int bs,
                                     double* __restrict__ out) {
    const int64_t total = int64_t(n) * bs;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(t / bs), e = int(t - int64_t(i) * bs);
        out[t] = x[size_t(idx[i]) * bs + e];
    }
}

int grid1(int64_t n, int threads, const Ctx& ctx) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, int64_t(ctx.num_sms) * 32)));
}

}  // namespace

void launch_restrict(Ctx& ctx, const Transfer& T, const double* rf, double* rc) {
    const int64_t total = int64_t(T.n_coarse) * T.bs;
    if (!total) return;
    if (T.max_children <= 64 && size_t(T.max_children) * T.bs * 8 <= 48 * 1024) {
        const int threads = T.bs <= 32 ? 32 : T.bs <= 64 ? 64 : T.bs <= 128 ? 128 : 256;
        restrict_cta_kernel<<<std::max(1, std::min(T.n_coarse, ctx.num_sms * 16)), threads,
                              size_t(T.max_children) * T.bs * 8, ctx.stream>>>(
            T.child_ptr.as<int>(), T.child_list.as<int>(), T.orth.as<int>(), T.K.as<double>(), rf, rc, T.n_coarse,
            T.bss, T.ncomp, T.max_children);
        after_launch("restrict_cta_kernel");
        return;
    }
    restrict_kernel<<<grid1(total, 256, ctx), 256, 0, ctx.stream>>>(
        T.child_ptr.as<int>(), T.child_list.as<int>(), T.orth.as<int>(), T.K.as<double>(), rf, rc,
        T.n_coarse, T.bss, T.ncomp);
    after_launch("restrict_kernel");
}

void launch_prolong_add(Ctx& ctx, const Transfer& T, const double* xc, double* xf) {
    const int64_t total = int64_t(T.n_fine) * T.bs;
    if (!total) return;
    if (T.bs * 8 <= 48 * 1024) {
        const int threads = std::min(256, std::max(32, ((T.max_children * T.bs + 31) / 32) * 32));
        prolong_cta_kernel<<<std::max(1, std::min(T.n_coarse, ctx.num_sms * 16)), threads, size_t(T.bs) * 8,
                             ctx.stream>>>(T.child_ptr.as<int>(), T.child_list.as<int>(), T.orth.as<int>(),
                                           T.K.as<double>(), xc, xf, T.n_coarse, T.bss, T.ncomp);
        after_launch("prolong_cta_kernel");
        return;
    }
    prolong_kernel<<<grid1(total, 256, ctx), 256, 0, ctx.stream>>>(
        T.parent.as<int>(), T.orth.as<int>(), T.K.as<double>(), xc, xf, T.n_fine, T.bss, T.ncomp);
    after_launch("prolong_kernel");
}

void launch_pinv_apply(Ctx& ctx, const DenseEig& E, double tol, const double* b, double* x) {
    const int n = E.n;
    if (!n) return;
    const double cut = tol * E.lmax;
    if (n <= 3072) {
        pinv_cta_kernel<<<1, 1024, sizeof(double) * 2 * n, ctx.stream>>>(E.Vr.as<double>(), E.Vc.as<double>(),
                                                                        E.lambda.as<double>(), b, x, n, cut);
        after_launch("pinv_cta_kernel");
        return;
    }
    pinv_t_kernel<<<div_up(n, 128), 128, 0, ctx.stream>>>(E.Vr.as<double>(), E.lambda.as<double>(),
                                                         b, E.t.as<double>(), n, cut);
    after_launch("pinv_t_kernel");
    pinv_x_kernel<<<div_up(n, 128), 128, 0, ctx.stream>>>(E.Vc.as<double>(), E.t.as<double>(), x, n);
    after_launch("pinv_x_kernel");
}

void launch_project_constants(Ctx& ctx, double* v, int N, int bs, const int* comp_offsets,
                              int ncomp, double kval, bool strict_order) {
    if (!ncomp) return;
    if (strict_order) {
        project_strict_kernel<<<1, 32, 0, ctx.stream>>>(v, N, bs, comp_offsets, ncomp, kval);
        after_launch("project_strict_kernel");
    } else {
        project_fast_kernel<<<ncomp, 1024, 0, ctx.stream>>>(v, N, bs, comp_offsets, ncomp, kval);
        after_launch("project_fast_kernel");
    }
}

void launch_gather_blocks(Ctx& ctx, const double* x, const int* idx, int n, int bs, double* out) {
    if (n <= 0) return;
    gather_blocks_kernel<<<grid1(int64_t(n) * bs, 256, ctx), 256, 0, ctx.stream>>>(x, idx, n, bs, out);
    after_launch("gather_blocks_kernel");
}

void launch_axpy(Ctx& ctx, int64_t n, double alpha, const double* x, double* y) {
    if (!n) return;
    axpy_kernel<<<grid1(n, 256, ctx), 256, 0, ctx.stream>>>(n, alpha, x, y);
    after_launch("axpy_kernel");
}

void launch_fill(Ctx& ctx, int64_t n, double v, double* y) {
    if (!n) return;
    fill_kernel<<<grid1(n, 256, ctx), 256, 0, ctx.stream>>>(n, v, y);
    after_launch("fill_kernel");
}

void launch_dot(Ctx& ctx, int64_t n, const double* a, const double* b, double* d_out) {
    // partials live right after d_out in the context's reduction scratch
    double* part = d_out + 1;
    dot_partial_kernel<<<kDotBlocks, 256, 0, ctx.stream>>>(n, a, b, part);
    after_launch("dot_partial_kernel");
    dot_final_kernel<<<1, 32, 0, ctx.stream>>>(part, kDotBlocks, d_out);
    after_launch("dot_final_kernel");
}

}  // namespace ldgmg_b200
