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
#include <cstdlib>
#include <string>
#include <type_traits>

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

/// Restriction, one THREAD per (parent p, child q, output o = (c, j)): the
/// per-child sum s_q = 0 + K_o[0,j] src_q[c,0] + K_o[1,j] src_q[c,1] + ... is
/// one BSS-long chain whose 2*BSS operands are all loaded up front (BSS
/// compile-time, fully unrolled), so a parent costs ~3 memory round trips
/// (child_ptr -> child ids -> K / residual blocks) + one chain; the s_q meet
/// in shared memory and thread o sums them in child order,
/// acc = 0 + s_1 + s_2 + ... (restrict_kernel's bits).  `ppc` parents per CTA.
template <int BSS>
__global__ void __launch_bounds__(256) restrict_item_kernel(const int* __restrict__ child_ptr,
                                                            const int* __restrict__ child,
                                                            const int* __restrict__ corth,
                                                            const double* __restrict__ K,
                                                            const double* __restrict__ rf, double* __restrict__ rc,
                                                            int n_coarse, int bss_rt, int ncomp, int maxch, int ppc,
                                                            double* __restrict__ zero_xc) {
    extern __shared__ double ssum[];  // ppc x maxch x BS
    const int bss = BSS > 0 ? BSS : bss_rt;
    const int BS = bss * ncomp, bb = bss * bss, per = maxch * BS;
    pdl_launch_dependents();
    pdl_wait();
    for (int p0 = blockIdx.x * ppc; p0 < n_coarse; p0 += gridDim.x * ppc) {
        for (int t = threadIdx.x; t < ppc * per; t += blockDim.x) {
            const int lp = t / per, r = t - lp * per, q = r / BS, o = r - q * BS;
            const int p = p0 + lp;
            if (p >= n_coarse) continue;
            const int q0 = __ldg(child_ptr + p), nch = __ldg(child_ptr + p + 1) - q0;
            if (q >= nch) continue;
            const int f = __ldg(child + q0 + q), ot = __ldg(corth + q0 + q);
            const double* src = rf + size_t(f) * BS;
            double sq;
            if (ot < 0) {
                sq = src[o];
            } else {
                const int c = o / bss, j = o - c * bss;
                const double* Ko = K + size_t(ot) * bb + j;
                const double* sc = src + c * bss;
                sq = 0.0;
                if constexpr (BSS > 0) {
                    double kv[BSS], xv[BSS];
#pragma unroll
                    for (int i = 0; i < BSS; ++i) {
                        kv[i] = __ldg(Ko + i * BSS);
                        xv[i] = sc[i];
                    }
#pragma unroll
                    for (int i = 0; i < BSS; ++i) sq = madd_rn(sq, kv[i], xv[i]);
                } else {
#pragma unroll 9
                    for (int i = 0; i < bss; ++i) sq = madd_rn(sq, __ldg(Ko + size_t(i) * bss), sc[i]);
                }
            }
            ssum[t] = sq;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < ppc * BS; t += blockDim.x) {
            const int lp = t / BS, o = t - lp * BS, p = p0 + lp;
            if (p >= n_coarse) continue;
            const int nch = __ldg(child_ptr + p + 1) - __ldg(child_ptr + p);
            const double* ss = ssum + size_t(lp) * per + o;
            double acc = 0.0;
            for (int q = 0; q < nch; ++q) acc = __dadd_rn(acc, ss[q * BS]);
            rc[size_t(p) * BS + o] = acc;
            if (zero_xc) zero_xc[size_t(p) * BS + o] = 0.0;  // the coarse iterate starts at 0
        }
        __syncthreads();
    }
}

/// Prolongation, one THREAD per fine entry (f, ii = (c, i)):
/// xf[ii] += 0 + K_o[i,0] xc_p[c,0] + K_o[i,1] xc_p[c,1] + ...  (prolong_kernel's
/// bits).  K is read transposed (Kt[j,i]) so the threads of one child
/// (consecutive i) load consecutive words; xc loads broadcast.
template <int BSS>
__global__ void __launch_bounds__(256) prolong_flat_kernel(const int* __restrict__ parent,
                                                           const int* __restrict__ orth,
                                                           const double* __restrict__ Kt,
                                                           const double* __restrict__ xc,
                                                           double* __restrict__ xf, int n_fine, int bss_rt,
                                                           int ncomp) {
    const int bss = BSS > 0 ? BSS : bss_rt;
    const int BS = bss * ncomp, bb = bss * bss;
    const int64_t total = int64_t(n_fine) * BS;
    const int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const bool live = o < total;
    const int f = live ? int(o / BS) : 0;
    const int ii = int(o - int64_t(f) * BS), c = ii / bss, i = ii - c * bss;
    const int p = __ldg(parent + f), ot = __ldg(orth + f);
    pdl_launch_dependents();
    pdl_wait();
    if (!live) return;
    const double* src = xc + size_t(p) * BS + c * bss;
    const double old = xf[o];
    if (ot < 0) {
        xf[o] = __dadd_rn(old, xc[size_t(p) * BS + ii]);
        return;
    }
    const double* Kc = Kt + size_t(ot) * bb + i;
    double s = 0.0;
    if constexpr (BSS > 0) {
        double kv[BSS], xv[BSS];
#pragma unroll
        for (int jj = 0; jj < BSS; ++jj) {
            kv[jj] = __ldg(Kc + jj * BSS);
            xv[jj] = src[jj];
        }
#pragma unroll
        for (int jj = 0; jj < BSS; ++jj) s = madd_rn(s, kv[jj], xv[jj]);
    } else {
#pragma unroll 9
        for (int jj = 0; jj < bss; ++jj) s = madd_rn(s, __ldg(Kc + size_t(jj) * bss), src[jj]);
    }
    xf[o] = __dadd_rn(old, s);
}

/// Transfers of a REGULAR hierarchy (children of p are NCH p + o, o the
/// orthant): "K-stationary" kernels.  Thread (o, j) keeps column j of K_o
/// (restriction) or row i of K_o (prolongation) in registers for the whole
/// kernel and streams PB parents at a time through shared memory, so every
/// multiply-add needs one broadcast shared-memory operand and nothing else;
/// the arithmetic (and the bits) are restrict_kernel's / prolong_kernel's.
template <int BSS, int NCH, int PB>
__global__ void __launch_bounds__(NCH * BSS) restrict_ks_kernel(const double* __restrict__ K,
                                                               const double* __restrict__ rf, double* __restrict__ rc,
                                                               int n_coarse, int ncomp, double* __restrict__ zero_xc) {
    extern __shared__ double sm[];  // sx: PB x NCH x BS, ss: PB x NCH x BS
    const int BS = BSS * ncomp;
    double* sx = sm;
    double* ss = sm + size_t(PB) * NCH * BS;
    const int t = threadIdx.x, o = t / BSS, j = t - o * BSS;
    double kc[BSS];
#pragma unroll
    for (int i = 0; i < BSS; ++i) kc[i] = __ldg(K + size_t(o) * BSS * BSS + i * BSS + j);
    pdl_launch_dependents();
    pdl_wait();
    for (int p0 = blockIdx.x * PB; p0 < n_coarse; p0 += gridDim.x * PB) {
        const int np = min(PB, n_coarse - p0);
        // children of p0..p0+np-1 are one contiguous run of fine blocks
        const double* src = rf + size_t(p0) * NCH * BS;
        for (int e = t; e < np * NCH * BS; e += NCH * BSS) sx[e] = src[e];
        __syncthreads();
        for (int lp = 0; lp < np; ++lp)
            for (int c = 0; c < ncomp; ++c) {
                const double* xv = sx + (size_t(lp) * NCH + o) * BS + c * BSS;
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < BSS; ++i) s = madd_rn(s, kc[i], xv[i]);
                ss[(size_t(lp) * NCH + o) * BS + c * BSS + j] = s;
            }
        __syncthreads();
        for (int e = t; e < np * BS; e += NCH * BSS) {
            const int lp = e / BS, oo = e - lp * BS;
            const double* sp = ss + size_t(lp) * NCH * BS + oo;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < NCH; ++q) acc = __dadd_rn(acc, sp[q * BS]);
            rc[size_t(p0) * BS + e] = acc;
            if (zero_xc) zero_xc[size_t(p0) * BS + e] = 0.0;  // the coarse iterate starts at 0
        }
        __syncthreads();
    }
}

template <int BSS, int NCH, int PB>
__global__ void __launch_bounds__(NCH * BSS) prolong_ks_kernel(const double* __restrict__ K,
                                                              const double* __restrict__ xc, double* __restrict__ xf,
                                                              int n_coarse, int ncomp) {
    extern __shared__ double sm[];  // PB x BS coarse blocks
    const int BS = BSS * ncomp;
    const int t = threadIdx.x, o = t / BSS, i = t - o * BSS;
    double kr[BSS];
#pragma unroll
    for (int jj = 0; jj < BSS; ++jj) kr[jj] = __ldg(K + size_t(o) * BSS * BSS + i * BSS + jj);
    pdl_launch_dependents();
    pdl_wait();
    for (int p0 = blockIdx.x * PB; p0 < n_coarse; p0 += gridDim.x * PB) {
        const int np = min(PB, n_coarse - p0);
        for (int e = t; e < np * BS; e += NCH * BSS) sm[e] = xc[size_t(p0) * BS + e];
        __syncthreads();
        for (int lp = 0; lp < np; ++lp)
            for (int c = 0; c < ncomp; ++c) {
                const double* xv = sm + size_t(lp) * BS + c * BSS;
                double* dst = xf + (size_t(p0 + lp) * NCH + o) * BS + c * BSS + i;
                const double old = *dst;
                double s = 0.0;
#pragma unroll
                for (int jj = 0; jj < BSS; ++jj) s = madd_rn(s, kr[jj], xv[jj]);
                *dst = __dadd_rn(old, s);
            }
        __syncthreads();
    }
}

/// Bottom pseudoinverse streaming V through shared memory: KC rows of the
/// row-major Vr (then of Vc) per TMA bulk copy, double buffered; thread i
/// keeps its sequential k-ascending chain (reference order) for up to 3
/// columns.  The V arrays carry tail padding for the even-size copies.
__global__ void __launch_bounds__(1024) pinv_stream_kernel(const double* __restrict__ Vr,
                                                           const double* __restrict__ Vc,
                                                           const double* __restrict__ lam,
                                                           const double* __restrict__ b, double* __restrict__ x,
                                                           int n, double cut, int KC) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[2];
    const int tid = threadIdx.x, NT = blockDim.x;
    const int nv = (n + 1) & ~1;
    double* sb = sm;            // b, then reused for nothing
    double* st = sm + nv;       // t
    double* ring = st + nv;     // 2 x KC x n
    const size_t chunk = size_t(KC) * n;
    const int nchunks = (n + KC - 1) / KC;
    if (tid == 0) {
        mbar_init(bars + 0, 1);
        mbar_init(bars + 1, 1);
        fence_mbar_init();
    }
    pdl_launch_dependents();
    pdl_wait();
    for (int i = tid; i < n; i += NT) sb[i] = b[i];
    __syncthreads();
    uint32_t phases = 0u;  // bit s: parity to wait for on bars[s]
    for (int pass = 0; pass < 2; ++pass) {
        const double* Vm = pass == 0 ? Vr : Vc;
        const double* vin = pass == 0 ? sb : st;
        auto issue = [&](int c) {
            const int rows = min(KC, n - c * KC);
            const uint32_t bytes = uint32_t(((size_t(rows) * n + 1) & ~size_t(1)) * sizeof(double));
            double* dst = ring + size_t(c & 1) * chunk;
            mbar_arrive_expect_tx(bars + (c & 1), bytes);
            bulk_g2s(dst, Vm + size_t(c) * chunk, bytes, bars + (c & 1));
        };
        if (tid == 0) {
            fence_proxy_async();
            issue(0);
            if (nchunks > 1) issue(1);
        }
        double acc[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c < nchunks; ++c) {
            const int slot = c & 1;
            mbar_wait(bars + slot, (phases >> slot) & 1u);
            phases ^= 1u << slot;
            const double* rows = ring + size_t(slot) * chunk;
            const int k0 = c * KC, kr = min(KC, n - k0);
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int i = tid + u * NT;
                if (i < n) {
                    double s = acc[u];
                    for (int k = 0; k < kr; ++k) s = madd_rn(s, rows[size_t(k) * n + i], vin[k0 + k]);
                    acc[u] = s;
                }
            }
            __syncthreads();  // every thread is done with this slot
            if (tid == 0 && c + 2 < nchunks) {
                fence_proxy_async();
                issue(c + 2);
            }
        }
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int i = tid + u * NT;
            if (i < n) {
                if (pass == 0) {
                    const double l = lam[i];
                    st[i] = fabs(l) <= cut ? 0.0 : acc[u] / l;
                } else {
                    x[i] = acc[u];
                }
            }
        }
        __syncthreads();
    }
}

/// t_i = cut(sum_k V(k,i) b_k) / lambda_i ; Vr row-major: V(k,i) at k*n+i.
/// Large bottoms (n >= 1536, C5 48^3: n = 2916): one thread per output, the
/// k-ascending chain fed by batches of 32 independent V loads (coalesced
/// across the warp), so each thread keeps 32 loads in flight instead of
/// one: the GEMV is latency-bound by construction (the sum order is fixed).
constexpr int kPinvBatch = 32;
/// read-only load kept in program order (asm volatile), so a batch of them
/// is issued before the chain consumes the first
__device__ __forceinline__ double ldg_ordered(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__global__ void __launch_bounds__(64) pinv_t_kernel(const double* __restrict__ Vr, const double* __restrict__ lam,
                                                    const double* __restrict__ b, double* __restrict__ t, int n,
                                                    double cut) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    pdl_launch_dependents();
    pdl_wait();
    if (i >= n) return;
    double s = 0.0;
    int k = 0;
    for (; k + kPinvBatch <= n; k += kPinvBatch) {
        double v[kPinvBatch];
#pragma unroll
        for (int u = 0; u < kPinvBatch; ++u) v[u] = ldg_ordered(Vr + size_t(k + u) * n + i);
#pragma unroll
        for (int u = 0; u < kPinvBatch; ++u) s = madd_rn(s, v[u], __ldg(b + k + u));
    }
    for (; k < n; ++k) s = madd_rn(s, __ldg(Vr + size_t(k) * n + i), __ldg(b + k));
    const double l = lam[i];
    t[i] = fabs(l) <= cut ? 0.0 : s / l;
}

/// x_i = sum_k V(i,k) t_k ; Vc column-major: V(i,k) at k*n+i.
__global__ void __launch_bounds__(64) pinv_x_kernel(const double* __restrict__ Vc, const double* __restrict__ t,
                                                    double* __restrict__ x, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    pdl_launch_dependents();
    pdl_wait();
    if (i >= n) return;
    double s = 0.0;
    int k = 0;
    for (; k + kPinvBatch <= n; k += kPinvBatch) {
        double v[kPinvBatch];
#pragma unroll
        for (int u = 0; u < kPinvBatch; ++u) v[u] = ldg_ordered(Vc + size_t(k + u) * n + i);
#pragma unroll
        for (int u = 0; u < kPinvBatch; ++u) s = madd_rn(s, v[u], __ldg(t + k + u));
    }
    for (; k < n; ++k) s = madd_rn(s, __ldg(Vc + size_t(k) * n + i), __ldg(t + k));
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

/// Fast projection over the whole GPU with a fixed shape (kProjParts
/// contiguous element ranges, fixed trees), so the result is deterministic
/// and independent of the device: partials, then every CTA re-sums the
/// partials in the same order and applies the update to its range.
constexpr int kProjParts = 256;
__global__ void __launch_bounds__(256) project_partial_kernel(const double* __restrict__ v, int N, int bs,
                                                              const int* __restrict__ offs, double kval,
                                                              double* __restrict__ part, int k0 = 0, int ebase = 0) {
    __shared__ double red[8];
    pdl_launch_dependents();
    pdl_wait();
    const int k = k0 + blockIdx.x, c = blockIdx.y, off = offs[c];
    const int e0 = int(int64_t(k) * N / kProjParts), e1 = int(int64_t(k + 1) * N / kProjParts);
    double s = 0.0;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) s = madd_rn(s, v[size_t(e - ebase) * bs + off], kval);
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t = __dadd_rn(t, red[w]);
        part[c * kProjParts + k] = t;
    }
}
__global__ void __launch_bounds__(256) project_apply_kernel(double* __restrict__ v, int N, int bs,
                                                            const int* __restrict__ offs, double kval,
                                                            const double* __restrict__ part, int k0 = 0,
                                                            int ebase = 0) {
    __shared__ double red[8];
    __shared__ double md;
    pdl_launch_dependents();
    pdl_wait();
    const int k = k0 + blockIdx.x, c = blockIdx.y, off = offs[c];
    double s = part[c * kProjParts + threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t = __dadd_rn(t, red[w]);
        md = -t;
    }
    __syncthreads();
    const double m = md;
    const int e0 = int(int64_t(k) * N / kProjParts), e1 = int(int64_t(k + 1) * N / kProjParts);
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        double& xv = v[size_t(e - ebase) * bs + off];
        xv = __dadd_rn(xv, __dmul_rn(m, kval));
    }
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

namespace {
/// parents per K-stationary step of the regular-hierarchy transfer kernels
constexpr int kTransferPB = 8;
}  // namespace

void launch_restrict(Ctx& ctx, const Transfer& T, const double* rf, double* rc, double* zero_xc) {
    const int64_t total = int64_t(T.n_coarse) * T.bs;
    if (!total) return;
    if (T.regular) {
        bool done = true;
        auto go = [&](auto pbc) {
            constexpr int PB = decltype(pbc)::value;
            const int grid = std::max(1, std::min(div_up(T.n_coarse, PB), ctx.num_sms * 8));
            const size_t smem = sizeof(double) * 2 * PB * (size_t(1) << T.dim) * T.bs;
            auto launch = [&](auto kern, int threads) {
                ensure_dyn_smem(kern, smem);
                launch_pdl_small(kern, dim3(grid), dim3(threads), smem, ctx.stream, T.K.as<double>(), rf, rc,
                                 T.n_coarse, T.ncomp, zero_xc);
            };
            if (T.dim == 3 && T.bss == 27) launch(restrict_ks_kernel<27, 8, PB>, 216);
            else if (T.dim == 3 && T.bss == 8) launch(restrict_ks_kernel<8, 8, PB>, 64);
            else if (T.dim == 2 && T.bss == 16) launch(restrict_ks_kernel<16, 4, PB>, 64);
            else if (T.dim == 2 && T.bss == 25) launch(restrict_ks_kernel<25, 4, PB>, 100);
            else if (T.dim == 2 && T.bss == 9) launch(restrict_ks_kernel<9, 4, PB>, 36);
            else done = false;
        };
        go(std::integral_constant<int, kTransferPB>{});
        if (done) {
            after_launch("restrict_ks_kernel");
            return;
        }
    }
    const int per = std::max(1, T.max_children) * T.bs;
    if (size_t(per) * 8 <= 48 * 1024) {
        const int ppc = std::max(1, 256 / per);
        const int threads = std::min(256, ((ppc * per + 31) / 32) * 32);
        const int grid = std::max(1, std::min(div_up(T.n_coarse, ppc), ctx.num_sms * 32));
        const size_t smem = sizeof(double) * size_t(ppc) * per;
        auto launch = [&](auto kern) {
            launch_pdl_small(kern, dim3(grid), dim3(threads), smem, ctx.stream, T.child_ptr.as<int>(),
                       T.child_list.as<int>(), T.child_orth.as<int>(), T.K.as<double>(), rf, rc, T.n_coarse, T.bss,
                       T.ncomp, std::max(1, T.max_children), ppc, zero_xc);
        };
        switch (T.bss) {
            case 16: launch(restrict_item_kernel<16>); break;
            case 25: launch(restrict_item_kernel<25>); break;
            case 27: launch(restrict_item_kernel<27>); break;
            default: launch(restrict_item_kernel<0>); break;
        }
        after_launch("restrict_item_kernel");
        return;
    }
    if (zero_xc)  // the fallback kernels below do not zero
        LDGMG_CUDA(cudaMemsetAsync(zero_xc, 0, sizeof(double) * size_t(total), ctx.stream));
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
    if (T.regular) {
        bool done = true;
        auto go = [&](auto pbc) {
            constexpr int PB = decltype(pbc)::value;
            const int grid = std::max(1, std::min(div_up(T.n_coarse, PB), ctx.num_sms * 8));
            const size_t smem = sizeof(double) * PB * T.bs;
            auto launch = [&](auto kern, int threads) {
                ensure_dyn_smem(kern, smem);
                launch_pdl_small(kern, dim3(grid), dim3(threads), smem, ctx.stream, T.K.as<double>(), xc, xf,
                                 T.n_coarse, T.ncomp);
            };
            if (T.dim == 3 && T.bss == 27) launch(prolong_ks_kernel<27, 8, PB>, 216);
            else if (T.dim == 3 && T.bss == 8) launch(prolong_ks_kernel<8, 8, PB>, 64);
            else if (T.dim == 2 && T.bss == 16) launch(prolong_ks_kernel<16, 4, PB>, 64);
            else if (T.dim == 2 && T.bss == 25) launch(prolong_ks_kernel<25, 4, PB>, 100);
            else if (T.dim == 2 && T.bss == 9) launch(prolong_ks_kernel<9, 4, PB>, 36);
            else done = false;
        };
        go(std::integral_constant<int, kTransferPB>{});
        if (done) {
            after_launch("prolong_ks_kernel");
            return;
        }
    }
    {
        const int grid = div_up(total, 256);
        auto launch = [&](auto kern) {
            launch_pdl_small(kern, dim3(grid), dim3(256), 0, ctx.stream, T.parent.as<int>(), T.orth.as<int>(),
                       T.Kt.as<double>(), xc, xf, T.n_fine, T.bss, T.ncomp);
        };
        switch (T.bss) {
            case 16: launch(prolong_flat_kernel<16>); break;
            case 25: launch(prolong_flat_kernel<25>); break;
            case 27: launch(prolong_flat_kernel<27>); break;
            default: launch(prolong_flat_kernel<0>); break;
        }
        after_launch("prolong_flat_kernel");
    }
}

void launch_pinv_apply(Ctx& ctx, const DenseEig& E, double tol, const double* b, double* x) {
    const int n = E.n;
    if (!n) return;
    const double cut = tol * E.lmax;
    constexpr int big = 1536;  // above: one thread per output, batched V loads
    if (n < big) {
        // KC rows of V per stage, two stages, within ~200 KB of shared memory
        const size_t vec = size_t((n + 1) & ~1) * 2;
        int KC = int(std::min<size_t>(size_t(n), ((200 * 1024 / 8 - vec - 2) / (2 * size_t(n)))));
        KC &= ~1;
        if (KC >= 2) {
            const size_t smem = sizeof(double) * (vec + size_t(2) * KC * n + 2);
            ensure_dyn_smem(pinv_stream_kernel, size_t(smem));
            static bool once = (max_carveout(pinv_stream_kernel), true);
            (void)once;
            launch_pdl_small(pinv_stream_kernel, dim3(1), dim3(1024), smem, ctx.stream, E.Vr.as<double>(),
                       E.Vc.as<double>(), E.lambda.as<double>(), b, x, n, cut, KC);
            after_launch("pinv_stream_kernel");
            return;
        }
    }
    launch_pdl_small(pinv_t_kernel, dim3(div_up(n, 64)), dim3(64), 0, ctx.stream, E.Vr.as<double>(),
                     E.lambda.as<double>(), b, E.t.as<double>(), n, cut);
    after_launch("pinv_t_kernel");
    launch_pdl_small(pinv_x_kernel, dim3(div_up(n, 64)), dim3(64), 0, ctx.stream, E.Vc.as<double>(),
                     E.t.as<double>(), x, n);
    after_launch("pinv_x_kernel");
}

void launch_project_constants(Ctx& ctx, double* v, int N, int bs, const int* comp_offsets,
                              int ncomp, double kval, bool strict_order, double* scratch) {
    if (!ncomp) return;
    if (strict_order) {
        project_strict_kernel<<<1, 32, 0, ctx.stream>>>(v, N, bs, comp_offsets, ncomp, kval);
        after_launch("project_strict_kernel");
    } else if (scratch && N >= kProjParts) {
        static bool once = (max_carveout(project_partial_kernel), max_carveout(project_apply_kernel), true);
        (void)once;
        launch_pdl_small(project_partial_kernel, dim3(kProjParts, ncomp), dim3(256), 0, ctx.stream,
                   static_cast<const double*>(v), N, bs, comp_offsets, kval, scratch, 0, 0);
        after_launch("project_partial_kernel");
        launch_pdl_small(project_apply_kernel, dim3(kProjParts, ncomp), dim3(256), 0, ctx.stream, v, N, bs, comp_offsets,
                   kval, static_cast<const double*>(scratch), 0, 0);
        after_launch("project_apply_kernel");
    } else {
        project_fast_kernel<<<ncomp, 1024, 0, ctx.stream>>>(v, N, bs, comp_offsets, ncomp, kval);
        after_launch("project_fast_kernel");
    }
}

/// Fast projection over a rank's element slice [r0, r1): the ranges of the
/// 256 fixed global ranges that lie inside the slice (the slice must be a
/// union of ranges); same per-range trees as launch_project_constants.
static void slice_ranges(int N, int r0, int r1, int& k0, int& nk) {
    k0 = -1;
    nk = 0;
    for (int k = 0; k < kProjParts; ++k) {
        const int e0 = int(int64_t(k) * N / kProjParts), e1 = int(int64_t(k + 1) * N / kProjParts);
        if (e0 >= r0 && e1 <= r1 && e1 > e0) {
            if (k0 < 0) k0 = k;
            ++nk;
        } else if ((e0 < r1 && e1 > r0) && !(e0 >= r0 && e1 <= r1)) {
            fail(LDGMG_ERR_INVALID_ARGUMENT, "project: rank slice is not a union of the 256 projection ranges");
        }
    }
}

void launch_project_partials_slice(Ctx& ctx, const double* v, int N, int r0, int r1, int bs, const int* offs,
                                   int ncomp, double kval, double* part) {
    int k0, nk;
    slice_ranges(N, r0, r1, k0, nk);
    if (!nk || !ncomp) return;
    project_partial_kernel<<<dim3(nk, ncomp), 256, 0, ctx.stream>>>(v, N, bs, offs, kval, part, k0, r0);
    after_launch("project_partial_kernel");
}

void launch_project_apply_slice(Ctx& ctx, double* v, int N, int r0, int r1, int bs, const int* offs, int ncomp,
                                double kval, const double* part) {
    int k0, nk;
    slice_ranges(N, r0, r1, k0, nk);
    if (!nk || !ncomp) return;
    project_apply_kernel<<<dim3(nk, ncomp), 256, 0, ctx.stream>>>(v, N, bs, offs, kval, part, k0, r0);
    after_launch("project_apply_kernel");
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
