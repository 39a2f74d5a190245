// Krylov accelerators around the GPU V-cycle (krylov.hpp:35-306): the
// reference's measurement protocol.  Preconditioned CG with the V-norm
// residual and left-preconditioned full GMRES (MGS Arnoldi + Givens), the
// log-linear rate fit, and estimate_eta.  Vectors stay on the device; the
// small Hessenberg / Givens recurrences run on the host exactly as in the
// reference.  Dot products use the fixed-shape tree reduction, or the
// reference's sequential order when the hierarchy is in strict-order mode
// (then CG/GMRES are bit-identical to the reference).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#include "core.hpp"
#include "krylov.hpp"
#include "mg.hpp"

namespace ldgmg_b200 {

namespace {

__global__ void dot_strict_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                                  double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s = madd_rn(s, a[i], b[i]);
        *out = s;
    }
}

__global__ void scale_kernel(int64_t n, double alpha, double* __restrict__ x) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        x[i] = __dmul_rn(x[i], alpha);
}

/// p = z + beta p   (krylov.hpp:160)
__global__ void xpby_kernel(int64_t n, const double* __restrict__ z, double beta, double* __restrict__ p) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

int grid_n(int64_t n, const Ctx& ctx) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(ctx.num_sms) * 16)));
}

struct Ops {
    Ctx& ctx;
    Mg& mg;
    int64_t n;
    DevBuf red;
    double* h_red;
    Ops(Ctx& c, Mg& m, int64_t n_) : ctx(c), mg(m), n(n_), red(sizeof(double) * 1024) {
        LDGMG_CUDA(cudaMallocHost(&h_red, sizeof(double) * 2));
    }
    ~Ops() { cudaFreeHost(h_red); }
    double dot(const double* a, const double* b) {
        if (mg.strict_order) {
            dot_strict_kernel<<<1, 32, 0, ctx.stream>>>(n, a, b, red.as<double>());
            after_launch("dot_strict_kernel");
        } else {
            launch_dot(ctx, n, a, b, red.as<double>());
        }
        LDGMG_CUDA(cudaMemcpyAsync(h_red, red.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
        return h_red[0];
    }
    void axpy(double alpha, const double* x, double* y) { launch_axpy(ctx, n, alpha, x, y); }
    void scale(double alpha, double* x) {
        scale_kernel<<<grid_n(n, ctx), 256, 0, ctx.stream>>>(n, alpha, x);
        after_launch("scale_kernel");
    }
    void copy(double* dst, const double* src) {
        LDGMG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx.stream));
    }
    void spmv(const double* x, double* y) {
        RowPass p;
        p.A = mg.A[0];
        p.mode = MODE_SPMV;
        p.x = x;
        p.y = y;
        p.nrows = mg.A[0]->brows;
        launch_rowpass(ctx, p);
    }
    void precond(const double* r, double* z) { mg.apply(ctx, r, z); }
};

}  // namespace

void fit_rate(SolveReport& rep) {
    const auto& r = rep.residuals;
    rep.rho = 0.0;
    rep.eta = 0.0;
    rep.low_confidence = true;
    rep.classification = 0;
    if (r.empty() || r[0] <= 0.0) return;
    const double floor = 1e-13 * r[0];
    int K = 0;
    while (K + 1 < int(r.size()) && r[K + 1] > floor) ++K;
    double slope;
    if (K >= 2) {
        double sx = 0, sy = 0, sxx = 0, sxy = 0;
        for (int k = 1; k <= K; ++k) {
            const double x = k, y = std::log(r[k]);
            sx += x;
            sy += y;
            sxx += x * x;
            sxy += x * y;
        }
        slope = (K * sxy - sx * sy) / (K * sxx - sx * sx);
        rep.low_confidence = K < 3;
    } else if (int(r.size()) >= 2) {
        slope = std::log(std::max(r[1], 1e-300)) - std::log(r[0]);
    } else {
        return;
    }
    rep.rho = std::exp(slope);
    if (rep.rho >= 1.0) {
        rep.eta = std::numeric_limits<double>::infinity();
        rep.classification = 2;
        return;
    }
    rep.eta = std::log(0.1) / std::log(rep.rho);
    rep.classification = rep.eta < 2.0 ? 0 : rep.eta < 10.0 ? 1 : 2;
}

/// pcg (krylov.hpp:117-164), zero initial guess; b, x device vectors.
SolveReport pcg(Ctx& ctx, Mg& mg, const double* b, double* x, double tol, int maxit) {
    if (!mg.symmetric()) fail(LDGMG_ERR_INVALID_ARGUMENT, "pcg: preconditioner plan is not symmetric");
    const int64_t n = int64_t(mg.A[0]->brows) * mg.bs;
    Ops op(ctx, mg, n);
    SolveReport rep;
    DevBuf r(sizeof(double) * n), z(sizeof(double) * n), p(sizeof(double) * n), Ap(sizeof(double) * n);
    LDGMG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, ctx.stream));
    op.copy(r.as<double>(), b);
    op.precond(r.as<double>(), z.as<double>());
    double rz = op.dot(r.as<double>(), z.as<double>());
    const double r0 = std::sqrt(std::max(rz, 0.0));
    rep.residuals.push_back(r0);
    if (r0 == 0.0) {
        rep.converged = true;
        fit_rate(rep);
        return rep;
    }
    op.copy(p.as<double>(), z.as<double>());
    for (int it = 1; it <= maxit; ++it) {
        op.spmv(p.as<double>(), Ap.as<double>());
        const double pAp = op.dot(p.as<double>(), Ap.as<double>());
        if (pAp <= 0.0) {
            rep.breakdown = true;
            break;
        }
        const double alpha = rz / pAp;
        op.axpy(alpha, p.as<double>(), x);
        op.axpy(-alpha, Ap.as<double>(), r.as<double>());
        op.precond(r.as<double>(), z.as<double>());
        const double rz_new = op.dot(r.as<double>(), z.as<double>());
        const double rk = std::sqrt(std::max(rz_new, 0.0));
        rep.residuals.push_back(rk);
        rep.iterations = it;
        if (rz_new < 0.0) {
            rep.breakdown = true;
            break;
        }
        if (rk <= tol * r0) {
            rep.converged = true;
            break;
        }
        const double beta = rz_new / rz;
        rz = rz_new;
        xpby_kernel<<<grid_n(n, ctx), 256, 0, ctx.stream>>>(n, z.as<double>(), beta, p.as<double>());
        after_launch("xpby_kernel");
    }
    fit_rate(rep);
    return rep;
}

/// gmres_left (krylov.hpp:169-251), zero initial guess.
SolveReport gmres_left(Ctx& ctx, Mg& mg, const double* b, double* x, double tol, int maxit) {
    const int64_t n = int64_t(mg.A[0]->brows) * mg.bs;
    Ops op(ctx, mg, n);
    SolveReport rep;
    LDGMG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, ctx.stream));
    DevBuf basis(sizeof(double) * n * size_t(maxit + 1)), w(sizeof(double) * n), t(sizeof(double) * n);
    auto V = [&](int i) { return basis.as<double>() + size_t(i) * n; };
    op.precond(b, V(0));
    const double g0 = std::sqrt(op.dot(V(0), V(0)));
    rep.residuals.push_back(g0);
    if (g0 == 0.0) {
        rep.converged = true;
        fit_rate(rep);
        return rep;
    }
    op.scale(1.0 / g0, V(0));
    int nbasis = 1;
    std::vector<double> H(size_t(maxit + 1) * maxit, 0.0), gamma(maxit + 1, 0.0), cs(maxit), sn(maxit);
    auto h = [&](int i, int j) -> double& { return H[size_t(j) * (maxit + 1) + i]; };
    gamma[0] = g0;
    int m = 0;
    for (int j = 0; j < maxit; ++j) {
        op.spmv(V(j), t.as<double>());
        op.precond(t.as<double>(), w.as<double>());
        const double pre_norm = std::sqrt(op.dot(w.as<double>(), w.as<double>()));
        for (int i = 0; i <= j; ++i) {
            const double hv = op.dot(w.as<double>(), V(i));
            h(i, j) = hv;
            op.axpy(-hv, V(i), w.as<double>());
        }
        const double hn = std::sqrt(op.dot(w.as<double>(), w.as<double>()));
        h(j + 1, j) = hn;
        const bool happy = hn <= 1e-14 * pre_norm;
        if (!happy) {
            op.scale(1.0 / hn, w.as<double>());
            op.copy(V(nbasis), w.as<double>());
            ++nbasis;
        }
        for (int i = 0; i < j; ++i) {
            const double tv = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
            h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
            h(i, j) = tv;
        }
        const double d = std::hypot(h(j, j), h(j + 1, j));
        if (d == 0.0) {
            cs[j] = 1.0;
            sn[j] = 0.0;
        } else {
            cs[j] = h(j, j) / d;
            sn[j] = h(j + 1, j) / d;
        }
        h(j, j) = d;
        h(j + 1, j) = 0.0;
        gamma[j + 1] = -sn[j] * gamma[j];
        gamma[j] = cs[j] * gamma[j];
        m = j + 1;
        const double rk = std::abs(gamma[j + 1]);
        rep.residuals.push_back(rk);
        rep.iterations = m;
        if (happy) {
            rep.breakdown = true;
            rep.converged = true;
            break;
        }
        if (rk <= tol * g0) {
            rep.converged = true;
            break;
        }
    }
    std::vector<double> y(m, 0.0);
    for (int i = m - 1; i >= 0; --i) {
        double s = gamma[i];
        for (int k = i + 1; k < m; ++k) s -= h(i, k) * y[k];
        y[i] = h(i, i) != 0.0 ? s / h(i, i) : 0.0;
    }
    for (int i = 0; i < m; ++i) op.axpy(y[i], V(i), x);
    fit_rate(rep);
    return rep;
}

/// estimate_eta (krylov.hpp:279-306): seeded uniform rhs, kernel projected
/// out (kernel vectors are orthonormal constant fields, so the reference's
/// orthonormalize() returns them unchanged), zero guess, CG or GMRES.
SolveReport estimate_eta(Ctx& ctx, Mg& mg, int kind, uint64_t seed, double tol, int maxit) {
    const int N = mg.A[0]->brows, bs = mg.bs;
    const int64_t n = int64_t(N) * bs;
    std::vector<double> b(n);
    std::mt19937_64 rng(seed);
    for (auto& v : b) {
        const double u = double(rng() >> 11) * 0x1.0p-53;
        v = 2.0 * u - 1.0;
    }
    // kernel_basis (ldg_core.hpp:64-78), orthonormalize (krylov.hpp:254-265:
    // disjoint constant fields, so only the renormalisation touches the bits)
    // and dot/axpy (blockla.hpp:60-68), all in the reference's order
    double kv = 1.0 / std::sqrt(double(N));
    {
        double s = 0.0;
        for (int e = 0; e < N; ++e) s += kv * kv;
        const double nrm = std::sqrt(s);
        if (nrm > 1e-10) kv = kv * (1.0 / nrm);
    }
    for (int off : mg.kernel_offsets_host) {
        double d = 0.0;
        for (int64_t i = 0; i < n; ++i) d += b[i] * ((i % bs) == off ? kv : 0.0);
        for (int64_t i = 0; i < n; ++i) b[i] += -d * ((i % bs) == off ? kv : 0.0);
    }
    DevBuf db(sizeof(double) * n), dx(sizeof(double) * n);
    h2d(ctx, db.p, b.data(), sizeof(double) * n);
    return kind == 0 ? pcg(ctx, mg, db.as<double>(), dx.as<double>(), tol, maxit)
                     : gmres_left(ctx, mg, db.as<double>(), dx.as<double>(), tol, maxit);
}

}  // namespace ldgmg_b200
