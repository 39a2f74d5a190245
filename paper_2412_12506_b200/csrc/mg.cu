// Smoothers, transfers, the multigrid hierarchy and the V-cycle driver
// (host orchestration of the device kernels; every operator application is a
// bsr_kernels.cu row pass).  Mirrors smoothers.hpp:373-534 and
// multigrid.hpp:45-274 of the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <vector>

#include "core.hpp"
#include "host_eig.hpp"
#include "mg.hpp"

#include <cusolverDn.h>
#include <string>

namespace ldgmg_b200 {

// ------------------------------------------------------------- colouring
/// Greedy colouring in ascending element order (smoothers.hpp:63-84),
/// restated; rejects non-symmetric patterns with the reference's messages.
std::vector<int> colour_mesh_host(const Bsr& A) {
    if (A.brows != A.bcols) fail(LDGMG_ERR_INVALID_ARGUMENT, "colour_mesh: matrix not block-square");
    auto find = [&](int i, int j) {
        for (int k = A.hptr[i]; k < A.hptr[i + 1]; ++k)
            if (A.hcol[k] == j) return k;
        return -1;
    };
    for (int i = 0; i < A.brows; ++i)
        for (int k = A.hptr[i]; k < A.hptr[i + 1]; ++k)
            if (find(A.hcol[k], i) < 0) fail(LDGMG_ERR_INVALID_ARGUMENT, "colour_mesh: pattern is not symmetric");
    std::vector<int> colour(A.brows, -1);
    std::vector<char> used;
    int ncol = 0;
    for (int e = 0; e < A.brows; ++e) {
        used.assign(size_t(ncol) + 1, 0);
        for (int k = A.hptr[e]; k < A.hptr[e + 1]; ++k) {
            const int j = A.hcol[k];
            if (j != e && colour[j] >= 0) used[colour[j]] = 1;
        }
        int c = 0;
        while (used[c]) ++c;
        colour[e] = c;
        ncol = std::max(ncol, c + 1);
    }
    return colour;
}

// ------------------------------------------------------- diagonal factors
void upload_factors(Ctx& ctx, DiagFactors& F, int N, int bs, const double* V, const double* lambda,
                    const double* s) {
    F.n = N;
    F.bs = bs;
    F.ld = bs | 1;
    F.vstride = even_up(int64_t(bs) * F.ld);
    std::vector<double> hv(size_t(N) * F.vstride, 0.0), lmax(N, 0.0);
    for (int e = 0; e < N; ++e) {
        const double* Ve = V + size_t(e) * bs * bs;
        double* dst = hv.data() + size_t(e) * F.vstride;
        for (int a = 0; a < bs; ++a)
            for (int b = 0; b < bs; ++b) dst[size_t(a) * F.ld + b] = Ve[size_t(a) * bs + b];
        double m = 0.0;  // cwiseAbs().maxCoeff(), blockla.hpp:332
        for (int i = 0; i < bs; ++i) m = std::max(m, std::abs(lambda[size_t(e) * bs + i]));
        lmax[e] = bs ? m : 0.0;
    }
    F.V.alloc(sizeof(double) * hv.size());
    F.lambda.alloc(sizeof(double) * size_t(N) * bs);
    F.scale.alloc(sizeof(double) * size_t(N) * bs);
    F.lmax.alloc(sizeof(double) * N);
    h2d(ctx, F.V.p, hv.data(), F.V.bytes);
    h2d(ctx, F.lambda.p, lambda, F.lambda.bytes);
    h2d(ctx, F.scale.p, s, F.scale.bytes);
    h2d(ctx, F.lmax.p, lmax.data(), F.lmax.bytes);
    (void)ctx;
}

void compute_factors(Ctx& ctx, const Bsr& A, DiagFactors& F) {
    static int host = -1;
    if (host < 0) {
        const char* e = getenv("LDGMG_HOST_FACTORS");
        host = e && atoi(e) ? 1 : 0;
    }
    if (host)
        compute_factors_host(ctx, A, F);
    else
        compute_factors_gpu(ctx, A, F);
}

/// factor_diagonal (smoothers.hpp:464-494): power-of-two equilibration
/// s_i = 2^-(ex/2) of |D_ii| (frexp exponent), then eig(s D s).
void compute_factors_host(Ctx& ctx, const Bsr& A, DiagFactors& F) {
    const int N = A.brows, bs = A.rbs;
    std::vector<int> dk(N, -1);
    for (int e = 0; e < N; ++e) {
        for (int k = A.hptr[e]; k < A.hptr[e + 1]; ++k)
            if (A.hcol[k] == e) dk[e] = k;
        if (dk[e] < 0) fail(LDGMG_ERR_RUNTIME, "Smoother: missing diagonal block");
    }
    // fetch the diagonal blocks in reference (row-major) layout
    std::vector<double> all(size_t(A.nnzb) * bs * bs);
    std::vector<int> hp(A.hptr), hc(A.hcol);
    bsr_download(ctx, A, nullptr, nullptr, all.data());
    std::vector<double> V(size_t(N) * bs * bs), lam(size_t(N) * bs), sc(size_t(N) * bs);
    std::vector<int> bad(N, 0);
    parallel_for(N, [&](int lo, int hi) {
        std::vector<double> D(size_t(bs) * bs);
        for (int e = lo; e < hi; ++e) {
            const double* v = all.data() + size_t(dk[e]) * bs * bs;
            double* s = sc.data() + size_t(e) * bs;
            for (int i = 0; i < bs; ++i) {
                const double d = std::abs(v[size_t(i) * bs + i]);
                if (d > 0.0) {
                    int ex = 0;
                    std::frexp(d, &ex);
                    s[i] = std::ldexp(1.0, -(ex / 2));
                } else {
                    s[i] = 1.0;
                }
            }
            // column-major s D s ((s_i D_ij) s_j, as the shim's diag products)
            double norm2 = 0.0, asym2 = 0.0;
            for (int j = 0; j < bs; ++j)
                for (int i = 0; i < bs; ++i) {
                    D[size_t(j) * bs + i] = (s[i] * v[size_t(i) * bs + j]) * s[j];
                    norm2 += D[size_t(j) * bs + i] * D[size_t(j) * bs + i];
                }
            for (int j = 0; j < bs; ++j)
                for (int i = 0; i < bs; ++i) {
                    const double t = D[size_t(j) * bs + i] - D[size_t(i) * bs + j];
                    asym2 += t * t;
                }
            if (std::sqrt(asym2) > 1e-13 * std::max(1e-300, std::sqrt(norm2))) {
                bad[e] = 1;
                continue;
            }
            sym_eig_host(bs, D.data(), lam.data() + size_t(e) * bs, V.data() + size_t(e) * bs * bs);
        }
    });
    for (int e = 0; e < N; ++e)
        if (bad[e]) fail(LDGMG_ERR_INVALID_ARGUMENT, "sym_eig: matrix is not symmetric");
    upload_factors(ctx, F, N, bs, V.data(), lam.data(), sc.data());
}

// ------------------------------------------- processor-block GS schedule
/// Wavefronts of the sequential processor-block GS sweep (smoothers.hpp:
/// 426-436): rows 0..n_rows-1 are relaxed in ascending (reverse: descending)
/// order within their partition, reading in-partition neighbours live and
/// everything else (other partitions; columns >= n_cols_own, i.e. a rank's
/// frozen ghosts) from the sweep-start snapshot.  Row e goes one wavefront
/// after every in-partition neighbour it reads that precedes it
/// (read-after-write) and after every earlier row that reads it
/// (write-after-read: that row must see the OLD x_e; implied by the first
/// rule on symmetric patterns, explicit so any pattern is exact).  Relaxing
/// one wavefront per launch reproduces the sequential sweep bit for bit.
void pgs_wavefronts(int n_rows, const int* ptr, const int* col, const int* part_of, int n_cols_own, bool reverse,
                    std::vector<int>& rows, std::vector<int>& level_ptr) {
    const int N = n_rows;
    auto inpart = [&](int e, int j) { return j < n_cols_own && j != e && part_of[j] == part_of[e]; };
    std::vector<int> lev(N, 0), need(N, 0);
    int nlev = N ? 1 : 0;
    for (int i = 0; i < N; ++i) {
        const int e = reverse ? N - 1 - i : i;
        int l = need[e];
        for (int k = ptr[e]; k < ptr[e + 1]; ++k) {
            const int j = col[k];
            if (inpart(e, j) && (reverse ? j > e : j < e)) l = std::max(l, lev[j] + 1);
        }
        lev[e] = l;
        nlev = std::max(nlev, l + 1);
        for (int k = ptr[e]; k < ptr[e + 1]; ++k) {
            const int j = col[k];
            if (inpart(e, j) && (reverse ? j < e : j > e)) need[j] = std::max(need[j], l + 1);
        }
    }
    level_ptr.assign(nlev + 1, 0);
    std::vector<int> cnt(nlev, 0);
    for (int e = 0; e < N; ++e) ++cnt[lev[e]];
    for (int l = 0; l < nlev; ++l) level_ptr[l + 1] = level_ptr[l] + cnt[l];
    rows.resize(N);
    std::vector<int> fill(level_ptr.begin(), level_ptr.end() - 1);
    for (int e = 0; e < N; ++e) rows[fill[lev[e]]++] = e;
}

// --------------------------------------------------------------- smoother
void Smoother::init_common(Ctx& ctx) {
    N = A->brows;
    bs = A->rbs;
    if (A->brows != A->bcols || A->rbs != A->cbs)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "Smoother: operator must be block-square");
    if (cfg.kind == LDGMG_COLOURED_GS) cfg.omega = 1.0;  // smoothers.hpp:380
    if (cfg.kind == LDGMG_COLOURED_GS) {
        colour = colour_mesh_host(*A);
        ncolours = N ? 1 + *std::max_element(colour.begin(), colour.end()) : 0;
        std::vector<int> rows;
        colour_ptr.assign(ncolours + 1, 0);
        for (int c = 0; c < ncolours; ++c) {
            for (int e = 0; e < N; ++e)
                if (colour[e] == c) rows.push_back(e);
            colour_ptr[c + 1] = int(rows.size());
        }
        colour_rows.alloc(sizeof(int) * std::max<size_t>(1, rows.size()));
        if (!rows.empty())
            h2d(ctx, colour_rows.p, rows.data(), sizeof(int) * rows.size());
    }
    if (cfg.kind == LDGMG_PROC_BLOCK_GS) {
        // partition_ranges (smoothers.hpp:87-94) and part_of (:383-386)
        const int P = cfg.partitions;
        if (P < 1 || P > N)
            fail(LDGMG_ERR_INVALID_ARGUMENT, "partition_ranges: partition count must lie in [1, N]");
        std::vector<int> part_of(N);
        for (int p = 0; p < P; ++p)
            for (int e = int(int64_t(p) * N / P); e < int(int64_t(p + 1) * N / P); ++e) part_of[e] = p;
        part.alloc(sizeof(int) * std::max(1, N));
        h2d(ctx, part.p, part_of.data(), sizeof(int) * N);
        // The reference sweeps every partition sequentially (forward:
        // ascending, reverse: descending), reading in-partition neighbours
        // live and the others from a snapshot (smoothers.hpp:426-436).  An
        // element therefore depends only on its in-partition neighbours that
        // precede it in the sweep; relaxing the wavefronts of that DAG one
        // launch at a time reproduces the sequential result bit for bit.
        for (int d = 0; d < 2; ++d) {
            std::vector<int> rows;
            pgs_wavefronts(N, A->hptr.data(), A->hcol.data(), part_of.data(), N, d == 1, rows, sched_ptr[d]);
            sched_rows[d].alloc(sizeof(int) * std::max(1, N));
            if (N) h2d(ctx, sched_rows[d].p, rows.data(), sizeof(int) * N);
        }
    }
    if (cfg.kind == LDGMG_SAI && cfg.level < 0)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "pattern_power: negative power");
    snap.alloc(sizeof(double) * std::max<int64_t>(1, int64_t(N) * bs));
    (void)ctx;
}

void Smoother::apply(Ctx& ctx, const double* b, double* x, int sweep, bool r_ready, const double* r_in) const {
    switch (cfg.kind) {
        case LDGMG_JACOBI: {
            LDGMG_CUDA(cudaMemcpyAsync(snap.p, x, sizeof(double) * size_t(N) * bs,
                                       cudaMemcpyDeviceToDevice, ctx.stream));
            RowPass p;
            p.A = A;
            p.mode = MODE_RELAX;
            p.x = snap.as<double>();
            p.b = b;
            p.xe = x;
            p.y = x;
            p.nrows = N;
            p.F = &F;
            p.omega = cfg.omega;
            launch_rowpass(ctx, p);
            break;
        }
        case LDGMG_COLOURED_GS: {
            for (int ci = 0; ci < ncolours; ++ci) {
                const int c = sweep == LDGMG_SWEEP_FORWARD ? ci : ncolours - 1 - ci;
                RowPass p;
                p.A = A;
                p.mode = MODE_RELAX;
                p.x = x;
                p.b = b;
                p.xe = x;
                p.y = x;
                p.rows = colour_rows.as<int>() + colour_ptr[c];
                p.nrows = colour_ptr[c + 1] - colour_ptr[c];
                p.F = &F;
                p.omega = 1.0;
                launch_rowpass(ctx, p);
            }
            break;
        }
        case LDGMG_PROC_BLOCK_GS: {
            LDGMG_CUDA(cudaMemcpyAsync(snap.p, x, sizeof(double) * size_t(N) * bs,
                                       cudaMemcpyDeviceToDevice, ctx.stream));
            const int d = sweep == LDGMG_SWEEP_FORWARD ? 0 : 1;
            for (size_t l = 0; l + 1 < sched_ptr[d].size(); ++l) {
                RowPass p;
                p.A = A;
                p.mode = MODE_RELAX;
                p.x = x;
                p.x_alt = snap.as<double>();
                p.part = part.as<int>();
                p.b = b;
                p.xe = x;
                p.y = x;
                p.rows = sched_rows[d].as<int>() + sched_ptr[d][l];
                p.nrows = sched_ptr[d][l + 1] - sched_ptr[d][l];
                p.F = &F;
                p.omega = cfg.omega;
                launch_rowpass(ctx, p);
            }
            break;
        }
        case LDGMG_SAI: {
            const double* r = r_in ? r_in : snap.as<double>();
            if (!r_ready && !r_in) {
                RowPass p;
                p.A = A;
                p.mode = MODE_RESIDUAL;
                p.x = x;
                p.b = b;
                p.y = snap.as<double>();
                p.nrows = N;
                launch_rowpass(ctx, p);
            }
            RowPass q;
            q.A = sweep == LDGMG_SWEEP_FORWARD ? B.get() : &bsr_transpose_for_sweep(ctx, *B);
            q.mode = MODE_ADD;
            q.x = r;
            q.xe = x;
            q.y = x;
            q.nrows = N;
            launch_rowpass(ctx, q);
            break;
        }
        default:
            fail(LDGMG_ERR_INVALID_ARGUMENT, "Smoother: unsupported kind");
    }
}

void Smoother::apply_sweeps(Ctx& ctx, const double* b, double* x, int sweep, int nu, bool r_ready,
                            bool x_zero) const {
    if (cfg.kind != LDGMG_JACOBI || nu < 1) {
        // SAI from x = 0 (the coarse levels' pre-smoothing): the first
        // residual b - A 0 is b bit for bit (every block product is +0 and
        // b - (+0) = b), so the sweep reads b instead of a residual pass
        const double* r0 = x_zero && cfg.kind == LDGMG_SAI ? b : nullptr;
        for (int i = 0; i < nu; ++i) apply(ctx, b, x, sweep, r_ready && i == 0, i == 0 ? r0 : nullptr);
        return;
    }
    // Jacobi: ping-pong between x and the snapshot buffer instead of copying
    // x before every sweep -- the relax pass reads every input (neighbours
    // and x_e) from `src` and writes `dst`, exactly the reference's sweep
    // from a snapshot (smoothers.hpp:411-416), so the bits are unchanged; an
    // odd count ends with one copy back.
    double* bufs[2] = {x, snap.as<double>()};
    for (int i = 0; i < nu; ++i) {
        RowPass p;
        p.A = A;
        p.mode = MODE_RELAX;
        p.x = bufs[i & 1];
        p.b = b;
        p.xe = bufs[i & 1];
        p.y = bufs[(i + 1) & 1];
        p.nrows = N;
        p.F = &F;
        p.omega = cfg.omega;
        launch_rowpass(ctx, p);
    }
    if (nu & 1)
        LDGMG_CUDA(cudaMemcpyAsync(x, snap.p, sizeof(double) * size_t(N) * bs, cudaMemcpyDeviceToDevice, ctx.stream));
}

double Smoother::bytes_per_apply() const {
    const double W = 8.0;
    const double nb = double(A->nnzb);
    if (cfg.kind == LDGMG_SAI) return W * (double(bs) * bs * (nb + double(B->nnzb)) + 6.0 * N * bs);
    const double sweep = W * (double(bs) * bs * (nb - N) + (double(bs) * bs + 2.0 * bs) * N + 3.0 * N * bs);
    return sweep;
}

// --------------------------------------------------------------- transfer
std::unique_ptr<Transfer> transfer_create(Ctx& ctx, int n_fine, int n_coarse, const int* parent_of,
                                          const int* orthant_of, int dim, int bss, int ncomp,
                                          const double* K) {
    require(n_fine >= 0 && n_coarse >= 0 && bss > 0 && ncomp > 0, "transfer: bad shape");
    require(dim == 2 || dim == 3, "transfer: dim must be 2 or 3");
    auto T = std::make_unique<Transfer>();
    T->n_fine = n_fine;
    T->n_coarse = n_coarse;
    T->dim = dim;
    T->bss = bss;
    T->ncomp = ncomp;
    T->bs = bss * ncomp;
    T->hparent.assign(parent_of, parent_of + n_fine);
    T->horth.assign(orthant_of, orthant_of + n_fine);
    std::vector<int> cptr(n_coarse + 1, 0), clist(n_fine);
    for (int f = 0; f < n_fine; ++f) {
        require(parent_of[f] >= 0 && parent_of[f] < n_coarse, "transfer: parent out of range");
        require(orthant_of[f] >= -1 && orthant_of[f] < (1 << dim), "transfer: orthant out of range");
        ++cptr[parent_of[f] + 1];
    }
    for (int p = 0; p < n_coarse; ++p) cptr[p + 1] += cptr[p];
    std::vector<int> fill(cptr.begin(), cptr.end() - 1);
    for (int f = 0; f < n_fine; ++f) clist[fill[parent_of[f]]++] = f;  // ascending f per parent
    for (int p = 0; p < n_coarse; ++p) T->max_children = std::max(T->max_children, cptr[p + 1] - cptr[p]);
    const size_t nk = size_t(1) << dim;
    T->parent.alloc(sizeof(int) * std::max(1, n_fine));
    T->orth.alloc(sizeof(int) * std::max(1, n_fine));
    T->child_ptr.alloc(sizeof(int) * (n_coarse + 1));
    T->child_list.alloc(sizeof(int) * std::max(1, n_fine));
    T->K.alloc(sizeof(double) * nk * bss * bss);
    h2d(ctx, T->parent.p, parent_of, sizeof(int) * n_fine);
    h2d(ctx, T->orth.p, orthant_of, sizeof(int) * n_fine);
    h2d(ctx, T->child_ptr.p, cptr.data(), sizeof(int) * cptr.size());
    h2d(ctx, T->child_list.p, clist.data(), sizeof(int) * n_fine);
    h2d(ctx, T->K.p, K, T->K.bytes);
    {
        const int nc = 1 << dim;
        bool reg = n_fine == n_coarse * nc;
        for (int f = 0; reg && f < n_fine; ++f) reg = parent_of[f] == f / nc && orthant_of[f] == f % nc;
        T->regular = reg;
    }
    std::vector<int> corth(n_fine);
    for (int q = 0; q < n_fine; ++q) corth[q] = orthant_of[clist[q]];
    T->child_orth.alloc(sizeof(int) * std::max(1, n_fine));
    h2d(ctx, T->child_orth.p, corth.data(), sizeof(int) * n_fine);
    std::vector<double> Kt(nk * bss * bss);
    for (size_t o = 0; o < nk; ++o)
        for (int i = 0; i < bss; ++i)
            for (int j = 0; j < bss; ++j)
                Kt[o * bss * bss + size_t(j) * bss + i] = K[o * bss * bss + size_t(i) * bss + j];
    T->Kt.alloc(sizeof(double) * Kt.size());
    h2d(ctx, T->Kt.p, Kt.data(), T->Kt.bytes);
    return T;
}

// -------------------------------------------------------------- multigrid
void Mg::init(Ctx& ctx) {
    require(depth >= 1, "multigrid: empty hierarchy");
    require(cfg.nu1 >= 0 && cfg.nu2 >= 0, "multigrid: smoothing counts must be nonnegative");
    if (depth < cfg.min_depth)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "multigrid: hierarchy depth below the configured minimum");
    if (A.back()->brows > cfg.bottom_max_elements)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "multigrid: bottom level exceeds the element budget");
    bs = A[0]->rbs;
    for (int l = 0; l < depth; ++l) {
        if (A[l]->rbs != bs || A[l]->cbs != bs || A[l]->brows != A[l]->bcols)
            fail(LDGMG_ERR_INVALID_ARGUMENT, "multigrid: level assembler changed the discretization");
        // check_level (multigrid.hpp:201-204): every stored (i, j) has a stored (j, i)
        const Bsr& L = *A[l];
        for (int i = 0; i < L.brows; ++i)
            for (int k = L.hptr[i]; k < L.hptr[i + 1]; ++k) {
                const int j = L.hcol[k];
                const int* b0 = L.hcol.data() + L.hptr[j];
                const int* b1 = L.hcol.data() + L.hptr[j + 1];
                if (std::find(b0, b1, i) == b1)
                    fail(LDGMG_ERR_INVALID_ARGUMENT, "multigrid: level operator pattern not symmetric");
            }
        if (l + 1 < depth) {
            require(T[l] != nullptr, "multigrid: missing transfer");
            require(T[l]->n_fine == A[l]->brows && T[l]->n_coarse == A[l + 1]->brows && T[l]->bs == bs,
                    "multigrid: transfer shape mismatch");
        }
    }
    // level buffers: r[l] fine residual, x/b for coarse levels
    r.resize(depth);
    xl.resize(depth);
    bl.resize(depth);
    for (int l = 0; l < depth; ++l) {
        const size_t n = sizeof(double) * std::max<int64_t>(1, int64_t(A[l]->brows) * bs);
        r[l].alloc(n);
        if (l > 0) {
            xl[l].alloc(n);
            bl[l].alloc(n);
        }
    }
    bp.alloc(sizeof(double) * std::max<int64_t>(1, int64_t(A[0]->brows) * bs));
    // kernel vectors (ldg_core.hpp:64-78): constant mode 0 of each component
    std::vector<int> offs;
    if (kernel_constants)
        for (int c = 0; c < (system_kind == LDGMG_SYSTEM_SCALAR ? 1 : dim); ++c) offs.push_back(c * bs_scalar);
    if (kernel_pressure) offs.push_back(dim * bs_scalar);
    nkernel = int(offs.size());
    kernel_offsets_host = offs;
    kernel_offs.alloc(sizeof(int) * std::max<size_t>(1, offs.size()));
    if (!offs.empty())
        h2d(ctx, kernel_offs.p, offs.data(), sizeof(int) * offs.size());
    kval = 1.0 / std::sqrt(double(A[0]->brows));
    red.alloc(sizeof(double) * 1024);
    LDGMG_CUDA(cudaMallocHost(&h_red, sizeof(double) * 4));
    (void)ctx;
}

/// Dense symmetric eigensolve of a LARGE bottom operator at setup time
/// (cuSOLVER dsyevd on the device; the host tred2/tql2 takes ~19 s at
/// n = 2916).  Same contract as sym_eig_host: eigenvalues ascending,
/// eigenvectors as the columns of V (column-major).  Setup only.
void sym_eig_device(Ctx& ctx, int n, const double* A, double* lambda, double* V) {
    cusolverDnHandle_t h = nullptr;
    auto ck = [](cusolverStatus_t st, const char* what) {
        if (st != CUSOLVER_STATUS_SUCCESS) fail(LDGMG_ERR_RUNTIME, std::string("sym_eig: ") + what + " failed");
    };
    ck(cusolverDnCreate(&h), "cusolverDnCreate");
    struct Guard {
        cusolverDnHandle_t h;
        ~Guard() { cusolverDnDestroy(h); }
    } guard{h};
    ck(cusolverDnSetStream(h, ctx.stream), "cusolverDnSetStream");
    DevBuf dA(sizeof(double) * size_t(n) * n), dW(sizeof(double) * n), dinfo(sizeof(int));
    h2d(ctx, dA.p, A, dA.bytes);
    int lwork = 0;
    ck(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA.as<double>(), n,
                                   dW.as<double>(), &lwork),
       "dsyevd_bufferSize");
    DevBuf work(sizeof(double) * std::max(1, lwork));
    ck(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA.as<double>(), n, dW.as<double>(),
                        work.as<double>(), lwork, dinfo.as<int>()),
       "dsyevd");
    int info = 0;
    d2h(ctx, &info, dinfo.p, sizeof(int));
    if (info != 0) fail(LDGMG_ERR_RUNTIME, "sym_eig: eigensolver failed");
    d2h(ctx, lambda, dW.p, sizeof(double) * n);
    d2h(ctx, V, dA.p, dA.bytes);
}

void Mg::set_bottom(Ctx& ctx, const double* V, const double* lambda) {
    const Bsr& Ab = *A.back();
    const int n = Ab.brows * bs;
    std::vector<double> Vc(size_t(n) * n), lam(n);
    if (V && lambda) {
        std::memcpy(Vc.data(), V, sizeof(double) * Vc.size());
        std::memcpy(lam.data(), lambda, sizeof(double) * n);
    } else {
        // dense bottom operator (to_dense, blockla.hpp:241-251), eig on host
        std::vector<double> vals(size_t(Ab.nnzb) * bs * bs), D(size_t(n) * n, 0.0);
        bsr_download(ctx, Ab, nullptr, nullptr, vals.data());
        for (int i = 0; i < Ab.brows; ++i)
            for (int k = Ab.hptr[i]; k < Ab.hptr[i + 1]; ++k)
                for (int rr = 0; rr < bs; ++rr)
                    for (int c = 0; c < bs; ++c)
                        D[size_t(Ab.hcol[k] * bs + c) * n + size_t(i) * bs + rr] =
                            vals[size_t(k) * bs * bs + size_t(rr) * bs + c];
        double nrm = 0.0, asym = 0.0;
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                nrm += D[size_t(j) * n + i] * D[size_t(j) * n + i];
                const double t = D[size_t(j) * n + i] - D[size_t(i) * n + j];
                asym += t * t;
            }
        if (std::sqrt(asym) > 1e-13 * std::max(1e-300, std::sqrt(nrm)))
            fail(LDGMG_ERR_INVALID_ARGUMENT, "sym_eig: matrix is not symmetric");
        static const int gpu_min = getenv("LDGMG_GPU_EIG_MIN") ? atoi(getenv("LDGMG_GPU_EIG_MIN")) : 1024;
        if (n >= gpu_min && gpu_min >= 0)
            sym_eig_device(ctx, n, D.data(), lam.data(), Vc.data());  // large bottoms (C5 48^3: n = 2916)
        else
            sym_eig_host(n, D.data(), lam.data(), Vc.data());
    }
    std::vector<double> Vr(size_t(n) * n);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) Vr[size_t(i) * n + k] = Vc[size_t(k) * n + i];
    bottom.n = n;
    bottom.lmax = 0.0;
    for (double l : lam) bottom.lmax = std::max(bottom.lmax, std::abs(l));
    // +2: tail padding for the even-sized bulk copies of pinv_stream_kernel
    bottom.Vc.alloc(sizeof(double) * (Vc.size() + 2));
    bottom.Vr.alloc(sizeof(double) * (Vr.size() + 2));
    bottom.lambda.alloc(sizeof(double) * std::max(1, n));
    bottom.t.alloc(sizeof(double) * std::max(1, n));
    h2d(ctx, bottom.Vc.p, Vc.data(), sizeof(double) * Vc.size());
    h2d(ctx, bottom.Vr.p, Vr.data(), sizeof(double) * Vr.size());
    h2d(ctx, bottom.lambda.p, lam.data(), sizeof(double) * n);
}

void Mg::v_cycle(Ctx& ctx, int l, double* x, const double* b, bool r0_ready) {
    if (l + 1 == depth) {
        launch_pinv_apply(ctx, bottom, cfg.bottom_tol, b, x);
        return;
    }
    const Smoother& S = *sm[l];
    // coarse levels start from x = 0 (zeroed by the restriction)
    S.apply_sweeps(ctx, b, x, cfg.pre, cfg.nu1, r0_ready, l > 0 && x == xl[l].as<double>());
    RowPass p;
    p.A = A[l];
    p.mode = MODE_RESIDUAL;
    p.x = x;
    p.b = b;
    p.y = r[l].as<double>();
    p.nrows = A[l]->brows;
    launch_rowpass(ctx, p);
    launch_restrict(ctx, *T[l], r[l].as<double>(), bl[l + 1].as<double>(), xl[l + 1].as<double>());
    v_cycle(ctx, l + 1, xl[l + 1].as<double>(), bl[l + 1].as<double>());
    launch_prolong_add(ctx, *T[l], xl[l + 1].as<double>(), x);
    S.apply_sweeps(ctx, b, x, cfg.post, cfg.nu2);
}

void Mg::project(Ctx& ctx, double* v) {
    launch_project_constants(ctx, v, A[0]->brows, bs, kernel_offs.as<int>(), nkernel, kval, strict_order,
                             red.as<double>());
}

double* Mg::r0_buffer() const {
    if (depth < 2 || cfg.nu1 < 1 || sm.empty() || !sm[0] || sm[0]->cfg.kind != LDGMG_SAI) return nullptr;
    return sm[0]->snap.as<double>();
}

void Mg::cycle(Ctx& ctx, double* x, const double* b, bool r0_ready) {
    require(!r0_ready || r0_buffer(), "multigrid: no level-0 residual to start from");
    v_cycle(ctx, 0, x, b, r0_ready);
    project(ctx, x);
}

void Mg::apply(Ctx& ctx, const double* b, double* x) {
    const size_t n = sizeof(double) * size_t(A[0]->brows) * bs;
    LDGMG_CUDA(cudaMemsetAsync(x, 0, n, ctx.stream));
    if (nkernel == 0) {
        v_cycle(ctx, 0, x, b);
        return;
    }
    LDGMG_CUDA(cudaMemcpyAsync(bp.p, b, n, cudaMemcpyDeviceToDevice, ctx.stream));
    project(ctx, bp.as<double>());
    v_cycle(ctx, 0, x, bp.as<double>());
    project(ctx, x);
}

void Mg::cycles(Ctx& ctx, double* x, const double* b, int n, bool r0_ready) {
    if (n <= 0) return;
    require(n == 1 || !r0_ready, "multigrid: a precomputed residual serves one cycle");
    if (!warm) {  // first run un-captured: sets kernel attributes, lazy transposes
        cycle(ctx, x, b, r0_ready);
        --n;
        warm = true;
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    if (n <= 0) return;
    Graph* G = nullptr;
    for (auto& g : graphs)
        if (g.x == x && g.b == b && g.s == ctx.stream && g.r0 == r0_ready) G = &g;
    if (!G) {
        Graph ng{x, b, ctx.stream, nullptr, 0, r0_ready};
        cudaGraph_t graph;
        const int64_t c0 = launch_counter().load();
        // capture on a private non-blocking stream (the context stream may be
        // the legacy default stream, which cannot be captured)
        if (!cap_stream) LDGMG_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
        LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
        Ctx cctx = ctx;
        cctx.stream = cap_stream;
        LDGMG_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
        try {
            cycle(cctx, x, b, r0_ready);
        } catch (...) {
            // leave the capture stream usable: end (and drop) the partial capture
            cudaGraph_t partial = nullptr;
            cudaStreamEndCapture(cap_stream, &partial);
            if (partial) cudaGraphDestroy(partial);
            cudaGetLastError();
            launch_counter().fetch_sub(launch_counter().load() - c0);
            throw;
        }
        LDGMG_CUDA(cudaStreamEndCapture(cap_stream, &graph));
        // captured launches did not run; they are counted per graph launch
        ng.nkernels = launch_counter().load() - c0;
        launch_counter().fetch_sub(ng.nkernels);
        LDGMG_CUDA(cudaGraphInstantiate(&ng.exec, graph, 0));
        LDGMG_CUDA(cudaGraphDestroy(graph));
        graphs.push_back(ng);
        G = &graphs.back();
    }
    for (int i = 0; i < n; ++i) {
        LDGMG_CUDA(cudaGraphLaunch(G->exec, ctx.stream));
        launch_counter().fetch_add(G->nkernels, std::memory_order_relaxed);
    }
}

void Mg::invalidate_graphs() {
    // the next cycles() runs un-captured once more: a new smoother may need
    // lazy setup (B^T views, kernel attributes) that cannot run under capture
    warm = false;
    for (auto& gr : graphs) cudaGraphExecDestroy(gr.exec);
    graphs.clear();
    if (solve_exec) cudaGraphExecDestroy(solve_exec);
    solve_exec = nullptr;
}

double Mg::dof_updates_per_cycle() const {
    double s = 0.0;
    for (int l = 0; l + 1 < depth; ++l) s += double(cfg.nu1 + cfg.nu2) * A[l]->brows * bs;
    return s;
}

double Mg::bytes_per_cycle() const {
    const double W = 8.0;
    double s = 0.0;
    for (int l = 0; l + 1 < depth; ++l) {
        const double N = A[l]->brows, Nc = A[l + 1]->brows;
        s += double(cfg.nu1 + cfg.nu2) * sm[l]->bytes_per_apply();
        if (l > 0 && cfg.nu1 > 0 && sm[l]->cfg.kind == LDGMG_SAI)  // first coarse sweep from x = 0: no residual pass
            s -= W * (double(bs) * bs * double(A[l]->nnzb) + 3.0 * bs * N);
        s += W * (double(bs) * bs * double(A[l]->nnzb) + 3.0 * bs * N);  // residual
        s += W * (bs * N + bs * Nc) + W * (bs * Nc + 2.0 * bs * N);      // transfers
    }
    s += W * 2.0 * double(bottom.n) * bottom.n;
    return s;
}

Mg::~Mg() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (h_red) cudaFreeHost(h_red);
    if (h_stage) cudaFreeHost(h_stage);
    if (h_stage_x) cudaFreeHost(h_stage_x);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    if (ev_snap) cudaEventDestroy(ev_snap);
    if (ev_d2h) cudaEventDestroy(ev_d2h);
    if (solve_exec) cudaGraphExecDestroy(solve_exec);
    if (cap_side) cudaStreamDestroy(cap_side);
    for (auto e : cap_ev)
        if (e) cudaEventDestroy(e);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (sai_cache) sai_cache_free(sai_cache);
}

}  // namespace ldgmg_b200
