// TEST INFRASTRUCTURE -- the CPU oracle.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load the library this
// file builds (oracle/_ref/libldgmg_ref.so).  It is never part of the product.
//
// A thin C API over the UNMODIFIED reference headers (/root/reference/proj/
// include/ldgmg, compiled in place by oracle/Makefile against oracle/shim).
// Every entry point forwards to the reference function it names; the only
// logic added here is
//   * the problem catalogue glue (the harness' assembler lambdas,
//     harness.hpp:74-98) plus extension A2 (curved phases re-tested on every
//     level), applied identically in the product setup;
//   * re-derivations of three PRIVATE Multigrid/Smoother members from the
//     same public reference functions the class uses: the per-element
//     diagonal factors (smoothers.hpp:464-494 -> sym_eig), the coarsening
//     maps (multigrid.hpp:168-189 -> coarsen) and the injection matrices
//     (probed through the public interpolate_add, multigrid.hpp:104-123).
#include <ldgmg/krylov.hpp>
#include <ldgmg/ldg_scalar.hpp>
#include <ldgmg/ldg_stokes.hpp>
#include <ldgmg/multigrid.hpp>

#include "../include/ldgmg_b200.h"

#include <chrono>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <atomic>
#include <thread>

using namespace ldgmg;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return LDGMG_ERR_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return LDGMG_ERR_LOGIC;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return LDGMG_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LDGMG_ERR_RUNTIME;
    }
}

BoundaryKind bc_of(int k) {
    switch (k) {
        case LDGMG_BC_PERIODIC: return BoundaryKind::Periodic;
        case LDGMG_BC_DIRICHLET: return BoundaryKind::Dirichlet;
        case LDGMG_BC_NEUMANN: return BoundaryKind::Neumann;
    }
    throw std::invalid_argument("ref: unknown boundary kind");
}

SmootherConfig smoother_of(const ldgmg_smoother_config& c) {
    SmootherConfig s;
    s.kind = static_cast<SmootherKind>(c.kind);
    s.omega = c.omega;
    s.partitions = c.partitions;
    s.level = c.level;
    s.zeta = c.zeta;
    s.cache = c.cache != 0;
    return s;
}

MultigridConfig mg_of(const ldgmg_mg_config& c) {
    MultigridConfig m;
    m.smoother = smoother_of(c.smoother);
    m.pre = c.pre == LDGMG_SWEEP_FORWARD ? Sweep::Forward : Sweep::Reverse;
    m.post = c.post == LDGMG_SWEEP_FORWARD ? Sweep::Forward : Sweep::Reverse;
    m.nu1 = c.nu1;
    m.nu2 = c.nu2;
    m.bottom_max_elements = c.bottom_max_elements;
    m.bottom_tol = c.bottom_tol;
    m.min_depth = c.min_depth;
    return m;
}

bool inside_curved(const ldgmg_problem_spec& s, const Element& e, int dim) {
    double acc = 0.0;
    for (int a = 0; a < dim; ++a) {
        const double c = 0.5 * (e.lo(a) + e.hi(a));
        const double r = s.phase_shape == LDGMG_PHASE_BALL ? s.radii[0] : s.radii[a];
        const double t = (c - s.center[a]) / r;
        acc += t * t;
    }
    return acc < 1.0;
}

/// Problem glue: fine mesh + per-level assembler (harness.hpp:74-98 shape).
struct Built {
    Mesh mesh;
    LevelAssembler assemble;
};

Built build(const ldgmg_problem_spec& s) {
    std::array<BoundaryKind, 6> bc{};
    for (int i = 0; i < 6; ++i) bc[i] = bc_of(s.bc[i]);
    Built out;
    out.mesh = build_uniform(s.n, s.dim, bc);
    PhaseGeometry geom = PhaseGeometry::single(s.mu_out, s.rho_out);
    const bool curved = s.phase_shape == LDGMG_PHASE_BALL || s.phase_shape == LDGMG_PHASE_ELLIPSE;
    if (s.phase_shape == LDGMG_PHASE_BOXES) {
        geom.regions.clear();
        geom.regions.push_back({{s.center[0], s.center[1], s.center[2]},
                                {s.radii[0], s.radii[1], s.radii[2]}, s.mu_in, s.rho_in});
        geom.regions.push_back({{0, 0, 0}, {1, 1, 1}, s.mu_out, s.rho_out});
        assign_phases(out.mesh, geom);
    }
    const ldgmg_problem_spec spec = s;
    out.assemble = [spec, geom, curved](const Mesh& m0) -> System {
        Mesh m = m0;
        PhaseGeometry g = geom;
        if (curved) {
            // Extension A2: phase by centroid test on this level's mesh.
            bool any_in = false, any_out = false;
            for (const Element& e : m.elements)
                (inside_curved(spec, e, m.dim) ? any_in : any_out) = true;
            g.regions.clear();
            if (any_in) g.regions.push_back({{0, 0, 0}, {1, 1, 1}, spec.mu_in, spec.rho_in});
            if (any_out) g.regions.push_back({{0, 0, 0}, {1, 1, 1}, spec.mu_out, spec.rho_out});
            for (Element& e : m.elements)
                e.phase = (inside_curved(spec, e, m.dim) || !any_out) ? 0 : (any_in ? 1 : 0);
            m.n_phases = (int)g.regions.size();
        }
        if (spec.kind == LDGMG_SYSTEM_SCALAR) {
            ScalarProblem P;
            P.mesh = m;
            P.phases = g;
            P.degree = spec.degree;
            P.beta = spec.beta;
            return assemble_scalar(P);
        }
        StokesProblem P;
        P.mesh = m;
        P.phases = g;
        P.degree = spec.degree;
        P.gamma = spec.gamma;
        P.beta = spec.beta;
        P.beta_p = spec.beta_p;
        P.delta = spec.delta;
        return assemble_stokes(P);
    };
    return out;
}

struct RefMg {
    ldgmg_problem_spec spec;
    Built built;
    std::unique_ptr<Multigrid> mg;
};

void copy_csr(const BlockCsr& A, int* ptr, int* col, double* val) {
    if (ptr) std::memcpy(ptr, A.ptr.data(), sizeof(int) * A.ptr.size());
    if (col) std::memcpy(col, A.col.data(), sizeof(int) * A.col.size());
    if (val) std::memcpy(val, A.val.data(), sizeof(double) * A.val.size());
}

BlockVec vec_in(const double* p, int n, int bs) {
    BlockVec v(n, bs);
    std::memcpy(v.data.data(), p, sizeof(double) * v.data.size());
    return v;
}

BlockCsr csr_in(int brows, int bcols, int rbs, int cbs, const int* ptr, const int* col,
                const double* val) {
    BlockCsr A;
    A.brows = brows;
    A.bcols = bcols;
    A.row_bs = rbs;
    A.col_bs = cbs;
    A.ptr.assign(ptr, ptr + brows + 1);
    A.col.assign(col, col + A.ptr[brows]);
    A.val.assign(val, val + size_t(A.ptr[brows]) * rbs * cbs);
    return A;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_mg_create(const ldgmg_problem_spec* spec, const ldgmg_mg_config* cfg) {
    RefMg* h = nullptr;
    const int rc = guard([&] {
        auto r = std::make_unique<RefMg>();
        r->spec = *spec;
        r->built = build(*spec);
        r->mg = std::make_unique<Multigrid>(r->built.mesh, r->built.assemble, mg_of(*cfg));
        h = r.release();
    });
    return rc == 0 ? h : nullptr;
}

void ref_mg_destroy(void* h) { delete static_cast<RefMg*>(h); }

/// A least-squares cache shared across hierarchies (MultigridConfig::cache,
/// multigrid.hpp:35): the reference's own way of building several
/// hierarchies of one problem without repeating the SAI solves.
void* ref_cache_new(void) { return new SaiCache(); }
void ref_cache_free(void* c) { delete static_cast<SaiCache*>(c); }
long long ref_cache_entries(void* c) { return (long long)static_cast<SaiCache*>(c)->entries(); }

void* ref_mg_create_shared(const ldgmg_problem_spec* spec, const ldgmg_mg_config* cfg, void* cache) {
    RefMg* h = nullptr;
    const int rc = guard([&] {
        auto r = std::make_unique<RefMg>();
        r->spec = *spec;
        r->built = build(*spec);
        MultigridConfig mc = mg_of(*cfg);
        mc.cache = static_cast<SaiCache*>(cache);
        r->mg = std::make_unique<Multigrid>(r->built.mesh, r->built.assemble, mc);
        h = r.release();
    });
    return rc == 0 ? h : nullptr;
}

/// `ncycles` Multigrid::cycle calls on each of `nh` INDEPENDENT hierarchies,
/// hierarchy i on its own thread with its own x (the reference's run_cells
/// parallelism, harness.hpp:305-327: each cell owns its hierarchy).  Wall
/// seconds from the common start to the last thread's end.
int ref_cycles_multi(void* const* hs, int nh, const double* b, int ncycles, double* seconds) {
    return guard([&] {
        if (nh < 1) throw std::invalid_argument("ref_cycles_multi: no hierarchies");
        const System& S = static_cast<RefMg*>(hs[0])->mg->system(0);
        const BlockVec bv = vec_in(b, S.n_elements(), S.block_size());
        std::atomic<int> ready{0};
        std::atomic<bool> go{false};
        std::chrono::steady_clock::time_point t0;
        std::vector<std::thread> pool;
        std::vector<std::string> errs(nh);
        for (int t = 0; t < nh; ++t)
            pool.emplace_back([&, t] {
                try {
                    const Multigrid& mg = *static_cast<RefMg*>(hs[t])->mg;
                    BlockVec x(S.n_elements(), S.block_size());
                    ready.fetch_add(1);
                    while (!go.load()) std::this_thread::yield();
                    for (int c = 0; c < ncycles; ++c) mg.cycle(x, bv);
                } catch (const std::exception& e) {
                    errs[t] = e.what();
                }
            });
        while (ready.load() < nh) std::this_thread::yield();
        t0 = std::chrono::steady_clock::now();
        go.store(true);
        for (auto& th : pool) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

int ref_mg_depth(void* h) { return static_cast<RefMg*>(h)->mg->depth(); }

int ref_level_shape(void* h, int lvl, int* N, int* bs, long long* nnzb) {
    return guard([&] {
        const System& S = static_cast<RefMg*>(h)->mg->system(lvl);
        *N = S.n_elements();
        *bs = S.block_size();
        *nnzb = (long long)S.A.col.size();
    });
}

int ref_level_matrix(void* h, int lvl, int* ptr, int* col, double* val) {
    return guard([&] { copy_csr(static_cast<RefMg*>(h)->mg->system(lvl).A, ptr, col, val); });
}

int ref_level_rhs(void* h, int lvl, double* b) {
    return guard([&] {
        const System& S = static_cast<RefMg*>(h)->mg->system(lvl);
        std::memcpy(b, S.b.data.data(), sizeof(double) * S.b.data.size());
    });
}

int ref_system_info(void* h, int* dim, int* ncomp, int* bs_scalar, int* kc, int* kp,
                    int* nvel) {
    return guard([&] {
        const System& S = static_cast<RefMg*>(h)->mg->system(0);
        *dim = S.dim;
        *ncomp = S.n_comp;
        *bs_scalar = S.bs_scalar;
        *kc = S.kernel_constants;
        *kp = S.kernel_pressure;
        *nvel = S.n_velocity();
    });
}

/// parent_of / orthant_of of level lvl -> lvl+1: the same coarsen() call the
/// hierarchy made (multigrid.hpp:175, deterministic).
int ref_level_transfer(void* h, int lvl, int* parent, int* orth) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        if (lvl + 1 >= mg.depth()) throw std::invalid_argument("ref: bottom level has no transfer");
        const Coarsening c = coarsen(mg.mesh(lvl));
        std::memcpy(parent, c.parent_of.data(), sizeof(int) * c.parent_of.size());
        std::memcpy(orth, c.orthant_of.data(), sizeof(int) * c.orthant_of.size());
    });
}

/// Injection matrices K_o (row-major bs_scalar^2 each, 2^dim of them), read
/// back column by column through the public interpolate_add on level 0.
int ref_injection(void* h, double* K) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        if (mg.depth() < 2) throw std::invalid_argument("ref: need two levels to probe injection");
        const System& S0 = mg.system(0);
        const System& S1 = mg.system(1);
        const int bs = S0.bs_scalar, BS = S0.block_size(), nch = 1 << S0.dim;
        const Coarsening c = coarsen(mg.mesh(0));
        for (int j = 0; j < bs; ++j) {
            BlockVec xc(S1.n_elements(), BS), xf(S0.n_elements(), BS);
            xc.block(0)[j] = 1.0;
            mg.interpolate_add(0, xc, xf);
            for (int f = 0; f < S0.n_elements(); ++f) {
                if (c.parent_of[f] != 0) continue;
                const int o = c.orthant_of[f];
                for (int i = 0; i < bs; ++i) K[(size_t(o) * bs + i) * bs + j] = xf.block(f)[i];
            }
        }
        (void)nch;
    });
}

/// Per-element diagonal factors exactly as Smoother::factor_diagonal
/// (smoothers.hpp:464-494) computes them: V column-major bs*bs, lambda, s.
int ref_diag_factors(void* h, int lvl, double* V, double* lam, double* sc) {
    return guard([&] {
        const System& S = static_cast<RefMg*>(h)->mg->system(lvl);
        const int N = S.n_elements(), bs = S.block_size();
        Eigen::MatrixXd D(bs, bs);
        for (int e = 0; e < N; ++e) {
            const int k = S.A.find(e, e);
            if (k < 0) throw std::runtime_error("Smoother: missing diagonal block");
            const double* v = S.A.block(k);
            for (int i = 0; i < bs; ++i)
                for (int j = 0; j < bs; ++j) D(i, j) = v[i * bs + j];
            Eigen::VectorXd s(bs);
            for (int i = 0; i < bs; ++i) {
                const double d = std::abs(D(i, i));
                if (d > 0.0) {
                    int ex = 0;
                    std::frexp(d, &ex);
                    s[i] = std::ldexp(1.0, -(ex / 2));
                } else {
                    s[i] = 1.0;
                }
            }
            const SymEig eig = sym_eig(s.asDiagonal() * D * s.asDiagonal());
            std::memcpy(V + size_t(e) * bs * bs, eig.V.data(), sizeof(double) * bs * bs);
            std::memcpy(lam + size_t(e) * bs, eig.lambda.data(), sizeof(double) * bs);
            std::memcpy(sc + size_t(e) * bs, s.data(), sizeof(double) * bs);
        }
    });
}

int ref_colours(void* h, int lvl, int* colour, int* ncol) {
    return guard([&] {
        const Smoother& sm = static_cast<RefMg*>(h)->mg->smoother(lvl);
        const auto& c = sm.colours();
        if (colour) std::memcpy(colour, c.data(), sizeof(int) * c.size());
        *ncol = sm.n_colours();
    });
}

int ref_sai_nnzb(void* h, int lvl, long long* nnzb) {
    return guard([&] {
        *nnzb = (long long)static_cast<RefMg*>(h)->mg->smoother(lvl).sai_matrix().col.size();
    });
}

int ref_sai_matrix(void* h, int lvl, int* ptr, int* col, double* val) {
    return guard(
        [&] { copy_csr(static_cast<RefMg*>(h)->mg->smoother(lvl).sai_matrix(), ptr, col, val); });
}

static void stats_out(const SaiStats& st, ldgmg_sai_stats* out) {
    std::memset(out, 0, sizeof(*out));
    out->rank_deficient_columns = st.rank_deficient_columns;
    out->cache_hits = (int64_t)st.cache_hits;
    out->cache_misses = (int64_t)st.cache_misses;
    out->n_shapes = (int)st.ls_dims.size();
    int i = 0;
    for (const auto& [shape, count] : st.ls_dims) {
        if (i >= 8) break;
        out->shape_rows[i] = shape.first;
        out->shape_cols[i] = shape.second;
        out->shape_count[i] = count;
        ++i;
    }
}

int ref_sai_stats(void* h, int lvl, ldgmg_sai_stats* out) {
    return guard([&] { stats_out(static_cast<RefMg*>(h)->mg->smoother(lvl).sai_stats(), out); });
}

int ref_bottom_size(void* h) {
    return (int)static_cast<RefMg*>(h)->mg->bottom_eig().lambda.size();
}

int ref_bottom(void* h, double* V, double* lam) {
    return guard([&] {
        const SymEig& e = static_cast<RefMg*>(h)->mg->bottom_eig();
        std::memcpy(V, e.V.data(), sizeof(double) * e.V.size());
        std::memcpy(lam, e.lambda.data(), sizeof(double) * e.lambda.size());
    });
}

int ref_kernel(void* h, int* nk, double* out) {
    return guard([&] {
        const auto k = kernel_basis(static_cast<RefMg*>(h)->mg->system(0));
        *nk = (int)k.size();
        if (out)
            for (size_t i = 0; i < k.size(); ++i)
                std::memcpy(out + i * k[i].size(), k[i].data.data(), sizeof(double) * k[i].size());
    });
}

int ref_spmv(void* h, int lvl, const double* x, double* y, int transpose) {
    return guard([&] {
        const System& S = static_cast<RefMg*>(h)->mg->system(lvl);
        const BlockVec xv = vec_in(x, S.n_elements(), S.block_size());
        BlockVec yv;
        if (transpose)
            spmv_transpose(S.A, xv, yv);
        else
            spmv(S.A, xv, yv);
        std::memcpy(y, yv.data.data(), sizeof(double) * yv.data.size());
    });
}

int ref_smoother_apply(void* h, int lvl, const double* b, double* x, int sweep) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        const System& S = mg.system(lvl);
        const BlockVec bv = vec_in(b, S.n_elements(), S.block_size());
        BlockVec xv = vec_in(x, S.n_elements(), S.block_size());
        mg.smoother(lvl).apply(bv, xv, sweep == LDGMG_SWEEP_FORWARD ? Sweep::Forward : Sweep::Reverse);
        std::memcpy(x, xv.data.data(), sizeof(double) * xv.data.size());
    });
}

int ref_restrict(void* h, int lvl, const double* rf, double* rc) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        const System& S = mg.system(lvl);
        const BlockVec r = vec_in(rf, S.n_elements(), S.block_size());
        const BlockVec c = mg.restrict_residual(lvl, r);
        std::memcpy(rc, c.data.data(), sizeof(double) * c.data.size());
    });
}

int ref_interpolate_add(void* h, int lvl, const double* xc, double* xf) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        const System& Sf = mg.system(lvl);
        const System& Sc = mg.system(lvl + 1);
        const BlockVec c = vec_in(xc, Sc.n_elements(), Sc.block_size());
        BlockVec f = vec_in(xf, Sf.n_elements(), Sf.block_size());
        mg.interpolate_add(lvl, c, f);
        std::memcpy(xf, f.data.data(), sizeof(double) * f.data.size());
    });
}

int ref_cycle(void* h, double* x, const double* b) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        const System& S = mg.system(0);
        const BlockVec bv = vec_in(b, S.n_elements(), S.block_size());
        BlockVec xv = vec_in(x, S.n_elements(), S.block_size());
        mg.cycle(xv, bv);
        std::memcpy(x, xv.data.data(), sizeof(double) * xv.data.size());
    });
}

int ref_apply(void* h, const double* b, double* x) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        const System& S = mg.system(0);
        const BlockVec y = mg.apply(vec_in(b, S.n_elements(), S.block_size()));
        std::memcpy(x, y.data.data(), sizeof(double) * y.data.size());
    });
}

/// Stationary solve (extension A7 protocol): x=0, cycle until
/// ||b-Ax||_2/||b||_2 <= tol; history[k] = relative residual after k cycles.
int ref_solve(void* h, const double* b, double* x, double tol, int maxit, double* history,
              int* iters) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        const System& S = mg.system(0);
        const BlockVec bv = vec_in(b, S.n_elements(), S.block_size());
        BlockVec xv(S.n_elements(), S.block_size());
        const double bn = norm2(bv);
        int it = 0;
        auto relres = [&] {
            BlockVec r = spmv(S.A, xv);
            for (size_t i = 0; i < r.size(); ++i) r.data[i] = bv.data[i] - r.data[i];
            return norm2(r) / bn;
        };
        double rr = relres();
        if (history) history[0] = rr;
        while (rr > tol && it < maxit) {
            mg.cycle(xv, bv);
            ++it;
            rr = relres();
            if (history) history[it] = rr;
        }
        *iters = it;
        std::memcpy(x, xv.data.data(), sizeof(double) * xv.data.size());
    });
}

/// `ncycles` V-cycles on each of `nthreads` independent copies of x (the
/// reference's own run_cells parallelism, harness.hpp:305-327); wall seconds.
int ref_cycles_parallel(void* h, const double* b, int ncycles, int nthreads, double* seconds) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        const System& S = mg.system(0);
        const BlockVec bv = vec_in(b, S.n_elements(), S.block_size());
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t)
            pool.emplace_back([&] {
                BlockVec x(S.n_elements(), S.block_size());
                for (int c = 0; c < ncycles; ++c) mg.cycle(x, bv);
            });
        for (auto& th : pool) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

int ref_random_rhs(int nblocks, int bs, unsigned long long seed, double* out) {
    return guard([&] {
        const BlockVec b = random_rhs(nblocks, bs, seed);
        std::memcpy(out, b.data.data(), sizeof(double) * b.data.size());
    });
}

int ref_eta(void* h, int kind, unsigned long long seed, double tol, int maxit, double* resid,
            int* nres, int* iters, int* converged, double* rho, double* eta) {
    return guard([&] {
        const Multigrid& mg = *static_cast<RefMg*>(h)->mg;
        EtaOptions eo;
        eo.seed = seed;
        eo.tol = tol;
        eo.maxit = maxit;
        const SolveReport rep =
            estimate_eta(mg.system(0), mg, kind == 0 ? KrylovKind::CG : KrylovKind::GMRES, eo);
        *nres = (int)rep.residuals.size();
        if (resid) std::memcpy(resid, rep.residuals.data(), sizeof(double) * rep.residuals.size());
        *iters = rep.iterations;
        *converged = rep.converged;
        *rho = rep.rho;
        *eta = rep.eta;
    });
}

// ---------------------------------------------- raw-matrix entry points
int ref_bsr_spmv(int brows, int bcols, int rbs, int cbs, const int* ptr, const int* col,
                 const double* val, const double* x, double* y, int transpose,
                 unsigned long long* mults) {
    return guard([&] {
        const BlockCsr A = csr_in(brows, bcols, rbs, cbs, ptr, col, val);
        const BlockVec xv = transpose ? vec_in(x, brows, rbs) : vec_in(x, bcols, cbs);
        BlockVec yv;
        block_mult_counter() = 0;
        if (transpose)
            spmv_transpose(A, xv, yv);
        else
            spmv(A, xv, yv);
        if (mults) *mults = block_mult_counter();
        std::memcpy(y, yv.data.data(), sizeof(double) * yv.data.size());
    });
}

/// dump_block_coo (blockla.hpp:253-268) of a raw matrix to `path`.
int ref_dump_block_coo(int brows, int bcols, int rbs, int cbs, const int* ptr, const int* col,
                       const double* val, const char* path) {
    return guard([&] {
        const BlockCsr A = csr_in(brows, bcols, rbs, cbs, ptr, col, val);
        std::ofstream os(path);
        if (!os) throw std::runtime_error("ref_dump_block_coo: cannot open output");
        dump_block_coo(A, os);
    });
}

int ref_pattern_power_nnz(int n, const int* ptr, const int* col, int level, long long* nnz) {
    return guard([&] {
        std::vector<double> val(static_cast<size_t>(ptr[n]), 1.0);
        const BlockCsr A = csr_in(n, n, 1, 1, ptr, col, val.data());
        const BlockPattern P = pattern_power(A, level);
        long long s = 0;
        for (const auto& r : P.rows) s += (long long)r.size();
        *nnz = s;
    });
}

int ref_pattern_power(int n, const int* ptr, const int* col, int level, int* pptr, int* pcol) {
    return guard([&] {
        std::vector<double> val(static_cast<size_t>(ptr[n]), 1.0);
        const BlockCsr A = csr_in(n, n, 1, 1, ptr, col, val.data());
        const BlockPattern P = pattern_power(A, level);
        pptr[0] = 0;
        for (int i = 0; i < n; ++i) {
            std::memcpy(pcol + pptr[i], P.rows[i].data(), sizeof(int) * P.rows[i].size());
            pptr[i + 1] = pptr[i] + (int)P.rows[i].size();
        }
    });
}

int ref_dense_lstsq(int m, int n, int nrhs, const double* M, const double* rhs, double* X,
                    int* deficient) {
    return guard([&] {
        Eigen::MatrixXd Mm(m, n), R(m, nrhs);
        std::memcpy(Mm.data(), M, sizeof(double) * m * n);
        std::memcpy(R.data(), rhs, sizeof(double) * m * nrhs);
        const LstsqResult r = dense_lstsq(Mm, R);
        std::memcpy(X, r.X.data(), sizeof(double) * n * nrhs);
        *deficient = r.rank_deficient;
    });
}

int ref_sym_eig(int n, const double* A, double* lam, double* V) {
    return guard([&] {
        Eigen::MatrixXd M(n, n);
        std::memcpy(M.data(), A, sizeof(double) * n * n);
        const SymEig e = sym_eig(M);
        std::memcpy(lam, e.lambda.data(), sizeof(double) * n);
        std::memcpy(V, e.V.data(), sizeof(double) * n * n);
    });
}

/// build_sai on a caller-supplied system (smoothers.hpp:259-367).  Two-phase:
/// returns a handle; query nnzb / matrix / stats, then free.
struct RefSai {
    BlockCsr B;
    SaiStats st;
};

void* ref_sai_build(int kind, int dim, int ncomp, int bs_scalar, int N, const int* ptr,
                    const int* col, const double* val, int level, double zeta, int cache) {
    RefSai* out = nullptr;
    const int rc = guard([&] {
        System S;
        S.kind = kind == LDGMG_SYSTEM_STOKES ? SystemKind::Stokes : SystemKind::Scalar;
        S.dim = dim;
        S.n_comp = ncomp;
        S.bs_scalar = bs_scalar;
        const int bs = ncomp * bs_scalar;
        S.A = csr_in(N, N, bs, bs, ptr, col, val);
        auto r = std::make_unique<RefSai>();
        SaiCache c;
        r->B = build_sai(S, level, zeta, cache ? &c : nullptr, &r->st);
        out = r.release();
    });
    return rc == 0 ? out : nullptr;
}
long long ref_sai_raw_nnzb(void* h) { return (long long)static_cast<RefSai*>(h)->B.col.size(); }
void ref_sai_raw_matrix(void* h, int* ptr, int* col, double* val) {
    copy_csr(static_cast<RefSai*>(h)->B, ptr, col, val);
}
void ref_sai_raw_stats(void* h, ldgmg_sai_stats* out) { stats_out(static_cast<RefSai*>(h)->st, out); }
void ref_sai_raw_free(void* h) { delete static_cast<RefSai*>(h); }

int ref_balance_vector(int kind, int dim, int ncomp, int bs_scalar, int N, const int* ptr,
                       const int* col, const double* val, double zeta, double* alpha) {
    return guard([&] {
        System S;
        S.kind = kind == LDGMG_SYSTEM_STOKES ? SystemKind::Stokes : SystemKind::Scalar;
        S.dim = dim;
        S.n_comp = ncomp;
        S.bs_scalar = bs_scalar;
        const int bs = ncomp * bs_scalar;
        S.A = csr_in(N, N, bs, bs, ptr, col, val);
        const auto a = balance_vector(S, zeta);
        std::memcpy(alpha, a.data(), sizeof(double) * a.size());
    });
}

int ref_colour_mesh(int N, const int* ptr, const int* col, int* colour) {
    return guard([&] {
        std::vector<double> val(static_cast<size_t>(ptr[N]), 1.0);
        const auto c = colour_mesh(csr_in(N, N, 1, 1, ptr, col, val.data()));
        std::memcpy(colour, c.data(), sizeof(int) * c.size());
    });
}

}  // extern "C"
