// ldgmg_b200.hpp -- C++ drop-in over the C ABI (ldgmg_b200.h).
//
// Re-exposes the B200 hot path with the reference's class and method names
// (blockla.hpp / smoothers.hpp / multigrid.hpp / krylov.hpp) in namespace
// ldgmg::gpu, mapping status codes back to the reference's exception types.
// Header-only; link libldgmg_b200.so.
//
// Two layers:
//  * always available: Context, DeviceBsr, DeviceVec, Smoother, Transfer,
//    Multigrid (device vectors, no reference types);
//  * when the reference headers are included first (LDGMG_MULTIGRID_HPP is
//    defined): ldgmg::gpu::Multigrid(Mesh, LevelAssembler, MultigridConfig)
//    with the reference constructor's semantics (mesh chain via the
//    reference's coarsen(), the caller's assembler per level, the same
//    validation and exceptions), and cycle / apply / smoother() / pcg /
//    gmres_left / estimate_eta on ldgmg::BlockVec.  This is the one-line switch
//    INTEGRATION.md describes.
#ifndef LDGMG_B200_HPP
#define LDGMG_B200_HPP

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ldgmg_b200.h"

namespace ldgmg {
namespace gpu {

/// Status -> the reference's exception types (blockla.hpp, smoothers.hpp).
inline void check(int status) {
    if (status == LDGMG_OK) return;
    const std::string msg = ldgmg_last_error();
    switch (status) {
        case LDGMG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case LDGMG_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

enum class Sweep { Forward = LDGMG_SWEEP_FORWARD, Reverse = LDGMG_SWEEP_REVERSE };

class Context {
  public:
    explicit Context(int device = 0) {
        ldgmg_ctx* c = nullptr;
        check(ldgmg_ctx_create(device, &c));
        h_.reset(c);
    }
    ldgmg_ctx* get() const { return h_.get(); }
    void synchronize() const { check(ldgmg_ctx_synchronize(h_.get())); }
    void set_stream(void* cuda_stream) { check(ldgmg_ctx_set_stream(h_.get(), cuda_stream)); }

  private:
    struct Del {
        void operator()(ldgmg_ctx* c) const { ldgmg_ctx_destroy(c); }
    };
    std::unique_ptr<ldgmg_ctx, Del> h_;
};

/// Device vector in the BlockVec layout (blockla.hpp:46-58).
class DeviceVec {
  public:
    DeviceVec(const Context& ctx, int nblocks, int bs) : ctx_(&ctx), nblocks(nblocks), bs(bs) {
        void* p = nullptr;
        check(ldgmg_device_alloc(ctx.get(), bytes(), &p));
        p_ = static_cast<double*>(p);
        set_zero();
    }
    DeviceVec(const DeviceVec&) = delete;
    DeviceVec& operator=(const DeviceVec&) = delete;
    DeviceVec(DeviceVec&& o) noexcept : ctx_(o.ctx_), nblocks(o.nblocks), bs(o.bs), p_(o.p_) { o.p_ = nullptr; }
    ~DeviceVec() {
        if (p_) ldgmg_device_free(ctx_->get(), p_);
    }
    size_t size() const { return size_t(nblocks) * bs; }
    size_t bytes() const { return size() * sizeof(double); }
    double* data() { return p_; }
    const double* data() const { return p_; }
    void upload(const double* host) { check(ldgmg_copy_h2d(ctx_->get(), p_, host, bytes())); }
    void download(double* host) const { check(ldgmg_copy_d2h(ctx_->get(), host, p_, bytes())); }
    void set_zero() {
        std::vector<double> z(size(), 0.0);
        upload(z.data());
    }

  private:
    const Context* ctx_;

  public:
    int nblocks, bs;

  private:
    double* p_ = nullptr;
};

/// Device BSR operator (BlockCsr, blockla.hpp:73-92).
class DeviceBsr {
  public:
    DeviceBsr(const Context& ctx, int brows, int bcols, int row_bs, int col_bs, const int* ptr, const int* col,
              const double* val)
        : ctx_(&ctx), brows(brows), bcols(bcols), row_bs(row_bs), col_bs(col_bs) {
        ldgmg_bsr* b = nullptr;
        check(ldgmg_bsr_upload(ctx.get(), brows, bcols, row_bs, col_bs, ptr, col, val, &b));
        h_.reset(b);
    }
    ldgmg_bsr* get() const { return h_.get(); }

  private:
    const Context* ctx_;
    struct Del {
        void operator()(ldgmg_bsr* b) const { ldgmg_bsr_destroy(b); }
    };
    std::unique_ptr<ldgmg_bsr, Del> h_;

  public:
    int brows, bcols, row_bs, col_bs;
};

/// spmv / spmv_transpose (blockla.hpp:136-176) on device vectors.
inline void spmv(const Context& ctx, const DeviceBsr& A, const DeviceVec& x, DeviceVec& y) {
    if (x.nblocks != A.bcols || x.bs != A.col_bs || y.nblocks != A.brows || y.bs != A.row_bs)
        throw std::invalid_argument("spmv: shape mismatch");
    check(ldgmg_spmv(ctx.get(), A.get(), x.data(), y.data()));
}
inline void spmv_transpose(const Context& ctx, const DeviceBsr& A, const DeviceVec& x, DeviceVec& y) {
    if (x.nblocks != A.brows || x.bs != A.row_bs || y.nblocks != A.bcols || y.bs != A.col_bs)
        throw std::invalid_argument("spmv_transpose: shape mismatch");
    check(ldgmg_spmv_transpose(ctx.get(), A.get(), x.data(), y.data()));
}

/// Smoother (smoothers.hpp:373-534); setup on the GPU.
class Smoother {
  public:
    Smoother(const Context& ctx, const DeviceBsr& A, const ldgmg_smoother_config& cfg,
             int system_kind = LDGMG_SYSTEM_SCALAR, int n_velocity = 0)
        : ctx_(&ctx), A_(&A) {
        ldgmg_smoother* s = nullptr;
        check(ldgmg_smoother_create(ctx.get(), A.get(), system_kind, n_velocity, &cfg, &s));
        h_ = s;
        own_ = true;
    }
    Smoother(const Context& ctx, ldgmg_smoother* view, int n, int bs) : ctx_(&ctx), h_(view), n_(n), bs_(bs) {}
    Smoother(const Smoother&) = delete;
    Smoother& operator=(const Smoother&) = delete;
    ~Smoother() {
        if (own_) ldgmg_smoother_destroy(h_);
    }
    void apply(const DeviceVec& b, DeviceVec& x, Sweep sweep) const {
        check(ldgmg_smoother_apply(ctx_->get(), h_, b.data(), x.data(), int(sweep)));
    }
    int n_colours() const {
        int n = 0;
        check(ldgmg_smoother_colours(h_, nullptr, &n));
        return n;
    }
    ldgmg_sai_stats sai_stats() const {
        ldgmg_sai_stats st{};
        check(ldgmg_smoother_sai_stats(h_, &st));
        return st;
    }
    ldgmg_smoother* get() const { return h_; }

  private:
    const Context* ctx_;
    const DeviceBsr* A_ = nullptr;
    ldgmg_smoother* h_ = nullptr;
    bool own_ = false;
    int n_ = 0, bs_ = 0;
};

/// Inter-level transfer (multigrid.hpp:104-149).
class Transfer {
  public:
    Transfer(const Context& ctx, int n_fine, int n_coarse, const int* parent_of, const int* orthant_of, int dim,
             int bs_scalar, int n_comp, const double* K)
        : ctx_(&ctx) {
        ldgmg_transfer* t = nullptr;
        check(ldgmg_transfer_create(ctx.get(), n_fine, n_coarse, parent_of, orthant_of, dim, bs_scalar, n_comp, K, &t));
        h_.reset(t);
    }
    ldgmg_transfer* get() const { return h_.get(); }
    void restrict_residual(const DeviceVec& rf, DeviceVec& rc) const {
        check(ldgmg_restrict(ctx_->get(), h_.get(), rf.data(), rc.data()));
    }
    void interpolate_add(const DeviceVec& xc, DeviceVec& xf) const {
        check(ldgmg_interpolate_add(ctx_->get(), h_.get(), xc.data(), xf.data()));
    }

  private:
    const Context* ctx_;
    struct Del {
        void operator()(ldgmg_transfer* t) const { ldgmg_transfer_destroy(t); }
    };
    std::unique_ptr<ldgmg_transfer, Del> h_;
};

/// Device-level V-cycle hierarchy over already assembled level operators.
class DeviceMultigrid {
  public:
    DeviceMultigrid(const Context& ctx, std::vector<std::unique_ptr<DeviceBsr>> levels,
                    std::vector<std::unique_ptr<Transfer>> transfers, int system_kind, int dim, int n_comp,
                    int bs_scalar, bool kernel_constants, bool kernel_pressure, const ldgmg_mg_config& cfg)
        : ctx_(&ctx), levels_(std::move(levels)), transfers_(std::move(transfers)) {
        std::vector<const ldgmg_bsr*> A;
        std::vector<const ldgmg_transfer*> T;
        for (auto& l : levels_) A.push_back(l->get());
        for (auto& t : transfers_) T.push_back(t->get());
        ldgmg_mg* m = nullptr;
        check(ldgmg_mg_create(ctx.get(), int(A.size()), A.data(), T.data(), system_kind, dim, n_comp, bs_scalar,
                              kernel_constants, kernel_pressure, &cfg, nullptr, nullptr, &m));
        h_.reset(m);
    }
    int depth() const { return ldgmg_mg_depth(h_.get()); }
    /// Sequential (reference-order) kernel projection and Krylov reductions:
    /// bit-identical to the reference on singular systems (periodic scalar,
    /// Stokes pressure).  Off: fixed-tree device reductions (deterministic,
    /// within 1e-13 of the reference, faster).
    void set_strict_order(bool strict) const { check(ldgmg_mg_set_strict_order(h_.get(), strict ? 1 : 0)); }
    void cycle(DeviceVec& x, const DeviceVec& b) const { check(ldgmg_mg_cycle(ctx_->get(), h_.get(), x.data(), b.data())); }
    void apply(const DeviceVec& b, DeviceVec& x) const { check(ldgmg_mg_apply(ctx_->get(), h_.get(), b.data(), x.data())); }
    void cycles(DeviceVec& x, const DeviceVec& b, int n) const {
        check(ldgmg_mg_cycles(ctx_->get(), h_.get(), x.data(), b.data(), n));
    }
    ldgmg_solve_report krylov(int kind, const DeviceVec& b, DeviceVec& x, std::vector<double>& residuals, double tol,
                              int maxit) const {
        residuals.assign(size_t(maxit) + 2, 0.0);
        ldgmg_solve_report r{};
        r.residuals = residuals.data();
        r.capacity = maxit + 2;
        check(ldgmg_krylov_solve(ctx_->get(), h_.get(), kind, b.data(), x.data(), tol, maxit, &r));
        residuals.resize(size_t(r.n_residuals));
        return r;
    }
    ldgmg_mg* get() const { return h_.get(); }
    const DeviceBsr& level(int l) const { return *levels_.at(size_t(l)); }

  private:
    const Context* ctx_;
    std::vector<std::unique_ptr<DeviceBsr>> levels_;
    std::vector<std::unique_ptr<Transfer>> transfers_;
    struct Del {
        void operator()(ldgmg_mg* m) const { ldgmg_mg_destroy(m); }
    };
    std::unique_ptr<ldgmg_mg, Del> h_;
};

}  // namespace gpu
}  // namespace ldgmg

// --------------------------------------------------------------------------
// Reference-typed drop-in (requires <ldgmg/multigrid.hpp> / <ldgmg/krylov.hpp>
// from the reference to be included before this header).
#if defined(LDGMG_MULTIGRID_HPP)
namespace ldgmg {
namespace gpu {

inline ldgmg_smoother_config to_c(const SmootherConfig& s) {
    ldgmg_smoother_config c{};
    c.kind = int(s.kind);
    c.omega = s.omega;
    c.partitions = s.partitions;
    c.level = s.level;
    c.zeta = s.zeta;
    c.cache = s.cache ? 1 : 0;
    return c;
}

inline ldgmg_mg_config to_c(const MultigridConfig& m) {
    ldgmg_mg_config c{};
    c.smoother = to_c(m.smoother);
    c.pre = m.pre == ldgmg::Sweep::Forward ? LDGMG_SWEEP_FORWARD : LDGMG_SWEEP_REVERSE;
    c.post = m.post == ldgmg::Sweep::Forward ? LDGMG_SWEEP_FORWARD : LDGMG_SWEEP_REVERSE;
    c.nu1 = m.nu1;
    c.nu2 = m.nu2;
    c.bottom_max_elements = m.bottom_max_elements;
    c.bottom_tol = m.bottom_tol;
    c.min_depth = m.min_depth;
    return c;
}

/// Drop-in for ldgmg::Multigrid (multigrid.hpp:45-274): same constructor and
/// solve interface; operators, smoothers and the V-cycle live on the B200.
class Multigrid {
  public:
    Multigrid(Mesh fine, const LevelAssembler& assemble, MultigridConfig cfg, const Context& ctx = default_ctx())
        : ctx_(&ctx), cfg_(cfg) {
        if (cfg.nu1 < 0 || cfg.nu2 < 0) throw std::invalid_argument("multigrid: smoothing counts must be nonnegative");
        // mesh chain: the reference's own coarsen() and phase rule (multigrid.hpp:168-194)
        meshes_.push_back(std::move(fine));
        std::vector<Coarsening> maps;
        for (;;) {
            const Mesh& m = meshes_.back();
            Coarsening c;
            try {
                c = coarsen(m);
            } catch (const std::invalid_argument&) {
                break;
            }
            bool phase_ok = true;
            for (int f = 0; f < (int)m.elements.size() && phase_ok; ++f)
                phase_ok = m.elements[f].phase == c.mesh.elements[c.parent_of[f]].phase;
            if (!phase_ok) break;
            maps.push_back(c);
            meshes_.push_back(c.mesh);
        }
        if ((int)meshes_.size() < cfg.min_depth)
            throw std::invalid_argument("multigrid: hierarchy depth below the configured minimum");
        if ((int)meshes_.back().elements.size() > cfg.bottom_max_elements)
            throw std::invalid_argument("multigrid: bottom level exceeds the element budget");
        std::vector<std::unique_ptr<DeviceBsr>> levels;
        for (const Mesh& m : meshes_) {
            systems_.push_back(assemble(m));
            const System& S = systems_.back();
            const System& S0 = systems_.front();
            if (S.dim != S0.dim || S.degree != S0.degree || S.n_comp != S0.n_comp || S.bs_scalar != S0.bs_scalar ||
                S.kind != S0.kind)
                throw std::invalid_argument("multigrid: level assembler changed the discretization");
            levels.push_back(std::make_unique<DeviceBsr>(ctx, S.A.brows, S.A.bcols, S.A.row_bs, S.A.col_bs,
                                                         S.A.ptr.data(), S.A.col.data(), S.A.val.data()));
        }
        const System& S0 = systems_.front();
        std::vector<double> K(size_t(1) << S0.dim);
        K.assign((size_t(1) << S0.dim) * size_t(S0.bs_scalar) * S0.bs_scalar, 0.0);
        check(ldgmg_injection_matrices(S0.dim, S0.degree, K.data()));
        std::vector<std::unique_ptr<Transfer>> transfers;
        for (size_t l = 0; l < maps.size(); ++l)
            transfers.push_back(std::make_unique<Transfer>(ctx, (int)maps[l].parent_of.size(),
                                                           (int)meshes_[l + 1].elements.size(),
                                                           maps[l].parent_of.data(), maps[l].orthant_of.data(),
                                                           S0.dim, S0.bs_scalar, S0.n_comp, K.data()));
        dev_ = std::make_unique<DeviceMultigrid>(ctx, std::move(levels), std::move(transfers),
                                                 S0.kind == SystemKind::Stokes ? LDGMG_SYSTEM_STOKES : LDGMG_SYSTEM_SCALAR,
                                                 S0.dim, S0.n_comp, S0.bs_scalar, S0.kernel_constants,
                                                 S0.kernel_pressure, to_c(cfg));
        // the drop-in promises the reference's bits: strict-order reductions
        // by default (set_strict_order(false) selects the fast tree)
        dev_->set_strict_order(true);
    }
    Multigrid(const Multigrid&) = delete;
    Multigrid& operator=(const Multigrid&) = delete;

    int depth() const { return (int)meshes_.size(); }
    const Mesh& mesh(int level = 0) const { return meshes_.at(size_t(level)); }
    const System& system(int level = 0) const { return systems_.at(size_t(level)); }
    const MultigridConfig& config() const { return cfg_; }
    bool symmetric() const { return symmetric_plan(cfg_.smoother, cfg_.pre, cfg_.post); }

    /// Multigrid::cycle (multigrid.hpp:82-85) on host vectors
    void cycle(BlockVec& x, const BlockVec& b) const {
        DeviceVec dx(*ctx_, x.nblocks, x.bs), db(*ctx_, b.nblocks, b.bs);
        dx.upload(x.data.data());
        db.upload(b.data.data());
        dev_->cycle(dx, db);
        dx.download(x.data.data());
    }
    /// Multigrid::apply (multigrid.hpp:90-101)
    BlockVec apply(const BlockVec& b) const {
        BlockVec x(b.nblocks, b.bs);
        DeviceVec dx(*ctx_, b.nblocks, b.bs), db(*ctx_, b.nblocks, b.bs);
        db.upload(b.data.data());
        dev_->apply(db, dx);
        dx.download(x.data.data());
        return x;
    }
    /// pcg (kind = LDGMG_KRYLOV_CG) / gmres_left (LDGMG_KRYLOV_GMRES),
    /// krylov.hpp:117-251, with this hierarchy as the preconditioner V
    std::pair<BlockVec, ldgmg_solve_report> solve(int kind, const BlockVec& b, std::vector<double>& residuals,
                                                  double tol = 1e-12, int maxit = 60) const {
        BlockVec x(b.nblocks, b.bs);
        DeviceVec dx(*ctx_, b.nblocks, b.bs), db(*ctx_, b.nblocks, b.bs);
        db.upload(b.data.data());
        const ldgmg_solve_report r = dev_->krylov(kind, db, dx, residuals, tol, maxit);
        dx.download(x.data.data());
        return {std::move(x), r};
    }
    const DeviceMultigrid& device() const { return *dev_; }
    void set_strict_order(bool strict) const { dev_->set_strict_order(strict); }

  private:
    static const Context& default_ctx() {
        static Context c(0);
        return c;
    }
    const Context* ctx_;
    MultigridConfig cfg_;
    std::vector<Mesh> meshes_;
    std::vector<System> systems_;
    std::unique_ptr<DeviceMultigrid> dev_;
};

}  // namespace gpu
}  // namespace ldgmg
#endif

#endif  // LDGMG_B200_HPP
