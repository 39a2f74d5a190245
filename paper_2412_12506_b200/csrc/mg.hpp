// Smoother / multigrid objects behind the C ABI handles.
#pragma once

#include <memory>
#include <vector>

#include "core.hpp"

namespace ldgmg_b200 {

std::vector<int> colour_mesh_host(const Bsr& A);
/// Processor-block GS wavefront schedule (see mg.cu).
void pgs_wavefronts(int n_rows, const int* ptr, const int* col, const int* part_of, int n_cols_own, bool reverse,
                    std::vector<int>& rows, std::vector<int>& level_ptr);
void upload_factors(Ctx& ctx, DiagFactors& F, int N, int bs, const double* V, const double* lambda,
                    const double* s);
void compute_factors(Ctx& ctx, const Bsr& A, DiagFactors& F);      // GPU (factors.cu) unless LDGMG_HOST_FACTORS=1
void compute_factors_host(Ctx& ctx, const Bsr& A, DiagFactors& F);  // host eig, multithreaded
void compute_factors_gpu(Ctx& ctx, const Bsr& A, DiagFactors& F);
std::unique_ptr<Transfer> transfer_create(Ctx& ctx, int n_fine, int n_coarse, const int* parent_of,
                                          const int* orthant_of, int dim, int bss, int ncomp,
                                          const double* K);

/// SAI build on the GPU (sai_build.cu): B on the pattern of A^level.
struct SaiResult {
    std::unique_ptr<Bsr> B;
    ldgmg_sai_stats stats{};
};
struct SaiCache;  // least-squares solution cache, shareable across builds
SaiCache* sai_cache_new();
void sai_cache_free(SaiCache* c);
/// `colmask` (optional, N entries): solve only the columns with a nonzero
/// entry (distributed setup: the rank's columns); the others stay empty.
SaiResult build_sai_gpu(Ctx& ctx, const Bsr& A, int system_kind, int n_velocity, int level,
                        double zeta, bool cache, SaiCache* shared, const std::vector<char>* colmask = nullptr);

struct Smoother {
    const Bsr* A = nullptr;
    ldgmg_smoother_config cfg{};
    int system_kind = LDGMG_SYSTEM_SCALAR, n_velocity = 0;
    int N = 0, bs = 0;
    DiagFactors F;
    std::vector<int> colour, colour_ptr;
    int ncolours = 0;
    DevBuf colour_rows;
    std::unique_ptr<Bsr> B;
    ldgmg_sai_stats stats{};
    DevBuf snap;  // Jacobi / processor-block GS snapshot, SAI residual scratch
    // processor-block GS: partition of each element, wavefront schedules
    // (rows grouped by level) for the forward [0] and reverse [1] sweeps
    DevBuf part, sched_rows[2];
    std::vector<int> sched_ptr[2];

    void init_common(Ctx& ctx);
    /// `r_ready`: SAI only -- `snap` already holds b - A x for this x (the
    /// caller's residual check computed it with the same kernel), so the
    /// sweep's own residual pass is skipped; the bits are unchanged.
    /// `r_in` (SAI only): a vector known to equal b - A x (e.g. b when x = 0).
    void apply(Ctx& ctx, const double* b, double* x, int sweep, bool r_ready = false,
               const double* r_in = nullptr) const;
    /// `nu` consecutive applications (the V-cycle's pre / post smoothing);
    /// Jacobi ping-pongs x with the snapshot buffer instead of copying;
    /// `x_zero`: x is exactly zero on entry (coarse levels).
    void apply_sweeps(Ctx& ctx, const double* b, double* x, int sweep, int nu, bool r_ready = false,
                      bool x_zero = false) const;
    double bytes_per_apply() const;
};

struct Mg {
    int depth = 0;
    std::vector<const Bsr*> A;
    std::vector<const Transfer*> T;
    std::vector<Smoother*> sm;
    // owned pieces (problem-built hierarchies / default smoothers)
    std::vector<std::unique_ptr<Bsr>> own_A;
    std::vector<std::unique_ptr<Transfer>> own_T;
    std::vector<std::unique_ptr<Smoother>> own_sm;
    ldgmg_mg_config cfg{};
    int system_kind = LDGMG_SYSTEM_SCALAR, dim = 2, n_comp = 1, bs_scalar = 1, bs = 1;
    int kernel_constants = 0, kernel_pressure = 0, n_velocity = 0;
    bool strict_order = false;  // reference-order (sequential) kernel projection
    std::vector<int> kernel_offsets_host;
    /// symmetric_plan (multigrid.hpp:41-43)
    bool symmetric() const { return cfg.smoother.kind == LDGMG_JACOBI || cfg.pre != cfg.post; }
    DenseEig bottom;
    std::vector<DevBuf> r, xl, bl;
    DevBuf bp, kernel_offs, red;
    int nkernel = 0;
    double kval = 0.0;
    double* h_red = nullptr;
    bool warm = false;
    struct Graph {
        double* x;
        const double* b;
        cudaStream_t s;
        cudaGraphExec_t exec;
        int64_t nkernels;
        bool r0;  // captured with the level-0 residual precomputed (cycle(..., r0_ready))
    };
    std::vector<Graph> graphs;
    cudaStream_t cap_stream = nullptr;
    SaiCache* sai_cache = nullptr;  // shared across levels (multigrid.hpp:60)
    // ldgmg_mg_solve_host scratch (cached so the graph of (x, b) is reused)
    DevBuf solve_b, solve_x, solve_r, solve_xs;
    double* h_stage = nullptr;    // pinned staging for host -> device
    double* h_stage_x = nullptr;  // pinned landing buffer of the iterate snapshots
    cudaStream_t d2h_stream = nullptr;
    cudaEvent_t ev_snap = nullptr, ev_d2h = nullptr;
    // device-resident solve loop (capi.cu build_solve_graph): prologue + a
    // conditional WHILE node whose body is cycle -> snapshot -> check
    cudaGraphExec_t solve_exec = nullptr;
    int solve_cap = 0;          // history capacity the graph was built for
    int64_t solve_npro = 0, solve_nbody = 0;  // kernels per prologue / per loop body
    /// drop every captured graph (after a change the captures baked in)
    void invalidate_graphs();
    bool solve_graph_bad = false;
    DevBuf solve_red, solve_state;
    cudaStream_t cap_side = nullptr;
    cudaEvent_t cap_ev[2] = {nullptr, nullptr};

    void init(Ctx& ctx);
    void set_bottom(Ctx& ctx, const double* V, const double* lambda);
    void v_cycle(Ctx& ctx, int l, double* x, const double* b, bool r0_ready = false);
    void project(Ctx& ctx, double* v);
    void cycle(Ctx& ctx, double* x, const double* b, bool r0_ready = false);
    void apply(Ctx& ctx, const double* b, double* x);
    void cycles(Ctx& ctx, double* x, const double* b, int n, bool r0_ready = false);
    /// Level-0 residual buffer the first pre-smoothing sweep can start from
    /// (SAI smoother with nu1 >= 1), nullptr when the smoother has none.
    double* r0_buffer() const;
    double dof_updates_per_cycle() const;
    double bytes_per_cycle() const;
    ~Mg();
};

}  // namespace ldgmg_b200
