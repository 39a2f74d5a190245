// C++ drop-in check: the reference's ldgmg::Multigrid vs ldgmg::gpu::Multigrid
// (include/ldgmg_b200.hpp) built from the SAME Mesh / LevelAssembler /
// MultigridConfig -- the one-line switch of INTEGRATION.md.  Built by
// `make -C oracle dropin` (needs the reference headers), run on a B200 by
// tests/test_gpu_dropin_cpp.py.  Prints one "PASS"/"FAIL" line per case.
#include <ldgmg/krylov.hpp>
#include <ldgmg/ldg_scalar.hpp>
#include <ldgmg/ldg_stokes.hpp>
#include <ldgmg/multigrid.hpp>

#include "../../include/ldgmg_b200.hpp"

#include <cstdio>
#include <random>

using namespace ldgmg;

static std::array<BoundaryKind, 6> sides(BoundaryKind k) { return {k, k, k, k, k, k}; }

static double rel(const BlockVec& a, const BlockVec& b) {
    double d = 0, n = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        d += (a.data[i] - b.data[i]) * (a.data[i] - b.data[i]);
        n += b.data[i] * b.data[i];
    }
    return std::sqrt(d / std::max(n, 1e-300));
}

static int run(const char* name, const Mesh& mesh, const LevelAssembler& asmb, const MultigridConfig& cfg) {
    const Multigrid ref(mesh, asmb, cfg);
    const gpu::Multigrid dev(mesh, asmb, cfg);
    int bad = ref.depth() != dev.depth();
    const System& S = ref.system(0);
    BlockVec b = random_rhs(S.n_elements(), S.block_size(), 3);
    for (const BlockVec& k : kernel_basis(S)) axpy(-dot(b, k), k, b);
    BlockVec xr(S.n_elements(), S.block_size()), xg = xr;
    for (int it = 0; it < 3; ++it) {
        ref.cycle(xr, b);
        dev.cycle(xg, b);
    }
    const double e1 = rel(xg, xr);
    const double e2 = rel(dev.apply(b), ref.apply(b));
    std::vector<double> res;
    auto [x, rep] = dev.solve(LDGMG_KRYLOV_GMRES, b, res, 1e-10, 60);
    const SolveReport want = gmres_left(S.A, b, preconditioner(ref), 1e-10, 60).second;
    bad |= e1 > 1e-12 || e2 > 1e-12 || std::abs(rep.iterations - want.iterations) > 0;
    std::printf("%s %s depth=%d cycle_rel=%.3g apply_rel=%.3g gmres_its=%d/%d\n", bad ? "FAIL" : "PASS", name,
                dev.depth(), e1, e2, rep.iterations, want.iterations);
    return bad;
}

int main() {
    int bad = 0;
    {
        ScalarProblem P;
        P.mesh = build_uniform(16, 2, sides(BoundaryKind::Dirichlet));
        P.degree = 2;
        LevelAssembler a = [P](const Mesh& m) {
            ScalarProblem Q = P;
            Q.mesh = m;
            return assemble_scalar(Q);
        };
        MultigridConfig cfg;
        cfg.smoother = SmootherConfig::coloured_gs();
        bad |= run("scalar2d-dirichlet-gs", P.mesh, a, cfg);
        cfg.smoother = SmootherConfig::sai(1);
        bad |= run("scalar2d-dirichlet-sai1", P.mesh, a, cfg);
    }
    {
        ScalarProblem P;
        P.mesh = build_uniform(8, 3, sides(BoundaryKind::Periodic));
        P.degree = 2;
        LevelAssembler a = [P](const Mesh& m) {
            ScalarProblem Q = P;
            Q.mesh = m;
            return assemble_scalar(Q);
        };
        MultigridConfig cfg;
        cfg.smoother = SmootherConfig::sai(1);
        bad |= run("scalar3d-periodic-sai1", P.mesh, a, cfg);
    }
    {
        StokesProblem P;
        P.mesh = build_uniform(8, 2, sides(BoundaryKind::Periodic));
        P.degree = 2;
        P.gamma = 1.0;
        LevelAssembler a = [P](const Mesh& m) {
            StokesProblem Q = P;
            Q.mesh = m;
            return assemble_stokes(Q);
        };
        MultigridConfig cfg;
        cfg.smoother = SmootherConfig::sai(1, 0.13);
        bad |= run("stokes2d-stress-sai1", P.mesh, a, cfg);
    }
    // exceptions map back to the reference's types
    try {
        ScalarProblem P;
        P.mesh = build_uniform(8, 2, sides(BoundaryKind::Periodic));
        MultigridConfig cfg;
        cfg.nu1 = -1;
        gpu::Multigrid dev(P.mesh, [P](const Mesh& m) { ScalarProblem Q = P; Q.mesh = m; return assemble_scalar(Q); }, cfg);
        std::printf("FAIL no exception for nu1<0\n");
        bad = 1;
    } catch (const std::invalid_argument&) {
        std::printf("PASS invalid_argument for nu1<0\n");
    }
    return bad;
}
