// Krylov accelerators around the GPU V-cycle (krylov.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "core.hpp"

namespace ldgmg_b200 {

struct Mg;

/// SolveReport (krylov.hpp:38-47)
struct SolveReport {
    std::vector<double> residuals;
    int iterations = 0;
    bool converged = false;
    bool breakdown = false;
    double rho = 0.0;
    double eta = 0.0;
    int classification = 0;  // 0 fast, 1 slow, 2 nonconvergent
    bool low_confidence = false;
};

void fit_rate(SolveReport& rep);
SolveReport pcg(Ctx& ctx, Mg& mg, const double* b, double* x, double tol, int maxit);
SolveReport gmres_left(Ctx& ctx, Mg& mg, const double* b, double* x, double tol, int maxit);
SolveReport estimate_eta(Ctx& ctx, Mg& mg, int kind, uint64_t seed, double tol, int maxit);

}  // namespace ldgmg_b200
