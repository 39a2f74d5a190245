// Built-in host setup (see setup.hpp).  Restates, for uniform Morton meshes,
//   basis.hpp:23-134       Legendre modes, Gauss-Legendre rule, tables
//   mesh.hpp:171-314,412   Morton roots, faces, coarsening
//   ldg_core.hpp:84-586    traces, face blocks, G_k, E, L^T D R products
//   ldg_scalar.hpp:83-125  A = sum_k G_k^T M_mu G_k + E
//   ldg_stokes.hpp:73-280  saddle operator, pressure penalty, unsteady term
//   multigrid.hpp:168-241  level chain and injection matrices
// with the reference's accumulation order so results are bit-identical.
#include "setup.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "host_eig.hpp"

namespace ldgmg_b200 {

namespace {

// ------------------------------------------------------------------ basis
std::pair<double, double> legendre(int k, double x) {
    double p0 = 1.0, d0 = 0.0;
    if (k == 0) return {p0, d0};
    double p1 = x, d1 = 1.0;
    for (int n = 1; n < k; ++n) {
        const double p2 = ((2 * n + 1) * x * p1 - n * p0) / (n + 1);
        const double d2 = d0 + (2 * n + 1) * p1;
        p0 = p1;
        d0 = d1;
        p1 = p2;
        d1 = d2;
    }
    return {p1, d1};
}
double mode_val(int k, double x) { return std::sqrt((2 * k + 1) / 2.0) * legendre(k, x).first; }
double mode_dval(int k, double x) { return std::sqrt((2 * k + 1) / 2.0) * legendre(k, x).second; }

void gauss_legendre(int npts, std::vector<double>& x, std::vector<double>& w) {
    x.assign(npts, 0.0);
    w.assign(npts, 0.0);
    for (int i = 0; i < (npts + 1) / 2; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (npts + 0.5));
        for (int it = 0; it < 100; ++it) {
            auto [p, d] = legendre(npts, t);
            const double dt = p / d;
            t -= dt;
            if (std::abs(dt) < 1e-15) break;
        }
        auto [p, d] = legendre(npts, t);
        (void)p;
        const int j = npts - 1 - i;
        x[i] = -std::abs(t);
        x[j] = std::abs(t);
        w[i] = w[j] = 2.0 / ((1.0 - t * t) * d * d);
    }
    if (npts % 2 == 1) x[npts / 2] = 0.0;
}

double mass_scalar(double h, int dim) {
    double m = 1.0;
    for (int a = 0; a < dim; ++a) m *= 0.5 * h;
    return m;
}

struct Basis {
    int degree = 1, dim = 2, p1 = 2, bs = 4;
    std::vector<double> nodes, weights, val, dval, end_val;
    Basis(int degree_, int dim_) : degree(degree_), dim(dim_) {
        if (degree < 1 || degree > 8) throw std::invalid_argument("basis: degree out of range");
        if (dim != 2 && dim != 3) throw std::invalid_argument("basis: dim must be 2 or 3");
        p1 = degree + 1;
        bs = 1;
        for (int a = 0; a < dim; ++a) bs *= p1;
        gauss_legendre(p1, nodes, weights);
        val.resize(p1 * p1);
        dval.resize(p1 * p1);
        end_val.resize(p1 * 2);
        for (int m = 0; m < p1; ++m) {
            for (int q = 0; q < p1; ++q) {
                val[m * p1 + q] = mode_val(m, nodes[q]);
                dval[m * p1 + q] = mode_dval(m, nodes[q]);
            }
            end_val[m * 2 + 0] = mode_val(m, -1.0);
            end_val[m * 2 + 1] = mode_val(m, +1.0);
        }
    }
    std::array<int, 3> decompose(int m) const {
        std::array<int, 3> ix{0, 0, 0};
        for (int a = 0; a < dim; ++a) {
            ix[a] = m % p1;
            m /= p1;
        }
        return ix;
    }
    int compose(const std::array<int, 3>& ix) const {
        int m = 0, stride = 1;
        for (int a = 0; a < dim; ++a) {
            m += ix[a] * stride;
            stride *= p1;
        }
        return m;
    }
};

// ------------------------------------------------------------------- mesh
enum FaceKind { F_INTERIOR = 0, F_DIRICHLET = 1, F_NEUMANN = 2 };

struct Face {
    int left = -1, right = -1, axis = 0, kind = F_INTERIOR, side = 0;
    std::array<double, 3> lo{0, 0, 0};
    double size = 0;
};

struct LevelMesh {
    int dim = 2, n = 2, level = 1;
    int bc[6];
    double h = 0.5;
    std::vector<std::array<int, 3>> idx;  // Morton order
    std::vector<int> phase;
    // extension A1: the elements are the in-range cells
    // of the 2^level grid, in its Morton order; Morton code -> element index
    // (empty: the identity, n a power of two on the reference's path)
    std::vector<int> code2elem;

    bool periodic(int a) const { return bc[2 * a] == LDGMG_BC_PERIODIC; }
    int n_elements() const { return int(idx.size()); }
    double lo(int e, int a) const { return idx[e][a] * h; }
    double hi(int e, int a) const { return (idx[e][a] + 1) * h; }
    int element_at(const std::array<int, 3>& ix) const {
        int code = 0;
        for (int b = 0; b < level; ++b)
            for (int a = 0; a < dim; ++a) code |= ((ix[a] >> b) & 1) << (b * dim + a);
        return code2elem.empty() ? code : code2elem[code];
    }
    /// Faces of element e in the reference's canonical local order
    /// (element_face_table, ldg_core.hpp:287-309): axis-major, lower first.
    void faces_of(int e, std::vector<Face>& out) const {
        out.clear();
        for (int a = 0; a < dim; ++a) {
            for (int upper = 0; upper < 2; ++upper) {
                Face f;
                f.axis = a;
                f.size = h;
                std::array<int, 3> nb = idx[e];
                const bool at_end = upper ? idx[e][a] == n - 1 : idx[e][a] == 0;
                if (at_end && !periodic(a)) {
                    const int kind = bc[2 * a + upper];
                    f.left = e;
                    f.right = -1;
                    f.kind = kind == LDGMG_BC_DIRICHLET ? F_DIRICHLET : F_NEUMANN;
                    f.side = upper ? +1 : -1;
                    for (int t = 0; t < dim; ++t) f.lo[t] = lo(e, t);
                    f.lo[a] = upper ? hi(e, a) : lo(e, a);
                    out.push_back(f);
                    continue;
                }
                nb[a] = upper ? (idx[e][a] + 1) % n : (idx[e][a] + n - 1) % n;
                const int j = element_at(nb);
                // interior faces are emitted by their lower-side element
                const int lower_el = upper ? e : j;
                f.left = lower_el;
                f.right = upper ? j : e;
                f.kind = F_INTERIOR;
                for (int t = 0; t < dim; ++t) f.lo[t] = lo(lower_el, t);
                f.lo[a] = hi(lower_el, a);
                out.push_back(f);
            }
        }
    }
};

/// build_uniform (mesh.hpp:143-183): Morton-ordered uniform mesh.  any_n
/// (extension A1): n need not be a power of two -- the elements are the cells
/// of the bounding 2^ceil(log2 n) grid with every index < n, kept in that
/// grid's Morton order (so 2^d siblings stay contiguous whenever n is even
/// and the order stays monotone along every axis), h = 1/n.  For a power of
/// two this is exactly the reference's mesh.
LevelMesh uniform_mesh(int n, int dim, const int* bc, bool any_n = false) {
    LevelMesh m;
    m.dim = dim;
    m.n = n;
    if (n < 2) throw std::invalid_argument("mesh: need at least 2 elements per axis");
    const bool pow2 = (n & (n - 1)) == 0;
    if (!pow2 && !any_n) throw std::invalid_argument("mesh: element count per axis must be a power of two");
    m.level = 0;
    while ((1 << m.level) < n) ++m.level;
    m.h = pow2 ? std::ldexp(1.0, -m.level) : 1.0 / n;
    for (int i = 0; i < 6; ++i) m.bc[i] = bc[i];
    for (int a = 0; a < dim; ++a)
        if ((bc[2 * a] == LDGMG_BC_PERIODIC) != (bc[2 * a + 1] == LDGMG_BC_PERIODIC))
            throw std::invalid_argument("mesh: periodic boundaries must pair opposite sides");
    const int side = 1 << m.level;
    const int64_t codes = dim == 2 ? int64_t(side) * side : int64_t(side) * side * side;
    const int64_t total = dim == 2 ? int64_t(n) * n : int64_t(n) * n * n;
    if (total > (int64_t(1) << 30)) throw std::invalid_argument("mesh: too many elements");
    m.idx.reserve(size_t(total));
    if (any_n) m.code2elem.assign(size_t(codes), -1);
    for (int64_t code = 0; code < codes; ++code) {
        std::array<int, 3> ix{0, 0, 0};
        for (int b = 0; b < m.level; ++b)
            for (int a = 0; a < dim; ++a) ix[a] |= int((code >> (b * dim + a)) & 1) << b;
        bool in = true;
        for (int a = 0; a < dim; ++a) in &= ix[a] < n;
        if (!in) continue;
        if (any_n) m.code2elem[size_t(code)] = int(m.idx.size());
        m.idx.push_back(ix);
    }
    m.phase.assign(size_t(total), 0);
    return m;
}

// ------------------------------------------------------------ phases
struct Region {
    std::array<double, 3> lo{0, 0, 0}, hi{1, 1, 1};
    double mu = 1, rho = 1;
};

bool inside_curved(const ldgmg_problem_spec& s, const LevelMesh& m, int e) {
    double acc = 0.0;
    for (int a = 0; a < m.dim; ++a) {
        const double c = 0.5 * (m.lo(e, a) + m.hi(e, a));
        const double r = s.phase_shape == LDGMG_PHASE_BALL ? s.radii[0] : s.radii[a];
        const double t = (c - s.center[a]) / r;
        acc += t * t;
    }
    return acc < 1.0;
}

/// assign_phases (mesh.hpp:461-488) for the box catalogue geometry.
void assign_box_phases(LevelMesh& m, const std::vector<Region>& regs) {
    const double eps = 1e-12;
    for (int e = 0; e < m.n_elements(); ++e) {
        int match = -1;
        for (int r = 0; r < int(regs.size()) && match < 0; ++r) {
            bool inside = true;
            for (int a = 0; a < m.dim; ++a) {
                const double c = 0.5 * (m.lo(e, a) + m.hi(e, a));
                if (c < regs[r].lo[a] - eps || c > regs[r].hi[a] + eps) inside = false;
            }
            if (inside) match = r;
        }
        if (match < 0) throw std::invalid_argument("assign_phases: regions do not cover the domain");
        for (const auto& reg : regs)
            for (int a = 0; a < m.dim; ++a) {
                if (m.lo(e, a) < reg.lo[a] - eps && m.hi(e, a) > reg.lo[a] + eps)
                    throw std::invalid_argument("assign_phases: element straddles a region boundary");
                if (m.lo(e, a) < reg.hi[a] - eps && m.hi(e, a) > reg.hi[a] + eps)
                    throw std::invalid_argument("assign_phases: element straddles a region boundary");
            }
        m.phase[e] = match;
    }
}

// --------------------------------------------------------- assembly ctx
struct Ctx {
    const LevelMesh* mesh;
    const Basis* B;
    int dim, bs, p1;
    double beta;
    std::vector<double> msc, mu, rho;
    // row-restricted assembly (distributed setup): rows of the operator to
    // build (`rows`), and the rows of G / E they need (`grows` = rows plus
    // their face neighbours).  Empty vectors = every row.  Each built row is
    // bit-identical to the full assembly (same per-row accumulation).
    std::vector<char> rows, grows;
    bool want(int e) const { return rows.empty() || rows[e]; }
    bool want_g(int e) const { return grows.empty() || grows[e]; }

    int donor(const Face& f) const { return mu[f.right] > mu[f.left] ? f.right : f.left; }
    double penalty_tau(const Face& f) const {
        const double m = f.right >= 0 ? std::min(mu[f.left], mu[f.right]) : mu[f.left];
        return beta * m / f.size;
    }
};

/// LDGMG_SETUP_TIMING=1: wall time of the assembly phases on stderr.
struct PhaseTimer {
    bool on;
    std::chrono::steady_clock::time_point t;
    const char* what;
    explicit PhaseTimer(const char* w) : what(w) {
        const char* e = std::getenv("LDGMG_SETUP_TIMING");
        on = e && std::atoi(e);
        t = std::chrono::steady_clock::now();
    }
    void stamp(const char* phase) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[assembly %s] %-18s %8.3f s\n", what, phase,
                     std::chrono::duration<double>(now - t).count());
        t = now;
    }
};

struct FaceQ {
    int nq = 0;
    std::vector<double> w;
};

FaceQ face_quad(const Ctx& c, const Face& f) {
    FaceQ q;
    const int nt = c.dim - 1;
    q.nq = 1;
    for (int t = 0; t < nt; ++t) q.nq *= c.p1;
    q.w.resize(q.nq);
    double area = 1.0;
    for (int t = 0; t < nt; ++t) area *= 0.5 * f.size;
    for (int flat = 0; flat < q.nq; ++flat) {
        int rem = flat;
        double wq = area;
        for (int a = 0; a < c.dim; ++a) {
            if (a == f.axis) continue;
            const int qa = rem % c.p1;
            rem /= c.p1;
            wq *= c.B->weights[qa];
        }
        q.w[flat] = wq;
    }
    return q;
}

/// trace_values (ldg_core.hpp:179-223)
void trace_values(const Ctx& c, const Face& f, int e, int refside, std::vector<double>& out) {
    const LevelMesh& m = *c.mesh;
    int nq = 1;
    for (int t = 0; t < c.dim - 1; ++t) nq *= c.p1;
    out.assign(size_t(nq) * c.bs, 0.0);
    double v1[2][8 * 8];
    int slots = 0;
    const double elsize = m.h;
    for (int a = 0; a < c.dim; ++a) {
        if (a == f.axis) continue;
        for (int qa = 0; qa < c.p1; ++qa) {
            const double xi =
                (2.0 * (f.lo[a] - m.lo(e, a)) + f.size * (c.B->nodes[qa] + 1.0)) / elsize - 1.0;
            for (int mm = 0; mm < c.p1; ++mm) v1[slots][mm * c.p1 + qa] = mode_val(mm, xi);
        }
        ++slots;
    }
    const int endside = refside > 0 ? 1 : 0;
    for (int flat = 0; flat < nq; ++flat) {
        int qslot[2] = {0, 0};
        int rem = flat;
        for (int t = 0; t < c.dim - 1; ++t) {
            qslot[t] = rem % c.p1;
            rem /= c.p1;
        }
        for (int i = 0; i < c.bs; ++i) {
            const auto ix = c.B->decompose(i);
            double v = c.B->end_val[ix[f.axis] * 2 + endside];
            int slot = 0;
            for (int a = 0; a < c.dim; ++a) {
                if (a == f.axis) continue;
                v *= v1[slot][ix[a] * c.p1 + qslot[slot]];
                ++slot;
            }
            out[size_t(flat) * c.bs + i] = v;
        }
    }
}

/// face_block (ldg_core.hpp:268-280)
void face_block(const FaceQ& fq, const std::vector<double>& test, const std::vector<double>& donor,
                int bs, std::vector<double>& out) {
    out.assign(size_t(bs) * bs, 0.0);
    for (int q = 0; q < fq.nq; ++q) {
        const double wq = fq.w[q];
        const double* tv = test.data() + size_t(q) * bs;
        const double* dv = donor.data() + size_t(q) * bs;
        for (int i = 0; i < bs; ++i) {
            const double ti = wq * tv[i];
            for (int j = 0; j < bs; ++j) out[size_t(i) * bs + j] += ti * dv[j];
        }
    }
}

/// One block row under construction: columns kept in insertion-independent
/// ascending order (std::map, like BlockBuilder::freeze).
struct Row {
    std::map<int, std::vector<double>> cells;
    double* at(int j, int nb) {
        auto& cell = cells[j];
        if (cell.empty()) cell.assign(size_t(nb), 0.0);
        return cell.data();
    }
    void add(int j, const double* b, double scale, int nb) {
        double* dst = at(j, nb);
        for (int k = 0; k < nb; ++k) dst[k] += scale * b[k];
    }
};

/// Frozen block rows (CSR per row, ascending columns).
struct Rows {
    int bs = 0;
    std::vector<std::vector<int>> cols;
    std::vector<std::vector<double>> vals;  // row-major blocks, concatenated
    void freeze_row(int r, const Row& row) {
        cols[r].clear();
        vals[r].clear();
        for (const auto& [j, b] : row.cells) {
            cols[r].push_back(j);
            vals[r].insert(vals[r].end(), b.begin(), b.end());
        }
    }
    void resize(int n, int bs_) {
        bs = bs_;
        cols.assign(n, {});
        vals.assign(n, {});
    }
    const double* block(int r, int k) const { return vals[r].data() + size_t(k) * bs * bs; }
};

/// G_k (ldg_core.hpp:313-375), all k at once, threaded over rows.
void gradient_rows(const Ctx& c, std::array<Rows, 3>& G) {
    const int N = c.mesh->n_elements(), bs = c.bs, p1 = c.p1;
    std::vector<double> S(size_t(p1) * p1, 0.0);
    for (int a = 0; a < p1; ++a)
        for (int b = 0; b < p1; ++b) {
            double s = 0.0;
            for (int q = 0; q < p1; ++q) s += c.B->weights[q] * c.B->dval[a * p1 + q] * c.B->val[b * p1 + q];
            S[size_t(a) * p1 + b] = s;
        }
    for (int k = 0; k < c.dim; ++k) G[k].resize(N, bs);
    parallel_for(N, [&](int lo, int hi) {
        std::vector<Face> faces;
        std::vector<double> VE, VD, M;
        for (int e = lo; e < hi; ++e) {
            if (!c.want_g(e)) continue;
            std::array<Row, 3> rows;
            const double scal = 2.0 / c.mesh->h;
            for (int k = 0; k < c.dim; ++k) {
                double* blk = rows[k].at(e, bs * bs);
                for (int i = 0; i < bs; ++i) {
                    auto ix = c.B->decompose(i);
                    const int ia = ix[k];
                    for (int jb = 0; jb < p1; ++jb) {
                        ix[k] = jb;
                        blk[size_t(i) * bs + c.B->compose(ix)] -= scal * S[size_t(ia) * p1 + jb];
                    }
                }
            }
            c.mesh->faces_of(e, faces);
            for (const Face& f : faces) {
                if (f.kind == F_DIRICHLET) continue;
                const FaceQ fq = face_quad(c, f);
                if (f.kind == F_NEUMANN) {
                    trace_values(c, f, e, f.side, VE);
                    face_block(fq, VE, VE, bs, M);
                    rows[f.axis].add(e, M.data(), f.side / c.msc[e], bs * bs);
                    continue;
                }
                const int sigma = e == f.left ? +1 : -1;
                const int d = c.donor(f);
                trace_values(c, f, e, sigma, VE);
                if (d == e) {
                    face_block(fq, VE, VE, bs, M);
                } else {
                    trace_values(c, f, d, d == f.left ? +1 : -1, VD);
                    face_block(fq, VE, VD, bs, M);
                }
                rows[f.axis].add(d, M.data(), sigma / c.msc[e], bs * bs);
            }
            for (int k = 0; k < c.dim; ++k) G[k].freeze_row(e, rows[k]);
        }
    });
}

/// E (ldg_core.hpp:412-439) or the Stokes pressure penalty E_p
/// (ldg_stokes.hpp:73-98) when `pressure` is set.
void penalty_rows(const Ctx& c, bool pressure, double beta_p, double delta, Rows& E) {
    const int N = c.mesh->n_elements(), bs = c.bs;
    E.resize(N, bs);
    parallel_for(N, [&](int lo, int hi) {
        std::vector<Face> faces;
        std::vector<double> VE, VO, M;
        for (int e = lo; e < hi; ++e) {
            if (!c.want(e)) continue;
            Row row;
            c.mesh->faces_of(e, faces);
            for (const Face& f : faces) {
                double tau;
                if (pressure) {
                    if (f.kind != F_INTERIOR) continue;
                    const double mu_f = std::max(c.mu[f.left], c.mu[f.right]);
                    const double rho_f = std::max(c.rho[f.left], c.rho[f.right]);
                    const double denom = mu_f + (delta > 0 ? rho_f * f.size * f.size / delta : 0.0);
                    tau = beta_p * f.size / denom;
                    if (tau == 0.0) continue;
                } else {
                    if (f.kind == F_NEUMANN) continue;
                    tau = c.penalty_tau(f);
                }
                const FaceQ fq = face_quad(c, f);
                if (f.kind == F_DIRICHLET) {
                    trace_values(c, f, e, f.side, VE);
                    face_block(fq, VE, VE, bs, M);
                    row.add(e, M.data(), tau, bs * bs);
                    continue;
                }
                const int other = e == f.left ? f.right : f.left;
                trace_values(c, f, e, e == f.left ? +1 : -1, VE);
                trace_values(c, f, other, other == f.left ? +1 : -1, VO);
                face_block(fq, VE, VE, bs, M);
                row.add(e, M.data(), tau, bs * bs);
                face_block(fq, VE, VO, bs, M);
                row.add(other, M.data(), -tau, bs * bs);
            }
            E.freeze_row(e, row);
        }
    });
}

/// Column adjacency of L (rows ascending), self row rotated to the front:
/// the source order of accumulate_AtDB (ldg_core.hpp:555-571).
std::vector<std::vector<std::pair<int, int>>> column_sources(const Rows& L, int N) {
    std::vector<std::vector<std::pair<int, int>>> src(N);
    for (int r = 0; r < N; ++r)
        for (int k = 0; k < int(L.cols[r].size()); ++k) src[L.cols[r][k]].push_back({r, k});
    for (int e = 0; e < N; ++e) {
        auto& s = src[e];
        for (size_t i = 0; i < s.size(); ++i)
            if (s[i].first == e && i != 0) {
                std::rotate(s.begin(), s.begin() + i, s.begin() + i + 1);
                break;
            }
    }
    return src;
}

/// dst_row(e) += sum_sources d_r * (B1^T B2)   (ldg_core.hpp:547-586; the
/// product summed k ascending then scaled, as the Eigen shim evaluates it)
void at_d_b_row(int e, const std::vector<std::pair<int, int>>& sources, const Rows& L, const Rows& R,
                const std::vector<double>& d, int bs, Row& dst, std::vector<double>& tmp) {
    tmp.resize(size_t(bs) * bs);
    for (const auto& [r, k1] : sources) {
        const double* B1 = L.block(r, k1);
        for (int k2 = 0; k2 < int(R.cols[r].size()); ++k2) {
            const double* B2 = R.block(r, k2);
            for (int j = 0; j < bs; ++j)
                for (int i = 0; i < bs; ++i) {
                    double s = 0.0;
                    for (int k = 0; k < bs; ++k) s += B1[size_t(k) * bs + i] * B2[size_t(k) * bs + j];
                    tmp[size_t(i) * bs + j] = d[r] * s;
                }
            double* out = dst.at(R.cols[r][k2], bs * bs);
            for (int i = 0; i < bs; ++i)
                for (int j = 0; j < bs; ++j) out[size_t(i) * bs + j] += tmp[size_t(i) * bs + j];
        }
    }
    (void)e;
}

void rows_to_csr(const Rows& R, int N, HostCsr& A) {
    A.brows = N;
    A.bs = R.bs;
    A.ptr.assign(N + 1, 0);
    for (int r = 0; r < N; ++r) A.ptr[r + 1] = A.ptr[r] + int(R.cols[r].size());
    A.col.resize(A.ptr[N]);
    A.val.resize(size_t(A.ptr[N]) * R.bs * R.bs);
    parallel_for(N, [&](int lo, int hi) {
        for (int r = lo; r < hi; ++r) {
            std::copy(R.cols[r].begin(), R.cols[r].end(), A.col.begin() + A.ptr[r]);
            std::copy(R.vals[r].begin(), R.vals[r].end(), A.val.begin() + size_t(A.ptr[r]) * R.bs * R.bs);
        }
    });
}

bool has_kind(const LevelMesh& m, int bc_kind) {
    for (int a = 0; a < m.dim; ++a)
        if (!m.periodic(a) && (m.bc[2 * a] == bc_kind || m.bc[2 * a + 1] == bc_kind)) return true;
    return false;
}

/// assemble_scalar (ldg_scalar.hpp:83-125), operator part
void assemble_scalar(const Ctx& c, HostCsr& A) {
    const int N = c.mesh->n_elements(), bs = c.bs;
    PhaseTimer tm("scalar");
    std::array<Rows, 3> G;
    gradient_rows(c, G);
    tm.stamp("gradient rows");
    Rows E;
    penalty_rows(c, false, 0.0, 0.0, E);
    tm.stamp("penalty rows");
    std::vector<double> dmu(N);
    for (int e = 0; e < N; ++e) dmu[e] = c.mu[e] * c.msc[e];
    std::array<std::vector<std::vector<std::pair<int, int>>>, 3> src;
    for (int k = 0; k < c.dim; ++k) src[k] = column_sources(G[k], N);
    Rows out;
    out.resize(N, bs);
    parallel_for(N, [&](int lo, int hi) {
        std::vector<double> tmp;
        for (int e = lo; e < hi; ++e) {
            if (!c.want(e)) continue;
            Row row;
            for (int k = 0; k < c.dim; ++k) at_d_b_row(e, src[k][e], G[k], G[k], dmu, bs, row, tmp);
            for (int kk = 0; kk < int(E.cols[e].size()); ++kk) row.add(E.cols[e][kk], E.block(e, kk), 1.0, bs * bs);
            out.freeze_row(e, row);
        }
    });
    tm.stamp("G^T D G + E");
    rows_to_csr(out, N, A);
    tm.stamp("csr");
}

/// assemble_stokes (ldg_stokes.hpp:102-192), operator part
void assemble_stokes(const Ctx& c, double gamma, double beta_p, double delta, HostCsr& A) {
    const int N = c.mesh->n_elements(), bsv = c.bs, dim = c.dim;
    const int BS = (dim + 1) * bsv;
    const bool unsteady = delta > 0;
    PhaseTimer tm("stokes");
    std::array<Rows, 3> G;
    gradient_rows(c, G);
    tm.stamp("gradient rows");
    Rows Ev, Ep;
    penalty_rows(c, false, 0.0, 0.0, Ev);
    penalty_rows(c, true, beta_p, delta, Ep);
    tm.stamp("penalty rows");
    std::vector<double> dmu(N);
    for (int e = 0; e < N; ++e) dmu[e] = c.mu[e] * c.msc[e];
    std::array<std::vector<std::vector<std::pair<int, int>>>, 3> src;
    for (int k = 0; k < dim; ++k) src[k] = column_sources(G[k], N);
    // visc = sum_k G_k^T M_mu G_k + Ev ; cross[i][j] = G_j^T M_mu G_i
    Rows visc;
    visc.resize(N, bsv);
    std::array<std::array<Rows, 3>, 3> cross;
    if (gamma != 0.0)
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) cross[i][j].resize(N, bsv);
    parallel_for(N, [&](int lo, int hi) {
        std::vector<double> tmp;
        for (int e = lo; e < hi; ++e) {
            if (!c.want(e)) continue;
            Row row;
            for (int k = 0; k < dim; ++k) at_d_b_row(e, src[k][e], G[k], G[k], dmu, bsv, row, tmp);
            for (int kk = 0; kk < int(Ev.cols[e].size()); ++kk)
                row.add(Ev.cols[e][kk], Ev.block(e, kk), 1.0, bsv * bsv);
            visc.freeze_row(e, row);
            if (gamma != 0.0)
                for (int i = 0; i < dim; ++i)
                    for (int j = 0; j < dim; ++j) {
                        Row cr;
                        at_d_b_row(e, src[j][e], G[j], G[i], dmu, bsv, cr, tmp);
                        cross[i][j].freeze_row(e, cr);
                    }
        }
    });
    tm.stamp("G^T D G (+cross)");
    // Scatter into the saddle layout, per destination row, in the
    // reference's global insertion order (ldg_stokes.hpp:149-191).
    // Pressure-velocity blocks come from G_i columns: (cc, r) gets -(G_i^T)msc_r.
    std::array<std::vector<std::vector<std::pair<int, int>>>, 3> gsrc;
    for (int i = 0; i < dim; ++i) gsrc[i] = column_sources(G[i], N);  // (r, k) with col == cc
    Rows out;
    out.resize(N, BS);
    parallel_for(N, [&](int lo, int hi) {
        std::vector<double> tr(size_t(bsv) * bsv);
        for (int r0 = lo; r0 < hi; ++r0) {
            if (!c.want(r0)) continue;
            Row row;
            auto add_sub = [&](int E2, int ci, int cj, const double* small, double s) {
                double* dst = row.at(E2, BS * BS);
                for (int a = 0; a < bsv; ++a) {
                    double* drow = dst + size_t(ci * bsv + a) * BS + cj * bsv;
                    const double* srow = small + size_t(a) * bsv;
                    for (int b = 0; b < bsv; ++b) drow[b] += s * srow[b];
                }
            };
            for (int k = 0; k < int(visc.cols[r0].size()); ++k)
                for (int i = 0; i < dim; ++i) add_sub(visc.cols[r0][k], i, i, visc.block(r0, k), 1.0);
            if (gamma != 0.0)
                for (int i = 0; i < dim; ++i)
                    for (int j = 0; j < dim; ++j) {
                        const Rows& C = cross[i][j];
                        for (int k = 0; k < int(C.cols[r0].size()); ++k)
                            add_sub(C.cols[r0][k], i, j, C.block(r0, k), gamma);
                    }
            // pressure coupling (ldg_stokes.hpp:169-180): every (sub-block, cell)
            // receives exactly one contribution, so only the values matter
            for (int i = 0; i < dim; ++i) {
                for (const auto& [r, kk] : gsrc[i][r0]) {  // G_i(r, r0): (i, p) of cell (r0, r)
                    const double* B = G[i].block(r, kk);
                    for (int a = 0; a < bsv; ++a)
                        for (int b = 0; b < bsv; ++b) tr[size_t(a) * bsv + b] = B[size_t(b) * bsv + a];
                    add_sub(r, i, dim, tr.data(), -c.msc[r]);
                }
                for (int k = 0; k < int(G[i].cols[r0].size()); ++k)
                    add_sub(G[i].cols[r0][k], dim, i, G[i].block(r0, k), -c.msc[r0]);
            }
            for (int k = 0; k < int(Ep.cols[r0].size()); ++k) add_sub(Ep.cols[r0][k], dim, dim, Ep.block(r0, k), -1.0);
            if (unsteady) {
                const double m = c.rho[r0] * c.msc[r0] / delta;
                double* dst = row.at(r0, BS * BS);
                for (int i = 0; i < dim; ++i)
                    for (int a = 0; a < bsv; ++a) dst[size_t(i * bsv + a) * BS + i * bsv + a] += m;
            }
            out.freeze_row(r0, row);
        }
    });
    tm.stamp("saddle scatter");
    rows_to_csr(out, N, A);
    tm.stamp("csr");
}

}  // namespace

namespace {
/// Rows within `hops` face-graph steps of the element range [r0, r1).
std::vector<char> halo_rows(const LevelMesh& m, int r0, int r1, int hops) {
    const int N = m.n_elements();
    std::vector<char> in(N, 0);
    std::vector<int> frontier, next;
    for (int e = r0; e < r1; ++e) {
        in[e] = 1;
        frontier.push_back(e);
    }
    std::vector<Face> faces;
    for (int h = 0; h < hops && !frontier.empty(); ++h) {
        next.clear();
        for (int e : frontier) {
            m.faces_of(e, faces);
            for (const Face& f : faces) {
                if (f.kind != F_INTERIOR) continue;
                const int o = f.left == e ? f.right : f.left;
                if (!in[o]) {
                    in[o] = 1;
                    next.push_back(o);
                }
            }
        }
        frontier.swap(next);
    }
    return in;
}
/// rows plus their face neighbours (the G / E rows an operator row needs)
std::vector<char> with_neighbours(const LevelMesh& m, const std::vector<char>& rows) {
    std::vector<char> g(rows);
    std::vector<Face> faces;
    for (int e = 0; e < m.n_elements(); ++e) {
        if (!rows[e]) continue;
        m.faces_of(e, faces);
        for (const Face& f : faces)
            if (f.kind == F_INTERIOR) g[f.left == e ? f.right : f.left] = 1;
    }
    return g;
}

// ------------------------------------------------ deferred (device) assembly
/// Stored-block table of the program: the rows of the given Rows objects
/// concatenated (bsv^2 doubles per block); base[t][r] = first block of row r.
struct BlockTable {
    std::vector<std::vector<int64_t>> base;
    int64_t total = 0;
    void add(const Rows& R) {
        std::vector<int64_t> b(R.cols.size() + 1, 0);
        for (size_t r = 0; r < R.cols.size(); ++r) b[r + 1] = b[r] + int64_t(R.cols[r].size());
        for (auto& v : b) v += total;
        total = b.back();
        base.push_back(std::move(b));
    }
    int id(int t, int r, int k) const { return int(base[t][r] + k); }
};

void fill_blocks(const std::vector<const Rows*>& rows, LevelProgram& P, int bsv) {
    int64_t total = 0;
    for (const Rows* R : rows)
        for (const auto& c : R->cols) total += int64_t(c.size());
    P.blocks.resize(size_t(total) * bsv * bsv);
    std::vector<int64_t> off;
    int64_t o = 0;
    for (const Rows* R : rows)
        for (size_t r = 0; r < R->cols.size(); ++r) {
            off.push_back(o);
            o += int64_t(R->cols[r].size());
        }
    size_t idx = 0;
    for (const Rows* R : rows) {
        const size_t base = idx;
        parallel_for(int(R->cols.size()), [&](int lo, int hi) {
            for (int r = lo; r < hi; ++r)
                std::copy(R->vals[r].begin(), R->vals[r].end(), P.blocks.begin() + off[base + r] * bsv * bsv);
        });
        idx += R->cols.size();
    }
}

/// One recorded inner block: prods (b1, b2, d) in accumulation order, then
/// an optional stored block added with scale 1.
struct SymCell {
    std::vector<int> b1, b2;
    std::vector<double> d;
    int add = -1;
};
using SymRow = std::map<int, SymCell>;

/// at_d_b_row, recorded: the same source / block visiting order.
void sym_at_d_b_row(const std::vector<std::pair<int, int>>& sources, const Rows& L, int tL, const Rows& R, int tR,
                    const BlockTable& T, const std::vector<double>& d, SymRow& dst) {
    for (const auto& [r, k1] : sources)
        for (int k2 = 0; k2 < int(R.cols[r].size()); ++k2) {
            SymCell& cell = dst[R.cols[r][k2]];
            cell.b1.push_back(T.id(tL, r, k1));
            cell.b2.push_back(T.id(tR, r, k2));
            cell.d.push_back(d[r]);
        }
}

/// Appends the inner blocks of `rows` (row-major in row, ascending columns)
/// to the program; returns, per row, the inner ids of its cells.
std::vector<std::vector<std::pair<int, int>>> emit_inner(std::vector<SymRow>& rows, LevelProgram& P) {
    std::vector<std::vector<std::pair<int, int>>> ids(rows.size());
    for (size_t r = 0; r < rows.size(); ++r)
        for (auto& [j, cell] : rows[r]) {
            const int id = int(P.inner_ptr.size()) - 1;
            ids[r].push_back({j, id});
            P.prod_b1.insert(P.prod_b1.end(), cell.b1.begin(), cell.b1.end());
            P.prod_b2.insert(P.prod_b2.end(), cell.b2.begin(), cell.b2.end());
            P.prod_d.insert(P.prod_d.end(), cell.d.begin(), cell.d.end());
            P.inner_ptr.push_back(int64_t(P.prod_b1.size()));
            P.inner_add.push_back(cell.add);
        }
    return ids;
}

struct Term {
    int kind, idx;
    double scale;
};

/// program_scalar: assemble_scalar (ldg_scalar.hpp:83-125) recorded.
void program_scalar(const Ctx& c, LevelProgram& P) {
    const int N = c.mesh->n_elements(), bs = c.bs;
    std::array<Rows, 3> G;
    gradient_rows(c, G);
    Rows E;
    penalty_rows(c, false, 0.0, 0.0, E);
    std::vector<double> dmu(N);
    for (int e = 0; e < N; ++e) dmu[e] = c.mu[e] * c.msc[e];
    std::array<std::vector<std::vector<std::pair<int, int>>>, 3> src;
    for (int k = 0; k < c.dim; ++k) src[k] = column_sources(G[k], N);
    BlockTable T;
    std::vector<const Rows*> tabs;
    for (int k = 0; k < c.dim; ++k) {
        T.add(G[k]);
        tabs.push_back(&G[k]);
    }
    const int tE = c.dim;
    T.add(E);
    tabs.push_back(&E);
    P.n = N;
    P.bs = P.bsv = bs;
    P.ncomp = 1;
    fill_blocks(tabs, P, bs);
    std::vector<SymRow> rows(N);
    parallel_for(N, [&](int lo, int hi) {
        for (int e = lo; e < hi; ++e) {
            if (!c.want(e)) continue;
            for (int k = 0; k < c.dim; ++k) sym_at_d_b_row(src[k][e], G[k], k, G[k], k, T, dmu, rows[e]);
            for (int kk = 0; kk < int(E.cols[e].size()); ++kk) rows[e][E.cols[e][kk]].add = T.id(tE, e, kk);
        }
    });
    const auto ids = emit_inner(rows, P);
    P.ptr.assign(N + 1, 0);
    for (int e = 0; e < N; ++e) {
        P.ptr[e + 1] = P.ptr[e] + int(ids[e].size());
        for (const auto& [j, id] : ids[e]) {
            P.col.push_back(j);
            P.term_kind.push_back(3);
            P.term_idx.push_back(id);
            P.term_scale.push_back(1.0);
            P.term_ptr.push_back(int64_t(P.term_kind.size()));
        }
    }
}

/// program_stokes: assemble_stokes (ldg_stokes.hpp:102-192) recorded.
void program_stokes(const Ctx& c, double gamma, double beta_p, double delta, LevelProgram& P) {
    const int N = c.mesh->n_elements(), bsv = c.bs, dim = c.dim, nc = dim + 1;
    const bool unsteady = delta > 0;
    std::array<Rows, 3> G;
    gradient_rows(c, G);
    Rows Ev, Ep;
    penalty_rows(c, false, 0.0, 0.0, Ev);
    penalty_rows(c, true, beta_p, delta, Ep);
    std::vector<double> dmu(N);
    for (int e = 0; e < N; ++e) dmu[e] = c.mu[e] * c.msc[e];
    std::array<std::vector<std::vector<std::pair<int, int>>>, 3> src;
    for (int k = 0; k < dim; ++k) src[k] = column_sources(G[k], N);
    BlockTable T;
    std::vector<const Rows*> tabs;
    for (int k = 0; k < dim; ++k) {
        T.add(G[k]);
        tabs.push_back(&G[k]);
    }
    const int tEv = dim, tEp = dim + 1;
    T.add(Ev);
    tabs.push_back(&Ev);
    T.add(Ep);
    tabs.push_back(&Ep);
    P.n = N;
    P.bsv = bsv;
    P.ncomp = nc;
    P.bs = nc * bsv;
    fill_blocks(tabs, P, bsv);
    // inner blocks: visc rows, then cross[i][j] rows
    std::vector<SymRow> visc(N);
    std::vector<std::vector<SymRow>> cross(gamma != 0.0 ? dim * dim : 0, std::vector<SymRow>(N));
    parallel_for(N, [&](int lo, int hi) {
        for (int e = lo; e < hi; ++e) {
            if (!c.want(e)) continue;
            for (int k = 0; k < dim; ++k) sym_at_d_b_row(src[k][e], G[k], k, G[k], k, T, dmu, visc[e]);
            for (int kk = 0; kk < int(Ev.cols[e].size()); ++kk) visc[e][Ev.cols[e][kk]].add = T.id(tEv, e, kk);
            if (gamma != 0.0)
                for (int i = 0; i < dim; ++i)
                    for (int j = 0; j < dim; ++j)
                        sym_at_d_b_row(src[j][e], G[j], j, G[i], i, T, dmu, cross[i * dim + j][e]);
        }
    });
    const auto vids = emit_inner(visc, P);
    std::vector<std::vector<std::vector<std::pair<int, int>>>> cids;
    for (auto& cr : cross) cids.push_back(emit_inner(cr, P));
    std::array<std::vector<std::vector<std::pair<int, int>>>, 3> gsrc;
    for (int i = 0; i < dim; ++i) gsrc[i] = column_sources(G[i], N);
    // final rows: per cell the sub-block term lists in the saddle scatter's order
    using CellTerms = std::vector<std::vector<Term>>;  // [sub-block] -> terms
    std::vector<std::map<int, CellTerms>> fin(N);
    parallel_for(N, [&](int lo, int hi) {
        for (int r0 = lo; r0 < hi; ++r0) {
            if (!c.want(r0)) continue;
            auto& row = fin[r0];
            auto add = [&](int cell, int ci, int cj, Term t) {
                auto& ct = row[cell];
                if (ct.empty()) ct.resize(size_t(nc) * nc);
                ct[size_t(ci) * nc + cj].push_back(t);
            };
            for (const auto& [j, id] : vids[r0])
                for (int i = 0; i < dim; ++i) add(j, i, i, {0, id, 1.0});
            if (gamma != 0.0)
                for (int i = 0; i < dim; ++i)
                    for (int j = 0; j < dim; ++j)
                        for (const auto& [cc, id] : cids[size_t(i) * dim + j][r0]) add(cc, i, j, {0, id, gamma});
            for (int i = 0; i < dim; ++i) {
                for (const auto& [r, kk] : gsrc[i][r0]) add(r, i, dim, {2, T.id(i, r, kk), -c.msc[r]});
                for (int k = 0; k < int(G[i].cols[r0].size()); ++k)
                    add(G[i].cols[r0][k], dim, i, {1, T.id(i, r0, k), -c.msc[r0]});
            }
            for (int k = 0; k < int(Ep.cols[r0].size()); ++k) add(Ep.cols[r0][k], dim, dim, {1, T.id(tEp, r0, k), -1.0});
            if (unsteady) {
                const double m = c.rho[r0] * c.msc[r0] / delta;
                for (int i = 0; i < dim; ++i) add(r0, i, i, {4, 0, m});
            }
        }
    });
    P.ptr.assign(N + 1, 0);
    for (int r0 = 0; r0 < N; ++r0) {
        P.ptr[r0 + 1] = P.ptr[r0] + int(fin[r0].size());
        for (auto& [cell, ct] : fin[r0]) {
            P.col.push_back(cell);
            for (const auto& terms : ct) {
                for (const Term& t : terms) {
                    P.term_kind.push_back(t.kind);
                    P.term_idx.push_back(t.idx);
                    P.term_scale.push_back(t.scale);
                }
                P.term_ptr.push_back(int64_t(P.term_kind.size()));
            }
        }
    }
}

}  // namespace

void problem_build(const ldgmg_problem_spec& s, int min_depth, int bottom_max_elements, Problem& P) {
    problem_build_partial(s, min_depth, bottom_max_elements, 1, 0, 0, 0, P);
}

void problem_build_partial(const ldgmg_problem_spec& s, int min_depth, int bottom_max_elements, int nranks,
                           int rank, int halo_hops, int min_rows_per_rank, Problem& P, bool deferred, bool any_n) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(LDGMG_ERR_INVALID_ARGUMENT, "partition: bad rank / rank count");
    if (halo_hops < 0) fail(LDGMG_ERR_INVALID_ARGUMENT, "partition: negative halo");
    if (s.dim != 2 && s.dim != 3) fail(LDGMG_ERR_INVALID_ARGUMENT, "mesh: dim must be 2 or 3");
    if (s.kind != LDGMG_SYSTEM_SCALAR && s.kind != LDGMG_SYSTEM_STOKES)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "problem: unknown system kind");
    const int degree_cap = s.dim == 2 ? 5 : 3;
    if (s.degree < 1 || s.degree > degree_cap)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "ldg: polynomial degree out of supported range");
    if (s.kind == LDGMG_SYSTEM_STOKES) {
        if (s.gamma != 0.0 && s.gamma != 1.0) fail(LDGMG_ERR_INVALID_ARGUMENT, "stokes: gamma must be 0 or 1");
        if (s.beta_p < 0) fail(LDGMG_ERR_INVALID_ARGUMENT, "stokes: beta_p must be >= 0");
    }
    P.spec = s;
    P.kind = s.kind;
    P.dim = s.dim;
    P.degree = s.degree;
    const Basis B(s.degree, s.dim);
    P.bs_scalar = B.bs;
    P.n_comp = s.kind == LDGMG_SYSTEM_SCALAR ? 1 : s.dim + 1;

    // region table
    std::vector<Region> regs;
    const bool curved = s.phase_shape == LDGMG_PHASE_BALL || s.phase_shape == LDGMG_PHASE_ELLIPSE;
    if (s.phase_shape == LDGMG_PHASE_BOXES) {
        Region in;
        in.lo = {s.center[0], s.center[1], s.center[2]};
        in.hi = {s.radii[0], s.radii[1], s.radii[2]};
        in.mu = s.mu_in;
        in.rho = s.rho_in;
        Region out;
        out.mu = s.mu_out;
        out.rho = s.rho_out;
        regs = {in, out};
    } else if (!curved) {
        Region one;
        one.mu = s.mu_out;
        one.rho = s.rho_out;
        regs = {one};
    }

    // mesh chain (multigrid.hpp:168-194)
    std::vector<LevelMesh> meshes;
    meshes.push_back(uniform_mesh(s.n, s.dim, s.bc, any_n));
    if (s.phase_shape == LDGMG_PHASE_BOXES) assign_box_phases(meshes[0], regs);
    for (;;) {
        const LevelMesh& m = meshes.back();
        if (m.n < 4) break;  // coarsen: uniform mesh already at n=2
        if (m.n & 1) break;  // A1: an odd count has no sibling groups (48 -> 24 -> 12 -> 6 -> 3)
        LevelMesh cm = uniform_mesh(m.n / 2, m.dim, m.bc, any_n);
        const int group = 1 << m.dim;
        bool phase_ok = true;
        for (int p = 0; p < cm.n_elements(); ++p) {
            cm.phase[p] = m.phase[size_t(p) * group];
            for (int c = 0; c < group; ++c) phase_ok &= m.phase[size_t(p) * group + c] == cm.phase[p];
        }
        if (!phase_ok) break;
        meshes.push_back(std::move(cm));
    }
    if (int(meshes.size()) < min_depth)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "multigrid: hierarchy depth below the configured minimum");
    if (meshes.back().n_elements() > bottom_max_elements)
        fail(LDGMG_ERR_INVALID_ARGUMENT, "multigrid: bottom level exceeds the element budget");

    P.levels.clear();
    P.levels.resize(meshes.size());
    bool partial_prefix = true;
    for (size_t l = 0; l < meshes.size(); ++l) {
        LevelMesh& m = meshes[l];
        std::vector<Region> lregs = regs;
        if (curved) {
            bool any_in = false, any_out = false;
            for (int e = 0; e < m.n_elements(); ++e) (inside_curved(s, m, e) ? any_in : any_out) = true;
            lregs.clear();
            Region in, out;
            in.mu = s.mu_in;
            in.rho = s.rho_in;
            out.mu = s.mu_out;
            out.rho = s.rho_out;
            if (any_in) lregs.push_back(in);
            if (any_out) lregs.push_back(out);
            for (int e = 0; e < m.n_elements(); ++e)
                m.phase[e] = (inside_curved(s, m, e) || !any_out) ? 0 : (any_in ? 1 : 0);
        }
        Ctx c;
        c.mesh = &m;
        c.B = &B;
        c.dim = s.dim;
        c.bs = B.bs;
        c.p1 = B.p1;
        c.beta = s.beta > 0 ? s.beta : 4.0 * s.degree * s.degree;
        const int N = m.n_elements();
        c.msc.resize(N);
        c.mu.resize(N);
        c.rho.resize(N);
        std::vector<int> owned(lregs.size(), 0);
        for (int e = 0; e < N; ++e) {
            if (m.phase[e] < 0 || m.phase[e] >= int(lregs.size()))
                fail(LDGMG_ERR_INVALID_ARGUMENT, "ldg: element phase outside the region table");
            ++owned[m.phase[e]];
            c.msc[e] = mass_scalar(m.h, s.dim);
            c.mu[e] = lregs[m.phase[e]].mu;
            c.rho[e] = lregs[m.phase[e]].rho;
        }
        for (int o : owned)
            if (o == 0) fail(LDGMG_ERR_INVALID_ARGUMENT, "ldg: phase region owns no elements");
        ProblemLevel& L = P.levels[l];
        L.n = m.n;
        L.phase = m.phase;
        L.partial = false;
        // distributed levels (the same rule as parallel.DistMultigrid): the
        // rank's range plus `halo_hops` face layers; smaller levels in full
        // the partitioned levels are a prefix of the hierarchy, and a level is
        // partitioned only if no rank boundary splits a sibling group of its
        // restriction (parallel.partition_depth applies the same rule)
        bool aligned = true;
        for (int q = 1; q < nranks; ++q)
            aligned &= int(int64_t(q) * N / nranks) % (1 << s.dim) == 0;
        partial_prefix = partial_prefix && nranks > 1 && N >= nranks * min_rows_per_rank && l + 1 < meshes.size() &&
                         aligned;
        if (partial_prefix) {
            const int r0 = int(int64_t(rank) * N / nranks), r1 = int(int64_t(rank + 1) * N / nranks);
            c.rows = halo_rows(m, r0, r1, halo_hops);
            c.grows = with_neighbours(m, c.rows);
            L.partial = true;
        }
        L.deferred = deferred;
        if (s.kind == LDGMG_SYSTEM_SCALAR) {
            if (deferred)
                program_scalar(c, L.prog);
            else
                assemble_scalar(c, L.A);
        } else {
            if (has_kind(m, LDGMG_BC_NEUMANN) && s.gamma == 0.0)
                fail(LDGMG_ERR_INVALID_ARGUMENT, "stokes: stress boundary conditions require the stress form");
            if (deferred)
                program_stokes(c, s.gamma, s.beta_p, s.delta, L.prog);
            else
                assemble_stokes(c, s.gamma, s.beta_p, s.delta, L.A);
        }
        if (deferred) {  // shape of the (device-built) operator for the level queries
            L.A.brows = L.prog.n;
            L.A.bs = L.prog.bs;
            L.A.ptr = L.prog.ptr;
            L.A.col = L.prog.col;
        }
        if (l + 1 < meshes.size()) {
            const int group = 1 << s.dim;
            L.parent_of.resize(N);
            L.orthant_of.resize(N);
            for (int f = 0; f < N; ++f) {
                L.parent_of[f] = f / group;
                int orth = 0;
                for (int a = 0; a < s.dim; ++a) orth |= (m.idx[f][a] & 1) << a;
                L.orthant_of[f] = orth;
            }
        }
    }
    const LevelMesh& fine = meshes[0];
    if (s.kind == LDGMG_SYSTEM_SCALAR) {
        P.kernel_constants = !has_kind(fine, LDGMG_BC_DIRICHLET);
        P.kernel_pressure = 0;
    } else {
        P.kernel_constants = !has_kind(fine, LDGMG_BC_DIRICHLET) && !(s.delta > 0);
        P.kernel_pressure = !has_kind(fine, LDGMG_BC_NEUMANN);
    }

    P.inject = injection_matrices(s.dim, s.degree);
}

/// build_injection (multigrid.hpp:212-241): 1D maps T[s]_ij = sum_q w_q P_i(x_q)
/// P_j((x_q + 2s - 1)/2), Kronecker products over the child orthants.
std::vector<double> injection_matrices(int dim, int degree) {
    const Basis B(degree, dim);
    const int p1 = B.p1, bs = B.bs;
    std::array<std::vector<double>, 2> T;
    for (int sd = 0; sd < 2; ++sd) {
        T[sd].assign(size_t(p1) * p1, 0.0);
        for (int i = 0; i < p1; ++i)
            for (int j = 0; j < p1; ++j) {
                double acc = 0.0;
                for (int q = 0; q < p1; ++q)
                    acc += B.weights[q] * B.val[i * p1 + q] * mode_val(j, 0.5 * (B.nodes[q] + 2.0 * sd - 1.0));
                T[sd][size_t(i) * p1 + j] = acc;
            }
    }
    const int nk = 1 << dim;
    std::vector<double> K(size_t(nk) * bs * bs, 0.0);
    for (int o = 0; o < nk; ++o)
        for (int i = 0; i < bs; ++i) {
            const auto ix = B.decompose(i);
            for (int j = 0; j < bs; ++j) {
                const auto jx = B.decompose(j);
                double v = 1.0;
                for (int a = 0; a < dim; ++a) v *= T[(o >> a) & 1][size_t(ix[a]) * p1 + jx[a]];
                K[(size_t(o) * bs + i) * bs + j] = v;
            }
        }
    return K;
}

}  // namespace ldgmg_b200
