// Host symmetric eigensolver used at SETUP time only (per-element diagonal
// factors when the caller does not supply them, and the bottom-level dense
// pseudoinverse).  Householder tridiagonalisation followed by the implicit
// QL iteration (the classic tred2/tql2 algorithm, restated here); eigenvalues
// ascending with eigenvectors as columns, like the reference's
// SelfAdjointEigenSolver contract (blockla.hpp:318-326).  The hot path never
// calls this.
#include "host_eig.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <cstring>
#include <thread>

namespace ldgmg_b200 {

namespace {

// a: n x n column-major symmetric (lower triangle used), overwritten by Q;
// d: diagonal, e: sub-diagonal (e[0] = 0 on exit).
void tred2(int n, std::vector<double>& V, std::vector<double>& d, std::vector<double>& e) {
    auto v = [&](int i, int j) -> double& { return V[size_t(j) * n + i]; };
    for (int j = 0; j < n; ++j) d[j] = v(n - 1, j);
    for (int i = n - 1; i > 0; --i) {
        double scale = 0.0, h = 0.0;
        for (int k = 0; k < i; ++k) scale += std::abs(d[k]);
        if (scale == 0.0) {
            e[i] = d[i - 1];
            for (int j = 0; j < i; ++j) {
                d[j] = v(i - 1, j);
                v(i, j) = 0.0;
                v(j, i) = 0.0;
            }
        } else {
            for (int k = 0; k < i; ++k) {
                d[k] /= scale;
                h += d[k] * d[k];
            }
            double f = d[i - 1];
            double g = std::sqrt(h);
            if (f > 0) g = -g;
            e[i] = scale * g;
            h -= f * g;
            d[i - 1] = f - g;
            for (int j = 0; j < i; ++j) e[j] = 0.0;
            for (int j = 0; j < i; ++j) {
                f = d[j];
                v(j, i) = f;
                g = e[j] + v(j, j) * f;
                for (int k = j + 1; k <= i - 1; ++k) {
                    g += v(k, j) * d[k];
                    e[k] += v(k, j) * f;
                }
                e[j] = g;
            }
            f = 0.0;
            for (int j = 0; j < i; ++j) {
                e[j] /= h;
                f += e[j] * d[j];
            }
            const double hh = f / (h + h);
            for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
            for (int j = 0; j < i; ++j) {
                f = d[j];
                g = e[j];
                for (int k = j; k <= i - 1; ++k) v(k, j) -= (f * e[k] + g * d[k]);
                d[j] = v(i - 1, j);
                v(i, j) = 0.0;
            }
        }
        d[i] = h;
    }
    for (int i = 0; i < n - 1; ++i) {
        v(n - 1, i) = v(i, i);
        v(i, i) = 1.0;
        const double h = d[i + 1];
        if (h != 0.0) {
            for (int k = 0; k <= i; ++k) d[k] = v(k, i + 1) / h;
            for (int j = 0; j <= i; ++j) {
                double g = 0.0;
                for (int k = 0; k <= i; ++k) g += v(k, i + 1) * v(k, j);
                for (int k = 0; k <= i; ++k) v(k, j) -= g * d[k];
            }
        }
        for (int k = 0; k <= i; ++k) v(k, i + 1) = 0.0;
    }
    for (int j = 0; j < n; ++j) {
        d[j] = v(n - 1, j);
        v(n - 1, j) = 0.0;
    }
    v(n - 1, n - 1) = 1.0;
    e[0] = 0.0;
}

bool tql2(int n, std::vector<double>& V, std::vector<double>& d, std::vector<double>& e) {
    auto v = [&](int i, int j) -> double& { return V[size_t(j) * n + i]; };
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    double f = 0.0, tst1 = 0.0;
    const double eps = std::ldexp(1.0, -52);
    for (int l = 0; l < n; ++l) {
        tst1 = std::max(tst1, std::abs(d[l]) + std::abs(e[l]));
        int m = l;
        while (m < n) {
            if (std::abs(e[m]) <= eps * tst1) break;
            ++m;
        }
        if (m == n) m = n - 1;
        if (m > l) {
            int iter = 0;
            do {
                if (++iter > 200) return false;
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = std::hypot(p, 1.0);
                if (p < 0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < n; ++i) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1.0, c2 = c, c3 = c;
                const double el1 = e[l + 1];
                double s = 0.0, s2 = 0.0;
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * p;
                    r = std::hypot(p, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = p / r;
                    p = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    for (int k = 0; k < n; ++k) {
                        h = v(k, i + 1);
                        v(k, i + 1) = s * v(k, i) + c * h;
                        v(k, i) = c * v(k, i) - s * h;
                    }
                }
                p = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * p;
                d[l] = c * p;
            } while (std::abs(e[l]) > eps * tst1);
        }
        d[l] = d[l] + f;
        e[l] = 0.0;
    }
    // ascending order
    for (int i = 0; i < n - 1; ++i) {
        int k = i;
        double p = d[i];
        for (int j = i + 1; j < n; ++j)
            if (d[j] < p) {
                k = j;
                p = d[j];
            }
        if (k != i) {
            d[k] = d[i];
            d[i] = p;
            for (int j = 0; j < n; ++j) std::swap(v(j, i), v(j, k));
        }
    }
    return true;
}

}  // namespace

void sym_eig_host(int n, const double* A, double* lambda, double* V) {
    if (n == 0) return;
    std::vector<double> Vm(A, A + size_t(n) * n), d(n), e(n);
    // symmetric input: use the lower triangle (column-major) like LAPACK 'L'
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < j; ++i) Vm[size_t(j) * n + i] = Vm[size_t(i) * n + j];
    tred2(n, Vm, d, e);
    if (!tql2(n, Vm, d, e)) throw std::runtime_error("sym_eig: solver failed");
    std::copy(d.begin(), d.end(), lambda);
    std::copy(Vm.begin(), Vm.end(), V);
}

void parallel_for(int n, const std::function<void(int, int)>& body) {
    unsigned hw = std::thread::hardware_concurrency();
    int nt = int(std::max(1u, std::min(hw ? hw : 1u, 64u)));
    nt = std::min(nt, std::max(1, n / 16));
    if (nt <= 1) {
        body(0, n);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) {
        const int lo = int(int64_t(n) * t / nt), hi = int(int64_t(n) * (t + 1) / nt);
        pool.emplace_back([&, lo, hi] { body(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kPerThread = size_t(1) << 20;
    unsigned hw = std::thread::hardware_concurrency();
    const int nt = int(std::min<size_t>(std::min(8u, std::max(1u, hw)), std::max<size_t>(1, bytes / kPerThread)));
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) {
        const size_t lo = bytes * t / nt, hi = bytes * (t + 1) / nt;
        pool.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
        });
    }
    std::memcpy(dst, src, bytes / nt);
    for (auto& th : pool) th.join();
}

}  // namespace ldgmg_b200
