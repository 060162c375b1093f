// lx_hostmath.cpp -- host-side scalar math of the LeXInt path (product side).
//
// Leja points (§2.1), phi_l and Newton divided differences
// (P:141).  O(M^2) scalar work independent of the grid size; the
// data-parallel path runs in the CUDA kernels.  Independent of oracle/.
#include "lx_hostmath.h"

#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

namespace lx {

// ----------------------------------------------------------------- phi_l
// phi_l(z) = sum_{k>=0} z^k / (k+l)!  evaluated by Horner for |z| < 2,
// phi_0 = exp and phi_{j+1} = (phi_j - 1/j!)/z otherwise.
static const double kInvFact[] = {1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0};

double phi(int l, double z) {
    if (std::fabs(z) < 2.0) {
        // coefficients 1/(k+l)! for k = 0..NT-1, Horner from the top
        constexpr int NT = 34;  // 2^34/34! ~ 1e-29
        double c[NT];
        double f = kInvFact[l];
        c[0] = f;
        for (int k = 1; k < NT; k++) {
            f /= (double)(k + l);
            c[k] = f;
        }
        double s = c[NT - 1];
        for (int k = NT - 2; k >= 0; k--) s = std::fma(s, z, c[k]);
        return s;
    }
    double p = std::exp(z);
    for (int j = 0; j < l; j++) p = (p - kInvFact[j]) / z;
    return p;
}

// ----------------------------------------------------------------- Leja points
// Greedy maximisation of prod_k |z - xi_k| on [-2, 2].  For j >= 2 the
// maximiser of each gap between consecutive sorted nodes is the root of
// g(z) = sum_k 1/(z - xi_k); found by safeguarded Newton (bisection
// fallback).  Best gap by log-product; ties within 1e-12 -> larger z.
static double g_val(const std::vector<double>& x, double z, double* dg) {
    double s = 0.0, s2 = 0.0;
    for (double xk : x) {
        const double r = 1.0 / (z - xk);
        s += r;
        s2 += r * r;
    }
    *dg = -s2;
    return s;
}

static double gap_max(const std::vector<double>& x, double a, double b) {
    double lo = a, hi = b, z = 0.5 * (a + b);
    for (int it = 0; it < 200; it++) {
        double dg;
        const double g = g_val(x, z, &dg);
        if (g == 0.0) return z;
        if (g > 0.0) lo = z; else hi = z;
        double zn = z - g / dg;
        if (!(zn > lo && zn < hi)) zn = 0.5 * (lo + hi);
        if (zn == z || hi - lo <= 4e-16 * std::max(1.0, std::fabs(z))) return zn;
        z = zn;
    }
    return z;
}

static std::mutex g_leja_mu;
static std::vector<double> g_leja;  // immutable prefix once computed

static void extend_leja(int count) {
    std::vector<double>& x = g_leja;
    if (x.empty()) x.push_back(2.0);
    if ((int)x.size() < count && x.size() == 1) x.push_back(-2.0);
    while ((int)x.size() < count) {
        std::vector<double> s = x;
        std::sort(s.begin(), s.end());
        double best_z = 0.0, best_L = -INFINITY;
        for (size_t gi = 0; gi + 1 < s.size(); gi++) {
            const double z = gap_max(x, s[gi], s[gi + 1]);
            double L = 0.0;
            for (double xk : x) L += std::log(std::fabs(z - xk));
            if (L > best_L + 1e-12 || (std::fabs(L - best_L) <= 1e-12 && z > best_z)) {
                best_L = L;
                best_z = z;
            }
        }
        x.push_back(best_z);
    }
}

int leja_points(int count, double* out) {
    if (count < 1 || count > 4096 || !out) return 1;
    std::lock_guard<std::mutex> lk(g_leja_mu);
    if ((int)g_leja.size() < count) extend_leja(count);
    std::copy(g_leja.begin(), g_leja.begin() + count, out);
    return 0;
}

// ----------------------------------------------------------------- divided differences
// Newton divided differences of h(xi) = phi_l(a*dt*(c + gamma*xi)) by the
// triangular recurrence, row-wise so the inner loop is independent per j.
int divided_differences(int l, const double* xi, int m, double dt, double c, double gamma, double a,
                        double* d) {
    if (m < 1 || !xi || !d) return 1;
    if (l < 0 || l > 4) return 4;
    const double s = a * dt;
    for (int k = 0; k < m; k++) d[k] = phi(l, s * (c + gamma * xi[k]));
    for (int i = 1; i < m; i++) {
        const double di = d[i - 1], xi_i = xi[i - 1];
        for (int j = i; j < m; j++) d[j] = (d[j] - di) / (xi[j] - xi_i);
    }
    for (int k = 0; k < m; k++)
        if (!std::isfinite(d[k])) return 6;
    return 0;
}

}  // namespace lx
