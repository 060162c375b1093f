/*
 * lxoracle.c -- CPU ORACLE for the LeXInt hot path (arxiv 2310.08344).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * The product (paper_2310_08344_b200/) never includes, links or calls it,
 * and this file includes nothing from the product.
 *
 * Plain, slow, obviously-correct fp64 C: plain loops, no blocking, no fusion,
 * no reordering beyond what the paper's definitions state.  Every function
 * cites the passage it follows:
 *   P:<line>  = /root/reference/PAPER.md line (section / equation / listing)
 *   S:<line>  = /root/reference/SPEC.md line
 *   R<k>      = reading k of DESIGN.md "Readings of the paper" (= SURVEY 8(c)).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): mpmath phi values, closed
 * forms, brute-force Leja greedy property, dense expm / augmented-matrix phi,
 * FFT-exact solutions of the circulant stencil operators, convergence orders.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

/* Parallel build (bench.py's all-core cpu_baseline only; -fopenmp): the element-wise loops below are
 * split over threads with `OC_PARFOR` and the pairwise norm evaluates the top 6 levels of its
 * recursion tree in parallel -- the same tree, so every result is bit-identical to the serial build
 * (tests/test_oracle_scalar.py checks it).  Without -fopenmp the pragmas vanish. */
#ifdef _OPENMP
#define OC_PARFOR _Pragma("omp parallel for schedule(static)")
#else
#define OC_PARFOR
#endif

#define OC_OK 0
#define OC_ERR_ARG 1
#define OC_ERR_UNSUPPORTED 4
#define OC_ERR_NOCONV 5
#define OC_ERR_NONFINITE 6

/* ------------------------------------------------------------------------- */
/* vector helpers ("vecops")                                          */
/* ------------------------------------------------------------------------- */

/* Pairwise sum of x[i]^2 over [lo, hi) (pairwise summation). */
static double sumsq_pairwise(const double *x, long lo, long hi)
{
    if (hi - lo <= 8) {
        double s = 0.0;
        for (long i = lo; i < hi; i++) s += x[i] * x[i];
        return s;
    }
    long mid = lo + (hi - lo) / 2;
    return sumsq_pairwise(x, lo, mid) + sumsq_pairwise(x, mid, hi);
}

#ifdef _OPENMP
/* leaves of the pairwise recursion at depth 6 (same midpoints as sumsq_pairwise) */
static void oc_leaves(long lo, long hi, int depth, long *los, long *his, int *k)
{
    if (depth == 6) { los[*k] = lo; his[*k] = hi; (*k)++; return; }
    long mid = lo + (hi - lo) / 2;
    oc_leaves(lo, mid, depth + 1, los, his, k);
    oc_leaves(mid, hi, depth + 1, los, his, k);
}
static double oc_combine(int depth, const double *leaf, int *k)
{
    if (depth == 6) return leaf[(*k)++];
    double a = oc_combine(depth + 1, leaf, k);
    double b = oc_combine(depth + 1, leaf, k);
    return a + b;
}
#endif

/* ||x||_2 / sqrt(N): "l2 norm normalised to sqrt(N)" (§2.2). */
double oc_l2norm_scaled(const double *x, long n)
{
    if (n <= 0) return 0.0;
#ifdef _OPENMP
    if (n >= 4096) {   /* every range above depth 6 has > 8 points: the serial recursion splits there too */
        long los[64], his[64];
        double leaf[64];
        int k = 0;
        oc_leaves(0, n, 0, los, his, &k);
        _Pragma("omp parallel for schedule(dynamic)")
        for (int i = 0; i < 64; i++) leaf[i] = sumsq_pairwise(x, los[i], his[i]);
        k = 0;
        return sqrt(oc_combine(0, leaf, &k) / (double)n);
    }
#endif
    return sqrt(sumsq_pairwise(x, 0, n) / (double)n);
}

/* ------------------------------------------------------------------------- */
/* phi_l scalar functions (§1)                                           */
/*   phi_0 = exp, phi_{l+1}(z) = (phi_l(z) - 1/l!)/z.                         */
/* Taylor phi_l(z) = sum_k z^k/(k+l)! for |z| < 2 (R: the recursion cancels   */
/* catastrophically near 0); exp + the recursion otherwise.                   */
/* ------------------------------------------------------------------------- */
static double factorial(int l)
{
    double f = 1.0;
    for (int i = 2; i <= l; i++) f *= (double)i;
    return f;
}

double oc_phi(int l, double z)
{
    if (l < 0) return NAN;
    if (fabs(z) < 2.0) {
        double term = 1.0 / factorial(l);   /* k = 0 term: 1/l! */
        double sum = term;
        for (int k = 1; k <= 60; k++) {
            term = term * z / (double)(k + l);
            sum += term;
            if (fabs(term) < 1e-18 * fabs(sum)) break;
        }
        return sum;
    }
    double p = exp(z);                       /* phi_0 */
    for (int j = 0; j < l; j++)              /* phi_{j+1} = (phi_j - 1/j!)/z */
        p = (p - 1.0 / factorial(j)) / z;
    return p;
}

/* ------------------------------------------------------------------------- */
/* Leja points on K = [-2, 2] (§2.1):                                    */
/*   prod_{k<j} |z_j - z_k| = max_{z in K} prod_{k<j} |z - z_k|,               */
/*   |z_0| = max |z|  ->  z_0 = +2 (R7: sign +).                               */
/* For j >= 2 every candidate lies strictly between two consecutive sorted    */
/* nodes; on such a gap log prod|z - xi_k| is concave, so its maximiser is    */
/* the root of g(z) = sum_k 1/(z - xi_k) (decreasing from +inf to -inf),      */
/* found by bisection.  The largest gap maximum wins; ties (|dL| <= 1e-12)    */
/* go to the larger z (R7).                                             */
/* ------------------------------------------------------------------------- */
static double leja_g(const double *xi, int j, double z)
{
    double s = 0.0;
    for (int k = 0; k < j; k++) s += 1.0 / (z - xi[k]);
    return s;
}

static double leja_logprod(const double *xi, int j, double z)
{
    double s = 0.0;
    for (int k = 0; k < j; k++) s += log(fabs(z - xi[k]));
    return s;
}

static int cmp_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

int oc_leja_points(int count, double *xi)
{
    if (count < 1 || !xi) return OC_ERR_ARG;
    xi[0] = 2.0;
    if (count == 1) return OC_OK;
    xi[1] = -2.0;                 /* argmax |z - 2| on [-2, 2] */
    double *sorted = (double *)malloc(sizeof(double) * (size_t)count);
    if (!sorted) return OC_ERR_ARG;
    for (int j = 2; j < count; j++) {
        memcpy(sorted, xi, sizeof(double) * (size_t)j);
        qsort(sorted, (size_t)j, sizeof(double), cmp_double);
        double best_z = 0.0, best_L = -INFINITY;
        for (int gidx = 0; gidx + 1 < j; gidx++) {
            double lo = sorted[gidx], hi = sorted[gidx + 1];
            for (int it = 0; it < 200; it++) {
                double mid = 0.5 * (lo + hi);
                if (mid <= lo || mid >= hi) break;
                double g = leja_g(xi, j, mid);
                if (g == 0.0) { lo = hi = mid; break; }   /* exact root */
                if (g > 0.0) lo = mid; else hi = mid;
            }
            double z = 0.5 * (lo + hi);
            double L = leja_logprod(xi, j, z);
            if (L > best_L + 1e-12 || (fabs(L - best_L) <= 1e-12 && z > best_z)) {
                best_L = L;
                best_z = z;
            }
        }
        xi[j] = best_z;
    }
    free(sorted);
    return OC_OK;
}

/* ------------------------------------------------------------------------- */
/* Divided differences (R8):                                     */
/*   d_k = h[xi_0, ..., xi_k] of h(xi) = phi_l(a * dt * (c + gamma * xi)),     */
/* by the triangular recurrence d[i:] = (d[i:] - d[i-1]) / (xi[i:] - xi[i-1]). */
/* a is the vertical coefficient (R14).                                 */
/* ------------------------------------------------------------------------- */
int oc_divided_differences(int l, const double *xi, int m, double dt, double c,
                           double gamma, double a, double *d)
{
    if (m < 1 || !xi || !d) return OC_ERR_ARG;
    if (l < 0 || l > 4) return OC_ERR_UNSUPPORTED;
    for (int k = 0; k < m; k++) d[k] = oc_phi(l, a * dt * (c + gamma * xi[k]));
    for (int i = 1; i < m; i++)
        for (int j = i; j < m; j++)
            d[j] = (d[j] - d[i - 1]) / (xi[j] - xi[i - 1]);
    for (int k = 0; k < m; k++)
        if (!isfinite(d[k])) return OC_ERR_NONFINITE;
    return OC_OK;
}

/* ------------------------------------------------------------------------- */
/* Problems (R5, R10, R16).                                         */
/*   f(u) = diff * lap(u) + nu * sum_d D_d u + react * (u - u^3)               */
/*   lap : second-order centred 5-/7-point Laplacian                   */
/*   D_d : third-order upwind, +x-biased (R10):                                */
/*         (-u[i+2] + 6u[i+1] - 3u[i] - 2u[i-1]) / (6 dx)                      */
/*   periodic on [-1,1)^ndim, row-major, dim 0 slowest.                */
/*   J(u) v = diff * lap(v) + nu * sum_d D_d v + react * (1 - 3u^2) v (exact,  */
/*   R13).  Nonlinear remainder F(x) = f(x) - J(u) x with the linear  */
/*   part cancelled exactly (R18):  F(x) = g(x) - g'(u) x,  g(x) = react(x-x^3)*/
/* ------------------------------------------------------------------------- */
typedef struct {
    int ndim;        /* 2 or 3 */
    long n[3];       /* points per dimension; n[2] = 1 when ndim = 2 */
    double dx[3];    /* grid spacing per dimension */
    double diff;     /* diffusion coefficient */
    double nu;       /* advection velocity */
    double react;    /* Allen-Cahn reaction weight (0 or 1) */
    double flux;     /* Burgers flux weight beta: f += (beta/2) sum_d D_d(u^2) (Problem III) */
    const double *source;  /* optional time-independent source S (Problem II); NULL = none */
} oc_problem;

static long oc_npoints(const oc_problem *pb)
{
    long N = 1;
    for (int d = 0; d < pb->ndim; d++) N *= pb->n[d];
    return N;
}

static long wrap(long i, long n)
{
    while (i < 0) i += n;
    while (i >= n) i -= n;
    return i;
}

/* index of the point at (i0, i1, i2) with periodic wrap */
static long pidx(const oc_problem *pb, long i0, long i1, long i2)
{
    long n1 = pb->n[1], n2 = pb->ndim == 3 ? pb->n[2] : 1;
    i0 = wrap(i0, pb->n[0]);
    i1 = wrap(i1, n1);
    i2 = pb->ndim == 3 ? wrap(i2, n2) : 0;
    return (i0 * n1 + i1) * n2 + i2;
}

/* value of y at offset o along dimension d from point (i0,i1,i2) */
static double at(const oc_problem *pb, const double *y, long i0, long i1, long i2, int d, long o)
{
    if (d == 0) return y[pidx(pb, i0 + o, i1, i2)];
    if (d == 1) return y[pidx(pb, i0, i1 + o, i2)];
    return y[pidx(pb, i0, i1, i2 + o)];
}

/* Linear constant-coefficient part: w = diff * lap(y) + nu * sum_d D_d y. */
static void apply_linear(const oc_problem *pb, const double *y, double *w)
{
    long n0 = pb->n[0], n1 = pb->n[1], n2 = pb->ndim == 3 ? pb->n[2] : 1;
    OC_PARFOR
    for (long i0 = 0; i0 < n0; i0++)
        for (long i1 = 0; i1 < n1; i1++)
            for (long i2 = 0; i2 < n2; i2++) {
                double lap = 0.0, adv = 0.0;
                for (int d = 0; d < pb->ndim; d++) {
                    double h = pb->dx[d];
                    double um1 = at(pb, y, i0, i1, i2, d, -1);
                    double u0 = at(pb, y, i0, i1, i2, d, 0);
                    double up1 = at(pb, y, i0, i1, i2, d, 1);
                    double up2 = at(pb, y, i0, i1, i2, d, 2);
                    lap += (up1 - 2.0 * u0 + um1) / (h * h);
                    adv += (-up2 + 6.0 * up1 - 3.0 * u0 - 2.0 * um1) / (6.0 * h);
                }
                w[pidx(pb, i0, i1, i2)] = pb->diff * lap + pb->nu * adv;
            }
}

/* Slab form of J(u) y for the emulated slab decomposition:
 * y_gh holds rows -1 .. n_loc+1 of dimension 0 (one ghost row before, two after,
 * filled by the caller from the neighbouring slabs); w (rows 0..n_loc-1) gets
 * J(u) y with NO wrap along dimension 0 (the ghost rows replace it) and periodic
 * wrap along the other dimensions.  u: local rows only (NULL if react == 0). */
void oc_jac_apply_slab(const oc_problem *pb, long n_loc, const double *u, const double *y_gh, double *w)
{
    long n1 = pb->n[1], n2 = pb->ndim == 3 ? pb->n[2] : 1;
    long row = n1 * n2;
    for (long i0 = 0; i0 < n_loc; i0++)
        for (long i1 = 0; i1 < n1; i1++)
            for (long i2 = 0; i2 < n2; i2++) {
                double lap = 0.0, adv = 0.0;
                for (int d = 0; d < pb->ndim; d++) {
                    double h = pb->dx[d], v[4];
                    for (int o = -1; o <= 2; o++) {
                        long a0 = i0, a1 = i1, a2 = i2;
                        if (d == 0) a0 += o;
                        if (d == 1) a1 = wrap(i1 + o, n1);
                        if (d == 2) a2 = wrap(i2 + o, n2);
                        v[o + 1] = y_gh[(a0 + 1) * row + a1 * n2 + a2];
                    }
                    lap += (v[2] - 2.0 * v[1] + v[0]) / (h * h);
                    adv += (-v[3] + 6.0 * v[2] - 3.0 * v[1] - 2.0 * v[0]) / (6.0 * h);
                }
                long idx = i0 * row + i1 * n2 + i2;
                w[idx] = pb->diff * lap + pb->nu * adv;
                if (pb->react != 0.0) w[idx] += pb->react * (1.0 - 3.0 * u[idx] * u[idx]) * y_gh[row + idx];
            }
    /* (flux problems are not supported by the slab emulation) */
}

/* sum_d D_d w (third-order upwind, +x-biased, R10) of a pointwise field w */
static void apply_upwind_sum(const oc_problem *pb, const double *w, double *out)
{
    long n0 = pb->n[0], n1 = pb->n[1], n2 = pb->ndim == 3 ? pb->n[2] : 1;
    OC_PARFOR
    for (long i0 = 0; i0 < n0; i0++)
        for (long i1 = 0; i1 < n1; i1++)
            for (long i2 = 0; i2 < n2; i2++) {
                double adv = 0.0;
                for (int d = 0; d < pb->ndim; d++) {
                    double h = pb->dx[d];
                    double um1 = at(pb, w, i0, i1, i2, d, -1);
                    double u0 = at(pb, w, i0, i1, i2, d, 0);
                    double up1 = at(pb, w, i0, i1, i2, d, 1);
                    double up2 = at(pb, w, i0, i1, i2, d, 2);
                    adv += (-up2 + 6.0 * up1 - 3.0 * u0 - 2.0 * um1) / (6.0 * h);
                }
                out[pidx(pb, i0, i1, i2)] = adv;
            }
}

/* Burgers flux part of f and J (Problem III): (beta/2) sum_d D_d(u^2) and its exact
 * Jacobian beta sum_d D_d(u y) (R13).  out += beta * scale * sum_d D_d(a .* b). */
static void add_flux(const oc_problem *pb, const double *a, const double *b, double scale, double *out)
{
    long N = oc_npoints(pb);
    double *w = (double *)malloc(sizeof(double) * (size_t)N);
    double *t = (double *)malloc(sizeof(double) * (size_t)N);
    for (long i = 0; i < N; i++) w[i] = a[i] * b[i];
    apply_upwind_sum(pb, w, t);
    for (long i = 0; i < N; i++) out[i] += pb->flux * scale * t[i];
    free(w);
    free(t);
}

/* f(u) (Eq. (1); problems P:559; R16) */
void oc_rhs(const oc_problem *pb, const double *u, double *f)
{
    long N = oc_npoints(pb);
    apply_linear(pb, u, f);
    if (pb->flux != 0.0) add_flux(pb, u, u, 0.5, f);     /* (beta/2) sum_d D_d(u^2) */
    if (pb->react != 0.0)
        for (long i = 0; i < N; i++) f[i] += pb->react * (u[i] - u[i] * u[i] * u[i]);
    if (pb->source)   /* Problem II: f(u) = A u + S */
        for (long i = 0; i < N; i++) f[i] += pb->source[i];
}

/* w = J(u) y, exact Jacobian (R13). u may be NULL when react == 0. */
void oc_jac_apply(const oc_problem *pb, const double *u, const double *y, double *w)
{
    long N = oc_npoints(pb);
    apply_linear(pb, y, w);
    if (pb->flux != 0.0) add_flux(pb, u, y, 1.0, w);     /* beta sum_d D_d(u y) */
    if (pb->react != 0.0)
        OC_PARFOR
        for (long i = 0; i < N; i++) w[i] += pb->react * (1.0 - 3.0 * u[i] * u[i]) * y[i];
}

/* F(x) = f(x) - J(u) x  =  g(x) - g'(u) x  (R18).  A source S would add the same
 * constant to every F(x); it cancels in every difference F(x) - F(u) the integrators use,
 * so it is left out (R21). */
void oc_nonlinear_remainder(const oc_problem *pb, const double *u, const double *x, double *out)
{
    long N = oc_npoints(pb);
    for (long i = 0; i < N; i++) {
        if (pb->react != 0.0) {
            double g = pb->react * (x[i] - x[i] * x[i] * x[i]);
            double gp = pb->react * (1.0 - 3.0 * u[i] * u[i]);
            out[i] = g - gp * x[i];
        } else {
            out[i] = 0.0;
        }
    }
    if (pb->flux != 0.0) {
        /* Burgers: F(x) = sum_d D_d(beta/2 x^2 - beta u x)  (f(x) - J(u)x, diffusion and linear
         * advection cancelled exactly, R18) */
        double *w = (double *)malloc(sizeof(double) * (size_t)N);
        double *t = (double *)malloc(sizeof(double) * (size_t)N);
        for (long i = 0; i < N; i++) w[i] = 0.5 * pb->flux * x[i] * x[i] - pb->flux * u[i] * x[i];
        apply_upwind_sum(pb, w, t);
        for (long i = 0; i < N; i++) out[i] += t[i];
        free(w);
        free(t);
    }
}

/* Spectral bound |lambda_max| (R9, R16): Fourier symbol of the constant part
 * at theta = pi in every dimension, sum_d (4 diff/dx_d^2 + 4|nu|/(3 dx_d)),
 * plus the Gershgorin shift of the reaction, react * max(0, 3 max u^2 - 1). */
double oc_spectrum_bound(const oc_problem *pb, const double *u)
{
    double vmax = fabs(pb->nu);
    if (pb->flux != 0.0 && u) {   /* Burgers: frozen-coefficient speed |nu| + |beta| max|u| (R23) */
        long N = oc_npoints(pb);
        double m = 0.0;
        for (long i = 0; i < N; i++) if (u[i] * u[i] > m) m = u[i] * u[i];
        vmax = fabs(pb->nu) + fabs(pb->flux) * sqrt(m);
    }
    double b = 0.0;
    for (int d = 0; d < pb->ndim; d++) {
        double h = pb->dx[d];
        b += 4.0 * pb->diff / (h * h) + 4.0 * vmax / (3.0 * h);
    }
    if (pb->react != 0.0 && u) {
        long N = oc_npoints(pb);
        double m = 0.0;
        for (long i = 0; i < N; i++) if (u[i] * u[i] > m) m = u[i] * u[i];
        double s = 3.0 * m - 1.0;
        if (s > 0.0) b += pb->react * s;
    }
    return b;
}

/* Power iteration (R9): v_0 = ones + e_0; k_pw iterations of
 * w = J v, estimate = ||w|| / ||v||, v = w / ||w||.  Returns the last estimate. */
double oc_power_iteration(const oc_problem *pb, const double *u, int iters)
{
    long N = oc_npoints(pb);
    double *v = (double *)malloc(sizeof(double) * (size_t)N);
    double *w = (double *)malloc(sizeof(double) * (size_t)N);
    if (!v || !w) { free(v); free(w); return NAN; }
    for (long i = 0; i < N; i++) v[i] = 1.0;
    v[0] += 1.0;
    double est = 0.0;
    for (int k = 0; k < iters; k++) {
        oc_jac_apply(pb, u, v, w);
        double nw = oc_l2norm_scaled(w, N), nv = oc_l2norm_scaled(v, N);
        est = nw / nv;
        for (long i = 0; i < N; i++) v[i] = w[i] / nw;
    }
    free(v);
    free(w);
    return est;
}

/* ------------------------------------------------------------------------- */
/* Real Leja interpolation (Eq. (2); P:155 stopping rule;           */
/* listings alg:leja_exp_int, alg:leja_phi_nl_int, alg:leja_phi; R1-R6, R14). */
/*                                                                             */
/*   y_0 = v,  p_0^{(k)} = d_0^{(k)} y_0                                        */
/*   for m = 1, 2, ...:                                                        */
/*     y_m = y_{m-1} * ((z - c)/gamma - xi_{m-1})   with z -> J(u)             */
/*     p_m^{(k)} = p_{m-1}^{(k)} + d_m^{(k)} y_m        (active k only)        */
/*     accumulator k converges when                                            */
/*        ||d_m^{(k)} y_m|| <= rtol ||p_m^{(k)}|| + atol  (norms / sqrt(N))    */
/*     and is frozen; stop when all K have converged (iters = m).             */
/*   coeffs a_k: p^{(k)} ~ phi_l(a_k dt J(u)) v  (vertical).    */
/*   margins[0] = min_k thr/err at acceptance; margins[1] = min over the      */
/*   rejected checks of err/thr (how far the decisions were from flipping).   */
/* ------------------------------------------------------------------------- */
/* ------------------------------------------------------------------------- */
/* Black-box right-hand side (P:120-133 listing alg:RHS):    */
/* the method only calls f.  Jacobian-vector products by forward finite        */
/* differences ("computed numerically using finite differences"):       */
/*   J(u) y ~ (f(u + eps y) - f(u)) / eps,                                     */
/*   eps = sqrt(DBL_EPSILON) (1 + ||u||_inf) / ||y||_inf   (reading R25),       */
/* J(u) y = 0 when y = 0.  For a LINEAR f (Problem I, P:161-171 real_Leja_exp  */
/* with RHS = A) the operator is applied as f(y) itself (OC_JAC_LINEAR_F).     */
/* ------------------------------------------------------------------------- */
#define OC_JAC_EXACT 0
#define OC_JAC_FD 1
#define OC_JAC_LINEAR_F 2
#define OC_FD_EPS0 1.4901161193847656e-08   /* sqrt(DBL_EPSILON) = 2^-26 */

static double maxabs(const double *x, long N)
{
    double m = 0.0;
    for (long i = 0; i < N; i++) if (fabs(x[i]) > m) m = fabs(x[i]);
    return m;
}

/* w = J(u) y by forward differences; f_u = f(u) (unscaled). */
void oc_jac_apply_fd(const oc_problem *pb, const double *u, const double *f_u, const double *y, double *w)
{
    long N = oc_npoints(pb);
    double ymax = maxabs(y, N);
    if (ymax == 0.0) {
        for (long i = 0; i < N; i++) w[i] = 0.0;
        return;
    }
    double eps = OC_FD_EPS0 * (1.0 + maxabs(u, N)) / ymax;
    double *t = (double *)malloc(sizeof(double) * (size_t)N);
    double *ft = (double *)malloc(sizeof(double) * (size_t)N);
    for (long i = 0; i < N; i++) t[i] = u[i] + eps * y[i];
    oc_rhs(pb, t, ft);
    for (long i = 0; i < N; i++) w[i] = (ft[i] - f_u[i]) / eps;
    free(t);
    free(ft);
}

/* F(x) = f(x) - J(u) x with the finite-difference J (the listing's
 * Nonlinear_remainder(RHS, u, x, NL_x), alg:exprb32 P:530-531), literally. */
void oc_nonlinear_remainder_fd(const oc_problem *pb, const double *u, const double *f_u, const double *x,
                               double *out)
{
    long N = oc_npoints(pb);
    double *fx = (double *)malloc(sizeof(double) * (size_t)N);
    double *jx = (double *)malloc(sizeof(double) * (size_t)N);
    oc_rhs(pb, x, fx);
    oc_jac_apply_fd(pb, u, f_u, x, jx);
    for (long i = 0; i < N; i++) out[i] = fx[i] - jx[i];
    free(fx);
    free(jx);
}

static void jac_mode_apply(const oc_problem *pb, int mode, const double *u, const double *f_u, const double *y,
                           double *w)
{
    if (mode == OC_JAC_FD) oc_jac_apply_fd(pb, u, f_u, y, w);
    else if (mode == OC_JAC_LINEAR_F) oc_rhs(pb, y, w);
    else oc_jac_apply(pb, u, y, w);
}

int oc_real_leja_phi_ex(const oc_problem *pb, int jac_mode, const double *u_lin, const double *f_u,
                        const double *v, double **outs, const double *coeffs, int K, double dt, double c,
                        double gamma, int l, double rtol, double atol, const double *xi,
                        int max_nodes, int *iters, double *margins);

int oc_real_leja_phi(const oc_problem *pb, const double *u_lin, const double *v,
                     double **outs, const double *coeffs, int K, double dt, double c,
                     double gamma, int l, double rtol, double atol, const double *xi,
                     int max_nodes, int *iters, double *margins)
{
    return oc_real_leja_phi_ex(pb, OC_JAC_EXACT, u_lin, NULL, v, outs, coeffs, K, dt, c, gamma, l, rtol, atol,
                               xi, max_nodes, iters, margins);
}

/* jac_mode: OC_JAC_EXACT (J(u_lin) exact), OC_JAC_FD (J(u_lin) by differences of f;
 * f_u = f(u_lin) or NULL to compute it here), OC_JAC_LINEAR_F (operator = f itself). */
int oc_real_leja_phi_ex(const oc_problem *pb, int jac_mode, const double *u_lin, const double *f_u,
                        const double *v, double **outs, const double *coeffs, int K, double dt, double c,
                        double gamma, int l, double rtol, double atol, const double *xi,
                        int max_nodes, int *iters, double *margins)
{
    if (iters) *iters = 0;
    if (margins) { margins[0] = INFINITY; margins[1] = INFINITY; }
    if (K < 1 || K > 4 || !pb || !v || !outs || !coeffs || !xi || max_nodes < 2) return OC_ERR_ARG;
    if (l < 0 || l > 4) return OC_ERR_UNSUPPORTED;
    if (!(gamma > 0.0) && dt != 0.0) return OC_ERR_ARG;
    for (int k = 0; k < K; k++)
        if (!(coeffs[k] > 0.0 && coeffs[k] <= 1.0) || (k > 0 && !(coeffs[k] > coeffs[k - 1])))
            return OC_ERR_ARG;

    long N = oc_npoints(pb);
    double *y = (double *)malloc(sizeof(double) * (size_t)N);
    double *w = (double *)malloc(sizeof(double) * (size_t)N);
    double *d = (double *)malloc(sizeof(double) * (size_t)max_nodes * (size_t)K);
    if (!y || !w || !d) { free(y); free(w); free(d); return OC_ERR_ARG; }

    int status = OC_OK;
    double *fu_own = NULL;
    if (jac_mode == OC_JAC_FD && !f_u) {
        if (!u_lin) { free(y); free(w); free(d); return OC_ERR_ARG; }
        fu_own = (double *)malloc(sizeof(double) * (size_t)N);
        oc_rhs(pb, u_lin, fu_own);
        f_u = fu_own;
    }
    for (int k = 0; k < K; k++) {
        int s = oc_divided_differences(l, xi, max_nodes, dt, c, gamma, coeffs[k], d + (size_t)k * max_nodes);
        if (s != OC_OK) { status = s; goto done; }
    }

    int active[4] = {0, 0, 0, 0};
    OC_PARFOR
    for (long i = 0; i < N; i++) y[i] = v[i];
    for (int k = 0; k < K; k++) {
        active[k] = 1;
        OC_PARFOR
        for (long i = 0; i < N; i++) outs[k][i] = d[(size_t)k * max_nodes + 0] * v[i];
    }

    status = OC_ERR_NOCONV;
    for (int m = 1; m < max_nodes; m++) {
        jac_mode_apply(pb, jac_mode, u_lin, f_u, y, w);      /* w = J y */
        OC_PARFOR
        for (long i = 0; i < N; i++)                         /* Eq. (2) */
            y[i] = (w[i] - c * y[i]) / gamma - xi[m - 1] * y[i];
        double ny = oc_l2norm_scaled(y, N);
        int n_active = 0;
        for (int k = 0; k < K; k++) {
            if (!active[k]) continue;
            double dm = d[(size_t)k * max_nodes + m];
            OC_PARFOR
            for (long i = 0; i < N; i++) outs[k][i] = outs[k][i] + dm * y[i];
            double np = oc_l2norm_scaled(outs[k], N);
            double err = fabs(dm) * ny;
            double thr = rtol * np + atol;
            if (!isfinite(err) || !isfinite(thr)) { status = OC_ERR_NONFINITE; if (iters) *iters = m; goto done; }
            if (err <= thr) {
                active[k] = 0;
                if (margins) { double r = err > 0.0 ? thr / err : INFINITY; if (r < margins[0]) margins[0] = r; }
            } else {
                n_active++;
                if (margins) { double r = err / thr; if (r < margins[1]) margins[1] = r; }
            }
        }
        if (iters) *iters = m;
        if (n_active == 0) { status = OC_OK; break; }
    }
done:
    free(y);
    free(w);
    free(d);
    free(fu_own);
    return status;
}

/* ------------------------------------------------------------------------- */
/* Exponential integrators (listings alg:Ros_Eu, alg:exprb32;      */
/* EXPRB43 and EPIRK4s3A tableaux from P:83's citations, R17).                */
/*   method 0 Rosenbrock-Euler, 1 EXPRB32, 2 EXPRB43, 3 EPIRK4s3A, 4 EXPRB42,    */
/*   5 EPIRK5P1, 6 EXPRB53s3, 7 EXPRB54s4, 8 EPIRK4s3B, 9 EPIRK4s3.             */
/* u_low may be NULL for Rosenbrock-Euler (non-embedded, err = 0).            */
/* ------------------------------------------------------------------------- */
static void axpby(double a, const double *x, double b, const double *y, double *z, long N)
{
    for (long i = 0; i < N; i++) z[i] = a * x[i] + b * y[i];
}

/* F(x): analytic (R18) for the exact-Jacobian contract, literal f(x) - J_FD(u) x
 * for the black-box finite-difference mode. */
static void remainder_mode(const oc_problem *pb, int jac_mode, const double *u, const double *fu_raw,
                           const double *x, double *out)
{
    if (jac_mode == OC_JAC_FD) oc_nonlinear_remainder_fd(pb, u, fu_raw, x, out);
    else oc_nonlinear_remainder(pb, u, x, out);
}

int oc_step_ex(const oc_problem *pb, int jac_mode, int method, const double *u, double *u_low,
               double *u_high, double *err, double dt, double c, double gamma, double rtol, double atol,
               const double *xi, int max_nodes, int *iters)
{
    long N = oc_npoints(pb);
    int it = 0, total = 0, s = OC_OK;
    if (err) *err = 0.0;
    if (iters) *iters = 0;
    if (method < 0 || method > 9) return OC_ERR_ARG;
    if (jac_mode != OC_JAC_EXACT && jac_mode != OC_JAC_FD) return OC_ERR_ARG;
    size_t bytes = sizeof(double) * (size_t)N;
    double *fu_raw = NULL;
    double *f_u = (double *)malloc(bytes);
    double *t1 = (double *)malloc(bytes), *t2 = (double *)malloc(bytes), *t3 = (double *)malloc(bytes);
    double *t4 = (double *)malloc(bytes), *t5 = (double *)malloc(bytes), *t6 = (double *)malloc(bytes);
    double *t7 = (double *)malloc(bytes), *t8 = (double *)malloc(bytes);
    if (!f_u || !t1 || !t2 || !t3 || !t4 || !t5 || !t6 || !t7 || !t8) { s = OC_ERR_ARG; goto out; }

    /* f_u = RHS(u) * dt  (alg:Ros_Eu P:468-469) */
    oc_rhs(pb, u, f_u);
    if (jac_mode == OC_JAC_FD) {   /* unscaled f(u) for the difference quotients */
        fu_raw = (double *)malloc(bytes);
        if (!fu_raw) { s = OC_ERR_ARG; goto out; }
        memcpy(fu_raw, f_u, bytes);
    }
    for (long i = 0; i < N; i++) f_u[i] = dt * f_u[i];

    if (method == 0) {
        /* u_exprb2 = u + phi_1(J dt) f_u dt */
        double one = 1.0;
        double *o[1] = {t1};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, o, &one, 1, dt, c, gamma, 1, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        axpby(1.0, u, 1.0, t1, u_high, N);
        if (u_low) axpby(1.0, u, 1.0, t1, u_low, N);
    } else if (method == 1) {
        /* EXPRB32 (alg:exprb32 P:512-540) */
        double one = 1.0;
        double *o[1] = {t1};                                  /* u_flux */
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, o, &one, 1, dt, c, gamma, 1, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        axpby(1.0, u, 1.0, t1, u_low, N);                     /* u_exprb2 = a */
        remainder_mode(pb, jac_mode, u, fu_raw, u, t2);                 /* NL_u */
        remainder_mode(pb, jac_mode, u, fu_raw, u_low, t3);             /* NL_a */
        axpby(dt, t3, -dt, t2, t4, N);                        /* R_a = (NL_a - NL_u) dt */
        double *o3[1] = {t5};                                 /* u_nl_3 */
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t4, o3, &one, 1, dt, c, gamma, 3, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        axpby(1.0, u_low, 2.0, t5, u_high, N);                /* u_exprb3 = a + 2 u_nl_3 */
        for (long i = 0; i < N; i++) t6[i] = 2.0 * t5[i];      /* error_vector */
        if (err) *err = oc_l2norm_scaled(t6, N);
    } else if (method == 4) {
        /* EXPRB42 (Luan 2017, cited at P:83; reading R22):
         *   a = u + 3/4 h phi_1(3/4 hJ) f(u)
         *   u_{n+1} = u + h phi_1(hJ) f(u) + 32/9 h phi_3(hJ) D_a,   D_a = dt (F(a) - F(u))
         * non-embedded (u_low = u_high, err = 0). */
        double cf[2] = {0.75, 1.0};
        double *pv[2] = {t1, t2};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, pv, cf, 2, dt, c, gamma, 1, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        axpby(1.0, u, 0.75, t1, t3, N);                       /* a */
        remainder_mode(pb, jac_mode, u, fu_raw, u, t4);                 /* NL_u */
        remainder_mode(pb, jac_mode, u, fu_raw, t3, t5);                /* NL_a */
        axpby(dt, t5, -dt, t4, t6, N);                        /* D_a */
        for (long i = 0; i < N; i++) t6[i] = (32.0 / 9.0) * t6[i];
        double one = 1.0;
        double *o3[1] = {t7};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t6, o3, &one, 1, dt, c, gamma, 3, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) u_high[i] = u[i] + t2[i] + t7[i];
        if (u_low) for (long i = 0; i < N; i++) u_low[i] = u_high[i];
    } else if (method == 5) {
        /* EPIRK5P1 (Tokman, Loffeld & Tranquilli 2012, cited at P:83 and run in Table 2, P:616-634;
         * reading R26), psi functions = (phi_1, phi_1, phi_3), R(x) = h (F(x) - F(u)):
         *   Y1 = u + a11 h phi_1(g11 hJ) f
         *   Y2 = u + a21 h phi_1(g21 hJ) f + a22 phi_1(g22 hJ) R(Y1)
         *   u+ = u + b1 h phi_1(g31 hJ) f + b2 phi_1(g32 hJ) R(Y1) + b3 phi_3(g33 hJ) (R(Y2) - 2 R(Y1))
         * embedded fourth-order solution (reading R33): the same with g32 -> 1/2, g33 -> 1,
         *   u4 = u + b1 h phi_1(hJ) f + b2 phi_1(hJ/2) R(Y1) + b3 phi_3(hJ) (R(Y2) - 2 R(Y1)). */
        const double a11 = 0.35129592695058193092, a21 = 0.84405472011657126298, a22 = 1.6905891609568963624;
        const double b1 = 1.0, b2 = 1.2727127317356892397, b3 = 2.2714599265422622275;
        const double g11 = 0.35129592695058193092, g21 = 0.84405472011657126298, g22 = 1.0;
        const double g31 = 1.0, g32 = 0.71111095364366870359, g33 = 0.62378111953371494809;
        double cf3[3] = {g11, g21, g31};                     /* vertical phi_1 on f h */
        double *pv[3] = {t1, t2, t3};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, pv, cf3, 3, dt, c, gamma, 1, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        remainder_mode(pb, jac_mode, u, fu_raw, u, t4);      /* NL_u */
        axpby(1.0, u, a11, t1, t5, N);                       /* Y1 */
        remainder_mode(pb, jac_mode, u, fu_raw, t5, t6);     /* NL_Y1 */
        axpby(dt, t6, -dt, t4, t5, N);                       /* R1 = h (F(Y1) - F(u)) */
        double cf2[3] = {0.5, g32, g22};                     /* vertical phi_1 on R1 (1/2: embedded) */
        double *qv[3] = {t8, t6, t7};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t5, qv, cf2, 3, dt, c, gamma, 1, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) t1[i] = u[i] + a21 * t2[i] + a22 * t7[i];   /* Y2 */
        remainder_mode(pb, jac_mode, u, fu_raw, t1, t2);     /* NL_Y2 */
        axpby(dt, t2, -dt, t4, t7, N);                       /* R2 */
        axpby(1.0, t7, -2.0, t5, t2, N);                     /* R2 - 2 R1 */
        double cf33[2] = {g33, 1.0};                         /* vertical phi_3 (1: embedded) */
        double *o3[2] = {t7, t1};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t2, o3, cf33, 2, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) u_high[i] = u[i] + b1 * t3[i] + b2 * t6[i] + b3 * t7[i];
        for (long i = 0; i < N; i++) t2[i] = u[i] + b1 * t3[i] + b2 * t8[i] + b3 * t1[i];   /* u4 */
        if (u_low) for (long i = 0; i < N; i++) u_low[i] = t2[i];
        for (long i = 0; i < N; i++) t1[i] = u_high[i] - t2[i];
        if (err) *err = oc_l2norm_scaled(t1, N);                            /* P:252, R20 */
    } else if (method == 6) {
        /* EXPRB53s3 (Luan & Ostermann 2014, cited at P:83; reading R27), D_x = h (F(x) - F(u)):
         *   U2 = u + c2 h phi_1(c2 hJ) f                                  c2 = 1/2
         *   U3 = u + c3 h phi_1(c3 hJ) f + (27/25 phi_3(c2 hJ) + 729/125 phi_3(c3 hJ)) D2   c3 = 9/10
         *   u5 = u + h phi_1(hJ) f + (18 phi_3 - 60 phi_4)(hJ) D2 + (-250/81 phi_3 + 500/27 phi_4)(hJ) D3
         *   u3 = u + h phi_1(hJ) f + 8 phi_3(hJ) D2        (embedded, order 3)
         *   err = ||u5 - u3|| */
        const double c2 = 0.5, c3 = 0.9;
        double cf3[3] = {c2, c3, 1.0};
        double *pv[3] = {t1, t2, t3};                        /* phi_1(c2 hJ) hf, phi_1(c3 hJ) hf, phi_1(hJ) hf */
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, pv, cf3, 3, dt, c, gamma, 1, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        remainder_mode(pb, jac_mode, u, fu_raw, u, t4);      /* NL_u */
        axpby(1.0, u, c2, t1, t5, N);                        /* U2 */
        remainder_mode(pb, jac_mode, u, fu_raw, t5, t6);
        axpby(dt, t6, -dt, t4, t5, N);                       /* D2 */
        double *qv[3] = {t1, t6, t7};                        /* phi_3(c2 hJ) D2, phi_3(c3 hJ) D2, phi_3(hJ) D2 */
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t5, qv, cf3, 3, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++)                         /* U3 */
            t1[i] = u[i] + c3 * t2[i] + (27.0 / 25.0) * t1[i] + (729.0 / 125.0) * t6[i];
        remainder_mode(pb, jac_mode, u, fu_raw, t1, t2);
        axpby(dt, t2, -dt, t4, t6, N);                       /* D3 */
        axpby(18.0, t5, -250.0 / 81.0, t6, t1, N);           /* w3 */
        axpby(-60.0, t5, 500.0 / 27.0, t6, t2, N);           /* w4 */
        double one = 1.0;
        double *o3[1] = {t4};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t1, o3, &one, 1, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *o4[1] = {t5};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t2, o4, &one, 1, dt, c, gamma, 4, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) u_high[i] = u[i] + t3[i] + t4[i] + t5[i];   /* u5 */
        for (long i = 0; i < N; i++) u_low[i] = u[i] + t3[i] + 8.0 * t7[i];      /* u3 */
        for (long i = 0; i < N; i++) t1[i] = u_high[i] - u_low[i];
        if (err) *err = oc_l2norm_scaled(t1, N);
    } else if (method == 8) {
        /* EPIRK4s3B (Rainwater & Tokman 2016, cited at P:83; reading R34), D_x = h (F(x) - F(u)):
         *   a  = u + 2/3 h phi_2(hJ/2) f;   b = u + h phi_2(3hJ/4) f
         *   u3 = u + h phi_1(hJ) f + phi_3(hJ) (54 D_a - 16 D_b)
         *   u4 = u3 + phi_4(hJ) (-324 D_a + 144 D_b)
         * vertical phi_2 {1/2, 3/4} on f_u, phi_1 on f_u; err = ||u4 - u3||. */
        double cf2[2] = {0.5, 0.75};
        double *qv[2] = {t1, t2};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, qv, cf2, 2, dt, c, gamma, 2, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double one = 1.0;
        double *o1[1] = {t3};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, o1, &one, 1, dt, c, gamma, 1, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *NLu = t4, *Da = t5, *Db = t6, *tmp = t7;
        remainder_mode(pb, jac_mode, u, fu_raw, u, NLu);
        axpby(1.0, u, 2.0 / 3.0, t1, u_low, N);               /* a */
        remainder_mode(pb, jac_mode, u, fu_raw, u_low, tmp);
        axpby(dt, tmp, -dt, NLu, Da, N);                      /* D_a */
        axpby(1.0, u, 1.0, t2, u_low, N);                     /* b */
        remainder_mode(pb, jac_mode, u, fu_raw, u_low, tmp);
        axpby(dt, tmp, -dt, NLu, Db, N);                      /* D_b */
        axpby(54.0, Da, -16.0, Db, tmp, N);                   /* w3 */
        axpby(-324.0, Da, 144.0, Db, NLu, N);                 /* w4 */
        double *o3[1] = {Da};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, tmp, o3, &one, 1, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *o4[1] = {Db};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, NLu, o4, &one, 1, dt, c, gamma, 4, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) u_low[i] = u[i] + t3[i] + Da[i];        /* u3 */
        for (long i = 0; i < N; i++) u_high[i] = u_low[i] + Db[i];           /* u4 */
        for (long i = 0; i < N; i++) tmp[i] = u_high[i] - u_low[i];
        if (err) *err = oc_l2norm_scaled(tmp, N);
    } else if (method == 7) {
        /* EXPRB54s4 (Luan & Ostermann 2014, cited at P:83; reading R31), D_x = h (F(x) - F(u)),
         * nodes c2 = 1/4, c3 = 1/2, c4 = 9/10:
         *   U2 = u + c2 h phi_1(c2 hJ) f
         *   U3 = u + c3 h phi_1(c3 hJ) f + 4 phi_3(c3 hJ) D2
         *   U4 = u + c4 h phi_1(c4 hJ) f + phi_3(c4 hJ)(5832/125 D2 - 729/125 D3)
         *                                 + phi_4(c4 hJ)(-157464/625 D2 + 39366/625 D3)
         *   u5 = u + h phi_1(hJ) f + phi_3(hJ)(18 D3 - 250/81 D4) + phi_4(hJ)(-60 D3 + 500/27 D4)
         *   u4 = u + h phi_1(hJ) f + phi_3(hJ)(64 D2 - 8 D3) + phi_4(hJ)(-384 D2 + 96 D3)   (embedded, order 4)
         *   err = ||u5 - u4|| */
        double cf4[4] = {0.25, 0.5, 0.9, 1.0};
        double *pv[4] = {t1, t2, t3, t7};                    /* phi_1(c hJ) hf, c = 1/4, 1/2, 9/10, 1 */
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, pv, cf4, 4, dt, c, gamma, 1, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        remainder_mode(pb, jac_mode, u, fu_raw, u, t4);      /* NL_u */
        axpby(1.0, u, 0.25, t1, t5, N);                      /* U2 */
        remainder_mode(pb, jac_mode, u, fu_raw, t5, t6);
        axpby(dt, t6, -dt, t4, t5, N);                       /* D2 */
        double half = 0.5, c4 = 0.9, one = 1.0;
        double *o1[1] = {t1};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t5, o1, &half, 1, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);                               /* phi_3(hJ/2) D2 */
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) t6[i] = u[i] + 0.5 * t2[i] + 4.0 * t1[i];     /* U3 */
        remainder_mode(pb, jac_mode, u, fu_raw, t6, u_low);
        axpby(dt, u_low, -dt, t4, t6, N);                    /* D3 */
        axpby(5832.0 / 125.0, t5, -729.0 / 125.0, t6, t1, N);
        axpby(-157464.0 / 625.0, t5, 39366.0 / 625.0, t6, t2, N);
        double *o2[1] = {u_low};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t1, o2, &c4, 1, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *o3[1] = {u_high};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t2, o3, &c4, 1, dt, c, gamma, 4, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) t1[i] = u[i] + 0.9 * t3[i] + u_low[i] + u_high[i];   /* U4 */
        remainder_mode(pb, jac_mode, u, fu_raw, t1, t2);
        axpby(dt, t2, -dt, t4, t3, N);                       /* D4 */
        axpby(64.0, t5, -8.0, t6, t1, N);                    /* embedded: 64 D2 - 8 D3, -384 D2 + 96 D3 */
        axpby(-384.0, t5, 96.0, t6, t2, N);
        double *o4[1] = {t4};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t1, o4, &one, 1, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *o5[1] = {u_low};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t2, o5, &one, 1, dt, c, gamma, 4, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) u_low[i] = u[i] + t7[i] + t4[i] + u_low[i];  /* u4 */
        axpby(18.0, t6, -250.0 / 81.0, t3, t1, N);           /* 18 D3 - 250/81 D4 */
        axpby(-60.0, t6, 500.0 / 27.0, t3, t2, N);           /* -60 D3 + 500/27 D4 */
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t1, o4, &one, 1, dt, c, gamma, 3, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *o6[1] = {t5};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, t2, o6, &one, 1, dt, c, gamma, 4, rtol, atol, xi,
                                max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) u_high[i] = u[i] + t7[i] + t4[i] + t5[i];   /* u5 */
        for (long i = 0; i < N; i++) t1[i] = u_high[i] - u_low[i];
        if (err) *err = oc_l2norm_scaled(t1, N);
    } else {
        /* EXPRB43 (method 2) / EPIRK4s3A (method 3) -- R17 tableaux -- / EPIRK4s3 (method 9, R35):
         *  EXPRB43:   a = u + 1/2 hphi_1(hJ/2) f;  b = u + hphi_1 f + hphi_1 D_a
         *             u3 = u + hphi_1 f + hphi_3 (16 D_a - 2 D_b)
         *             u4 = u3 + hphi_4 (-48 D_a + 12 D_b)
         *  EPIRK4s3A: a = u + 1/2 hphi_1(hJ/2) f;  b = u + 2/3 hphi_1(2hJ/3) f
         *             u3 = u + hphi_1 f + hphi_3 (32 D_a - 27/2 D_b)
         *             u4 = u3 + hphi_4 (-144 D_a + 81 D_b)
         *  EPIRK4s3:  a = u + 1/8 hphi_1(hJ/8) f;  b = u + 1/9 hphi_1(hJ/9) f
         *             u3 = u + hphi_1 f + phi_3 (-1024 D_a + 1458 D_b)
         *             u4 = u3 + phi_4 (27648 D_a - 34992 D_b)
         *  D_x = dt (F(x) - F(u)); vertical phi_1 on f_u. */
        int e4s3 = (method == 9);
        int epirk = (method == 3) || e4s3;
        double cf2[2] = {0.5, 1.0}, cf3[3] = {0.5, 2.0 / 3.0, 1.0}, cf9[3] = {1.0 / 9.0, 1.0 / 8.0, 1.0};
        double *pv[3] = {t1, t2, t3};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, f_u, pv, e4s3 ? cf9 : epirk ? cf3 : cf2, epirk ? 3 : 2, dt, c,
                             gamma, 1, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *p_half = t1, *p_one = epirk ? t3 : t2;
        double *NLu = t4, *Da = t5, *Db = t6, *tmp = t7;
        remainder_mode(pb, jac_mode, u, fu_raw, u, NLu);
        /* a = u + 1/2 p_half  (EPIRK4s3: u + 1/8 p_{1/8}, the second vertical output) */
        if (e4s3) axpby(1.0, u, 0.125, t2, u_low, N);
        else axpby(1.0, u, 0.5, p_half, u_low, N);
        remainder_mode(pb, jac_mode, u, fu_raw, u_low, tmp);
        axpby(dt, tmp, -dt, NLu, Da, N);                      /* D_a */
        if (e4s3) {
            /* b = u + 1/9 p_{1/9} (the first vertical output) */
            axpby(1.0, u, 1.0 / 9.0, t1, u_low, N);
        } else if (epirk) {
            /* b = u + 2/3 p_twothirds */
            axpby(1.0, u, 2.0 / 3.0, t2, u_low, N);
        } else {
            /* b = u + p_one + phi_1(hJ) D_a */
            double one = 1.0;
            double *o[1] = {u_high};
            s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, Da, o, &one, 1, dt, c, gamma, 1, rtol, atol, xi, max_nodes, &it, NULL);
            total += it;
            if (s) goto out;
            for (long i = 0; i < N; i++) u_low[i] = u[i] + p_one[i] + u_high[i];
        }
        remainder_mode(pb, jac_mode, u, fu_raw, u_low, tmp);
        axpby(dt, tmp, -dt, NLu, Db, N);                      /* D_b */
        double a3 = e4s3 ? -1024.0 : epirk ? 32.0 : 16.0, b3 = e4s3 ? 1458.0 : epirk ? -13.5 : -2.0;
        double a4 = e4s3 ? 27648.0 : epirk ? -144.0 : -48.0, b4 = e4s3 ? -34992.0 : epirk ? 81.0 : 12.0;
        axpby(a3, Da, b3, Db, tmp, N);                        /* w3 */
        axpby(a4, Da, b4, Db, NLu, N);                        /* w4 (NLu no longer needed) */
        double one = 1.0;
        double *o3[1] = {Da};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, tmp, o3, &one, 1, dt, c, gamma, 3, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        double *o4[1] = {Db};
        s = oc_real_leja_phi_ex(pb, jac_mode, u, fu_raw, NLu, o4, &one, 1, dt, c, gamma, 4, rtol, atol, xi, max_nodes, &it, NULL);
        total += it;
        if (s) goto out;
        for (long i = 0; i < N; i++) u_low[i] = u[i] + p_one[i] + Da[i];    /* u3 */
        for (long i = 0; i < N; i++) u_high[i] = u_low[i] + Db[i];          /* u4 */
        for (long i = 0; i < N; i++) tmp[i] = u_high[i] - u_low[i];
        if (err) *err = oc_l2norm_scaled(tmp, N);
    }
out:
    if (iters) *iters = total;
    free(f_u); free(t1); free(t2); free(t3); free(t4); free(t5); free(t6); free(t7); free(t8);
    free(fu_raw);
    return s;
}

/* Exact-Jacobian steps (R13, R18): the contract the device hot path follows. */
int oc_step(const oc_problem *pb, int method, const double *u, double *u_low, double *u_high,
            double *err, double dt, double c, double gamma, double rtol, double atol,
            const double *xi, int max_nodes, int *iters)
{
    return oc_step_ex(pb, OC_JAC_EXACT, method, u, u_low, u_high, err, dt, c, gamma, rtol, atol, xi, max_nodes,
                      iters);
}

/* ------------------------------------------------------------------------- */
/* Step-size control by the embedded error ("may be used to control the */
/* step sizes"; reading R32): the elementary controller                        */
/*   accept iff err <= tol;  h_new = h min(5, max(0.2, 0.9 (tol/err)^(1/(q+1)))) */
/* (err = 0 -> 5), q = order of the embedded (lower-order) solution; the last  */
/* step is clipped to land on t_end; a step whose Leja calls fail (NOCONV,     */
/* NONFINITE) counts as rejected with err = inf (factor 0.2).                  */
/* (c, gamma) from the Gershgorin / closed-                                    */
/* form bound of the current state.  u is overwritten with u(t_end).*/
/* log_dt / log_err / log_acc (max_steps entries each) record every attempt.   */
/* ------------------------------------------------------------------------- */
static int oc_embedded_order(int method)
{
    switch (method) {
    case 1: return 2;   /* EXPRB32: a */
    case 2: return 3;   /* EXPRB43: u_3 */
    case 3: return 3;   /* EPIRK4s3A: u_3 */
    case 6: return 3;   /* EXPRB53s3: u_3 */
    case 5: return 4;   /* EPIRK5P1: u_4 (R33) */
    case 7: return 4;   /* EXPRB54s4: u_4 */
    case 8: return 3;   /* EPIRK4s3B: u_3 (R34) */
    case 9: return 3;   /* EPIRK4s3: u_3 (R35) */
    default: return 0;  /* non-embedded */
    }
}

int oc_integrate_adaptive(const oc_problem *pb, int method, double *u, double t_end, double dt0, double tol,
                          double rtol, double atol, const double *xi, int max_nodes, int max_steps, int *accepted,
                          int *rejected, double *log_dt, double *log_err, int *log_acc, int *iters)
{
    int q = oc_embedded_order(method);
    if (q == 0 || !(dt0 > 0.0) || !(tol > 0.0) || !(t_end > 0.0)) return OC_ERR_ARG;
    long N = oc_npoints(pb);
    double *lo = (double *)malloc(sizeof(double) * (size_t)N), *hi = (double *)malloc(sizeof(double) * (size_t)N);
    if (!lo || !hi) { free(lo); free(hi); return OC_ERR_ARG; }
    double t = 0.0, h = dt0;
    int acc = 0, rej = 0, total = 0, s = OC_OK;
    for (int k = 0; k < max_steps && t < t_end; k++) {
        if (h > t_end - t) h = t_end - t;
        double bound = oc_spectrum_bound(pb, u);
        double eig = -1.05 * bound, c = eig / 2.0, gamma = -eig / 4.0;
        double err = 0.0;
        int it = 0;
        s = oc_step_ex(pb, OC_JAC_EXACT, method, u, lo, hi, &err, h, c, gamma, rtol, atol, xi, max_nodes, &it);
        total += it;
        if (s == OC_ERR_NOCONV || s == OC_ERR_NONFINITE) {   /* a failed step is a rejected one */
            err = INFINITY;
            s = OC_OK;
        }
        if (s) break;
        int ok = err <= tol;
        if (log_dt) log_dt[k] = h;
        if (log_err) log_err[k] = err;
        if (log_acc) log_acc[k] = ok;
        double fac = err > 0.0 ? 0.9 * pow(tol / err, 1.0 / (q + 1)) : 5.0;
        if (fac > 5.0) fac = 5.0;
        if (fac < 0.2) fac = 0.2;
        if (ok) {
            memcpy(u, hi, sizeof(double) * (size_t)N);
            t = (h == t_end - t) ? t_end : t + h;
            acc++;
        } else {
            rej++;
        }
        h = h * fac;
    }
    if (!s && t < t_end) s = OC_ERR_NOCONV;   /* step budget exhausted */
    if (accepted) *accepted = acc;
    if (rejected) *rejected = rej;
    if (iters) *iters = total;
    free(lo);
    free(hi);
    return s;
}
