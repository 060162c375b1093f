// lx_dev.cuh -- device helpers shared by the sm_100a kernel translation units (not part of the ABI):
// memory-order primitives, phi_l and the in-kernel Newton coefficients, deterministic reductions, the
// fused stencil tiles, the P:155 decision and the grid barrier.  Included by lx_k_*.cu and lx_kernels.cu.
#pragma once
#include "lx_internal.h"

#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

namespace lx {

#define FULL_MASK 0xffffffffu

// Bounds checks of the debug build (-DLX_DEBUG_BOUNDS; tools/debug_bounds.sh): a failed check prints the
// site and traps.  Compiled out of the product build.
#ifdef LX_DEBUG_BOUNDS
#define LX_DCHECK(cond, what)                                                                              \
    do {                                                                                                   \
        if (!(cond)) {                                                                                     \
            printf("LX_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x);                                                                           \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
#else
#define LX_DCHECK(cond, what) \
    do {                      \
    } while (0)
#endif

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// spin-wait read: relaxed (no L1 invalidation per poll); the waiter issues one fence_acquire() after
// it has seen the released value (relaxed load + fence.acq_rel = acquire pattern)
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ const double* rowp(const RowSrc& s, int r) {
    if ((unsigned)r < (unsigned)s.n_loc) return s.base + (long long)r * s.stride;
    if (s.ghost) return s.ghost + (long long)(r < 0 ? 0 : r - s.n_loc + 1) * s.stride;
    return s.base + (long long)(r < 0 ? r + s.n_loc : r - s.n_loc) * s.stride;
}

// phi_l with explicitly rounded operations (no FMA contraction), so every kernel
// that evaluates it -- and every coefficient derived from it -- is bitwise reproducible.
// Taylor terms use the constant reciprocals 1/n (one multiply instead of a division).
static __constant__ double c_inv_int[40] = {
    0.0, 1.0, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7, 1.0 / 8, 1.0 / 9, 1.0 / 10,
    1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19, 1.0 / 20,
    1.0 / 21, 1.0 / 22, 1.0 / 23, 1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28, 1.0 / 29, 1.0 / 30,
    1.0 / 31, 1.0 / 32, 1.0 / 33, 1.0 / 34, 1.0 / 35, 1.0 / 36, 1.0 / 37, 1.0 / 38, 1.0 / 39};

static __constant__ double c_inv_fact[6] = {1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0};

static __device__ double phi_dev(int l, double z) {
    const double* inv_fact = c_inv_fact;   // constant bank (a local array indexed by l would live in local memory)
    if (fabs(z) < 2.0) {   // Taylor: sum_k z^k/(k+l)!  (34 terms: 2^34/34! ~ 1e-29)
        double term = inv_fact[l], s = term;
#pragma unroll
        for (int k = 1; k < 34; k++) {
            term = __dmul_rn(term, __dmul_rn(z, c_inv_int[k + l]));
            s = __dadd_rn(s, term);
        }
        return s;
    }
    double p = exp(z);
    for (int j = 0; j < l; j++) p = __ddiv_rn(__dsub_rn(p, inv_fact[j]), z);
    return p;
}

__device__ __forceinline__ double coef_arg(double a, double dt, double c, double gamma, double x) {
    // a*dt*(c + gamma*x), explicitly rounded (no contraction)
    return __dmul_rn(__dmul_rn(a, dt), __dadd_rn(c, __dmul_rn(gamma, x)));
}

__device__ __forceinline__ double P_c(const LejaParams& P) { return P.cg_dev ? P.cg_dev[0] : P.cc; }
__device__ __forceinline__ double P_g(const LejaParams& P) { return P.cg_dev ? P.cg_dev[1] : P.cgamma; }
__device__ __forceinline__ double P_alpha(const LejaParams& P) {
    return P.cg_dev ? (P.cdt == 0.0 ? 0.0 : 1.0 / P.cg_dev[1]) : P.alpha;
}

__device__ __forceinline__ double coef_h(const LejaParams& P, int k, int j) {
    return phi_dev(P.lk[k], coef_arg(P.ak[k], P.cdt, P_c(P), P_g(P), P.xi[j]));
}

// one step of the recurrence: (d - d_i) * 1/(xi_j - xi_i), explicitly rounded
__device__ __forceinline__ double dd_step(double d, double di, double r) { return __dmul_rn(__dsub_rn(d, di), r); }

__device__ __forceinline__ double coef_fold(const LejaParams& P, int K, int k, int j) {
    double d = coef_h(P, k, j);
    const int M = P.max_nodes;
    const double* tab = P.table + 1 + k;
    const double* Rc = P.R + j;
    int i = 0;
    for (; i + 4 <= j; i += 4) {
        const double t0 = tab[(size_t)i * (1 + K)], t1 = tab[(size_t)(i + 1) * (1 + K)];
        const double t2 = tab[(size_t)(i + 2) * (1 + K)], t3 = tab[(size_t)(i + 3) * (1 + K)];
        const double r0 = Rc[(size_t)i * M], r1 = Rc[(size_t)(i + 1) * M];
        const double r2 = Rc[(size_t)(i + 2) * M], r3 = Rc[(size_t)(i + 3) * M];
        d = dd_step(d, t0, r0);
        d = dd_step(d, t1, r1);
        d = dd_step(d, t2, r2);
        d = dd_step(d, t3, r3);
    }
    for (; i < j; i++) d = dd_step(d, tab[(size_t)i * (1 + K)], Rc[(size_t)i * M]);
    return d;
}

// d_0, d_1, d_2 of accumulator k: computed by lane 0 of every warp, broadcast by shuffle
// (all lanes of the warp must call it).
__device__ __forceinline__ void coef_first3(const LejaParams& P, int k, double& d0, double& d1, double& d2) {
    const int M = P.max_nodes;
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
    if ((threadIdx.x & 31) == 0) {
        e0 = coef_h(P, k, 0);
        e1 = M > 1 ? dd_step(coef_h(P, k, 1), e0, P.R[1]) : 0.0;
        e2 = M > 2 ? dd_step(dd_step(coef_h(P, k, 2), e0, P.R[2]), e1, P.R[M + 2]) : 0.0;
    }
    d0 = __shfl_sync(0xffffffffu, e0, 0);
    d1 = __shfl_sync(0xffffffffu, e1, 0);
    d2 = __shfl_sync(0xffffffffu, e2, 0);
}

// Coefficient warp: write rows 0..2 (prologue) or row j (>= 3) of the table.
template <int K>
__device__ __forceinline__ void coef_write_row(const LejaParams& P, int j, int lane, int active, const double* dk) {
    if (j >= P.max_nodes) return;
    double* row = P.table + (size_t)j * (1 + K);
    if (lane == 0) row[0] = (j == 0 || P.cdt == 0.0) ? 0.0 : (-P_c(P) / P_g(P) - P.xi[j - 1]);
    if (lane < K && ((active >> lane) & 1)) {
        double v = 0.0;
        if (dk) {   // select by unrolled compare: an array indexed by the lane would live in local memory
#pragma unroll
            for (int k = 0; k < K; k++)
                if (lane == k) v = dk[k];
        } else {
            v = coef_fold(P, K, lane, j);
        }
        row[1 + lane] = v;
    }
}

__device__ __forceinline__ double coef_beta(const LejaParams& P, int m) {
    return (P.cdt == 0.0) ? 0.0 : (-P_c(P) / P_g(P) - P.xi[m - 1]);
}

// Deterministic block reduction of n values: xor-butterfly inside warps, then
// warps summed in index order by thread 0.  Result valid in thread 0.
template <int N>
__device__ __forceinline__ void block_reduce(double (&v)[N], double (*s_red)[kSlot]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < N; i++) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[i] += __shfl_xor_sync(FULL_MASK, v[i], off);
    }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N; i++) s_red[warp][i] = v[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < N; i++) {
            double s = s_red[0][i];
            for (int w = 1; w < kWarps; w++) s += s_red[w][i];
            v[i] = s;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double nl_rem(double react, double x, double u) {
    // F(x) = g(x) - g'(u) x,  g(x) = react (x - x^3)    (reading R18)
    const double g = react * (x - x * x * x);
    const double gp = react * (1.0 - 3.0 * u * u);
    return g - gp * x;
}

enum TileMode { M_LEJA = 0, M_POWER = 1, M_RHS = 2, M_REM = 3 };

// One warp work unit of the 2D stencil (64 columns x kRT rows).
template <int K, bool DIAG, bool FIRST, int MODE, bool RO>
__device__ __forceinline__ void tile2d(const LejaParams& P, const RowSrc& src, double* __restrict__ dst,
                                       int unit, int lane, double beta, const double* d0, const double* dm,
                                       int active, double scale, double& sy, double* sp) {
    const int b = unit % P.nb;
    const int rb = unit / P.nb;
    const int n1 = P.n1;
    const int j0 = b * 64 + 2 * lane;
    const bool valid = j0 < n1;
    const int last = min(31, ((n1 - b * 64) >> 1) - 1);
    const int i0 = rb * kRT;
    const int nout = min(kRT, P.n_loc - i0);
    const Stencil& S = P.st;

    double2 w[kRT + 3];
#pragma unroll
    for (int t = 0; t < kRT + 3; t++) {
        w[t] = make_double2(0.0, 0.0);
        if (valid && t < nout + 3) {
            const double* rp = rowp(src, i0 - 1 + t) + j0;
            w[t] = RO ? ldg2(rp) : ld2(rp);
        }
    }
    double hl[kRT];
    double2 hr[kRT];
#pragma unroll
    for (int t = 0; t < kRT; t++) {
        hl[t] = 0.0;
        hr[t] = make_double2(0.0, 0.0);
        if (t < nout) {
            const double* rp = rowp(src, i0 + t);
            if (lane == 0) {
                const int jl = (j0 == 0) ? n1 - 1 : j0 - 1;
                hl[t] = RO ? __ldg(rp + jl) : rp[jl];
            }
            if (lane == last) {
                int jr = j0 + 2;
                if (jr >= n1) jr -= n1;
                hr[t] = RO ? ldg2(rp + jr) : ld2(rp + jr);
            }
        }
    }
    constexpr int KK = K > 0 ? K : 1;
    double2 pv[kRT][KK];
    double2 uu[kRT];
#pragma unroll
    for (int t = 0; t < kRT; t++) {
        const long long off = (long long)(i0 + t) * n1 + j0;
        if (MODE == M_LEJA && !FIRST) {
#pragma unroll
            for (int k = 0; k < KK; k++) {
                pv[t][k] = make_double2(0.0, 0.0);
                if (valid && t < nout && ((active >> k) & 1)) pv[t][k] = ld2(P.p[k] + off);
            }
        }
        uu[t] = make_double2(0.0, 0.0);
        if (DIAG && valid && t < nout) uu[t] = ldg2(P.u + off);
    }

#pragma unroll
    for (int t = 0; t < kRT; t++) {
        if (t < nout) {  // uniform across the warp
            const double2 yc = w[t + 1], up = w[t], dn1 = w[t + 2], dn2 = w[t + 3];
            double left = __shfl_up_sync(FULL_MASK, yc.y, 1);
            double r1 = __shfl_down_sync(FULL_MASK, yc.x, 1);
            double r2 = __shfl_down_sync(FULL_MASK, yc.y, 1);
            if (lane == 0) left = hl[t];
            if (lane == last) {
                r1 = hr[t].x;
                r2 = hr[t].y;
            }
            // A y at (i, j0) and (i, j0+1): fixed summation order
            double ax = S.c0 * yc.x;
            ax = fma(S.m1[0], up.x, ax);
            ax = fma(S.p1[0], dn1.x, ax);
            ax = fma(S.p2[0], dn2.x, ax);
            ax = fma(S.m1[1], left, ax);
            ax = fma(S.p1[1], yc.y, ax);
            ax = fma(S.p2[1], r1, ax);
            double ay = S.c0 * yc.y;
            ay = fma(S.m1[0], up.y, ay);
            ay = fma(S.p1[0], dn1.y, ay);
            ay = fma(S.p2[0], dn2.y, ay);
            ay = fma(S.m1[1], yc.x, ay);
            ay = fma(S.p1[1], r1, ay);
            ay = fma(S.p2[1], r2, ay);
            if (DIAG) {
                ax = fma(fma(S.qb, uu[t].x * uu[t].x, S.qa), yc.x, ax);
                ay = fma(fma(S.qb, uu[t].y * uu[t].y, S.qa), yc.y, ay);
            }
            double2 yn;
            if (MODE == M_POWER) {
                yn.x = scale * ax;
                yn.y = scale * ay;
            } else if (MODE == M_RHS) {
                // f(u)*scale = scale*(A u + react*(u - u^3) [+ S])
                double fx = fma(S.react, yc.x - yc.x * yc.x * yc.x, ax);
                double fy = fma(S.react, yc.y - yc.y * yc.y * yc.y, ay);
                if (P.source && valid) {
                    const double2 sv = ldg2(P.source + (long long)(i0 + t) * n1 + j0);
                    fx += sv.x;
                    fy += sv.y;
                }
                yn.x = scale * fx;
                yn.y = scale * fy;
            } else {
                yn.x = fma(scale, ax, beta * yc.x);   // M_LEJA: scale = alpha = 1/gamma
                yn.y = fma(scale, ay, beta * yc.y);
            }
            if (valid) {
                const long long off = (long long)(i0 + t) * n1 + j0;
                st2(dst + off, yn);
                sy = fma(yn.x, yn.x, sy);
                sy = fma(yn.y, yn.y, sy);
                if (MODE == M_LEJA) {
#pragma unroll
                    for (int k = 0; k < KK; k++) {
                        if ((active >> k) & 1) {
                            double2 pn;
                            if (FIRST) {
                                pn.x = fma(dm[k], yn.x, d0[k] * yc.x);
                                pn.y = fma(dm[k], yn.y, d0[k] * yc.y);
                            } else {
                                pn.x = fma(dm[k], yn.x, pv[t][k].x);
                                pn.y = fma(dm[k], yn.y, pv[t][k].y);
                            }
                            st2(P.p[k] + off, pn);
                            sp[k] = fma(pn.x, pn.x, sp[k]);
                            sp[k] = fma(pn.y, pn.y, sp[k]);
                        }
                    }
                }
            }
        }
    }
}


// One warp work unit of the 3D stencil: 64 contiguous k (dim 2) x one j row (dim 1)
// x kRT3 planes (dim 0).  i-neighbours from the plane window, j-neighbours from
// rows j-1, j+1, j+2 of the same plane (adjacent warps own adjacent j -> L1 hits),
// k-neighbours by shuffles + edge-lane halo loads.  Units: u = (pb*nb + b)*n1 + j.
template <int K, bool DIAG, bool FIRST, int MODE, bool RO>
__device__ __forceinline__ void tile3d(const LejaParams& P, const RowSrc& src, double* __restrict__ dst,
                                       int unit, int lane, double beta, const double* d0, const double* dm,
                                       int active, double scale, double& sy, double* sp) {
    const int n1 = P.n1, n2 = P.n2;
    const int j = unit % n1;
    const int t0 = unit / n1;
    const int b = t0 % P.nb;
    const int pb = t0 / P.nb;
    const int k0 = b * 64 + 2 * lane;
    const bool valid = k0 < n2;
    const int last = min(31, ((n2 - b * 64) >> 1) - 1);
    const int i0 = pb * kRT3;
    const int nout = min(kRT3, P.n_loc - i0);
    const int jm = (j == 0) ? n1 - 1 : j - 1;
    const int jp1 = (j + 1 >= n1) ? j + 1 - n1 : j + 1;
    const int jp2 = (j + 2 >= n1) ? j + 2 - n1 : j + 2;
    const Stencil& S = P.st;
    auto LD2 = [&](const double* q) { return RO ? ldg2(q) : ld2(q); };

    double2 w[kRT3 + 3];
#pragma unroll
    for (int t = 0; t < kRT3 + 3; t++) {
        w[t] = make_double2(0.0, 0.0);
        if (valid && t < nout + 3) w[t] = LD2(rowp(src, i0 - 1 + t) + (long long)j * n2 + k0);
    }
    double2 wm[kRT3], wp1[kRT3], wp2[kRT3];
    double hl[kRT3];
    double2 hr[kRT3];
#pragma unroll
    for (int t = 0; t < kRT3; t++) {
        wm[t] = wp1[t] = wp2[t] = hr[t] = make_double2(0.0, 0.0);
        hl[t] = 0.0;
        if (t < nout) {
            const double* pl = rowp(src, i0 + t);
            if (valid) {
                wm[t] = LD2(pl + (long long)jm * n2 + k0);
                wp1[t] = LD2(pl + (long long)jp1 * n2 + k0);
                wp2[t] = LD2(pl + (long long)jp2 * n2 + k0);
            }
            const double* rp = pl + (long long)j * n2;
            if (lane == 0) {
                const int kl = (k0 == 0) ? n2 - 1 : k0 - 1;
                hl[t] = RO ? __ldg(rp + kl) : rp[kl];
            }
            if (lane == last) {
                int kr = k0 + 2;
                if (kr >= n2) kr -= n2;
                hr[t] = LD2(rp + kr);
            }
        }
    }
    constexpr int KK = K > 0 ? K : 1;
    double2 pv[kRT3][KK];
    double2 uu[kRT3];
#pragma unroll
    for (int t = 0; t < kRT3; t++) {
        const long long off = ((long long)(i0 + t) * n1 + j) * n2 + k0;
        if (MODE == M_LEJA && !FIRST) {
#pragma unroll
            for (int k = 0; k < KK; k++) {
                pv[t][k] = make_double2(0.0, 0.0);
                if (valid && t < nout && ((active >> k) & 1)) pv[t][k] = ld2(P.p[k] + off);
            }
        }
        uu[t] = make_double2(0.0, 0.0);
        if (DIAG && valid && t < nout) uu[t] = ldg2(P.u + off);
    }
#pragma unroll
    for (int t = 0; t < kRT3; t++) {
        if (t < nout) {
            const double2 yc = w[t + 1], up = w[t], dn1 = w[t + 2], dn2 = w[t + 3];
            double left = __shfl_up_sync(FULL_MASK, yc.y, 1);
            double r1 = __shfl_down_sync(FULL_MASK, yc.x, 1);
            double r2 = __shfl_down_sync(FULL_MASK, yc.y, 1);
            if (lane == 0) left = hl[t];
            if (lane == last) {
                r1 = hr[t].x;
                r2 = hr[t].y;
            }
            double ax = S.c0 * yc.x;
            ax = fma(S.m1[0], up.x, ax);
            ax = fma(S.p1[0], dn1.x, ax);
            ax = fma(S.p2[0], dn2.x, ax);
            ax = fma(S.m1[1], wm[t].x, ax);
            ax = fma(S.p1[1], wp1[t].x, ax);
            ax = fma(S.p2[1], wp2[t].x, ax);
            ax = fma(S.m1[2], left, ax);
            ax = fma(S.p1[2], yc.y, ax);
            ax = fma(S.p2[2], r1, ax);
            double ay = S.c0 * yc.y;
            ay = fma(S.m1[0], up.y, ay);
            ay = fma(S.p1[0], dn1.y, ay);
            ay = fma(S.p2[0], dn2.y, ay);
            ay = fma(S.m1[1], wm[t].y, ay);
            ay = fma(S.p1[1], wp1[t].y, ay);
            ay = fma(S.p2[1], wp2[t].y, ay);
            ay = fma(S.m1[2], yc.x, ay);
            ay = fma(S.p1[2], r1, ay);
            ay = fma(S.p2[2], r2, ay);
            if (DIAG) {
                ax = fma(fma(S.qb, uu[t].x * uu[t].x, S.qa), yc.x, ax);
                ay = fma(fma(S.qb, uu[t].y * uu[t].y, S.qa), yc.y, ay);
            }
            double2 yn;
            if (MODE == M_POWER) {
                yn.x = scale * ax;
                yn.y = scale * ay;
            } else if (MODE == M_RHS) {
                double fx = fma(S.react, yc.x - yc.x * yc.x * yc.x, ax);
                double fy = fma(S.react, yc.y - yc.y * yc.y * yc.y, ay);
                if (P.source && valid) {
                    const double2 sv = ldg2(P.source + ((long long)(i0 + t) * n1 + j) * n2 + k0);
                    fx += sv.x;
                    fy += sv.y;
                }
                yn.x = scale * fx;
                yn.y = scale * fy;
            } else {
                yn.x = fma(scale, ax, beta * yc.x);   // M_LEJA: scale = alpha = 1/gamma
                yn.y = fma(scale, ay, beta * yc.y);
            }
            if (valid) {
                const long long off = ((long long)(i0 + t) * n1 + j) * n2 + k0;
                st2(dst + off, yn);
                sy = fma(yn.x, yn.x, sy);
                sy = fma(yn.y, yn.y, sy);
                if (MODE == M_LEJA) {
#pragma unroll
                    for (int k = 0; k < KK; k++) {
                        if ((active >> k) & 1) {
                            double2 pn;
                            if (FIRST) {
                                pn.x = fma(dm[k], yn.x, d0[k] * yc.x);
                                pn.y = fma(dm[k], yn.y, d0[k] * yc.y);
                            } else {
                                pn.x = fma(dm[k], yn.x, pv[t][k].x);
                                pn.y = fma(dm[k], yn.y, pv[t][k].y);
                            }
                            st2(P.p[k] + off, pn);
                            sp[k] = fma(pn.x, pn.x, sp[k]);
                            sp[k] = fma(pn.y, pn.y, sp[k]);
                        }
                    }
                }
            }
        }
    }
}


// Output of one row of the flux-form tile: y_m (or f, remainder, power iterate) at (i, j0..j0+1), its
// norm, and the Newton accumulators p_m = p_{m-1} + d_m y_m (Leja mode).
template <int K, bool FIRST, int MODE>
__device__ __forceinline__ void tile2d_flux_out(const LejaParams& P, double* __restrict__ dst, int i, int j0,
                                                bool valid, double2 yc, const double* res, const double2* pv,
                                                double beta, const double* d0, const double* dm, int active,
                                                double scale, double& sy, double* sp) {
    constexpr int KK = K > 0 ? K : 1;
    const int n1 = P.n1;
    double2 yn;
    if (MODE == M_POWER) {
        yn.x = scale * res[0];
        yn.y = scale * res[1];
    } else if (MODE == M_RHS) {
        double fx = res[0], fy = res[1];
        if (P.source && valid) {
            const double2 sv = ldg2(P.source + (long long)i * n1 + j0);
            fx += sv.x;
            fy += sv.y;
        }
        yn.x = scale * fx;
        yn.y = scale * fy;
    } else if (MODE == M_REM) {
        yn.x = res[0];
        yn.y = res[1];
    } else {
        yn.x = fma(scale, res[0], beta * yc.x);
        yn.y = fma(scale, res[1], beta * yc.y);
    }
    if (valid) {
        const long long off = (long long)i * n1 + j0;
        st2(dst + off, yn);
        sy = fma(yn.x, yn.x, sy);
        sy = fma(yn.y, yn.y, sy);
        if (MODE == M_LEJA) {
#pragma unroll
            for (int k = 0; k < KK; k++) {
                if ((active >> k) & 1) {
                    double2 pn;
                    if (FIRST) {
                        pn.x = fma(dm[k], yn.x, d0[k] * yc.x);
                        pn.y = fma(dm[k], yn.y, d0[k] * yc.y);
                    } else {
                        pn.x = fma(dm[k], yn.x, pv[k].x);
                        pn.y = fma(dm[k], yn.y, pv[k].y);
                    }
                    st2(P.p[k] + off, pn);
                    sp[k] = fma(pn.x, pn.x, sp[k]);
                    sp[k] = fma(pn.y, pn.y, sp[k]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Flux-form 2D tile (Problem III, viscous Burgers; exact Jacobian R13):
//   M_LEJA/M_POWER: A y = diff lap(y) + sum_d D_d((nu + beta u) y)      (J(u) y)
//   M_RHS:          f(u) = diff lap(u) + sum_d D_d((nu + beta/2 u) u) [+ react g(u) + S]
//   M_REM:          a2 * (dt F(x) - dt F(u)),  F(x) = sum_d D_d(beta/2 x^2 - beta u x) + g-part
// Two register windows (the field y/x and u) with the same row / shuffle / halo
// pattern as tile2d.  Single GPU (u is read with periodic wrap).  For M_REM the
// `beta` argument carries dt and `scale` carries a2.
// ---------------------------------------------------------------------------
template <int K, bool FIRST, int MODE, bool RO>
__device__ __forceinline__ void tile2d_flux(const LejaParams& P, const RowSrc& src, double* __restrict__ dst,
                                            int unit, int lane, double beta, const double* d0, const double* dm,
                                            int active, double scale, double& sy, double* sp) {
    constexpr bool TWO = (MODE != M_RHS);   // RHS: the coefficient field is the input itself
    const int b = unit % P.nb;
    const int rb = unit / P.nb;
    const int n1 = P.n1;
    const int j0 = b * 64 + 2 * lane;
    const bool valid = j0 < n1;
    const int last = min(31, ((n1 - b * 64) >> 1) - 1);
    const int i0 = rb * kRTF;
    const int nout = min(kRTF, P.n_loc - i0);
    const Stencil& S = P.st;
    const RowSrc us{P.u, nullptr, (long long)n1, P.n_loc, 0};
    auto LD2 = [&](const double* q) { return RO ? ldg2(q) : ld2(q); };
    auto LD1 = [&](const double* q) { return RO ? __ldg(q) : *q; };

    double2 w[kRTF + 3], uw[kRTF + 3];
#pragma unroll
    for (int t = 0; t < kRTF + 3; t++) {
        w[t] = uw[t] = make_double2(0.0, 0.0);
        if (valid && t < nout + 3) {
            w[t] = LD2(rowp(src, i0 - 1 + t) + j0);
            if (TWO) uw[t] = ldg2(rowp(us, i0 - 1 + t) + j0);
        }
    }
    double hl[kRTF], uhl[kRTF];
    double2 hr[kRTF], uhr[kRTF];
#pragma unroll
    for (int t = 0; t < kRTF; t++) {
        hl[t] = uhl[t] = 0.0;
        hr[t] = uhr[t] = make_double2(0.0, 0.0);
        if (t < nout) {
            const double* rp = rowp(src, i0 + t);
            const double* rq = rowp(us, i0 + t);
            const int jl = (j0 == 0) ? n1 - 1 : j0 - 1;
            int jr = j0 + 2;
            if (jr >= n1) jr -= n1;
            if (lane == 0) {
                hl[t] = LD1(rp + jl);
                if (TWO) uhl[t] = __ldg(rq + jl);
            }
            if (lane == last) {
                hr[t] = LD2(rp + jr);
                if (TWO) uhr[t] = ldg2(rq + jr);
            }
        }
    }
    constexpr int KK = K > 0 ? K : 1;
    double2 pv[kRTF][KK];
#pragma unroll
    for (int t = 0; t < kRTF; t++) {
        const long long off = (long long)(i0 + t) * n1 + j0;
        if (MODE == M_LEJA && !FIRST) {
#pragma unroll
            for (int k = 0; k < KK; k++) {
                pv[t][k] = make_double2(0.0, 0.0);
                if (valid && t < nout && ((active >> k) & 1)) pv[t][k] = ld2(P.p[k] + off);
            }
        }
    }
    const double nu = S.nu, bt = S.flux;
    // J y (Leja / power modes): the flux field G = (nu + beta u) y is evaluated once per point of the
    // window (in place of u) and its halo, instead of once per stencil use (7x); the same expression,
    // so the result is bitwise that of evaluating it at each use.  The reaction diagonal
    // qb u^2 + qa is kept for the output rows.
    constexpr bool PRE = (MODE == M_LEJA || MODE == M_POWER);
    double2 qd[kRTF];
    if (PRE) {
#pragma unroll
        for (int t = 0; t < kRTF; t++) {
            qd[t] = make_double2(0.0, 0.0);
            if (S.react != 0.0) {
                qd[t].x = fma(S.qb, uw[t + 1].x * uw[t + 1].x, S.qa);
                qd[t].y = fma(S.qb, uw[t + 1].y * uw[t + 1].y, S.qa);
            }
        }
#pragma unroll
        for (int t = 0; t < kRTF + 3; t++) {
            uw[t].x = (nu + bt * uw[t].x) * w[t].x;
            uw[t].y = (nu + bt * uw[t].y) * w[t].y;
        }
#pragma unroll
        for (int t = 0; t < kRTF; t++) {
            uhl[t] = (nu + bt * uhl[t]) * hl[t];
            uhr[t].x = (nu + bt * uhr[t].x) * hr[t].x;
            uhr[t].y = (nu + bt * uhr[t].y) * hr[t].y;
        }
    }
#pragma unroll
    for (int t = 0; t < kRTF; t++) {
        if (PRE && t < nout) {
            const double2 yc = w[t + 1], up = w[t], dn1 = w[t + 2];
            const double2 gc = uw[t + 1], gu = uw[t], gd1 = uw[t + 2], gd2 = uw[t + 3];
            double yl = __shfl_up_sync(FULL_MASK, yc.y, 1);
            double yr1 = __shfl_down_sync(FULL_MASK, yc.x, 1);
            double gl = __shfl_up_sync(FULL_MASK, gc.y, 1);
            double gr1 = __shfl_down_sync(FULL_MASK, gc.x, 1);
            double gr2 = __shfl_down_sync(FULL_MASK, gc.y, 1);
            if (lane == 0) {
                yl = hl[t];
                gl = uhl[t];
            }
            if (lane == last) {
                yr1 = hr[t].x;
                gr1 = uhr[t].x;
                gr2 = uhr[t].y;
            }
            double res[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const double y0 = h ? yc.y : yc.x;
                const double ymr = h ? up.y : up.x, ypr = h ? dn1.y : dn1.x;
                const double ymc = h ? yc.x : yl, ypc = h ? yr1 : yc.y;
                const double g0 = h ? gc.y : gc.x;
                const double gmr = h ? gu.y : gu.x, gpr = h ? gd1.y : gd1.x, gp2r = h ? gd2.y : gd2.x;
                const double gmc = h ? gc.x : gl, gpc = h ? gr1 : gc.y, gp2c = h ? gr2 : gr1;
                double adv = (S.a0[0] + S.a0[1]) * g0;
                adv = fma(S.am1[0], gmr, adv);
                adv = fma(S.ap1[0], gpr, adv);
                adv = fma(S.ap2[0], gp2r, adv);
                adv = fma(S.am1[1], gmc, adv);
                adv = fma(S.ap1[1], gpc, adv);
                adv = fma(S.ap2[1], gp2c, adv);
                double lap = S.dd0 * y0;
                lap = fma(S.dm1[0], ymr, lap);
                lap = fma(S.dp1[0], ypr, lap);
                lap = fma(S.dm1[1], ymc, lap);
                lap = fma(S.dp1[1], ypc, lap);
                double a = lap + adv;
                if (S.react != 0.0) a = fma(h ? qd[t].y : qd[t].x, y0, a);
                res[h] = a;
            }
            tile2d_flux_out<K, FIRST, MODE>(P, dst, i0 + t, j0, valid, yc, res, pv[t], beta, d0, dm, active,
                                            scale, sy, sp);
        } else if (!PRE && t < nout) {
            const double2 yc = w[t + 1], up = w[t], dn1 = w[t + 2], dn2 = w[t + 3];
            const double2 uc = TWO ? uw[t + 1] : yc, uu = TWO ? uw[t] : up;
            const double2 ud1 = TWO ? uw[t + 2] : dn1, ud2 = TWO ? uw[t + 3] : dn2;
            double yl = __shfl_up_sync(FULL_MASK, yc.y, 1);
            double yr1 = __shfl_down_sync(FULL_MASK, yc.x, 1);
            double yr2 = __shfl_down_sync(FULL_MASK, yc.y, 1);
            double ul = __shfl_up_sync(FULL_MASK, uc.y, 1);
            double ur1 = __shfl_down_sync(FULL_MASK, uc.x, 1);
            double ur2 = __shfl_down_sync(FULL_MASK, uc.y, 1);
            if (lane == 0) {
                yl = hl[t];
                ul = TWO ? uhl[t] : hl[t];
            }
            if (lane == last) {
                yr1 = hr[t].x;
                yr2 = hr[t].y;
                ur1 = TWO ? uhr[t].x : hr[t].x;
                ur2 = TWO ? uhr[t].y : hr[t].y;
            }
            // pointwise flux field w(y, u) at the stencil points
            auto wf = [&](double yv, double uv) -> double {
                if (MODE == M_RHS) return (nu + 0.5 * bt * uv) * uv;
                if (MODE == M_REM) return 0.5 * bt * yv * yv - bt * uv * yv;
                return (nu + bt * uv) * yv;
            };
            auto wu = [&](double uv) -> double { return -0.5 * bt * uv * uv; };   // M_REM: F(u) field
            // value at point x=(i,j0) and y=(i,j0+1)
            double res[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const double y0 = h ? yc.y : yc.x, u0 = h ? uc.y : uc.x;
                const double ymr = h ? up.y : up.x, ypr = h ? dn1.y : dn1.x, yp2r = h ? dn2.y : dn2.x;
                const double umr = h ? uu.y : uu.x, upr = h ? ud1.y : ud1.x, up2r = h ? ud2.y : ud2.x;
                const double ymc = h ? yc.x : yl, ypc = h ? yr1 : yc.y, yp2c = h ? yr2 : yr1;
                const double umc = h ? uc.x : ul, upc = h ? ur1 : uc.y, up2c = h ? ur2 : ur1;
                double adv = (S.a0[0] + S.a0[1]) * wf(y0, u0);
                adv = fma(S.am1[0], wf(ymr, umr), adv);
                adv = fma(S.ap1[0], wf(ypr, upr), adv);
                adv = fma(S.ap2[0], wf(yp2r, up2r), adv);
                adv = fma(S.am1[1], wf(ymc, umc), adv);
                adv = fma(S.ap1[1], wf(ypc, upc), adv);
                adv = fma(S.ap2[1], wf(yp2c, up2c), adv);
                if (MODE == M_REM) {
                    double advu = (S.a0[0] + S.a0[1]) * wu(u0);
                    advu = fma(S.am1[0], wu(umr), advu);
                    advu = fma(S.ap1[0], wu(upr), advu);
                    advu = fma(S.ap2[0], wu(up2r), advu);
                    advu = fma(S.am1[1], wu(umc), advu);
                    advu = fma(S.ap1[1], wu(upc), advu);
                    advu = fma(S.ap2[1], wu(up2c), advu);
                    const double Fx = adv + nl_rem(S.react, y0, u0);
                    const double Fu = advu + nl_rem(S.react, u0, u0);
                    res[h] = scale * (beta * Fx + (-beta) * Fu);   // a2 * (dt F(x) - dt F(u))
                } else {
                    double lap = S.dd0 * y0;
                    lap = fma(S.dm1[0], ymr, lap);
                    lap = fma(S.dp1[0], ypr, lap);
                    lap = fma(S.dm1[1], ymc, lap);
                    lap = fma(S.dp1[1], ypc, lap);
                    double a = lap + adv;
                    if (MODE == M_RHS) {
                        a = fma(S.react, y0 - y0 * y0 * y0, a);
                    } else if (S.react != 0.0) {
                        a = fma(fma(S.qb, u0 * u0, S.qa), y0, a);
                    }
                    res[h] = a;
                }
            }
            tile2d_flux_out<K, FIRST, MODE>(P, dst, i0 + t, j0, valid, yc, res, pv[t], beta, d0, dm, active,
                                            scale, sy, sp);
        }
    }
}

template <int NDIM, int K, bool DIAG, bool FIRST, int MODE, bool RO>
__device__ __forceinline__ void tile(const LejaParams& P, const RowSrc& src, double* __restrict__ dst, int unit,
                                     int lane, double beta, const double* d0, const double* dm, int active,
                                     double scale, double& sy, double* sp) {
    if (NDIM == 4)   // flux form (Burgers), 2D
        tile2d_flux<K, FIRST, MODE, RO>(P, src, dst, unit, lane, beta, d0, dm, active, scale, sy, sp);
    else if (NDIM == 2)
        tile2d<K, DIAG, FIRST, MODE, RO>(P, src, dst, unit, lane, beta, d0, dm, active, scale, sy, sp);
    else
        tile3d<K, DIAG, FIRST, MODE, RO>(P, src, dst, unit, lane, beta, d0, dm, active, scale, sy, sp);
}

// ---------------------------------------------------------------------------
// Stopping decision of P:155 for iteration m (shared by the persistent and the
// step kernels).  sums = {S_y, S_p^(0..K-1)} over the whole (global) grid.
// rec != nullptr: the single writer updates margins / per-accumulator iters.
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ void leja_decide(const LejaParams& P, int m, const double* sums, const double* dm,
                                            int& act, int& done, int& status, Record* rec) {
    const double N = P.N_glob;
    const double ny = sqrt(sums[0] / N);
    int nact = 0;
    done = 0;
    status = 0;
    for (int k = 0; k < K; k++) {
        if (!((act >> k) & 1)) continue;
        const double err = fabs(dm[k]) * ny;
        const double thr = P.rtol * sqrt(sums[1 + k] / N) + P.atol;
        if (!isfinite(err) || !isfinite(thr)) {
            status = 6;  // LX_ERR_NONFINITE
            break;
        }
        if (err <= thr) {
            act &= ~(1 << k);
            if (rec) {
                rec->iters_k[k] = m;
                const double r = err > 0.0 ? thr / err : INFINITY;
                if (r < rec->margin_accept) rec->margin_accept = r;
            }
        } else {
            nact++;
            if (rec) {
                const double r = err / thr;
                if (r < rec->margin_reject) rec->margin_reject = r;
            }
        }
    }
    if (status) done = 1;
    else if (nact == 0) done = 1;
    else if (m >= P.max_nodes - 1) { done = 1; status = 5; }  // LX_ERR_NOCONV
    if (done && rec) {
        rec->iters += m;
        rec->ncalls += 1;
        if (rec->status == 0) rec->status = status;
    }
}

// Power iteration: estimate ||w_m|| / ||v_{m-1}|| and the scale of v_m = w_m/||w_m||.
__device__ __forceinline__ void power_decide(const LejaParams& P, int m, double sumsq, int& done, int& status,
                                             double* est_out, double* scale_out, Record* rec) {
    const double N = P.N_glob;
    const double nw = sqrt(sumsq / N);
    const double nv = (m == 1) ? sqrt((N + 3.0) / N) : 1.0;
    const double est = nw / nv;
    *est_out = est;
    *scale_out = 1.0 / nw;
    done = 0;
    status = 0;
    if (!isfinite(nw) || nw == 0.0) { done = 1; status = 6; }
    if (m >= P.power_iters) done = 1;
    if (done && rec) {
        rec->est = est;
        rec->iters += m;
        rec->ncalls += 1;
        if (rec->status == 0) rec->status = status;
    }
}

// ---------------------------------------------------------------------------
// Grid barrier with the convergence decision taken by the last arriver.
// Returns (in smem) done / active for the next iteration.
// ---------------------------------------------------------------------------
template <int K, int MODE>
__device__ __forceinline__ void barrier_decide(const LejaParams& P, int m, unsigned gen0, const double* dm,
                                               int active, double (*s_red)[kSlot], int* s_flags) {
    // Grid barrier + device-side decision.  Arrival = one acq_rel atomic per CTA
    // (releases this CTA's y/p stores and its partial slot, ordered before it by
    // bar.sync); the last arriver sums the slots in fixed order, decides, and
    // publishes {generation, status, done, active} in ONE st.release of a 64-bit
    // word, which the waiters acquire (no further fences or control reads).
    constexpr int NV = (MODE == M_LEJA) ? 1 + K : 1;
    const int tid = threadIdx.x;
    Ctrl* ctrl = P.ctrl;
    const int par = m & 1;
    __syncthreads();
    if (tid == 0) {
        const unsigned t = atom_add_acq_rel(&ctrl->arrive, 1u);
        s_flags[0] = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_flags[0]) {
        double acc[NV];
#pragma unroll
        for (int i = 0; i < NV; i++) acc[i] = 0.0;
        for (int c = tid; c < (int)gridDim.x; c += kThreads) {
            const double* slot = P.partials + ((size_t)par * gridDim.x + c) * kSlot;
#pragma unroll
            for (int i = 0; i < NV; i++) acc[i] += __ldcg(slot + i);
        }
        block_reduce<NV>(acc, s_red);
        if (tid == 0) {
            Record* rec = P.rec;
            int done = 0, status = 0, act = active;
            double scale = 0.0;
            if (MODE == M_LEJA) {
                leja_decide<K>(P, m, acc, dm, act, done, status, rec);
            } else {
                power_decide(P, m, acc[0], done, status, &ctrl->est, &scale, rec);
                ctrl->scale = scale;
            }
            ctrl->arrive = 0u;
            const unsigned long long w = ((unsigned long long)(gen0 + (unsigned)m) << 32) |
                                         ((unsigned long long)(status & 0xffff) << 16) |
                                         ((unsigned long long)(done & 0xff) << 8) | (unsigned long long)(act & 0xff);
            st_release64(&ctrl->word, w);
            s_flags[1] = done;
            s_flags[2] = act;
            s_red[0][kSlot - 1] = scale;
        }
    } else if (tid == 0) {
        unsigned long long w = ld_relaxed64(&ctrl->word);
        int spins = 0;
        while ((int)((unsigned)(w >> 32) - gen0) < m) {
            if (++spins > 32) __nanosleep(32);
            if (spins > P.timeout_spins) {
                atomicExch(&P.rec->status, 10);  // LX_ERR_TIMEOUT
                w = (1ull << 8);
                break;
            }
            w = ld_relaxed64(&ctrl->word);
        }
        fence_acquire();
        s_flags[1] = (int)((w >> 8) & 0xff);
        s_flags[2] = (int)(w & 0xff);
        if (MODE == M_POWER) s_red[0][kSlot - 1] = *(volatile double*)&ctrl->scale;
    }
    __syncthreads();
}


// stencil of the constant-coefficient operator at the two columns of a lane (same order as tile2d)
__device__ __forceinline__ void stencil2(const Stencil& S, const double2 yc, const double2 up, const double2 dn1,
                                         const double2 dn2, double left, double r1, double r2, double& ax, double& ay) {
    // the 7 stencil terms summed as a short tree (dependent FMA chain 4 deep instead of 7: the two-step
    // kernel is latency-bound on this chain), the same order in every kernel that uses it
    const double ax0 = fma(S.m1[0], up.x, S.c0 * yc.x);
    const double ax1 = fma(S.p2[0], dn2.x, S.p1[0] * dn1.x);
    const double ax2 = fma(S.p1[1], yc.y, S.m1[1] * left);
    ax = (ax0 + ax1) + fma(S.p2[1], r1, ax2);
    const double ay0 = fma(S.m1[0], up.y, S.c0 * yc.y);
    const double ay1 = fma(S.p2[0], dn2.y, S.p1[0] * dn1.y);
    const double ay2 = fma(S.p1[1], r1, S.m1[1] * yc.x);
    ay = (ay0 + ay1) + fma(S.p2[1], r2, ay2);
}

// y_m = alpha (A + diag) y_{m-1} + beta y_{m-1} at one row of the lane's two columns.
// r1/r2 come from the next lane; lane 31 uses its halo pair h (columns c0+62, c0+63).
template <bool DIAG>
__device__ __forceinline__ double2 leja_row(const Stencil& S, double alpha, double beta, const double2 up,
                                            const double2 yc, const double2 dn1, const double2 dn2, const double2 h,
                                            const double2 uu, int lane) {
    const double left = __shfl_up_sync(FULL_MASK, yc.y, 1);
    double r1 = __shfl_down_sync(FULL_MASK, yc.x, 1);
    double r2 = __shfl_down_sync(FULL_MASK, yc.y, 1);
    if (lane == 31) {
        r1 = h.x;
        r2 = h.y;
    }
    double ax, ay;
    stencil2(S, yc, up, dn1, dn2, left, r1, r2, ax, ay);
    if (DIAG) {
        ax = fma(fma(S.qb, uu.x * uu.x, S.qa), yc.x, ax);
        ay = fma(fma(S.qb, uu.y * uu.y, S.qa), yc.y, ay);
    }
    return make_double2(fma(alpha, ax, beta * yc.x), fma(alpha, ay, beta * yc.y));
}

// xor-butterfly sum of N values over the warp (fixed order: every lane ends with the same bits)
template <int N>
__device__ __forceinline__ void warp_sum(double* v) {
#pragma unroll
    for (int i = 0; i < N; i++) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[i] += __shfl_xor_sync(FULL_MASK, v[i], off);
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ double2 lds2(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed32(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys32(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}


// Co-resident CTAs (kThreads each, no dynamic smem) of a kernel on a device: SMs x blocks per SM,
// cached per (device, kernel) -- occupancy queries cost host microseconds on every Leja call.
inline int coresident(int device, const void* kern) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({device, kern});
    if (it != cache.end()) return it->second;
    int nsm = 0, per = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kThreads, 0);
    if (per < 1) per = 1;
    cache[{device, kern}] = nsm * per;
    return nsm * per;
}

template <typename Kern>
inline int max_coresident(int device, Kern kern) {
    return coresident(device, (const void*)kern);
}


// Cross-rank step of the slab kernel's barrier (ONE thread: the last arriver of this rank's grid
// barrier).  The rank's NV partial sums go to slot [epoch & 1][rank] of EVERY rank's exchange header
// (peer stores), then a system-scope release of flag[rank] = epoch on every rank; once all ranks'
// flags reached the epoch, the NV sums are replaced by the rank-ordered totals (identical on every
// rank -> identical decisions; with one rank, 0 + x = x: bitwise the single-domain sums).  A rank can
// be at most one epoch ahead of another (it waits for everybody each epoch), so two parities suffice.
// Returns 0, or 10 (LX_ERR_TIMEOUT) if a peer did not arrive within P.timeout_ns.
template <int NV>
__device__ __forceinline__ int xrank_sum(const LejaParams& P, double* acc) {
    XHdr* me = P.xh[P.xrank];
    const unsigned long long e = me->epoch + 1;
    me->epoch = e;
    const int par = (int)(e & 1);
    for (int q = 0; q < P.xranks; q++) {
        double* slot = &P.xh[q]->part[par][P.xrank][0];
#pragma unroll
        for (int i = 0; i < NV; i++) slot[i] = acc[i];
    }
    __threadfence_system();
    for (int q = 0; q < P.xranks; q++) st_release_sys64(&P.xh[q]->flag[P.xrank], e);
    const unsigned long long t0 = globaltimer_ns();
    for (int q = 0; q < P.xranks; q++) {
        while (ld_acquire_sys64(&me->flag[q]) < e) {
            if (globaltimer_ns() - t0 > P.timeout_ns) return 10;
            __nanosleep(32);
        }
    }
#pragma unroll
    for (int i = 0; i < NV; i++) {
        double s = 0.0;
        for (int q = 0; q < P.xranks; q++) s += __ldcv(&me->part[par][q][i]);
        acc[i] = s;
    }
    return 0;
}


// Key of a Leja call's parameters (node count, phi index, dt, shift / scale, vertical coefficients,
// tolerances) for the ping-pong parity prediction.
template <int K>
__device__ __forceinline__ unsigned long long tb2_call_key(const LejaParams& P) {
    unsigned long long h = 1469598103934665603ull;
    auto mix = [&h](unsigned long long x) {
        h ^= x;
        h *= 1099511628211ull;
    };
    mix((unsigned long long)P.l | ((unsigned long long)K << 8) | ((unsigned long long)P.max_nodes << 16) |
        ((unsigned long long)P.active0 << 40));
#pragma unroll
    for (int k = 0; k < K; k++) mix((unsigned long long)P.lk[k]);
    // the spectrum enters through dt*gamma and c/gamma, bucketed (1/32 octave): a time loop whose (c, gamma)
    // drift from step to step (lx_integrate, the Gershgorin bound of a nonlinear problem) keeps its
    // predictions; they steer only the scheduling (results never depend on them)
    auto bucket = [](double x) -> unsigned long long {
        if (!(x > 0.0) || !isfinite(x)) return 0x8000000000000000ull | (unsigned long long)__double_as_longlong(x);
        return (unsigned long long)(long long)floor(32.0 * log2(x));
    };
    mix((unsigned long long)__double_as_longlong(P.cdt));
    mix(bucket(P.cdt * P_g(P)));
    mix(bucket(-P_c(P) / P_g(P)));
    mix((unsigned long long)__double_as_longlong(P.rtol));
    mix((unsigned long long)__double_as_longlong(P.atol));
#pragma unroll
    for (int k = 0; k < K; k++) mix((unsigned long long)__double_as_longlong(P.ak[k]));
    return h | 1ull;
}

}  // namespace lx
