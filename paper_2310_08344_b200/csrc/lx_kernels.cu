// lx_kernels.cu -- sm_100a fp64 kernels of the LeXInt hot path (arxiv 2310.08344): overview, the
// coefficient / shift kernels, the integrator stage kernels and the preload of every kernel.
// The Leja kernels live in lx_k_leja.cu (one pass per iteration), lx_k_tb2.cu (two per pass, single
// domain and slab), lx_k_3d.cu (3D shared-memory tiles); shared device code in lx_dev.cuh.
//
// k_leja2d : ONE persistent cooperative kernel per Leja call.  Each iteration m
//            is one fused HBM pass over the grid (Eq. (2)):
//               y_m  = alpha*(A y_{m-1}) + beta_m*y_{m-1}     (alpha = 1/gamma,
//                                                              beta_m = -c/gamma - xi_{m-1})
//               p_m^(k) = p_{m-1}^(k) + d_m^(k) y_m            (k < K, active only)
//               S_y = sum y_m^2,  S_p^(k) = sum (p_m^(k))^2    (partials per CTA)
//            then a grid barrier whose last arriver sums the CTA partials in a
//            fixed order and takes the stopping decision of P:155
//               |d_m| sqrt(S_y/N) <= rtol sqrt(S_p/N) + atol
//            on the device.  No host round trip per iteration.
// k_power2d: power iteration with the same machinery.
// k_stage  : fused stencil / pointwise stage kernels of the integrators
//             with deterministic last-block norm reductions.
//
// Work decomposition: a warp owns a unit = 64 contiguous columns (one double2
// per lane) x kRT rows; it loads rows i0-1 .. i0+kRT+1 of y (the +x-biased
// upwind stencil reaches i-1, i+1, i+2), takes column neighbours from warp
// shuffles (+2 edge-lane halo loads), and streams p.  Adjacent warps of a CTA
// own adjacent column bands of the same rows, so halo re-reads hit L1/L2.
#include "lx_dev.cuh"

namespace lx {





// ---------------------------------------------------------------------------
// Coefficient table on the device: beta_m = -c/gamma - xi_{m-1} and the Newton
// divided differences d_m^(k) of h_k(xi) = phi_l(a_k dt (c + gamma xi)) at the
// Leja points (reading R8: triangular recurrence
// d[i:] = (d[i:] - d[i-1]) / (xi[i:] - xi[i-1])).  One CTA per accumulator,
// thread j owns d_j; one barrier per recurrence step.  No host work, no H2D.
// ---------------------------------------------------------------------------

// Critical path per recurrence step: one bar.sync, one shared load of the
// published d_{i-1}, one subtract, one multiply by the precomputed reciprocal
// R[i-1][j] = 1/(xi_j - xi_{i-1}) (per-context table, prefetched 4 steps ahead).
// Thread j publishes d_j when it becomes final (step j).
__global__ void k_coef_tables(const double* xi, const double* R, int M, CoefJobs jobs, double dt, double c,
                              double gamma, const double* cg_dev, int* status) {
    extern __shared__ double dsh[];   // [M] published final values
    const CoefJob J = jobs.j[blockIdx.x];
    if (cg_dev) {
        c = cg_dev[0];
        gamma = cg_dev[1];
    }
    const int j = threadIdx.x;
    const bool own = j < M;
    const double xj = own ? xi[j] : 0.0;
    double dj = own ? phi_dev(J.l, coef_arg(J.a, dt, c, gamma, xj)) : 0.0;
    if (j == 0) dsh[0] = dj;   // d_0 = h(xi_0) is final
    double rr[4];
#pragma unroll
    for (int q = 0; q < 4; q++) rr[q] = (own && q + 1 < M && j > q) ? __ldg(R + (size_t)q * M + j) : 0.0;
    for (int i0 = 1; i0 < M; i0 += 4) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int i = i0 + q;
            if (i < M) {
                const double r = rr[q];
                const int ip = i + 3;   // row of step i + 4
                rr[q] = (own && ip + 1 < M && j > ip) ? __ldg(R + (size_t)ip * M + j) : 0.0;
                __syncthreads();
                const double di = dsh[i - 1];
                if (own && j >= i) {
                    dj = dd_step(dj, di, r);
                    if (j == i) dsh[j] = dj;
                }
            }
        }
    }
    if (own) {
        J.table[(size_t)j * (1 + J.K) + 1 + J.k] = dj;
        if (!isfinite(dj)) atomicExch(status, 6);
        if (J.k == 0) J.table[(size_t)j * (1 + J.K)] = (j == 0 || dt == 0.0) ? 0.0 : (-c / gamma - xi[j - 1]);
    }
}

cudaError_t launch_coef_tables(const double* xi, const double* R, int M, const CoefJobs& jobs, double dt, double c,
                               double gamma, const double* cg_dev, int* status, cudaStream_t s) {
    const int threads = ((M + 31) / 32) * 32;
    if (threads > 1024 || jobs.n < 1) return cudaErrorInvalidValue;
    k_coef_tables<<<jobs.n, threads, M * sizeof(double), s>>>(xi, R, M, jobs, dt, c, gamma, cg_dev, status);
    return cudaGetLastError();
}


__global__ void k_shift_scale(const unsigned long long* umax, ShiftArgs a, double* cg) {
    // the bound of oracle/lxoracle.c oc_spectrum_bound, operation by operation (no contraction)
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const double m2 = __longlong_as_double((long long)*umax);
        double vmax = fabs(a.nu);
        if (a.flux != 0.0) vmax = __dadd_rn(fabs(a.nu), __dmul_rn(fabs(a.flux), sqrt(m2)));
        double b = 0.0;
        for (int d = 0; d < a.ndim; d++) {
            const double h = a.h[d];
            b = __dadd_rn(b, __dadd_rn(__ddiv_rn(__dmul_rn(4.0, a.diff), __dmul_rn(h, h)),
                                       __ddiv_rn(__dmul_rn(4.0, vmax), __dmul_rn(3.0, h))));
        }
        if (a.react != 0.0) {
            const double sft = __dsub_rn(__dmul_rn(3.0, m2), 1.0);
            if (sft > 0.0) b = __dadd_rn(b, __dmul_rn(a.react, sft));
        }
        const double eig = __dmul_rn(-1.05, b);
        cg[0] = eig / 2.0;
        cg[1] = -eig / 4.0;
        cg[2] = b;
    }
}

cudaError_t launch_shift_scale(const unsigned long long* umax, const ShiftArgs& a, double* cg_out, cudaStream_t s) {
    k_shift_scale<<<1, 32, 0, s>>>(umax, a, cg_out);
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Stage kernels
// ---------------------------------------------------------------------------

// Deterministic last-block reduction of one value into rec->err = sqrt(S/N).
__device__ __forceinline__ void stage_reduce_err(const StageArgs& A, double v, double (*s_red)[kSlot],
                                                 int* s_last) {
    double vals[1] = {v};
    block_reduce<1>(vals, s_red);
    if (threadIdx.x == 0) {
        A.partials[blockIdx.x * kSlot] = vals[0];
        __threadfence();
        const unsigned t = atomicAdd(&A.ctrl->ticket, 1u);
        *s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (*s_last) {
        __threadfence();
        double acc[1] = {0.0};
        for (int c = threadIdx.x; c < (int)gridDim.x; c += kThreads) acc[0] += __ldcg(A.partials + c * kSlot);
        block_reduce<1>(acc, s_red);
        if (threadIdx.x == 0) {
            if (A.rank_part) A.rank_part[0] = acc[0];   // multi-rank: finalised after the allgather
            else A.rec->err = sqrt(acc[0] / A.N_glob);
            A.ctrl->ticket = 0u;
        }
    }
}

template <int OP>
__global__ void __launch_bounds__(kThreads) k_stage_pointwise(const __grid_constant__ StageArgs A) {
    // Each loop trip handles UN independent element pairs; all loads of the trip are issued
    // before any store (outputs may alias inputs element-wise, which blocks the compiler from
    // overlapping trips on its own), so every thread keeps UN x (inputs) 16-byte loads in flight.
    constexpr int UN = 4;
    constexpr int NIN = (OP == ST_LIN4_ERR) ? 5 : (OP == ST_FINAL4 || OP == ST_LIN4 || OP == ST_REMB_W34) ? 4 : (OP == ST_STAGE_REMAINDER) ? 4
                        : (OP == ST_SUM3 || OP == ST_LIN3 || OP == ST_REM2_W34) ? 3 : (OP == ST_MAXSQ) ? 1 : 2;
    __shared__ double s_red[kWarps][kSlot];
    __shared__ int s_last;
    const long long npair = (long long)A.n_loc * A.n1 * A.n2 / 2;
    const long long stride = (long long)gridDim.x * kThreads;
    double acc = 0.0;
    unsigned long long umax = 0ull;
    const double dt = A.dt, react = A.st.react;
    const double* in[5] = {};
    if (OP == ST_REMAINDER_DIFF) { in[0] = A.x0; in[1] = A.u; }
    else if (OP == ST_STAGE_REMAINDER) { in[0] = A.x0; in[1] = A.u; in[2] = A.x1; in[3] = A.x2; }
    else if (OP == ST_REM2_W34) { in[0] = A.u; in[1] = A.x1; in[2] = A.x2; }
    else if (OP == ST_REMB_W34) { in[0] = A.u; in[1] = A.x1; in[2] = A.x2; in[3] = A.x3; }
    else if (OP == ST_EXPRB32_A) { in[0] = A.x0; in[1] = A.x1; }
    else { in[0] = A.x0; in[1] = A.x1; in[2] = A.x2; in[3] = A.x3; }
    if (OP == ST_LIN4_ERR) in[4] = A.y1;
    for (long long i0 = (long long)blockIdx.x * kThreads + threadIdx.x; i0 < npair; i0 += UN * stride) {
        double2 v[UN][NIN];
#pragma unroll
        for (int q = 0; q < UN; q++) {
            const long long o = 2 * (i0 + q * stride);
            const bool ok = i0 + q * stride < npair;
#pragma unroll
            for (int t = 0; t < NIN; t++) {
                v[q][t] = make_double2(0.0, 0.0);
                if (ok && in[t]) v[q][t] = ld2(in[t] + o);
            }
        }
#pragma unroll
        for (int q = 0; q < UN; q++) {
            const long long o = 2 * (i0 + q * stride);
            if (i0 + q * stride >= npair) break;
            if (OP == ST_AXPBY) {
                const double2 x = v[q][0], y = v[q][1];
                st2(A.y0 + o, make_double2(A.a0 * x.x + A.a1 * y.x, A.a0 * x.y + A.a1 * y.y));
            } else if (OP == ST_REMAINDER_DIFF) {
                const double2 x = v[q][0], u = v[q][1];
                st2(A.y0 + o, make_double2(dt * nl_rem(react, x.x, u.x) + (-dt) * nl_rem(react, u.x, u.x),
                                           dt * nl_rem(react, x.y, u.y) + (-dt) * nl_rem(react, u.y, u.y)));
            } else if (OP == ST_STAGE_REMAINDER) {
                // s = x0 + a0*x1 + a1*x2 (not stored);  y0 = dt F(s) - dt F(u)
                const double2 x = v[q][0], u = v[q][1], p = v[q][2], r = v[q][3];
                const double sx = x.x + A.a0 * p.x + A.a1 * r.x;
                const double sy = x.y + A.a0 * p.y + A.a1 * r.y;
                const double Dx = dt * nl_rem(react, sx, u.x) + (-dt) * nl_rem(react, u.x, u.x);
                const double Dy = dt * nl_rem(react, sy, u.y) + (-dt) * nl_rem(react, u.y, u.y);
                st2(A.y0 + o, make_double2(A.a2 * Dx, A.a2 * Dy));
            } else if (OP == ST_REM2_W34) {
                // the two remainders (same expressions as ST_STAGE_REMAINDER with a1 = 0, a2 = 1) and the
                // final stage's two combinations (same expressions as ST_COMBINE2): D_a, D_b never touch HBM
                const double2 u = v[q][0], pa = v[q][1], pb = v[q][2];
                const double sax = u.x + A.a0 * pa.x, say = u.y + A.a0 * pa.y;
                const double sbx = u.x + A.a1 * pb.x, sby = u.y + A.a1 * pb.y;
                const double dax = dt * nl_rem(react, sax, u.x) + (-dt) * nl_rem(react, u.x, u.x);
                const double day = dt * nl_rem(react, say, u.y) + (-dt) * nl_rem(react, u.y, u.y);
                const double dbx = dt * nl_rem(react, sbx, u.x) + (-dt) * nl_rem(react, u.x, u.x);
                const double dby = dt * nl_rem(react, sby, u.y) + (-dt) * nl_rem(react, u.y, u.y);
                st2(A.y0 + o, make_double2(A.a2 * dax + A.a3 * dbx, A.a2 * day + A.a3 * dby));
                st2(A.y1 + o, make_double2(A.a4 * dax + A.a5 * dbx, A.a4 * day + A.a5 * dby));
            } else if (OP == ST_REMB_W34) {
                // ST_STAGE_REMAINDER (a2 = 1) for D_b and ST_COMBINE2 with D_a read back, in one pass
                const double2 u = v[q][0], p = v[q][1], r = v[q][2], da = v[q][3];
                const double sx = u.x + A.a0 * p.x + A.a1 * r.x;
                const double sy = u.y + A.a0 * p.y + A.a1 * r.y;
                const double dbx = dt * nl_rem(react, sx, u.x) + (-dt) * nl_rem(react, u.x, u.x);
                const double dby = dt * nl_rem(react, sy, u.y) + (-dt) * nl_rem(react, u.y, u.y);
                st2(A.y0 + o, make_double2(A.a2 * da.x + A.a3 * dbx, A.a2 * da.y + A.a3 * dby));
                st2(A.y1 + o, make_double2(A.a4 * da.x + A.a5 * dbx, A.a4 * da.y + A.a5 * dby));
            } else if (OP == ST_EXPRB32_A) {
                const double2 u = v[q][0], p = v[q][1];
                const double2 a = make_double2(u.x + p.x, u.y + p.y);
                st2(A.y1 + o, a);
                st2(A.y0 + o, make_double2(dt * nl_rem(react, a.x, u.x) + (-dt) * nl_rem(react, u.x, u.x),
                                           dt * nl_rem(react, a.y, u.y) + (-dt) * nl_rem(react, u.y, u.y)));
            } else if (OP == ST_COMBINE2) {
                const double2 x = v[q][0], y = v[q][1];
                st2(A.y0 + o, make_double2(A.a0 * x.x + A.a1 * y.x, A.a0 * x.y + A.a1 * y.y));
                st2(A.y1 + o, make_double2(A.a2 * x.x + A.a3 * y.x, A.a2 * x.y + A.a3 * y.y));
            } else if (OP == ST_FINAL4) {
                const double2 u = v[q][0], p1 = v[q][1], q3 = v[q][2], q4 = v[q][3];
                const double2 u3 = make_double2(u.x + p1.x + q3.x, u.y + p1.y + q3.y);
                const double2 u4 = make_double2(u3.x + q4.x, u3.y + q4.y);
                st2(A.y0 + o, u3);
                st2(A.y1 + o, u4);
                const double ex = u4.x - u3.x, ey = u4.y - u3.y;
                acc = fma(ex, ex, acc);
                acc = fma(ey, ey, acc);
            } else if (OP == ST_FINAL_EXPRB32) {
                const double2 a = v[q][0], qq = v[q][1];
                st2(A.y0 + o, make_double2(a.x + 2.0 * qq.x, a.y + 2.0 * qq.y));
                const double ex = 2.0 * qq.x, ey = 2.0 * qq.y;
                acc = fma(ex, ex, acc);
                acc = fma(ey, ey, acc);
            } else if (OP == ST_LIN3) {
                const double2 x = v[q][0], y = v[q][1], z = v[q][2];
                st2(A.y0 + o, make_double2(x.x + A.a0 * y.x + A.a1 * z.x, x.y + A.a0 * y.y + A.a1 * z.y));
            } else if (OP == ST_LIN4) {
                const double2 x = v[q][0], y = v[q][1], z = v[q][2], w = v[q][3];
                st2(A.y0 + o, make_double2(x.x + A.a0 * y.x + A.a1 * z.x + A.a2 * w.x,
                                           x.y + A.a0 * y.y + A.a1 * z.y + A.a2 * w.y));
            } else if (OP == ST_LIN4_ERR) {
                const double2 x = v[q][0], y = v[q][1], z = v[q][2], w = v[q][3], e = v[q][4];
                const double2 r = make_double2(x.x + A.a0 * y.x + A.a1 * z.x + A.a2 * w.x,
                                               x.y + A.a0 * y.y + A.a1 * z.y + A.a2 * w.y);
                st2(A.y0 + o, r);
                const double ex = r.x - e.x, ey = r.y - e.y;
                acc = fma(ex, ex, acc);
                acc = fma(ey, ey, acc);
            } else if (OP == ST_SUM3) {
                const double2 x = v[q][0], y = v[q][1], z = v[q][2];
                st2(A.y0 + o, make_double2(x.x + y.x + z.x, x.y + y.y + z.y));
            } else if (OP == ST_MAXSQ) {
                const double2 x = v[q][0];
                const double m2 = fmax(x.x * x.x, x.y * x.y);
                const unsigned long long bb = (unsigned long long)__double_as_longlong(m2);
                umax = bb > umax ? bb : umax;
            }
        }
    }
    if (OP == ST_FINAL4 || OP == ST_FINAL_EXPRB32 || OP == ST_LIN4_ERR) stage_reduce_err(A, acc, s_red, &s_last);
    if (OP == ST_MAXSQ) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o2 = __shfl_xor_sync(FULL_MASK, umax, off);
            umax = o2 > umax ? o2 : umax;
        }
        if ((threadIdx.x & 31) == 0 && umax) atomicMax(&A.ctrl->umax, umax);
    }
}

template <int NDIM>
// three CTAs per SM (<= 85 registers), grid = one wave of them: 4096^2 f 59.5 -> 50.5 us vs two per SM
__global__ void __launch_bounds__(kThreads, 3) k_rhs2d(const __grid_constant__ LejaParams P, double scale) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double sy = 0.0, sp[1] = {0.0};
    for (int unit = blockIdx.x * kWarps + warp; unit < P.nunits; unit += gridDim.x * kWarps)
        tile<NDIM, 0, false, false, M_RHS, true>(P, P.v, P.ydst[0], unit, lane, 0.0, nullptr, nullptr, 0, scale, sy, sp);
}

__global__ void k_fill_start(double* v, long long n, int add_e0) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] = (add_e0 && i == 0) ? 2.0 : 1.0;
}

cudaError_t launch_fill_start(double* v, long long n, bool add_e0, cudaStream_t s) {
    k_fill_start<<<256, 256, 0, s>>>(v, n, add_e0 ? 1 : 0);
    return cudaGetLastError();
}

static void* stage_kernel_ptr(int op) {
    switch (op) {
        case ST_AXPBY: return (void*)k_stage_pointwise<ST_AXPBY>;
        case ST_REMAINDER_DIFF: return (void*)k_stage_pointwise<ST_REMAINDER_DIFF>;
        case ST_STAGE_REMAINDER: return (void*)k_stage_pointwise<ST_STAGE_REMAINDER>;
        case ST_EXPRB32_A: return (void*)k_stage_pointwise<ST_EXPRB32_A>;
        case ST_COMBINE2: return (void*)k_stage_pointwise<ST_COMBINE2>;
        case ST_FINAL4: return (void*)k_stage_pointwise<ST_FINAL4>;
        case ST_FINAL_EXPRB32: return (void*)k_stage_pointwise<ST_FINAL_EXPRB32>;
        case ST_MAXSQ: return (void*)k_stage_pointwise<ST_MAXSQ>;
        case ST_SUM3: return (void*)k_stage_pointwise<ST_SUM3>;
        case ST_LIN3: return (void*)k_stage_pointwise<ST_LIN3>;
        case ST_LIN4: return (void*)k_stage_pointwise<ST_LIN4>;
        case ST_LIN4_ERR: return (void*)k_stage_pointwise<ST_LIN4_ERR>;
        case ST_REM2_W34: return (void*)k_stage_pointwise<ST_REM2_W34>;
        case ST_REMB_W34: return (void*)k_stage_pointwise<ST_REMB_W34>;
    }
    return nullptr;
}

// One full wave of resident CTAs (never more: a partial second wave doubles the time).
__global__ void __launch_bounds__(kThreads, 2) k_rem2d_flux(const __grid_constant__ LejaParams P, double dt, double a2,
                                                              double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double sy = 0.0, sp[1] = {0.0};
    for (int unit = blockIdx.x * kWarps + warp; unit < P.nunits; unit += gridDim.x * kWarps)
        tile2d_flux<0, false, M_REM, true>(P, P.v, out, unit, lane, dt, nullptr, nullptr, 0, a2, sy, sp);
}

cudaError_t launch_rem_flux(const LejaParams& P, double dt, double a2, double* out, cudaStream_t s) {
    k_rem2d_flux<<<P.grid, kThreads, 0, s>>>(P, dt, a2, out);
    return cudaGetLastError();
}

int stage_grid_size(int device, int op) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    void* k = stage_kernel_ptr(op);
    const int g = k ? coresident(device, k) : nsm;
    return g > 8 * nsm ? 8 * nsm : g;
}

cudaError_t launch_rhs(const LejaParams& P, double scale, cudaStream_t s) {
    if (P.ndim == 4) k_rhs2d<4><<<P.grid, kThreads, 0, s>>>(P, scale);
    else if (P.ndim == 3) k_rhs2d<3><<<P.grid, kThreads, 0, s>>>(P, scale);
    else k_rhs2d<2><<<P.grid, kThreads, 0, s>>>(P, scale);
    return cudaGetLastError();
}

cudaError_t launch_stage(int op, const StageArgs& A, cudaStream_t s) {
    const dim3 g(A.grid), b(kThreads);
    switch (op) {
        case ST_AXPBY: k_stage_pointwise<ST_AXPBY><<<g, b, 0, s>>>(A); break;
        case ST_REMAINDER_DIFF: k_stage_pointwise<ST_REMAINDER_DIFF><<<g, b, 0, s>>>(A); break;
        case ST_STAGE_REMAINDER: k_stage_pointwise<ST_STAGE_REMAINDER><<<g, b, 0, s>>>(A); break;
        case ST_EXPRB32_A: k_stage_pointwise<ST_EXPRB32_A><<<g, b, 0, s>>>(A); break;
        case ST_COMBINE2: k_stage_pointwise<ST_COMBINE2><<<g, b, 0, s>>>(A); break;
        case ST_FINAL4: k_stage_pointwise<ST_FINAL4><<<g, b, 0, s>>>(A); break;
        case ST_FINAL_EXPRB32: k_stage_pointwise<ST_FINAL_EXPRB32><<<g, b, 0, s>>>(A); break;
        case ST_MAXSQ: k_stage_pointwise<ST_MAXSQ><<<g, b, 0, s>>>(A); break;
        case ST_SUM3: k_stage_pointwise<ST_SUM3><<<g, b, 0, s>>>(A); break;
        case ST_LIN3: k_stage_pointwise<ST_LIN3><<<g, b, 0, s>>>(A); break;
        case ST_LIN4: k_stage_pointwise<ST_LIN4><<<g, b, 0, s>>>(A); break;
        case ST_LIN4_ERR: k_stage_pointwise<ST_LIN4_ERR><<<g, b, 0, s>>>(A); break;
        case ST_REM2_W34: k_stage_pointwise<ST_REM2_W34><<<g, b, 0, s>>>(A); break;
        case ST_REMB_W34: k_stage_pointwise<ST_REMB_W34><<<g, b, 0, s>>>(A); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t preload_leja();
cudaError_t preload_tb2();
cudaError_t preload_3d();

// Force every kernel of the library to be loaded now (cudaFuncGetAttributes loads a function under CUDA
// lazy loading).  Virtual ranks sharing one context run persistent kernels that spin on each other; a
// lazy load during that time needs the context to idle and would deadlock until the watchdog.
cudaError_t preload_kernels() {
    cudaError_t e = preload_leja();
    if (e == cudaSuccess) e = preload_tb2();
    if (e == cudaSuccess) e = preload_3d();
    if (e != cudaSuccess) return e;
    for (int op = ST_RHS_SCALED; op <= ST_LIN4; op++) {
        const void* k = stage_kernel_ptr(op);   // (ST_RHS_SCALED is a stencil kernel: k_rhs2d below)
        cudaFuncAttributes a;
        if (k && cudaFuncGetAttributes(&a, k) != cudaSuccess) return cudaGetLastError();
    }
    const void* fixed[] = {(const void*)k_coef_tables, (const void*)k_shift_scale, (const void*)k_fill_start,
                           (const void*)k_rem2d_flux, (const void*)k_rhs2d<2>, (const void*)k_rhs2d<3>,
                           (const void*)k_rhs2d<4>};
    for (const void* k : fixed) {
        cudaFuncAttributes a;
        if (cudaFuncGetAttributes(&a, k) != cudaSuccess) return cudaGetLastError();
    }
    return cudaSuccess;
}

}  // namespace lx
