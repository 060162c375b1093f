// lx_blackbox.cu -- sm_100a kernels of the black-box right-hand-side path.
//
// The paper's LeXInt only calls a user RHS functor f (listing alg:RHS) and forms
// Jacobian-vector products by finite differences: J(u) y ~ (f(u + eps y) - f(u)) / eps.
// Here the user's f is a host callback that enqueues device work on the context stream; every
// other step of the Leja iteration (Eq. (2)) and of the stopping test runs in
// the kernels below.  Per Leja iteration m:
//   k_bb_perturb(m)  : w = u + eps_m y_{m-1},  eps_m = 2^-26 (1 + ||u||_inf) / ||y_{m-1}||_inf   (R25)
//   user f(w) -> fw   (or f(y_{m-1}) for a linear black-box operator)
//   k_bb_update(m)   : J y = (fw - f(u)) / eps_m ; y_m = alpha J y + beta_m y_{m-1} ;
//                      p_k += d_m^(k) y_m ; per-CTA partials (sum y^2, sum p_k^2), max|y_m| ;
//                      the last CTA sums the partials in CTA order and takes the decision.
// All kernels return at entry once the decision says "done", so the host may enqueue one
// iteration ahead of the flag it reads.
#include <cuda_runtime.h>
#include <math.h>

#include "lx_internal.h"

namespace lx {

namespace {

constexpr double kFdEps0 = 1.4901161193847656e-08;   // 2^-26 = sqrt(DBL_EPSILON)  (R25)

__device__ __forceinline__ double u64_as_double(unsigned long long b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ unsigned long long double_as_u64(double x) {
    return (unsigned long long)__double_as_longlong(x);
}

// block sum of NV values (fixed order: warp butterfly, then warps in index order)
template <int NV>
__device__ __forceinline__ void block_sum(double* v, double (*s)[NV]) {
#pragma unroll
    for (int i = 0; i < NV; i++)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; i++) s[warp][i] = v[i];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; i++) {
            double a = 0.0;
            for (int w = 0; w < kWarps; w++) a += s[w][i];
            v[i] = a;
        }
    }
}

__device__ __forceinline__ double block_max(double v, double* s) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s[warp] = v;
    __syncthreads();
    double m = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kWarps; w++) m = fmax(m, s[w]);
    return m;
}

// 16-byte global accesses (cudaMalloc'd vectors and caller tensors are 16-byte aligned: lexint.h)
__device__ __forceinline__ double2 ld2g(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2g(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

__device__ __forceinline__ double fd_eps(const BbCtrl* c, int slot) {
    const double ym = u64_as_double(c->maxbits[slot]);
    if (ym == 0.0) return 0.0;                 // J(u) 0 = 0
    return kFdEps0 * (1.0 + u64_as_double(c->umaxbits)) / ym;
}

// p_k = d_0^(k) v ; max|v| -> maxbits[0] ; max|u| -> umaxbits (FD) ; decision state reset by the host
__global__ void __launch_bounds__(kThreads) k_bb_init(BbArgs A) {
    __shared__ double s[kWarps];
    double mv = 0.0, mu = 0.0;
    const long long N = A.N;
    const int K = A.K;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        const double v = A.y_in[i];
        mv = fmax(mv, fabs(v));
        if (A.u) mu = fmax(mu, fabs(A.u[i]));
        for (int k = 0; k < K; k++) A.p[k][i] = A.table[1 + k] * v;
    }
    mv = block_max(mv, s);
    __syncthreads();
    mu = block_max(mu, s);
    if (threadIdx.x == 0) {
        atomicMax(&A.ctrl->maxbits[0], double_as_u64(mv));
        if (A.u) atomicMax(&A.ctrl->umaxbits, double_as_u64(mu));
    }
}

// w = u + eps_m y_{m-1}; block 0 also clears the max slot iteration m will fill
__global__ void __launch_bounds__(kThreads) k_bb_perturb(BbArgs A, int m) {
    BbCtrl* c = A.ctrl;
    if (*(volatile int*)&c->done) return;
    const double eps = fd_eps(c, (m - 1) & 1);
    const long long N = A.N;
    const long long npair = N >> 1;
    // 4 element pairs per trip, all loads issued before the stores (bytes in flight for a 2-CTA/SM grid)
    constexpr int UN = 4;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < npair; i0 += UN * stride) {
        double2 u[UN], y[UN];
#pragma unroll
        for (int q = 0; q < UN; q++) {
            const long long i = i0 + q * stride;
            if (i < npair) {
                u[q] = ld2g(A.u + 2 * i);
                y[q] = ld2g(A.y_in + 2 * i);
            }
        }
#pragma unroll
        for (int q = 0; q < UN; q++) {
            const long long i = i0 + q * stride;
            if (i < npair)
                st2g(A.w + 2 * i, make_double2(__dadd_rn(u[q].x, __dmul_rn(eps, y[q].x)),
                                               __dadd_rn(u[q].y, __dmul_rn(eps, y[q].y))));
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (N & 1) A.w[N - 1] = __dadd_rn(A.u[N - 1], __dmul_rn(eps, A.y_in[N - 1]));
        c->maxbits[m & 1] = 0ull;
    }
}

template <int K>
__global__ void __launch_bounds__(kThreads) k_bb_update(BbArgs A, int m) {
    constexpr int NV = 1 + K;
    __shared__ double s_red[kWarps][NV];
    __shared__ double s_max[kWarps];
    __shared__ int s_last;
    BbCtrl* c = A.ctrl;
    if (*(volatile int*)&c->done) return;
    const int act = c->active;
    const double* row = A.table + (size_t)m * (1 + A.K);
    const double beta = row[0];
    double dm[K];
#pragma unroll
    for (int k = 0; k < K; k++) dm[k] = row[1 + k];
    const double alpha = A.alpha;
    const bool fd = A.mode == 1;
    const double eps = fd ? fd_eps(c, (m - 1) & 1) : 1.0;
    const double ieps = (fd && eps != 0.0) ? 1.0 / eps : 0.0;
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) acc[i] = 0.0;
    double my = 0.0;
    const long long N = A.N;
    // pairs (16-byte loads/stores), UN independent pairs per trip with every load issued before any
    // store; the scalar tail (odd N) afterwards
    constexpr int UN = 2;
    const long long npair = N >> 1;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < npair; i0 += UN * stride) {
        double2 yp[UN], fw[UN], fu[UN], pv[UN][K];
#pragma unroll
        for (int q = 0; q < UN; q++) {
            const long long i = i0 + q * stride;
            const bool ok = i < npair;
            yp[q] = ok ? ld2g(A.y_in + 2 * i) : make_double2(0.0, 0.0);
            fw[q] = ok ? ld2g(A.fw + 2 * i) : make_double2(0.0, 0.0);
            fu[q] = (ok && fd) ? ld2g(A.fu + 2 * i) : make_double2(0.0, 0.0);
#pragma unroll
            for (int k = 0; k < K; k++)
                pv[q][k] = (ok && ((act >> k) & 1)) ? ld2g(A.p[k] + 2 * i) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < UN; q++) {
            const long long i = i0 + q * stride;
            if (i >= npair) break;
            double jx, jyy;
            if (fd) {
                jx = (eps == 0.0) ? 0.0 : (fw[q].x - fu[q].x) * ieps;
                jyy = (eps == 0.0) ? 0.0 : (fw[q].y - fu[q].y) * ieps;
            } else {
                jx = fw[q].x;
                jyy = fw[q].y;
            }
            const double2 y = make_double2(fma(alpha, jx, beta * yp[q].x), fma(alpha, jyy, beta * yp[q].y));
            st2g(A.y_out + 2 * i, y);
            acc[0] = fma(y.x, y.x, acc[0]);
            acc[0] = fma(y.y, y.y, acc[0]);
            my = fmax(my, fmax(fabs(y.x), fabs(y.y)));
#pragma unroll
            for (int k = 0; k < K; k++) {
                if ((act >> k) & 1) {
                    const double2 p = make_double2(fma(dm[k], y.x, pv[q][k].x), fma(dm[k], y.y, pv[q][k].y));
                    st2g(A.p[k] + 2 * i, p);
                    acc[1 + k] = fma(p.x, p.x, acc[1 + k]);
                    acc[1 + k] = fma(p.y, p.y, acc[1 + k]);
                }
            }
        }
    }
    if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {   // odd tail element
        const long long i = N - 1;
        const double yp = A.y_in[i];
        double jy;
        if (fd) jy = (eps == 0.0) ? 0.0 : (A.fw[i] - A.fu[i]) * ieps;
        else jy = A.fw[i];
        const double y = fma(alpha, jy, beta * yp);
        A.y_out[i] = y;
        acc[0] = fma(y, y, acc[0]);
        my = fmax(my, fabs(y));
#pragma unroll
        for (int k = 0; k < K; k++) {
            if ((act >> k) & 1) {
                const double p = fma(dm[k], y, A.p[k][i]);
                A.p[k][i] = p;
                acc[1 + k] = fma(p, p, acc[1 + k]);
            }
        }
    }
    block_sum<NV>(acc, s_red);
    __syncthreads();
    my = block_max(my, s_max);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; i++) A.partials[(size_t)blockIdx.x * NV + i] = acc[i];
        atomicMax(&c->maxbits[m & 1], double_as_u64(my));
        __threadfence();
        const unsigned t = atomicAdd(&c->ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    // last CTA: fixed-order sum of the CTA partials, then the P:155 test (R3, R4)
    __threadfence();
    double sums[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) sums[i] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
        for (int i = 0; i < NV; i++) sums[i] += __ldcg(A.partials + (size_t)b * NV + i);
    block_sum<NV>(sums, s_red);
    if (threadIdx.x == 0) {
        c->ticket = 0u;
        Record* rec = A.rec;
        const double Ng = A.N_glob;
        const double ny = sqrt(sums[0] / Ng);
        int a = act, nact = 0, status = 0, done = 0;
        for (int k = 0; k < K; k++) {
            if (!((a >> k) & 1)) continue;
            const double err = fabs(dm[k]) * ny;
            const double thr = A.rtol * sqrt(sums[1 + k] / Ng) + A.atol;
            if (!isfinite(err) || !isfinite(thr)) { status = 6; break; }
            if (err <= thr) {
                a &= ~(1 << k);
                rec->iters_k[k] = m;
                const double r = err > 0.0 ? thr / err : INFINITY;
                if (r < rec->margin_accept) rec->margin_accept = r;
            } else {
                nact++;
                const double r = err / thr;
                if (r < rec->margin_reject) rec->margin_reject = r;
            }
        }
        if (status) done = 1;
        else if (nact == 0) done = 1;
        else if (m >= A.max_nodes - 1) { done = 1; status = 5; }
        c->active = a;
        c->m = m;
        if (done) {
            rec->iters += m;
            rec->ncalls += 1;
            if (rec->status == 0) rec->status = status;
            c->status = status;
            __threadfence_system();
            c->done = 1;
            if (A.done_host) *(volatile int*)A.done_host = m;
        }
    }
}

// max |x| -> ctrl->maxbits[2] (host clears it first)
__global__ void __launch_bounds__(kThreads) k_bb_maxabs(const double* x, long long N, BbCtrl* c) {
    __shared__ double s[kWarps];
    double mx = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
        mx = fmax(mx, fabs(x[i]));
    mx = block_max(mx, s);
    if (threadIdx.x == 0) atomicMax(&c->maxbits[2], double_as_u64(mx));
}

// FD remainder pieces (alg:exprb32 Nonlinear_remainder), eps from maxbits[2]:
//   PERTURB: y0 = u + eps x0 ;  REMAINDER: y0 = x0 - (x1 - fu) / eps   (F(x) = f(x) - J_FD(u) x)
__global__ void __launch_bounds__(kThreads) k_bb_fdpiece(BbLin L, int op) {
    const double ym = u64_as_double(L.ctrl->maxbits[2]);
    const double eps = ym == 0.0 ? 0.0 : kFdEps0 * (1.0 + u64_as_double(L.ctrl->umaxbits)) / ym;
    const long long N = L.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        if (op == 0) L.y0[i] = __dadd_rn(L.u[i], __dmul_rn(eps, L.x0[i]));
        else L.y0[i] = L.x0[i] - (eps == 0.0 ? 0.0 : (L.x1[i] - L.fu[i]) / eps);
    }
}

// y0 = a0 x0 + a1 x1 + a2 x2 + a3 x3 (absent inputs skipped, evaluated left to right)
__global__ void __launch_bounds__(kThreads) k_bb_lincomb(BbLin L) {
    const long long N = L.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        double s = L.a0 * L.x0[i];
        if (L.x1) s += L.a1 * L.x1[i];
        if (L.x2) s += L.a2 * L.x2[i];
        if (L.x3) s += L.a3 * L.x3[i];
        L.y0[i] = s;
    }
}

// rec->err = || a0 x0 + a1 x1 || / sqrt(N), CTA partials summed in CTA order by the last CTA
__global__ void __launch_bounds__(kThreads) k_bb_norm(BbLin L) {
    __shared__ double s_red[kWarps][1];
    __shared__ int s_last;
    double acc[1] = {0.0};
    const long long N = L.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        double e = L.a0 * L.x0[i];
        if (L.x1) e += L.a1 * L.x1[i];
        acc[0] = fma(e, e, acc[0]);
    }
    block_sum<1>(acc, s_red);
    if (threadIdx.x == 0) {
        L.partials[blockIdx.x] = acc[0];
        __threadfence();
        s_last = (atomicAdd(&L.ctrl->ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double t[1] = {0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) t[0] += __ldcg(L.partials + b);
    block_sum<1>(t, s_red);
    if (threadIdx.x == 0) {
        L.ctrl->ticket = 0u;
        L.rec->err = sqrt(t[0] / L.N_glob);
    }
}

// f(u) of the built-in problems for the black-box path (lx_builtin_rhs), evaluated literally in the
// order of the formulas (readings R10, R16, R24) with every operation explicitly
// rounded (no FMA contraction, divisions by h^2 and 6h):
//   lap_d = ((u_{+1} - 2 u_0) + u_{-1}) / (h h),   D_d(w) = ((((-w_{+2}) + 6 w_{+1}) - 3 w_0) - 2 w_{-1}) / (6 h)
//   f = (diff sum_d lap_d) + (nu sum_d D_d(u)) [+ (beta 1/2) sum_d D_d(u u)] [+ react (u - (u u) u)] [+ S]
// (sums over d in dimension order starting from 0).  The FD Jacobian (f(u + eps y) - f(u))/eps divides
// every rounding difference of f by eps ~ 1.5e-8 (R25); a deterministic, contraction-free f makes the
// black-box path reproducible bit for bit wherever its inputs are (SURVEY 8(f) f-1 "FMA-off").
__device__ __forceinline__ int lit_wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

__device__ __forceinline__ double lit_upwind(double wm1, double w0, double w1, double w2, double h6) {
    return __ddiv_rn(__dsub_rn(__dsub_rn(__dadd_rn(-w2, __dmul_rn(6.0, w1)), __dmul_rn(3.0, w0)), __dmul_rn(2.0, wm1)),
                     h6);
}

// grid: x over the contiguous dimension, y over the rows (i0, i1) -- no 64-bit index division.  The
// dimension loop is unrolled over NDIM, the four values per dimension are gathered from 32-bit row /
// column offsets, and h h, 6 h are rounded once per thread: the same rounded operations in the same
// order as the formula above, only the address arithmetic is cheaper.
template <int NDIM, bool FLUX>
__global__ void __launch_bounds__(kThreads) k_rhs_literal(RhsLit R) {
    // rows = all but the contiguous dimension (2D: dim 0; 3D: dims 0, 1)
    constexpr bool d3 = NDIM == 3;
    const int n0 = (int)R.n[0], n1 = (int)R.n[1];
    const int nrow = d3 ? n0 * n1 : n0;
    const int ninner = d3 ? (int)R.n[2] : n1;
    double hh[NDIM], h6[NDIM];
#pragma unroll
    for (int d = 0; d < NDIM; d++) {
        hh[d] = __dmul_rn(R.dx[d], R.dx[d]);
        h6[d] = __dmul_rn(6.0, R.dx[d]);
    }
    const double* __restrict__ in = R.in;
    for (int row = blockIdx.y; row < nrow; row += gridDim.y) {
        const int r0 = d3 ? row / n1 : row, r1 = d3 ? row - r0 * n1 : 0;
        // neighbour rows along the non-contiguous dimensions: row index of offset o = -1, +1, +2
        int rows[NDIM - 1][3];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const int o = q == 0 ? -1 : q;
            rows[0][q] = d3 ? lit_wrap(r0 + o, n0) * n1 + r1 : lit_wrap(r0 + o, n0);
            if (d3) rows[NDIM - 2][q] = r0 * n1 + lit_wrap(r1 + o, n1);
        }
        const size_t base = (size_t)row * ninner;
        for (int c = blockIdx.x * kThreads + threadIdx.x; c < ninner; c += gridDim.x * kThreads) {
            // v[d] = (w_{-1}, w_0, w_{+1}, w_{+2}) along dimension d
            double v[NDIM][4];
            const double u0 = __ldg(in + base + c);
#pragma unroll
            for (int d = 0; d < NDIM - 1; d++) {
                v[d][0] = __ldg(in + (size_t)rows[d][0] * ninner + c);
                v[d][1] = u0;
                v[d][2] = __ldg(in + (size_t)rows[d][1] * ninner + c);
                v[d][3] = __ldg(in + (size_t)rows[d][2] * ninner + c);
            }
            v[NDIM - 1][0] = __ldg(in + base + lit_wrap(c - 1, ninner));
            v[NDIM - 1][1] = u0;
            v[NDIM - 1][2] = __ldg(in + base + lit_wrap(c + 1, ninner));
            v[NDIM - 1][3] = __ldg(in + base + lit_wrap(c + 2, ninner));
            double lap = 0.0, adv = 0.0, flx = 0.0;
#pragma unroll
            for (int d = 0; d < NDIM; d++) {
                const double um1 = v[d][0], uc = v[d][1], up1 = v[d][2], up2 = v[d][3];
                lap = __dadd_rn(lap, __ddiv_rn(__dadd_rn(__dsub_rn(up1, __dmul_rn(2.0, uc)), um1), hh[d]));
                adv = __dadd_rn(adv, lit_upwind(um1, uc, up1, up2, h6[d]));
                if (FLUX)
                    flx = __dadd_rn(flx, lit_upwind(__dmul_rn(um1, um1), __dmul_rn(uc, uc), __dmul_rn(up1, up1),
                                                    __dmul_rn(up2, up2), h6[d]));
            }
            const size_t idx = base + c;
            double f = __dadd_rn(__dmul_rn(R.diff, lap), __dmul_rn(R.nu, adv));
            if (FLUX) f = __dadd_rn(f, __dmul_rn(__dmul_rn(R.flux, 0.5), flx));
            if (R.react != 0.0) f = __dadd_rn(f, __dmul_rn(R.react, __dsub_rn(u0, __dmul_rn(__dmul_rn(u0, u0), u0))));
            if (R.src) f = __dadd_rn(f, R.src[idx]);
            R.out[idx] = f;
        }
    }
}

}  // namespace

int bb_grid(int nsm) { return nsm * 2; }

cudaError_t launch_bb_init(const BbArgs& A, cudaStream_t s) {
    k_bb_init<<<A.grid, kThreads, 0, s>>>(A);
    return cudaGetLastError();
}
cudaError_t launch_bb_perturb(const BbArgs& A, int m, cudaStream_t s) {
    k_bb_perturb<<<A.grid, kThreads, 0, s>>>(A, m);
    return cudaGetLastError();
}
cudaError_t launch_bb_update(const BbArgs& A, int m, cudaStream_t s) {
    switch (A.K) {
        case 1: k_bb_update<1><<<A.grid, kThreads, 0, s>>>(A, m); break;
        case 2: k_bb_update<2><<<A.grid, kThreads, 0, s>>>(A, m); break;
        case 3: k_bb_update<3><<<A.grid, kThreads, 0, s>>>(A, m); break;
        case 4: k_bb_update<4><<<A.grid, kThreads, 0, s>>>(A, m); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
cudaError_t launch_bb_maxabs(const double* x, long long N, BbCtrl* c, int grid, cudaStream_t s) {
    k_bb_maxabs<<<grid, kThreads, 0, s>>>(x, N, c);
    return cudaGetLastError();
}
cudaError_t launch_bb_fdpiece(const BbLin& L, int op, cudaStream_t s) {
    k_bb_fdpiece<<<L.grid, kThreads, 0, s>>>(L, op);
    return cudaGetLastError();
}
cudaError_t launch_bb_lincomb(const BbLin& L, cudaStream_t s) {
    k_bb_lincomb<<<L.grid, kThreads, 0, s>>>(L);
    return cudaGetLastError();
}
cudaError_t launch_rhs_literal(const RhsLit& R, int grid, cudaStream_t s) {
    const long long nrow = R.ndim == 3 ? R.n[0] * R.n[1] : R.n[0];
    const long long ninner = R.ndim == 3 ? R.n[2] : R.n[1];
    const int gx = (int)((ninner + kThreads - 1) / kThreads);
    const int gy = (int)(nrow < 65535 ? nrow : 65535);
    (void)grid;
    const dim3 g(gx, gy);
    if (R.ndim == 3) {
        if (R.flux != 0.0) k_rhs_literal<3, true><<<g, kThreads, 0, s>>>(R);
        else k_rhs_literal<3, false><<<g, kThreads, 0, s>>>(R);
    } else {
        if (R.flux != 0.0) k_rhs_literal<2, true><<<g, kThreads, 0, s>>>(R);
        else k_rhs_literal<2, false><<<g, kThreads, 0, s>>>(R);
    }
    return cudaGetLastError();
}
cudaError_t launch_bb_norm(const BbLin& L, cudaStream_t s) {
    k_bb_norm<<<L.grid, kThreads, 0, s>>>(L);
    return cudaGetLastError();
}

cudaError_t preload_bb_kernels() {
    const void* ks[] = {(const void*)k_bb_init, (const void*)k_bb_perturb, (const void*)k_bb_update<1>,
                        (const void*)k_bb_update<2>, (const void*)k_bb_update<3>, (const void*)k_bb_update<4>,
                        (const void*)k_bb_maxabs, (const void*)k_bb_fdpiece, (const void*)k_bb_lincomb,
                        (const void*)k_bb_norm, (const void*)k_rhs_literal<2, false>, (const void*)k_rhs_literal<2, true>,
                        (const void*)k_rhs_literal<3, false>, (const void*)k_rhs_literal<3, true>};
    for (const void* k : ks) {
        cudaFuncAttributes a;
        const cudaError_t e = cudaFuncGetAttributes(&a, k);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace lx
