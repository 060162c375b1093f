// lx_k_leja.cu -- one-pass persistent Leja kernel (k_leja2d: one fused HBM pass per iteration,
// P:142-147 Eq. (2), device decision of P:155), power iteration (k_power2d), and the
// step-mode kernels of the per-iteration multi-rank protocol (k_leja2d_step, k_power2d_step).
#include "lx_dev.cuh"

namespace lx {

template <int NDIM, int K, bool DIAG>
__global__ void __launch_bounds__(kThreads, 2) k_leja2d(const __grid_constant__ LejaParams P) {
    __shared__ double s_red[kWarps][kSlot];
    __shared__ int s_flags[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // warp 0 of CTA 0 computes the Newton coefficients two iterations ahead; all
    // other warps share the stencil units
    const bool cwarp = (blockIdx.x == 0 && warp == 0);
    const int gw = blockIdx.x * kWarps + warp - 1;
    const int W = gridDim.x * kWarps - 1;
    unsigned gen0 = 0;
    if (tid == 0) gen0 = (unsigned)(ld_acquire64(&P.ctrl->word) >> 32);
    int active = P.active0;
    const int M = P.max_nodes;
    const double alpha = P_alpha(P);
    double d0[K], d1[K], d2[K];
#pragma unroll
    for (int k = 0; k < K; k++) coef_first3(P, k, d0[k], d1[k], d2[k]);
    if (cwarp && P.coef_gen) {
        coef_write_row<K>(P, 0, lane, active, d0);
        coef_write_row<K>(P, 1, lane, active, d1);
        coef_write_row<K>(P, 2, lane, active, d2);
    }
    double beta_n = coef_beta(P, 1), dm_n[K];
#pragma unroll
    for (int k = 0; k < K; k++) dm_n[k] = d1[k];
    for (int m = 1; m < M; m++) {
        const double beta = beta_n;
        double dm[K], sp[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            dm[k] = dm_n[k];
            sp[k] = 0.0;
        }
        double sy = 0.0;
        const int par = m & 1;
        double* dst = P.ydst[par];
        if (cwarp) {
            if (P.coef_gen && m + 2 < M) coef_write_row<K>(P, m + 2, lane, active, nullptr);
        } else if (m == 1) {
            for (int unit = gw; unit < P.nunits; unit += W)
                tile<NDIM, K, DIAG, true, M_LEJA, true>(P, P.v, dst, unit, lane, beta, d0, dm, active, alpha, sy, sp);
        } else {
            const RowSrc src = P.ysrc[par ^ 1];
            for (int unit = gw; unit < P.nunits; unit += W)
                tile<NDIM, K, DIAG, false, M_LEJA, false>(P, src, dst, unit, lane, beta, d0, dm, active, alpha, sy, sp);
        }
        double vals[1 + K];
        vals[0] = sy;
#pragma unroll
        for (int k = 0; k < K; k++) vals[1 + k] = sp[k];
        // coefficients of iteration m+1, fetched before the barrier: row m+1 was written during
        // iteration m-1 and released by barrier m-1
        if (m + 1 < M) {
            beta_n = coef_beta(P, m + 1);
#pragma unroll
            for (int k = 0; k < K; k++) dm_n[k] = (m + 1 == 2) ? d2[k] : P.table[(size_t)(m + 1) * (1 + K) + 1 + k];
        }
        block_reduce<1 + K>(vals, s_red);
        if (tid == 0) {
            double* slot = P.partials + ((size_t)par * gridDim.x + blockIdx.x) * kSlot;
#pragma unroll
            for (int i = 0; i < 1 + K; i++) slot[i] = vals[i];
        }
        barrier_decide<K, M_LEJA>(P, m, gen0, dm, active, s_red, s_flags);
        active = s_flags[2];
        if (s_flags[1]) break;
    }
}

template <int NDIM, bool DIAG>
__global__ void __launch_bounds__(kThreads, 2) k_power2d(const __grid_constant__ LejaParams P) {
    __shared__ double s_red[kWarps][kSlot];
    __shared__ int s_flags[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned gen0 = 0;
    if (tid == 0) gen0 = (unsigned)(ld_acquire64(&P.ctrl->word) >> 32);
    double scale = 1.0;
    for (int m = 1; m <= P.power_iters; m++) {
        double sy = 0.0, sp[1] = {0.0};
        const int par = m & 1;
        double* dst = P.ydst[par];
        const RowSrc src = (m == 1) ? P.v : P.ysrc[par ^ 1];
        for (int unit = blockIdx.x * kWarps + warp; unit < P.nunits; unit += gridDim.x * kWarps)
            tile<NDIM, 0, DIAG, false, M_POWER, false>(P, src, dst, unit, lane, 0.0, nullptr, nullptr, 0, scale, sy, sp);
        double vals[1] = {sy};
        block_reduce<1>(vals, s_red);
        if (tid == 0) P.partials[((size_t)par * gridDim.x + blockIdx.x) * kSlot] = vals[0];
        barrier_decide<0, M_POWER>(P, m, gen0, nullptr, 0, s_red, s_flags);
        scale = s_red[0][kSlot - 1];
        if (s_flags[1]) break;
    }
}


// ---------------------------------------------------------------------------
// Step mode (multi-rank slab decomposition): one launch per iteration m.
// Prologue: decision of iteration m-1 from the per-rank partials gathered by
// the transport (summed in rank order -> identical decision on every rank);
// body: tiles of iteration m; epilogue: CTA partials -> rank partial (fixed
// order, last-block ticket).  Speculative launches after convergence exit at
// entry (ctrl->done), so the host may enqueue iterations in chunks.
// ---------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void rank_reduce(const LejaParams& P, double (&vals)[NV], double (*s_red)[kSlot],
                                            int* s_last) {
    block_reduce<NV>(vals, s_red);
    if (threadIdx.x == 0) {
        double* slot = P.partials + (size_t)blockIdx.x * kSlot;
#pragma unroll
        for (int i = 0; i < NV; i++) slot[i] = vals[i];
        __threadfence();
        const unsigned t = atomicAdd(&P.ctrl->ticket, 1u);
        *s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (*s_last) {
        __threadfence();
        double acc[NV];
#pragma unroll
        for (int i = 0; i < NV; i++) acc[i] = 0.0;
        for (int c = threadIdx.x; c < (int)gridDim.x; c += kThreads) {
#pragma unroll
            for (int i = 0; i < NV; i++) acc[i] += __ldcg(P.partials + (size_t)c * kSlot + i);
        }
        block_reduce<NV>(acc, s_red);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int i = 0; i < NV; i++) P.rank_part[i] = acc[i];
            P.ctrl->ticket = 0u;
        }
    }
}

template <int NDIM, int K, bool DIAG>
__global__ void __launch_bounds__(kThreads, 2) k_leja2d_step(const __grid_constant__ LejaParams P, int m) {
    __shared__ double s_red[kWarps][kSlot];
    __shared__ int s_last;
    Ctrl* ctrl = P.ctrl;
    if (*(volatile int*)&ctrl->done) return;
    const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool cwarp = (blockIdx.x == 0 && warp == 0);   // coefficient warp: row m+2 of the table
    const int M = P.max_nodes;
    int active = P.active0;
    if (m >= 2) {
        const int prev = *(volatile int*)&ctrl->hist[m & 1];   // mask after iteration m-2
        double sums[1 + K];
#pragma unroll
        for (int i = 0; i < 1 + K; i++) {
            double s = 0.0;
            for (int r = 0; r < P.nranks; r++) s += P.gathered[r * kSlot + i];
            sums[i] = s;
        }
        double dmp[K];   // d_{m-1}: row written by launch 1 (m-1 <= 2) or launch m-3
#pragma unroll
        for (int k = 0; k < K; k++) dmp[k] = P.table[(size_t)(m - 1) * (1 + K) + 1 + k];
        int act = prev, done = 0, status = 0;
        leja_decide<K>(P, m - 1, sums, dmp, act, done, status, writer ? P.rec : nullptr);
        if (writer) {
            ctrl->hist[(m - 1) & 1] = act;
            if (done) {
                ctrl->status = status;
                ctrl->m = m - 1;
                ctrl->done = 1;
            }
        }
        if (done) return;
        active = act;
    }
    if (m >= M) return;   // decision-only launch
    double d0[K], dm[K], sp[K];
    if (m <= 2 || cwarp) {
        double e0[K], e1[K], e2[K];
#pragma unroll
        for (int k = 0; k < K; k++) coef_first3(P, k, e0[k], e1[k], e2[k]);
        if (cwarp && m == 1 && P.coef_gen) {
            coef_write_row<K>(P, 0, lane, active, e0);
            coef_write_row<K>(P, 1, lane, active, e1);
            coef_write_row<K>(P, 2, lane, active, e2);
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            d0[k] = e0[k];
            dm[k] = (m == 1) ? e1[k] : e2[k];
        }
    }
    if (m >= 3) {
#pragma unroll
        for (int k = 0; k < K; k++) {
            d0[k] = P.table[1 + k];
            dm[k] = P.table[(size_t)m * (1 + K) + 1 + k];   // written by launch m-2
        }
    }
#pragma unroll
    for (int k = 0; k < K; k++) sp[k] = 0.0;
    const double beta = coef_beta(P, m);
    const double alpha = P_alpha(P);
    double sy = 0.0;
    double* dst = P.ydst[m & 1];
    if (cwarp) {
        if (P.coef_gen && m + 2 < M) coef_write_row<K>(P, m + 2, lane, active, nullptr);
    } else {
        const int gw = blockIdx.x * kWarps + warp - 1;
        const int W = gridDim.x * kWarps - 1;
        if (m == 1) {
            for (int unit = gw; unit < P.nunits; unit += W)
                tile<NDIM, K, DIAG, true, M_LEJA, true>(P, P.v, dst, unit, lane, beta, d0, dm, active, alpha, sy, sp);
        } else {
            const RowSrc src = P.ysrc[(m - 1) & 1];
            for (int unit = gw; unit < P.nunits; unit += W)
                tile<NDIM, K, DIAG, false, M_LEJA, false>(P, src, dst, unit, lane, beta, d0, dm, active, alpha, sy, sp);
        }
    }
    double vals[1 + K];
    vals[0] = sy;
#pragma unroll
    for (int k = 0; k < K; k++) vals[1 + k] = sp[k];
    rank_reduce<1 + K>(P, vals, s_red, &s_last);
}

template <int NDIM, bool DIAG>
__global__ void __launch_bounds__(kThreads, 2) k_power2d_step(const __grid_constant__ LejaParams P, int m) {
    __shared__ double s_red[kWarps][kSlot];
    __shared__ int s_last;
    Ctrl* ctrl = P.ctrl;
    if (*(volatile int*)&ctrl->done) return;
    const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
    double scale = 1.0;
    if (m >= 2) {
        double s = 0.0;
        for (int r = 0; r < P.nranks; r++) s += P.gathered[r * kSlot];
        int done = 0, status = 0;
        double est;
        power_decide(P, m - 1, s, done, status, &est, &scale, writer ? P.rec : nullptr);
        if (done) {
            if (writer) {
                ctrl->status = status;
                ctrl->done = 1;
            }
            return;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double sy = 0.0, sp[1] = {0.0};
    const RowSrc src = (m == 1) ? P.v : P.ysrc[(m - 1) & 1];
    double* dst = P.ydst[m & 1];
    for (int unit = blockIdx.x * kWarps + warp; unit < P.nunits; unit += gridDim.x * kWarps)
        tile<NDIM, 0, DIAG, false, M_POWER, false>(P, src, dst, unit, lane, 0.0, nullptr, nullptr, 0, scale, sy, sp);
    double vals[1] = {sy};
    rank_reduce<1>(P, vals, s_red, &s_last);
}

__global__ void k_finalize_err(const double* gathered, int nranks, double N, Record* rec) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int r = 0; r < nranks; r++) s += gathered[r * kSlot];
        rec->err = sqrt(s / N);
    }
}

__global__ void k_max_u64(const unsigned long long* vals, int n, unsigned long long* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long m = 0ull;
        for (int i = 0; i < n; i++) m = vals[i] > m ? vals[i] : m;
        *out = m;
    }
}



template <int NDIM>
static void* leja_kernel_ptr_nd(int K, bool diag) {
    switch (K * 2 + (diag ? 1 : 0)) {
        case 2: return (void*)k_leja2d<NDIM, 1, false>;
        case 3: return (void*)k_leja2d<NDIM, 1, true>;
        case 4: return (void*)k_leja2d<NDIM, 2, false>;
        case 5: return (void*)k_leja2d<NDIM, 2, true>;
        case 6: return (void*)k_leja2d<NDIM, 3, false>;
        case 7: return (void*)k_leja2d<NDIM, 3, true>;
        case 8: return (void*)k_leja2d<NDIM, 4, false>;
        case 9: return (void*)k_leja2d<NDIM, 4, true>;
    }
    return nullptr;
}

static void* leja_kernel_ptr(int ndim, int K, bool diag) {
    if (ndim == 4) {   // flux form (Burgers, 2D); react handled at run time inside the tile
        switch (K) {
            case 1: return (void*)k_leja2d<4, 1, false>;
            case 2: return (void*)k_leja2d<4, 2, false>;
            case 3: return (void*)k_leja2d<4, 3, false>;
            case 4: return (void*)k_leja2d<4, 4, false>;
        }
        return nullptr;
    }
    return ndim == 3 ? leja_kernel_ptr_nd<3>(K, diag) : leja_kernel_ptr_nd<2>(K, diag);
}

int leja_grid_size(int device, int K, bool diag, int ndim, int nunits) {
    long long g = coresident(device, leja_kernel_ptr(ndim, K, diag));
    // never more CTAs than work: at least 2 units per warp for tiny grids
    long long need = (nunits + kWarps - 1) / kWarps;
    if (g > need) g = need > 0 ? need : 1;
    return (int)g;
}

cudaError_t launch_leja_persistent(const LejaParams& P, cudaStream_t s, bool diag) {
    void* kern = leja_kernel_ptr(P.ndim, P.K, diag);
    if (!kern) return cudaErrorInvalidValue;
    void* args[] = {(void*)&P};
    return cudaLaunchCooperativeKernel(kern, dim3(P.grid), dim3(kThreads), args, 0, s);
}

cudaError_t launch_power_persistent(const LejaParams& P, cudaStream_t s, bool diag) {
    void* kern = P.ndim == 4 ? (void*)k_power2d<4, false>
                 : P.ndim == 3 ? (diag ? (void*)k_power2d<3, true> : (void*)k_power2d<3, false>)
                               : (diag ? (void*)k_power2d<2, true> : (void*)k_power2d<2, false>);
    void* args[] = {(void*)&P};
    return cudaLaunchCooperativeKernel(kern, dim3(P.grid), dim3(kThreads), args, 0, s);
}


template <int NDIM>
static void* leja_step_ptr_nd(int K, bool diag) {
    switch (K * 2 + (diag ? 1 : 0)) {
        case 2: return (void*)k_leja2d_step<NDIM, 1, false>;
        case 3: return (void*)k_leja2d_step<NDIM, 1, true>;
        case 4: return (void*)k_leja2d_step<NDIM, 2, false>;
        case 5: return (void*)k_leja2d_step<NDIM, 2, true>;
        case 6: return (void*)k_leja2d_step<NDIM, 3, false>;
        case 7: return (void*)k_leja2d_step<NDIM, 3, true>;
        case 8: return (void*)k_leja2d_step<NDIM, 4, false>;
        case 9: return (void*)k_leja2d_step<NDIM, 4, true>;
    }
    return nullptr;
}

static void* leja_step_ptr(int ndim, int K, bool diag) {
    return ndim == 3 ? leja_step_ptr_nd<3>(K, diag) : leja_step_ptr_nd<2>(K, diag);
}

int step_grid_size(int device, int nunits) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    long long g = (long long)nsm * 2;
    long long need = (nunits + kWarps - 1) / kWarps;
    if (g > need) g = need > 0 ? need : 1;
    return (int)g;
}

cudaError_t launch_leja_step(const LejaParams& P, int m, cudaStream_t s, bool diag) {
    void* kern = leja_step_ptr(P.ndim, P.K, diag);
    if (!kern) return cudaErrorInvalidValue;
    void* args[] = {(void*)&P, (void*)&m};
    return cudaLaunchKernel(kern, dim3(P.grid), dim3(kThreads), args, 0, s);
}

cudaError_t launch_power_step(const LejaParams& P, int m, cudaStream_t s, bool diag) {
    void* kern = P.ndim == 3 ? (diag ? (void*)k_power2d_step<3, true> : (void*)k_power2d_step<3, false>)
                             : (diag ? (void*)k_power2d_step<2, true> : (void*)k_power2d_step<2, false>);
    void* args[] = {(void*)&P, (void*)&m};
    return cudaLaunchKernel(kern, dim3(P.grid), dim3(kThreads), args, 0, s);
}

cudaError_t launch_finalize_err(const double* gathered, int nranks, double N, Record* rec, cudaStream_t s) {
    k_finalize_err<<<1, 32, 0, s>>>(gathered, nranks, N, rec);
    return cudaGetLastError();
}

cudaError_t launch_max_u64(const unsigned long long* vals, int n, unsigned long long* out, cudaStream_t s) {
    k_max_u64<<<1, 32, 0, s>>>(vals, n, out);
    return cudaGetLastError();
}

cudaError_t preload_leja() {
    for (int K = 1; K <= kMaxK; K++)
        for (int d = 0; d < 2; d++) {
            for (int nd : {2, 3, 4}) {
                const void* k = leja_kernel_ptr(nd, K, d != 0);
                cudaFuncAttributes a;
                if (k && cudaFuncGetAttributes(&a, k) != cudaSuccess) return cudaGetLastError();
            }
            for (int nd : {2, 3}) {
                cudaFuncAttributes a;
                if (cudaFuncGetAttributes(&a, leja_step_ptr(nd, K, d != 0)) != cudaSuccess) return cudaGetLastError();
            }
        }
    const void* fixed[] = {(const void*)k_power2d<2, false>, (const void*)k_power2d<2, true>,
                           (const void*)k_power2d<3, false>, (const void*)k_power2d<3, true>,
                           (const void*)k_power2d<4, false>, (const void*)k_power2d_step<2, false>,
                           (const void*)k_power2d_step<2, true>, (const void*)k_power2d_step<3, false>,
                           (const void*)k_power2d_step<3, true>, (const void*)k_finalize_err, (const void*)k_max_u64};
    for (const void* k : fixed) {
        cudaFuncAttributes a;
        if (cudaFuncGetAttributes(&a, k) != cudaSuccess) return cudaGetLastError();
    }
    return cudaSuccess;
}

}  // namespace lx
