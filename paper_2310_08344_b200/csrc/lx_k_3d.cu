// lx_k_3d.cu -- 3D Leja kernel with shared-memory plane tiles (k_leja3d_smem).
#include "lx_dev.cuh"

namespace lx {

// ---------------------------------------------------------------------------
// 3D marching kernel with shared-memory plane tiles (single GPU; n1 % 8 == 0, n2 % 64 == 0).
// A CTA owns a (8 j-rows x 64 k) column of one run of TI3 planes and marches along i: every plane's
// tile of rows j0-1 .. j0+9 (11 rows: the j-neighbours j-1, j+1, j+2 of the 8 output rows) and
// columns k0-2 .. k0+65 is staged once by cp.async into a ring of 6 planes, so each y value is read
// from L2/HBM ~1.4 times (11/8 rows + run halos) instead of ~5.5 times by the warp-unit tile3d;
// i-, j- and k-neighbours all come from shared memory.  Same per-point FMA order as tile3d (bitwise
// equal results).  Newton coefficients come from the prebuilt table (k_coef_tables); the grid
// barrier and the P:155 decision are those of k_leja2d.
// ---------------------------------------------------------------------------
#ifndef LX_TI3
#define LX_TI3 64
#endif
constexpr int kTI3 = LX_TI3;             // planes per run
constexpr int kS3Cols = 68;              // k0-2 .. k0+65
constexpr int kS3J = 16;                 // output j-rows per CTA tile (2 per warp)
constexpr int kS3Rows = kS3J + 3;        // j0-1 .. j0+kS3J+1
constexpr int kS3Plane = kS3Rows * kS3Cols;   // doubles per staged plane
constexpr int kS3Depth = 6;              // ring of planes
constexpr int kS3Smem = kS3Depth * kS3Plane * 8;

__device__ __forceinline__ void s3_issue(const double* __restrict__ src, double* ring, int ip, int slot, int j0,
                                         int k0, int n0, int n1, int n2) {
    // kS3Rows rows x 34 16-byte pieces
    const int pl = ip < 0 ? ip + n0 : (ip >= n0 ? ip - n0 : ip);
    double* dst = ring + slot * kS3Plane;
    for (int t = threadIdx.x; t < kS3Rows * (kS3Cols / 2); t += kThreads) {
        const int r = t / (kS3Cols / 2), c2 = t - r * (kS3Cols / 2);
        int j = j0 - 1 + r;
        j = j < 0 ? j + n1 : (j >= n1 ? j - n1 : j);
        int k = k0 - 2 + 2 * c2;
        k = k < 0 ? k + n2 : (k >= n2 ? k - n2 : k);
        cp_async16(dst + r * kS3Cols + 2 * c2, src + ((size_t)pl * n1 + j) * n2 + k);
    }
}

template <int K, bool DIAG, bool FIRST>
__device__ __forceinline__ void s3_unit(const LejaParams& P, const double* __restrict__ src, double* __restrict__ dst,
                                        int cu, double* ring, int lane, int warp, double beta, const double* d0,
                                        const double* dm, int active, double alpha, double& sy, double* sp) {
    const int n0 = P.n_loc, n1 = P.n1, n2 = P.n2;
    const int njb = n1 / kS3J, nkb = n2 >> 6;
    const int jb = cu % njb;
    const int t0 = cu / njb;
    const int kb = t0 % nkb;
    const int ir = t0 / nkb;
    const int j0 = jb * kS3J, k0 = kb * 64;
    const int i0 = ir * kTI3, i1 = min(n0, i0 + kTI3);
    const Stencil& S = P.st;
    constexpr int KK = K > 0 ? K : 1;
    constexpr int RW = kS3J / kWarps;               // rows per warp
#pragma unroll
    for (int q = 0; q < 4; q++) {
        s3_issue(src, ring, i0 - 1 + q, q, j0, k0, n0, n1, n2);
        cp_async_commit();
    }
    const int kc = k0 + 2 * lane;
    // p / u of the next plane prefetched into registers one plane ahead (their latency off the barrier path);
    // K >= 3 keeps only u prefetched (the p registers would spill)
    constexpr bool PREF = K <= 2;
    constexpr int KP = PREF ? KK : 1;
    double2 pv[RW][KK], uu[RW], pvn[RW][KP], uun[RW];
    auto fetch_p = [&](int i, auto& pq) {
#pragma unroll
        for (int r = 0; r < RW; r++) {
            const long long off = ((long long)i * n1 + (j0 + warp + r * kWarps)) * n2 + kc;
#pragma unroll
            for (int k = 0; k < KK; k++) {
                pq[r][k] = make_double2(0.0, 0.0);
                if (!FIRST && i < i1 && ((active >> k) & 1)) pq[r][k] = ld2(P.p[k] + off);
            }
        }
    };
    auto fetch_u = [&](int i, double2 (&uq)[RW]) {
#pragma unroll
        for (int r = 0; r < RW; r++) {
            const long long off = ((long long)i * n1 + (j0 + warp + r * kWarps)) * n2 + kc;
            uq[r] = make_double2(0.0, 0.0);
            if (DIAG && i < i1) uq[r] = ldg2(P.u + off);
        }
    };
    if constexpr (PREF) fetch_p(i0, pv);
    fetch_u(i0, uu);
    for (int i = i0; i < i1; i++) {
        const int rel = i - i0 + 1;
        if (i + 3 <= i1 + 1) s3_issue(src, ring, i + 3, (rel + 3) % kS3Depth, j0, k0, n0, n1, n2);
        cp_async_commit();   // (possibly empty group: keeps the wait_group accounting uniform)
        if constexpr (PREF) fetch_p(i + 1, pvn);
        fetch_u(i + 1, uun);
        if constexpr (!PREF) fetch_p(i, pv);
        cp_async_wait<1>();
        __syncthreads();
        const uint32_t base = smem_u32(ring);
        auto at = [&](int pos, int row, int col) {
            return lds2(base + (uint32_t)(((pos % kS3Depth) * kS3Plane + row * kS3Cols + col) * 8));
        };
        const int cc = 2 + 2 * lane;
#pragma unroll
        for (int r = 0; r < RW; r++) {
            const int row = warp + r * kWarps + 1;     // staged row of output j
            const int j = j0 + row - 1;
            const double2 yc = at(rel, row, cc);
            const double2 up = at(rel - 1 + kS3Depth, row, cc);
            const double2 dn1 = at(rel + 1, row, cc);
            const double2 dn2 = at(rel + 2, row, cc);
            const double2 wm = at(rel, row - 1, cc);
            const double2 wp1 = at(rel, row + 1, cc);
            const double2 wp2 = at(rel, row + 2, cc);
            const double2 lf = at(rel, row, cc - 2);
            const double2 rt = at(rel, row, cc + 2);
            const double left = lf.y, r1 = rt.x, r2 = rt.y;
            const long long off = ((long long)i * n1 + j) * n2 + kc;
            double ax = S.c0 * yc.x;
            ax = fma(S.m1[0], up.x, ax);
            ax = fma(S.p1[0], dn1.x, ax);
            ax = fma(S.p2[0], dn2.x, ax);
            ax = fma(S.m1[1], wm.x, ax);
            ax = fma(S.p1[1], wp1.x, ax);
            ax = fma(S.p2[1], wp2.x, ax);
            ax = fma(S.m1[2], left, ax);
            ax = fma(S.p1[2], yc.y, ax);
            ax = fma(S.p2[2], r1, ax);
            double ay = S.c0 * yc.y;
            ay = fma(S.m1[0], up.y, ay);
            ay = fma(S.p1[0], dn1.y, ay);
            ay = fma(S.p2[0], dn2.y, ay);
            ay = fma(S.m1[1], wm.y, ay);
            ay = fma(S.p1[1], wp1.y, ay);
            ay = fma(S.p2[1], wp2.y, ay);
            ay = fma(S.m1[2], yc.x, ay);
            ay = fma(S.p1[2], r1, ay);
            ay = fma(S.p2[2], r2, ay);
            if (DIAG) {
                ax = fma(fma(S.qb, uu[r].x * uu[r].x, S.qa), yc.x, ax);
                ay = fma(fma(S.qb, uu[r].y * uu[r].y, S.qa), yc.y, ay);
            }
            double2 yn;
            yn.x = fma(alpha, ax, beta * yc.x);
            yn.y = fma(alpha, ay, beta * yc.y);
            st2(dst + off, yn);
            sy = fma(yn.x, yn.x, sy);
            sy = fma(yn.y, yn.y, sy);
#pragma unroll
            for (int k = 0; k < KK; k++) {
                if ((active >> k) & 1) {
                    double2 pn;
                    if (FIRST) {
                        pn.x = fma(dm[k], yn.x, d0[k] * yc.x);
                        pn.y = fma(dm[k], yn.y, d0[k] * yc.y);
                    } else {
                        pn.x = fma(dm[k], yn.x, pv[r][k].x);
                        pn.y = fma(dm[k], yn.y, pv[r][k].y);
                    }
                    st2(P.p[k] + off, pn);
                    sp[k] = fma(pn.x, pn.x, sp[k]);
                    sp[k] = fma(pn.y, pn.y, sp[k]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RW; r++) {
            uu[r] = uun[r];
            if constexpr (PREF) {
#pragma unroll
                for (int k = 0; k < KP; k++) pv[r][k] = pvn[r][k];
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();   // the ring is reused by the next unit
}

template <int K, bool DIAG>
__global__ void __launch_bounds__(kThreads, 2) k_leja3d_smem(const __grid_constant__ LejaParams P) {
    __shared__ double s_red[kWarps][kSlot];
    __shared__ int s_flags[4];
    extern __shared__ double s3_ring[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned gen0 = 0;
    if (tid == 0) gen0 = (unsigned)(ld_acquire64(&P.ctrl->word) >> 32);
    int active = P.active0;
    const int M = P.max_nodes;
    const double alpha = P_alpha(P);
    const int ncu = (P.n1 / kS3J) * (P.n2 >> 6) * ((P.n_loc + kTI3 - 1) / kTI3);
    double d0[K];
#pragma unroll
    for (int k = 0; k < K; k++) d0[k] = P.table[1 + k];
    double beta_n = coef_beta(P, 1), dm_n[K];
#pragma unroll
    for (int k = 0; k < K; k++) dm_n[k] = P.table[(size_t)(1 + K) + 1 + k];
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
        if (m == 1) {
            for (int cu = blockIdx.x; cu < ncu; cu += gridDim.x)
                s3_unit<K, DIAG, true>(P, P.v.base, dst, cu, s3_ring, lane, warp, beta, d0, dm, active, alpha, sy, sp);
        } else {
            const double* src = P.ydst[par ^ 1];
            for (int cu = blockIdx.x; cu < ncu; cu += gridDim.x)
                s3_unit<K, DIAG, false>(P, src, dst, cu, s3_ring, lane, warp, beta, d0, dm, active, alpha, sy, sp);
        }
        double vals[1 + K];
        vals[0] = sy;
#pragma unroll
        for (int k = 0; k < K; k++) vals[1 + k] = sp[k];
        if (m + 1 < M) {
            beta_n = coef_beta(P, m + 1);
#pragma unroll
            for (int k = 0; k < K; k++) dm_n[k] = P.table[(size_t)(m + 1) * (1 + K) + 1 + k];
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

static void* leja3d_smem_ptr(int K, bool diag) {
    switch (K * 2 + (diag ? 1 : 0)) {
        case 2: return (void*)k_leja3d_smem<1, false>;
        case 3: return (void*)k_leja3d_smem<1, true>;
        case 4: return (void*)k_leja3d_smem<2, false>;
        case 5: return (void*)k_leja3d_smem<2, true>;
        case 6: return (void*)k_leja3d_smem<3, false>;
        case 7: return (void*)k_leja3d_smem<3, true>;
        case 8: return (void*)k_leja3d_smem<4, false>;
        case 9: return (void*)k_leja3d_smem<4, true>;
    }
    return nullptr;
}

int leja3d_smem_units(int n0, int n1, int n2) { return (n1 / kS3J) * (n2 / 64) * ((n0 + kTI3 - 1) / kTI3); }

int leja3d_smem_grid_size(int device, int K, bool diag, int ncu) {
    void* kern = leja3d_smem_ptr(K, diag);
    if (!kern) return 0;
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({device, kern});
    int g;
    if (it != cache.end()) {
        g = it->second;
    } else {
        int nsm = 0, per = 0;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kS3Smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kThreads, kS3Smem);
        g = nsm * (per < 1 ? 1 : per);
        cache[{device, kern}] = g;
    }
    return g < ncu ? g : ncu;
}

cudaError_t launch_leja3d_smem(const LejaParams& P, cudaStream_t s, bool diag) {
    void* kern = leja3d_smem_ptr(P.K, diag);
    if (!kern) return cudaErrorInvalidValue;
    void* args[] = {(void*)&P};
    return cudaLaunchCooperativeKernel(kern, dim3(P.grid), dim3(kThreads), args, kS3Smem, s);
}

cudaError_t preload_3d() {
    for (int K = 1; K <= kMaxK; K++)
        for (int d = 0; d < 2; d++) {
            cudaFuncAttributes a;
            if (cudaFuncGetAttributes(&a, leja3d_smem_ptr(K, d != 0)) != cudaSuccess) return cudaGetLastError();
        }
    return cudaSuccess;
}

}  // namespace lx
