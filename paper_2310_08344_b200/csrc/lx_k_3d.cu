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

// ---------------------------------------------------------------------------
// f(u) dt on 3D grids (single domain, the smem kernel's shape) with the same shared-memory plane tiles as
// k_leja3d_smem (each u value read from L2 / HBM ~1.2 times instead of ~5.5 by the warp-tile k_rhs2d<3>):
// f(u) scale = scale (A u + react (u - u^3) [+ S]), the stencil in the FMA order of tile3d's M_RHS (16 B/pt,
// +8 with a source).  No grid-wide synchronisation: a plain launch over the CTA units.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2) k_rhs3d_smem(const __grid_constant__ LejaParams P, double scale) {
    extern __shared__ double s3_rhs_ring[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n0 = P.n_loc, n1 = P.n1, n2 = P.n2;
    const int njb = n1 / kS3J, nkb = n2 >> 6;
    const int ncu = njb * nkb * ((n0 + kTI3 - 1) / kTI3);
    const Stencil& S = P.st;
    constexpr int RW = kS3J / kWarps;
    const double* src = P.v.base;
    double* dst = P.ydst[0];
    for (int cu = blockIdx.x; cu < ncu; cu += gridDim.x) {
        const int jb = cu % njb, t0 = cu / njb, kb = t0 % nkb, ir = t0 / nkb;
        const int j0 = jb * kS3J, k0 = kb * 64;
        const int i0 = ir * kTI3, i1 = min(n0, i0 + kTI3);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            s3_issue(src, s3_rhs_ring, i0 - 1 + q, q, j0, k0, n0, n1, n2);
            cp_async_commit();
        }
        const int kc = k0 + 2 * lane;
        for (int i = i0; i < i1; i++) {
            const int rel = i - i0 + 1;
            if (i + 3 <= i1 + 1) s3_issue(src, s3_rhs_ring, i + 3, (rel + 3) % kS3Depth, j0, k0, n0, n1, n2);
            cp_async_commit();
            cp_async_wait<1>();
            __syncthreads();
            const uint32_t base = smem_u32(s3_rhs_ring);
            auto at = [&](int pos, int row, int col) {
                return lds2(base + (uint32_t)(((pos % kS3Depth) * kS3Plane + row * kS3Cols + col) * 8));
            };
            const int cc = 2 + 2 * lane;
#pragma unroll
            for (int r = 0; r < RW; r++) {
                const int row = warp + r * kWarps + 1;
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
                double fx = fma(S.react, yc.x - yc.x * yc.x * yc.x, ax);
                double fy = fma(S.react, yc.y - yc.y * yc.y * yc.y, ay);
                const long long off = ((long long)i * n1 + j) * n2 + kc;
                if (P.source) {
                    const double2 sv = ldg2(P.source + off);
                    fx += sv.x;
                    fy += sv.y;
                }
                st2(dst + off, make_double2(scale * fx, scale * fy));
            }
        }
        cp_async_wait<0>();
        __syncthreads();   // the ring is reused by the next unit
    }
}

cudaError_t launch_rhs3d_smem(const LejaParams& P, double scale, cudaStream_t s, int device) {
    static std::mutex mu;
    static std::map<int, int> cache;
    int g;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(device);
        if (it != cache.end()) {
            g = it->second;
        } else {
            int nsm = 0, per = 0;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
            cudaFuncSetAttribute((const void*)k_rhs3d_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kS3Smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)k_rhs3d_smem, kThreads, kS3Smem);
            g = nsm * (per < 1 ? 1 : per);
            cache[device] = g;
        }
    }
    const int ncu = leja3d_smem_units(P.n_loc, P.n1, P.n2);
    if (g > ncu) g = ncu;
    k_rhs3d_smem<<<g, kThreads, kS3Smem, s>>>(P, scale);
    return cudaGetLastError();
}

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

// ---------------------------------------------------------------------------
// 3D two-step kernel (2.5D temporal blocking, SURVEY 8(f) f-3 in 3D; constant-coefficient operators).
// One pass over the grid performs Leja iterations m = 2q+1 and m+1 (Eq. (2) twice).  A CTA owns a
// (16 j-rows x 64 k) column of a run of kTI3 planes and marches along i; its 16 warps have two roles,
// one barrier per plane step t:
//   stage A (warps 0..7): y_m on plane t over the halo-extended tile (rows j0-1 .. j0+17, columns
//            k0-2 .. k0+65: the j/k neighbours j-1, j+1, j+2 stage B needs) from the staged y_{m-1}
//            tiles (rows j0-2 .. j0+19, columns k0-4 .. k0+67; a cp.async ring of 5 planes that these
//            warps fill, plane t+4 into the slot of plane t-1) into a shared-memory ring of 5 y_m planes;
//            each thread keeps its own column's y_{m-1} at planes t-1, t, t+1 in registers and shares
//            the j-neighbours of its 3 consecutive rows; y_m never goes to HBM;
//   stage B (warps 8..15): y_{m+1} on plane t-3 over the 16 x 64 interior from the y_m planes t-4 .. t-1
//            finished in earlier steps (two rows per warp sharing their j-neighbours),
//            p_m = p_{m-1} + d_m y_m, p_{m+1} = p_m + d_{m+1} y_{m+1}, the norms of y_m, p_m, y_{m+1},
//            p_{m+1}; writes y_{m+1} and p.
// HBM per pass: read y_{m-1}, p; write y_{m+1}, p (32 B/pt for K = 1, +16 per further accumulator): half
// the bytes of two one-pass iterations.  Same per-point FMA order as k_leja3d_smem, so y and p are bitwise
// those of the one-pass kernel; only the norm summation order differs.  One grid barrier per pass; the
// last arriver decides m, then m+1.  An accumulator that converges at m got one term too many:
// it is rolled back, p_m = p_{m+1} - d_{m+1} y_{m+1} (within one rounding of the one-step value, as in
// the 2D two-step kernel), by the next pass's stage B or by the end-of-call fix-up.  Coefficients from
// the prebuilt table (k_coef_tables), as k_leja3d_smem.  n1 % 16 == 0, n2 % 64 == 0; no Allen-Cahn term.
// ---------------------------------------------------------------------------
constexpr int kB3J = 16;                        // output j-rows per tile
constexpr int kB3R1R = kB3J + 6, kB3R1C = 72;   // staged y_{m-1}: rows j0-2 .. j0+19, columns k0-4 .. k0+67
constexpr int kB3R1P = kB3R1R * kB3R1C;
constexpr int kB3R2R = kB3J + 3, kB3R2C = 68;   // y_m: rows j0-1 .. j0+17, columns k0-2 .. k0+65
constexpr int kB3R2P = kB3R2R * kB3R2C;
constexpr int kB3D = 5;                         // ring depth of both rings (planes)
constexpr int kB3Threads = 512, kB3Warps = kB3Threads / 32;   // 8 stage-A warps + 8 stage-B warps
constexpr int kB3Pieces = kB3R1R * (kB3R1C / 2);             // 16-B pieces of a staged plane (792)
constexpr int kB3PPT = (kB3Pieces + 255) / 256;              // pieces per stage-A thread (4)
static_assert(kB3J == 16 && kB3R2R == 19, "stage roles assume 16 output rows (19 y_m rows)");
constexpr int kB3SmemRings = kB3D * (kB3R1P + kB3R2P) * 8;
// + stage-B private staging of p_k / v / y_{m-1} (two rows x (K + 1) 16-B pieces per thread, two planes)
__host__ __device__ constexpr int b3_np(int K) { return 2 * (K + 1); }
__host__ __device__ constexpr int b3_smem(int K) { return kB3SmemRings + 2 * b3_np(K) * 16 * 256; }

__device__ __forceinline__ int b3_inc(int x, int n) { return x + 1 == n ? 0 : x + 1; }

// mbarrier helpers (CTA scope): the y_m ring's full / empty handshake between the two roles
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "LX_MBW_%=:\n"
        " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LX_MBW_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// named barrier of the 256 stage-A threads (the y_{m-1} ring is theirs alone)
__device__ __forceinline__ void bar_a() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// A y (before the alpha / beta scaling) at the two columns of a pair, k_leja3d_smem's FMA order
__device__ __forceinline__ double2 b3_apply(const Stencil& S, double2 yc, double2 up, double2 dn1, double2 dn2,
                                            double2 wm, double2 wp1, double2 wp2, double left, double2 rt) {
    // the 10 stencil terms summed per direction, then the three direction sums (dependent chain 6 deep
    // instead of 10: stage B, the kernel's critical path, is latency-bound on it)
    double x0 = fma(S.m1[0], up.x, S.c0 * yc.x);
    x0 = fma(S.p1[0], dn1.x, x0);
    x0 = fma(S.p2[0], dn2.x, x0);
    double x1 = S.m1[1] * wm.x;
    x1 = fma(S.p1[1], wp1.x, x1);
    x1 = fma(S.p2[1], wp2.x, x1);
    double x2 = S.m1[2] * left;
    x2 = fma(S.p1[2], yc.y, x2);
    x2 = fma(S.p2[2], rt.x, x2);
    double y0 = fma(S.m1[0], up.y, S.c0 * yc.y);
    y0 = fma(S.p1[0], dn1.y, y0);
    y0 = fma(S.p2[0], dn2.y, y0);
    double y1 = S.m1[1] * wm.y;
    y1 = fma(S.p1[1], wp1.y, y1);
    y1 = fma(S.p2[1], wp2.y, y1);
    double y2 = S.m1[2] * yc.x;
    y2 = fma(S.p1[2], rt.x, y2);
    y2 = fma(S.p2[2], rt.y, y2);
    return make_double2(x0 + (x1 + x2), y0 + (y1 + y2));
}

// Per-pass coefficients (shared memory): d_m, d_{m+1}, d_0 (first pass), d_{m-1} (rollback)
template <int K>
struct B3Coef {
    double ba, bb, alpha;
    double da[K], db[K], d0[K], dr[K];
};

// Stage A, main warps: R consecutive y_m rows a0 .. a0+R-1 of the pair column `lane` (R2 columns 2 lane,
// 2 lane + 1).  The own column's y_{m-1} at planes t-1, t, t+1 is kept in a register window (wu, wc, wd),
// so a row costs its k-neighbours and plane t+2; the j-neighbours of the R rows are the R centres plus
// three loads (R1 rows a0, a0+R+1, a0+R+2).
template <int R>
__device__ __forceinline__ void b3_stage_a(const Stencil& S, double alpha, double beta, uint32_t pc, uint32_t pd2,
                                           uint32_t pw, int a0, int lane, double2 (&wu)[3], double2 (&wc)[3],
                                           double2 (&wd)[3]) {
    constexpr uint32_t RB = kB3R1C * 8;
    const uint32_t cb = (uint32_t)a0 * RB + (uint32_t)((2 * lane + 2) * 8);   // R1 row a0 (= wm of row a0)
    double2 col[R + 3];
    col[0] = lds2(pc + cb);
#pragma unroll
    for (int r = 0; r < R; r++) col[1 + r] = wc[r];
    col[R + 1] = lds2(pc + cb + (R + 1) * RB);
    col[R + 2] = lds2(pc + cb + (R + 2) * RB);
#pragma unroll
    for (int r = 0; r < R; r++) {
        const uint32_t c = cb + (r + 1) * RB;
        const double2 dn2 = lds2(pd2 + c);
        const double2 lf = lds2(pc + c - 16);
        const double2 rt = lds2(pc + c + 16);
        const double2 yc = col[r + 1];
        const double2 ax = b3_apply(S, yc, wu[r], wd[r], dn2, col[r], col[r + 2], col[r + 3], lf.y, rt);
        const double yx = fma(alpha, ax.x, beta * yc.x), yy = fma(alpha, ax.y, beta * yc.y);
        const uint32_t o = pw + (uint32_t)((((a0 + r) * kB3R2C) + 2 * lane) * 8);
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(o), "d"(yx), "d"(yy) : "memory");
        wu[r] = yc;
        wc[r] = wd[r];
        wd[r] = dn2;
    }
}

// R1 byte offset of the centre of stage-A edge task e (warp 7): row e % 19, pair 32 + e / 19
__device__ __forceinline__ uint32_t b3_edge_c(int e) {
    const int a = e % kB3R2R, b = 32 + e / kB3R2R;
    return (uint32_t)(((a + 1) * kB3R1C + 2 * b + 2) * 8);
}

// Stage A, warp 7: the right-halo pairs 32, 33 (columns k0+62 .. k0+65) of all 19 rows (38 tasks, two per
// lane), own column's window as the main warps
__device__ __forceinline__ void b3_stage_a_edge(const Stencil& S, double alpha, double beta, uint32_t pc,
                                                uint32_t pd2, uint32_t pw, int lane, double2 (&wu)[3],
                                                double2 (&wc)[3], double2 (&wd)[3]) {
    constexpr uint32_t RB = kB3R1C * 8;
#pragma unroll
    for (int rnd = 0; rnd < 2; rnd++) {
        const int e = lane + 32 * rnd;
        if (e < 2 * kB3R2R) {
            const uint32_t c = b3_edge_c(e);
            const double2 yc = wc[rnd];
            const double2 dn2 = lds2(pd2 + c);
            const double2 wm = lds2(pc + c - RB);
            const double2 wp1 = lds2(pc + c + RB);
            const double2 wp2 = lds2(pc + c + 2 * RB);
            const double2 lf = lds2(pc + c - 16);
            const double2 rt = lds2(pc + c + 16);
            const double2 ax = b3_apply(S, yc, wu[rnd], wd[rnd], dn2, wm, wp1, wp2, lf.y, rt);
            const double yx = fma(alpha, ax.x, beta * yc.x), yy = fma(alpha, ax.y, beta * yc.y);
            const int a = e % kB3R2R, b = 32 + e / kB3R2R;
            const uint32_t o = pw + (uint32_t)((a * kB3R2C + 2 * b) * 8);
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(o), "d"(yx), "d"(yy) : "memory");
            wu[rnd] = yc;
            wc[rnd] = wd[rnd];
            wd[rnd] = dn2;
        }
    }
}

// Stage B (warps 8 .. 15, wb = warp - 8): y_{m+1} on plane s, output rows 2 wb, 2 wb + 1 (R2 rows
// 2 wb + 1, + 2); j-neighbours shared between the two rows; p_m, p_{m+1} and the four norms.
template <int K, bool FIRST, bool SLAB>
__device__ __forceinline__ void b3_stage_b(const LejaParams& P, const B3Coef<K>& C, double* __restrict__ dst,
                                           uint32_t pm1, uint32_t ps, uint32_t pn1, uint32_t pt, uint32_t cbB,
                                           long long off0, long long rstride, int act, int rbm, bool two,
                                           uint32_t pst, double* sums, double* x1, double* x2) {
    constexpr uint32_t RB2 = kB3R2C * 8;
    const Stencil& S = P.st;
    const double alpha = C.alpha, bb = C.bb;
    double2 col[5];
#pragma unroll
    for (int r = 0; r < 2; r++) {
        if (r == 0) {
#pragma unroll
            for (int i = 0; i < 4; i++) col[i] = lds2(ps + cbB + i * RB2);
        } else {
            col[4] = lds2(ps + cbB + 4 * RB2);
        }
        const uint32_t c = cbB + (r + 1) * RB2;
        const double2 up = lds2(pm1 + c);
        const double2 dn1 = lds2(pn1 + c);
        const double2 dn2 = lds2(pt + c);
        const double2 lf = lds2(ps + c - 16);
        const double2 rt = lds2(ps + c + 16);
        const double2 yc = col[r + 1];
        const double2 ax = b3_apply(S, yc, up, dn1, dn2, col[r], col[r + 2], col[r + 3], lf.y, rt);
        double2 yn;
        yn.x = fma(alpha, ax.x, bb * yc.x);
        yn.y = fma(alpha, ax.y, bb * yc.y);
        const long long off = off0 + r * rstride;
        LX_DCHECK(off >= 0 && off + 2 <= (long long)P.n_loc * P.n1 * P.n2, "stage B output offset");
        if (!two) yn = yc;   // one-iteration pass: y_m is the next pass's input
        st2(dst + off, yn);
        if (SLAB) {   // a boundary plane of y_{m+1}: also into the neighbour's ghost block (peer memory)
            LX_DCHECK(!x1 || off < 4 * (long long)P.n1 * P.n2, "ghost delivery up: plane < 4");
            LX_DCHECK(!x2 || off >= ((long long)P.n_loc - 2) * P.n1 * P.n2, "ghost delivery down: plane >= n-2");
            if (x1) st2(x1 + off, yn);
            if (x2) st2(x2 + off, yn);
        }
        sums[0] = fma(yc.x, yc.x, sums[0]);
        sums[0] = fma(yc.y, yc.y, sums[0]);
        sums[1 + K] = fma(yn.x, yn.x, sums[1 + K]);
        sums[1 + K] = fma(yn.y, yn.y, sums[1 + K]);
        // staged inputs of this thread (piece i at pst + 4096 i): p_k (i = r (K+1) + k), v / y_{m-1} (i = r (K+1) + K)
        double2 yo = make_double2(0.0, 0.0);
        if (FIRST || rbm) yo = lds2(pst + (uint32_t)((r * (K + 1) + K) * 4096));
#pragma unroll
        for (int k = 0; k < K; k++) {
            if ((act >> k) & 1) {
                double2 pm, pn;
                if (FIRST) {
                    pm.x = fma(C.da[k], yc.x, C.d0[k] * yo.x);
                    pm.y = fma(C.da[k], yc.y, C.d0[k] * yo.y);
                } else {
                    const double2 pin = lds2(pst + (uint32_t)((r * (K + 1) + k) * 4096));
                    pm.x = fma(C.da[k], yc.x, pin.x);
                    pm.y = fma(C.da[k], yc.y, pin.y);
                }
                sums[1 + k] = fma(pm.x, pm.x, sums[1 + k]);
                sums[1 + k] = fma(pm.y, pm.y, sums[1 + k]);
                pn = pm;
                if (two) {
                    pn.x = fma(C.db[k], yn.x, pm.x);
                    pn.y = fma(C.db[k], yn.y, pm.y);
                }
                sums[2 + K + k] = fma(pn.x, pn.x, sums[2 + K + k]);
                sums[2 + K + k] = fma(pn.y, pn.y, sums[2 + K + k]);
                st2(P.p[k] + off, pn);
            } else if (!FIRST && ((rbm >> k) & 1)) {
                const double2 pin = lds2(pst + (uint32_t)((r * (K + 1) + k) * 4096));
                double2 pr;
                pr.x = fma(-C.dr[k], yo.x, pin.x);
                pr.y = fma(-C.dr[k], yo.y, pin.y);
                st2(P.p[k] + off, pr);
            }
        }
    }
}

// One unit (16 j x 64 k column of a run of kTI3 planes).  Stage A computes y_m on planes t = i0-1 .. i1+1,
// stage B y_{m+1} on planes s = i0 .. i1-1 from y_m planes s-1 .. s+2.  The roles are decoupled: y_m ring
// slot (x - i0 + 2) % 5 of plane x has a "full" mbarrier (256 stage-A arrivals after its stores) and an
// "empty" one (256 stage-B arrivals after its last read, at s = x+1), so stage A runs up to two planes
// ahead of stage B and the stage-B warps run independently of each other; the stage-A warps keep one
// named barrier per plane for their own y_{m-1} ring.  Phase parities are tracked per slot (fb, eb).
template <int K, bool FIRST, bool SLAB>
__device__ __forceinline__ void b3_unit(const LejaParams& P, const double* __restrict__ src, double* __restrict__ dst,
                                        int cu, double* r1, double* r2, uint32_t bars, unsigned& ph,
                                        const B3Coef<K>& C, int act, int rbm, bool two, double* sums,
                                        const double* gsrc, double* xup, double* xdn, bool& peer) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n0 = P.n_loc, n1 = P.n1, n2 = P.n2;
    const int njb = n1 / kB3J, nkb = n2 >> 6;
    const int jb = cu % njb;
    const int t0 = cu / njb;
    const int kb = t0 % nkb;
    const int ir = t0 / nkb;
    const int j0 = jb * kB3J, k0 = kb * 64;
    const int i0 = ir * kTI3, i1 = min(n0, i0 + kTI3);
    const long long plane = (long long)n1 * n2;
    const uint32_t b1 = smem_u32(r1), b2 = smem_u32(r2);
    const uint32_t fullb = bars, emptyb = bars + kB3D * 8;
    constexpr uint32_t RB1 = kB3R1C * 8, RB2 = kB3R2C * 8;
    constexpr uint32_t SL1 = kB3R1P * 8, SL2 = kB3R2P * 8;   // slot bytes
    if (warp < 8) {
        const Stencil& S = P.st;
        // this thread's pieces of a staged plane (fixed per unit): global offset in the plane, smem offset
        int goff[kB3PPT];
        uint32_t soff[kB3PPT];
#pragma unroll
        for (int q = 0; q < kB3PPT; q++) {
            const int pc = tid + 256 * q;
            goff[q] = -1;
            soff[q] = 0;
            if (pc < kB3Pieces) {
                const int r = pc / (kB3R1C / 2), c2 = pc - r * (kB3R1C / 2);
                int j = j0 - 2 + r;
                j = j < 0 ? j + n1 : (j >= n1 ? j - n1 : j);
                int k = k0 - 4 + 2 * c2;
                k = k < 0 ? k + n2 : (k >= n2 ? k - n2 : k);
                goff[q] = j * n2 + k;
                soff[q] = (uint32_t)((r * kB3R1C + 2 * c2) * 8);
            }
        }
        // plane pl of y_{m-1}: periodic wrap (single domain) or, in the slab kernel, planes -2, -1, n .. n+3
        // from this rank's ghost block gsrc (slots 0, 1 = planes -2, -1; 2 .. 5 = planes n .. n+3)
        int pl = i0 - 2;
        if (!SLAB) {
            pl %= n0;
            if (pl < 0) pl += n0;
        }
        auto issue = [&](int slot) {
            const double* base;
            if (SLAB && (unsigned)pl >= (unsigned)n0) base = gsrc + (long long)(pl < 0 ? pl + 2 : pl - n0 + 2) * plane;
            else base = src + (long long)pl * plane;
            LX_DCHECK(SLAB ? (pl >= -2 && pl < n0 + 4) : (pl >= 0 && pl < n0), "stage A plane index");
            const uint32_t sb = b1 + (uint32_t)slot * SL1;
            LX_DCHECK(slot >= 0 && slot < kB3D, "stage A ring slot");
#pragma unroll
            for (int q = 0; q < kB3PPT; q++)
                if (goff[q] >= 0) {
                    LX_DCHECK(goff[q] + 2 <= plane && soff[q] + 16 <= SL1, "stage A piece offsets");
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + soff[q]), "l"(base + goff[q])
                                 : "memory");
                }
            pl = SLAB ? pl + 1 : b3_inc(pl, n0);
        };
#pragma unroll 1
        for (int q = 0; q < 5; q++) {   // planes i0-2 .. i0+2 -> slots 0..4
            issue(q);
            cp_async_commit();
        }
        cp_async_wait<2>();
        bar_a();
        // stage-A window: own column's y_{m-1} at planes t-1, t, t+1 (slots 0, 1, 2 for t = i0-1)
        double2 au[3], ac[3], ad[3];
        if (warp < 7) {
            const int a0 = warp < 6 ? 3 * warp : 18;
#pragma unroll
            for (int r = 0; r < 3; r++) {
                if (warp < 6 || r == 0) {
                    const uint32_t c = (uint32_t)(a0 + r + 1) * RB1 + (uint32_t)((2 * lane + 2) * 8);
                    au[r] = lds2(b1 + c);
                    ac[r] = lds2(b1 + SL1 + c);
                    ad[r] = lds2(b1 + 2 * SL1 + c);
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < 2; r++) {
                if (lane + 32 * r < 2 * kB3R2R) {
                    const uint32_t c = b3_edge_c(lane + 32 * r);
                    au[r] = lds2(b1 + c);
                    ac[r] = lds2(b1 + SL1 + c);
                    ad[r] = lds2(b1 + 2 * SL1 + c);
                }
            }
        }
        int sc = 1;   // slot of plane t (both rings)
        for (int t = i0 - 1; t <= i1 + 1; t++) {
            cp_async_wait<1>();   // plane t+2 has landed (t+3 may be in flight)
            bar_a();
            const int si = sc == 0 ? 4 : sc - 1;   // slot of plane t-1 <- plane t+4
            if (t + 4 <= i1 + 3) issue(si);
            cp_async_commit();
            const int s2 = sc >= 3 ? sc - 3 : sc + 2;   // slot of plane t+2
            const uint32_t pc = b1 + (uint32_t)sc * SL1, pd2 = b1 + (uint32_t)s2 * SL1;
            const uint32_t pw = b2 + (uint32_t)sc * SL2;
            mbar_wait(emptyb + sc * 8, ((ph >> (8 + sc)) & 1) ^ 1);   // stage B released the slot's previous plane
            ph ^= 1u << (8 + sc);
            if (warp < 6) b3_stage_a<3>(S, C.alpha, C.ba, pc, pd2, pw, 3 * warp, lane, au, ac, ad);
            else if (warp == 6) b3_stage_a<1>(S, C.alpha, C.ba, pc, pd2, pw, 18, lane, au, ac, ad);
            else b3_stage_a_edge(S, C.alpha, C.ba, pc, pd2, pw, lane, au, ac, ad);
            mbar_arrive(fullb + sc * 8);
            sc = b3_inc(sc, kB3D);
        }
        cp_async_wait<0>();
        bar_a();   // the y_{m-1} ring is refilled by the next unit
    } else {
        const int wb = warp - 8;
        const uint32_t cbB = (uint32_t)(2 * wb) * RB2 + (uint32_t)((2 * lane + 2) * 8);   // R2 row 2 wb, pair lane
        const long long rstride = n2;
        long long off0 = ((long long)i0 * n1 + (j0 + 2 * wb)) * n2 + k0 + 2 * lane;   // plane s
        // planes i0-1, i0, i0+1 (slots 1, 2, 3): wait for them once here (each fill is waited exactly once)
#pragma unroll
        for (int q = 1; q <= 3; q++) {
            mbar_wait(fullb + q * 8, (ph >> q) & 1);
            ph ^= 1u << q;
        }
        // per-thread staging of the plane's p_{m-1} (or v) / rollback operand, one plane ahead (cp.async;
        // each thread reads only its own pieces, so its own wait_group orders them)
        const uint32_t pbase = b2 + (uint32_t)kB3D * SL2 + (uint32_t)(tid - 256) * 16;
        constexpr uint32_t PSL = (uint32_t)b3_np(K) * 4096;   // staging slot bytes
        auto stage_in = [&](long long off, uint32_t d) {
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const long long o = off + r * rstride;
                LX_DCHECK(o >= 0 && o + 2 <= (long long)n0 * plane, "stage B staging offset");
                if (FIRST || rbm)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + (uint32_t)((r * (K + 1) + K) * 4096)),
                                 "l"(src + o)
                                 : "memory");
#pragma unroll
                for (int k = 0; k < K; k++)
                    if (!FIRST && (((act | rbm) >> k) & 1))
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + (uint32_t)((r * (K + 1) + k) * 4096)),
                                     "l"(P.p[k] + o)
                                     : "memory");
            }
        };
        stage_in(off0, pbase);
        cp_async_commit();
        uint32_t pslot = 0;
        int sb = 1;   // slot of plane s-1
        for (int s = i0; s < i1; s++) {
            const int s0 = b3_inc(sb, kB3D), s1 = b3_inc(s0, kB3D), s2 = b3_inc(s1, kB3D);
            if (s + 1 < i1) stage_in(off0 + plane, pbase + (pslot ^ PSL));
            cp_async_commit();
            cp_async_wait<1>();   // this plane's pieces have landed
            mbar_wait(fullb + s2 * 8, (ph >> s2) & 1);   // y_m plane s+2 (and, in order, s-1 .. s+1)
            ph ^= 1u << s2;
            // slab: planes 0 .. 3 go to rank-1's ghost planes n .. n+3 (slots 2 .. 5), planes n-2, n-1 to
            // rank+1's ghost planes -2, -1 (slots 0, 1); x + off addresses the ghost copy of dst + off
            double* x1 = nullptr;
            double* x2 = nullptr;
            if (SLAB) {
                if (s < 4) x1 = xup + 2 * plane;
                if (s >= n0 - 2) x2 = xdn + (2 - (long long)n0) * plane;
                peer |= (x1 != nullptr) | (x2 != nullptr);
            }
            b3_stage_b<K, FIRST, SLAB>(P, C, dst, b2 + (uint32_t)sb * SL2, b2 + (uint32_t)s0 * SL2,
                                       b2 + (uint32_t)s1 * SL2, b2 + (uint32_t)s2 * SL2, cbB, off0, rstride, act,
                                       rbm, two, pbase + pslot, sums, x1, x2);
            mbar_arrive(emptyb + sb * 8);   // plane s-1: last read
            sb = s0;
            off0 += plane;
            pslot ^= PSL;
        }
        cp_async_wait<0>();
        // planes i1-1, i1, i1+1 are not read again
#pragma unroll
        for (int q = 0; q < 3; q++) {
            mbar_arrive(emptyb + sb * 8);
            sb = b3_inc(sb, kB3D);
        }
    }
}

// Deterministic reduction over the 16 warps of a k_leja3d_tb2 CTA (result in thread 0)
template <int N>
__device__ __forceinline__ void b3_block_reduce(double (&v)[N], double (*s_red)[kSlot]) {
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
            double x = s_red[0][i];
            for (int w = 1; w < kB3Warps; w++) x += s_red[w][i];
            v[i] = x;
        }
    }
    __syncthreads();
}

// Grid barrier + the decisions of iterations m and m+1 (last arriver); word [63:32] gen0 + q + 1,
// [31:24] status, [23:16] rollback mask, [15:8] done, [7:0] active.
// SLAB: every thread that stored ghost planes into a neighbour fences them system-wide before the CTA
// arrives; the last arriver exchanges the rank's partial sums with every rank (xrank_sum), which also
// makes the barrier global: no rank starts pass q+1 (which overwrites the ghost planes its neighbours
// read in pass q-1 ... and reads the ones they wrote in pass q) before every rank finished pass q.
template <int K, bool SLAB>
__device__ __forceinline__ void b3_barrier_decide(const LejaParams& P, int q, int m, bool two, unsigned gen0,
                                                  const B3Coef<K>& C, int active, double (*s_red)[kSlot], int* s_flags,
                                                  bool peer, unsigned long long key, int pslot) {
    constexpr int NV = 2 * (1 + K);
    const int tid = threadIdx.x;
    Ctrl* ctrl = P.ctrl;
    const int par = q & 1;
    if (SLAB && peer) __threadfence_system();
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
        for (int c = tid; c < (int)gridDim.x; c += kB3Threads) {
            const double* slot = P.partials + ((size_t)par * gridDim.x + c) * kSlot;
#pragma unroll
            for (int i = 0; i < NV; i++) acc[i] += __ldcg(slot + i);
        }
        b3_block_reduce<NV>(acc, s_red);
        if (tid == 0) {
            Record* rec = P.rec;
            int done = 0, status = 0, act = active;
            if (SLAB && xrank_sum<NV>(P, acc)) {   // a peer did not arrive: LX_ERR_TIMEOUT on this rank
                atomicExch(&rec->status, 10);
                done = 1;
                status = 10;
            }
            if (!done) leja_decide<K>(P, m, acc, C.da, act, done, status, rec);
            const int rb = (two && status != 6 && status != 10) ? (active & ~act) : 0;
            int fm = m;
            if (!done) {
                // a one-iteration pass (predicted final iteration) that did not end the call simply continues
                if (two) leja_decide<K>(P, m + 1, acc + 1 + K, C.db, act, done, status, rec);
                fm = m + 1;
            }
            if (done && status != 10) {   // remember the final iteration for the next call with these parameters
                Tb2Ctl* tc = P.tc;
                const int slot = pslot >= 0 ? pslot : (int)(tc->pnext++ % (unsigned)kTb2Pred);
                tc->pkey[slot] = key;
                tc->pfin[slot] = (unsigned)fm;
            }
            ctrl->arrive = 0u;
            const unsigned long long w = ((unsigned long long)(gen0 + (unsigned)q + 1u) << 32) |
                                         ((unsigned long long)(status & 0xff) << 24) |
                                         ((unsigned long long)(rb & 0xff) << 16) |
                                         ((unsigned long long)(done & 0xff) << 8) | (unsigned long long)(act & 0xff);
            st_release64(&ctrl->word, w);
            s_flags[1] = done;
            s_flags[2] = act;
            s_flags[3] = rb;
        }
    } else if (tid == 0) {
        unsigned long long w = ld_relaxed64(&ctrl->word);
        int spins = 0;
        while ((int)((unsigned)(w >> 32) - gen0) < q + 1) {
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
        s_flags[3] = (int)((w >> 16) & 0xff);
    }
    __syncthreads();
}

// Prologue of the slab kernel: this rank's boundary planes of v into the neighbours' ghost blocks (planes
// 0 .. 3 -> rank-1's planes n .. n+3, planes n-2, n-1 -> rank+1's planes -2, -1), then a global barrier
// (grid barrier + an empty cross-rank exchange) so that pass 0 reads complete ghosts.  Generation gen0+1.
__device__ __forceinline__ void b3_slab_prologue(const LejaParams& P, unsigned gen0, int* s_flags) {
    const long long plane = (long long)P.n1 * P.n2, half = plane / 2;
    const int n = P.n_loc;
    for (long long t = (long long)blockIdx.x * kB3Threads + threadIdx.x; t < 6 * half;
         t += (long long)gridDim.x * kB3Threads) {
        const int pr = (int)(t / half);
        const long long o = 2 * (t - pr * half);
        const int src = pr < 4 ? pr : n - 6 + pr;
        LX_DCHECK(src >= 0 && src < n && o + 2 <= plane, "slab prologue plane");
        double* g = pr < 4 ? P.hup_v + (2 + pr) * plane : P.hdn_v + (pr - 4) * plane;
        st2(g + o, ld2(P.v.base + src * plane + o));
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        Ctrl* ctrl = P.ctrl;
        const unsigned t = atom_add_acq_rel(&ctrl->arrive, 1u);
        if (t == gridDim.x - 1) {
            double none[1] = {0.0};
            const int st = xrank_sum<0>(P, none);
            if (st) atomicExch(&P.rec->status, 10);
            ctrl->arrive = 0u;
            st_release64(&ctrl->word, ((unsigned long long)(gen0 + 1u) << 32) | (st ? (1ull << 8) : 0ull));
            s_flags[1] = st != 0;
        } else {
            unsigned long long w = ld_relaxed64(&ctrl->word);
            const unsigned long long t0 = globaltimer_ns();
            while ((int)((unsigned)(w >> 32) - gen0) < 1) {
                __nanosleep(32);
                if (globaltimer_ns() - t0 > P.timeout_ns + 1000000000ull) {
                    atomicExch(&P.rec->status, 10);
                    w = (1ull << 8);
                    break;
                }
                w = ld_relaxed64(&ctrl->word);
            }
            fence_acquire();
            s_flags[1] = (int)((w >> 8) & 0xff);
        }
    }
    __syncthreads();
}

template <int K, bool SLAB>
__global__ void __launch_bounds__(kB3Threads, 1) k_leja3d_tb2(const __grid_constant__ LejaParams P) {
    __shared__ double s_red[kB3Warps][kSlot];
    __shared__ int s_flags[4];
    extern __shared__ double b3_ring[];
    __shared__ __align__(8) unsigned long long s_bar[2 * kB3D];   // y_m ring: full[5], empty[5]
    double* r1 = b3_ring;
    double* r2 = b3_ring + kB3D * kB3R1P;
    const int tid = threadIdx.x;
    const uint32_t bars = smem_u32(s_bar);
    unsigned ph = 0;   // bits 0..4: full-barrier parities (stage B), 8..12: empty-barrier parities (stage A)
    if (tid == 0) {
        for (int q = 0; q < 2 * kB3D; q++) mbar_init(bars + q * 8, 256);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned gen0 = 0;
    if (tid == 0) gen0 = (unsigned)(ld_acquire64(&P.ctrl->word) >> 32);
    // final iteration of the last call with the same parameters (Tb2Ctl prediction table): a pass whose
    // FIRST iteration is predicted to end the call performs only that iteration (stage B then stores y_m,
    // not y_{m+1}), so a correct prediction needs no rollback; a wrong one continues at m + 1 next pass
    unsigned long long key = 0;
    __shared__ int s_pred[2];
    if (tid == 0) {
        key = tb2_call_key<K>(P);
        int fp = -1, ps = -1;
        for (int i = 0; i < kTb2Pred; i++)
            if (P.tc->pkey[i] == key) {
                fp = (int)P.tc->pfin[i];
                ps = i;
            }
        s_pred[0] = fp;
        s_pred[1] = ps;
    }
    if (SLAB) {
        b3_slab_prologue(P, gen0, s_flags);   // (syncs the block: s_pred visible)
        if (s_flags[1]) return;   // a peer never arrived (LX_ERR_TIMEOUT recorded)
        gen0 += 1u;
    }
    __syncthreads();
    const int fpred = s_pred[0], pslot = s_pred[1];
    int active = P.active0, rbm = 0;
    const int M = P.max_nodes;
    const int ncu = (P.n1 / kB3J) * (P.n2 >> 6) * ((P.n_loc + kTI3 - 1) / kTI3);
    // per-pass coefficients in shared memory (broadcast reads; registers are the scarce resource)
    __shared__ B3Coef<K> C;
    if (tid == 0) {
        C.alpha = P_alpha(P);
        for (int k = 0; k < K; k++) {
            C.d0[k] = P.table[1 + k];
            C.dr[k] = 0.0;
        }
    }
    int m = 1;   // first iteration of pass q
    for (int q = 0;; q++) {
        const bool two = m + 1 < M && m != fpred;
        if (tid == 0) {
            C.ba = coef_beta(P, m);
            C.bb = two ? coef_beta(P, m + 1) : 0.0;
            for (int k = 0; k < K; k++) {
                C.dr[k] = q ? C.db[k] : 0.0;
                C.da[k] = P.table[(size_t)m * (1 + K) + 1 + k];
                C.db[k] = two ? P.table[(size_t)(m + 1) * (1 + K) + 1 + k] : 0.0;
            }
        }
        __syncthreads();
        double sums[2 * (1 + K)];
#pragma unroll
        for (int i = 0; i < 2 * (1 + K); i++) sums[i] = 0.0;
        double* dst = P.ydst[q & 1];
        bool peer = false;
        // slab: y_{m-1}'s ghost planes (this rank's block) and the neighbours' ghost blocks of y_{m+1}
        const double* gsrc = SLAB ? (q == 0 ? P.gv : P.gy[(q - 1) & 1]) : nullptr;
        double* xup = SLAB ? P.hup[q & 1] : nullptr;
        double* xdn = SLAB ? P.hdn[q & 1] : nullptr;
        if (q == 0) {
            for (int cu = blockIdx.x; cu < ncu; cu += gridDim.x)
                b3_unit<K, true, SLAB>(P, P.v.base, dst, cu, r1, r2, bars, ph, C, active, 0, two, sums, gsrc, xup,
                                       xdn, peer);
        } else {
            const double* src = P.ydst[(q - 1) & 1];
            for (int cu = blockIdx.x; cu < ncu; cu += gridDim.x)
                b3_unit<K, false, SLAB>(P, src, dst, cu, r1, r2, bars, ph, C, active, rbm, two, sums, gsrc, xup,
                                        xdn, peer);
        }
        b3_block_reduce<2 * (1 + K)>(sums, s_red);
        if (tid == 0) {
            double* slot = P.partials + ((size_t)(q & 1) * gridDim.x + blockIdx.x) * kSlot;
#pragma unroll
            for (int i = 0; i < 2 * (1 + K); i++) slot[i] = sums[i];
        }
        b3_barrier_decide<K, SLAB>(P, q, m, two, gen0, C, active, s_red, s_flags, peer, key, pslot);
        active = s_flags[2];
        rbm = s_flags[3];
        if (s_flags[1]) {
            // end of the call: roll back accumulators that converged at m (p holds one term too many)
            if (rbm) {
                const size_t npair = (size_t)P.n_loc * P.n1 * P.n2 / 2;
                for (size_t i = (size_t)blockIdx.x * kB3Threads + tid; i < npair; i += (size_t)gridDim.x * kB3Threads) {
                    const double2 y = ld2(dst + 2 * i);
#pragma unroll
                    for (int k = 0; k < K; k++) {
                        if ((rbm >> k) & 1) {
                            double2 p = ld2(P.p[k] + 2 * i);
                            p.x = fma(-C.db[k], y.x, p.x);
                            p.y = fma(-C.db[k], y.y, p.y);
                            st2(P.p[k] + 2 * i, p);
                        }
                    }
                }
            }
            break;
        }
        m += two ? 2 : 1;
    }
}

static void* leja3d_tb2_ptr(int K, bool slab) {
    if (slab) {
        switch (K) {
            case 1: return (void*)k_leja3d_tb2<1, true>;
            case 2: return (void*)k_leja3d_tb2<2, true>;
            case 3: return (void*)k_leja3d_tb2<3, true>;
            case 4: return (void*)k_leja3d_tb2<4, true>;
        }
        return nullptr;
    }
    switch (K) {
        case 1: return (void*)k_leja3d_tb2<1, false>;
        case 2: return (void*)k_leja3d_tb2<2, false>;
        case 3: return (void*)k_leja3d_tb2<3, false>;
        case 4: return (void*)k_leja3d_tb2<4, false>;
    }
    return nullptr;
}

int leja3d_tb2_grid_size(int device, int K, int ncu, bool slab) {
    void* kern = leja3d_tb2_ptr(K, slab);
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
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, b3_smem(K));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kB3Threads, b3_smem(K));
        g = nsm * (per < 1 ? 1 : per);
        cache[{device, kern}] = g;
    }
    return g < ncu ? g : ncu;
}

cudaError_t launch_leja3d_tb2(const LejaParams& P, cudaStream_t s, bool slab) {
    void* kern = leja3d_tb2_ptr(P.K, slab);
    if (!kern) return cudaErrorInvalidValue;
    void* args[] = {(void*)&P};
    return cudaLaunchCooperativeKernel(kern, dim3(P.grid), dim3(kB3Threads), args, b3_smem(P.K), s);
}

cudaError_t preload_3d() {
    {
        cudaFuncAttributes a;
        if (cudaFuncGetAttributes(&a, (const void*)k_rhs3d_smem) != cudaSuccess) return cudaGetLastError();
    }
    for (int K = 1; K <= kMaxK; K++) {
        cudaFuncAttributes a;
        for (int sl = 0; sl < 2; sl++)
            if (cudaFuncGetAttributes(&a, leja3d_tb2_ptr(K, sl != 0)) != cudaSuccess) return cudaGetLastError();
        for (int d = 0; d < 2; d++)
            if (cudaFuncGetAttributes(&a, leja3d_smem_ptr(K, d != 0)) != cudaSuccess) return cudaGetLastError();
    }
    return cudaSuccess;
}

}  // namespace lx
