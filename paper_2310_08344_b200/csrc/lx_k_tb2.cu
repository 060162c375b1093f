// lx_k_tb2.cu -- the two-iterations-per-pass Leja kernel (k_leja2d_tb2) and its
// slab-decomposed instantiation over peer memory (SLAB).
#include "lx_dev.cuh"

namespace lx {

// ===========================================================================
// Temporal blocking: TWO Leja iterations per HBM pass.
//   pass (m, m+1): read y_{m-1}, p_{m-1};  y_m is formed in registers on a
//   widened halo (rows i0-1 .. i0+RT+1, columns j0-2 .. j0+61 of a 64-column
//   warp window whose 60 inner columns are outputs);  y_{m+1} and p_{m+1} are
//   written.  -> 32 B/pt per TWO iterations (16 B/pt per iteration) and one grid
//   barrier per two iterations.  Both iterations' norms are reduced, and the
//   stopping rule of P:155 is applied to m and then m+1 exactly as in the
//   one-step kernel (same decisions, same iteration counts).  If an accumulator
//   converges at the first iteration of a pass, its p_{m+1} is rolled back to
//   p_m = p_{m+1} - d_{m+1} y_{m+1} (<= 1 ulp from the one-step value) in the
//   next pass, or in a final pointwise pass when the call ends.
// ===========================================================================
// Shared-memory staging of the two-step kernel: per warp a ring of tb2_depth stages, one stage =
// the global rows one chunk consumes (16 B per lane per row, lane-private: every lane reads back only
// what its own cp.async wrote -> no warp synchronisation needed):
//   y_{m-1} rows i0+4 .. i0+RT+3 | halo pair of lane 31 for rows i0+2 .. i0+RT+1 |
//   p_k rows i0 .. i0+RT-1 (k < K) | u rows i0+2 .. i0+RT+1 (DIAG)
template <int K, bool DIAG>
struct Tb2Stage {
    static constexpr int RT = tb2_rt(K);
    static constexpr int Y = 0;
    static constexpr int H = RT * 32;
    static constexpr int PP = H + RT;
    static constexpr int U = PP + RT * K * 32;
    static constexpr int SIZE = U + (DIAG ? RT * 32 : 0);          // double2 per stage
    static constexpr int DEPTH = tb2_depth(K, DIAG);
    static constexpr int WARP = SIZE * DEPTH;                        // double2 per warp
};

// Row pointer of the two-step kernel: rows [0, n) of a local array; rows -2, -1, n .. n+3 by periodic
// wrap (single domain) or, in the slab kernel (SLAB), from the 6-row ghost block g (rows -2, -1, n,
// n+1, n+2, n+3), which the neighbouring ranks fill through peer memory.
template <bool SLAB>
__device__ __forceinline__ const double* tb2_row(const double* base, const double* g, int r, int n, int n1) {
    if (SLAB && (unsigned)r >= (unsigned)n) return g + (size_t)(r < 0 ? r + 2 : r - n + 2) * n1;
    return base + (size_t)(r < 0 ? r + n : (r >= n ? r - n : r)) * n1;
}

// Per-pass sources / destinations of the two-step kernel
struct Tb2Pass {
    const double* src;    // y_{m-1} (v on the first pass)
    const double* gsrc;   // its ghost block (SLAB)
    const double* gu;     // ghost block of u (SLAB, DIAG)
    double* dst;          // y_{m+1}
    double* hup;          // SLAB: ghost block of rank-1 receiving rows 0..3 of y_{m+1} (its rows n..n+3)
    double* hdn;          // SLAB: ghost block of rank+1 receiving rows n-2, n-1 (its rows -2, -1)
};

// stage the global rows of chunk ci into ring stage st (every lane: its own 16-byte pieces)
template <int K, bool DIAG, bool FIRST, bool SLAB>
__device__ __forceinline__ void tb2_issue(const LejaParams& P, const Tb2Pass& T, double2* __restrict__ ring, int ci,
                                          int st, int lane, int active, int rbmask) {
    using L = Tb2Stage<K, DIAG>;
    constexpr int RT = L::RT;
    constexpr int KK = K > 0 ? K : 1;
    const int n1 = P.n1, n = P.n_loc, nc = P.nrb;
    auto wrap = [n](int r) { return r < 0 ? r + n : (r >= n ? r - n : r); };
    auto colw = [n1](int c) { return c < 0 ? c + n1 : (c >= n1 ? c - n1 : c); };
    const int b = ci / nc;
    const int i0 = (ci - b * nc) * RT;
    const int jraw = b * kBand2 - 2 + 2 * lane;
    const int j = colw(jraw);
    double2* sg = ring + st * L::SIZE;
#pragma unroll
    for (int q = 0; q < RT; q++) {
        cp_async16(sg + L::Y + q * 32 + lane, tb2_row<SLAB>(T.src, T.gsrc, i0 + 4 + q, n, n1) + j);
        if (lane == 31) cp_async16(sg + L::H + q, tb2_row<SLAB>(T.src, T.gsrc, i0 + 2 + q, n, n1) + colw(jraw + 2));
        if (DIAG) cp_async16(sg + L::U + q * 32 + lane, tb2_row<SLAB>(P.u, T.gu, i0 + 2 + q, n, n1) + j);
    }
#pragma unroll
    for (int t = 0; t < RT; t++) {
#pragma unroll
        for (int k = 0; k < KK; k++) {
            const bool need = ((active >> k) & 1) ? !FIRST : (K > 1 && ((rbmask >> k) & 1));
            if (need) cp_async16(sg + L::PP + (t * K + k) * 32 + lane, P.p[k] + (size_t)wrap(i0 + t) * n1 + j);
        }
    }
}

// Temporally blocked pass over a contiguous range [cbeg, cend) of (band, chunk) work items in
// band-major order (chunk = RT rows of a 60-column band).  A warp marches down its rows with
// register windows: y_{m-1} rows [i0, i0+RT+4), y_m rows [i0-1, i0+RT+2), u rows [i0, i0+RT+2);
// per chunk it consumes RT new rows of y_{m-1} (and p, u) staged DEPTH-1 chunks ahead by
// cp.async, forms RT new rows of y_m (the 3-row halo recomputation happens only at a strip start)
// and writes RT rows of y_{m+1} and p_{m+1}.  Lanes 1..30 own the band's 60 output columns;
// lanes 0 and 31 carry halo columns.  Requires n_loc >= 16, n1 >= 64 (host-checked).
// SLAB: rows 0..3 and n-2, n-1 of y_{m+1} are also stored into the neighbours' ghost blocks (peer
// memory: the halo exchange overlaps the rest of the pass), followed by a system-scope fence.
template <int K, bool DIAG, bool FIRST, bool TWO, bool SLAB>
__device__ __forceinline__ void strip2d_tb2(const LejaParams& P, const Tb2Pass& T, int cbeg, int cend, int lane,
                                            double alpha, double b1, double b2, const double* d0, const double* da,
                                            const double* db, int active, int rbmask, const double* rbd,
                                            double (&acc)[2 * (1 + K)], double2* __restrict__ ring) {
    using L = Tb2Stage<K, DIAG>;
    constexpr int RT = L::RT, D = L::DEPTH;
    const int n1 = P.n1, n = P.n_loc, nc = P.nrb;
    const Stencil& S = P.st;
    auto colw = [n1](int c) { return c < 0 ? c + n1 : (c >= n1 ? c - n1 : c); };
    constexpr int KK = K > 0 ? K : 1;
    double2 aw[RT + 4], yw[RT + 3], uw[RT + 2];
    const double2 z2 = make_double2(0.0, 0.0);
    // prime the ring: chunks cbeg .. cbeg+D-2
#pragma unroll
    for (int d = 0; d < D - 1; d++) {
        if (cbeg + d < cend) tb2_issue<K, DIAG, FIRST, SLAB>(P, T, ring, cbeg + d, d, lane, active, rbmask);
        cp_async_commit();
    }
    int ci = cbeg, st = 0;
#pragma unroll 1
    while (ci < cend) {
        const int b = ci / nc;
        const int cseg = min(cend, (b + 1) * nc);   // this band's part of the range
        const int c0 = b * kBand2;
        const int jraw = c0 - 2 + 2 * lane;
        const int j = colw(jraw);
        const int jh = colw(jraw + 2);
        const bool outl = lane >= 1 && lane <= 30 && jraw < n1 && jraw < c0 + kBand2;
        {
            // strip start: y_{m-1} rows i0-2 .. i0+3 (direct loads), y_m rows i0-1 .. i0+1
            const int i0 = (ci - b * nc) * RT;
            double2 t6[6], h3[3], u3[3];
#pragma unroll
            for (int q = 0; q < 6; q++) t6[q] = ld2(tb2_row<SLAB>(T.src, T.gsrc, i0 - 2 + q, n, n1) + j);
#pragma unroll
            for (int q = 0; q < 3; q++) {
                h3[q] = (lane == 31) ? ld2(tb2_row<SLAB>(T.src, T.gsrc, i0 - 1 + q, n, n1) + jh) : z2;
                u3[q] = DIAG ? ldg2(tb2_row<SLAB>(P.u, T.gu, i0 - 1 + q, n, n1) + j) : z2;
            }
#pragma unroll
            for (int q = 0; q < 3; q++)
                yw[q] = leja_row<DIAG>(S, alpha, b1, t6[q], t6[q + 1], t6[q + 2], t6[q + 3], h3[q], u3[q], lane);
#pragma unroll
            for (int q = 0; q < 4; q++) aw[q] = t6[q + 2];
            uw[0] = u3[1];
            uw[1] = u3[2];
        }
#pragma unroll 1
        for (int i0 = (ci - b * nc) * RT; ci < cseg; ci++, i0 += RT) {
            // keep D-1 chunks in flight: stage chunk ci+D-1, then wait for chunk ci's group
            {
                int sn = st + D - 1;
                if (sn >= D) sn -= D;
                if (ci + D - 1 < cend) tb2_issue<K, DIAG, FIRST, SLAB>(P, T, ring, ci + D - 1, sn, lane, active, rbmask);
                cp_async_commit();
                cp_async_wait<D - 1>();
            }
            // shared-space loads (ld.shared, not generic): 32-bit address of this stage
            const uint32_t sgb = smem_u32(ring) + (uint32_t)(st * L::SIZE) * 16u;
            auto sg = [sgb](int i) { return lds2(sgb + (uint32_t)i * 16u); };
            if (++st == D) st = 0;
            const int nout = min(RT, n - i0);
            double2 ah[RT];
#pragma unroll
            for (int q = 0; q < RT; q++) {
                aw[4 + q] = sg(L::Y + q * 32 + lane);
                ah[q] = (lane == 31) ? sg(L::H + q) : z2;
                if (DIAG) uw[2 + q] = sg(L::U + q * 32 + lane);
            }
            // step 1: y_m rows i0+2 .. i0+RT+1
#pragma unroll
            for (int q = 0; q < RT; q++)
                yw[3 + q] = leja_row<DIAG>(S, alpha, b1, aw[1 + q], aw[2 + q], aw[3 + q], aw[4 + q], ah[q],
                                           DIAG ? uw[2 + q] : z2, lane);
            // step 2: y_{m+1} on the output rows; p updates and norms
#pragma unroll
            for (int t = 0; t < RT; t++) {
                if (t < nout) {
                    const double2 yc = yw[t + 1];
                    double2 zz = yc;
                    if (TWO) zz = leja_row<DIAG>(S, alpha, b2, yw[t], yc, yw[t + 2], yw[t + 3], z2, uw[t], lane);
                    if (outl) {
                        const size_t off = (size_t)(i0 + t) * n1 + j;
                        st2(T.dst + off, zz);
                        acc[0] = fma(yc.y, yc.y, fma(yc.x, yc.x, acc[0]));
                        if (TWO) acc[1 + K] = fma(zz.y, zz.y, fma(zz.x, zz.x, acc[1 + K]));
                        const double2 yprev = aw[t];   // y_{m-1} (= v on the first pass)
#pragma unroll
                        for (int k = 0; k < KK; k++) {
                            if ((active >> k) & 1) {
                                double2 pm;
                                if (FIRST) {
                                    pm.x = fma(da[k], yc.x, d0[k] * yprev.x);
                                    pm.y = fma(da[k], yc.y, d0[k] * yprev.y);
                                } else {
                                    const double2 pv = sg(L::PP + (t * K + k) * 32 + lane);
                                    pm.x = fma(da[k], yc.x, pv.x);
                                    pm.y = fma(da[k], yc.y, pv.y);
                                }
                                acc[1 + k] = fma(pm.y, pm.y, fma(pm.x, pm.x, acc[1 + k]));
                                double2 pn = pm;
                                if (TWO) {
                                    pn.x = fma(db[k], zz.x, pm.x);
                                    pn.y = fma(db[k], zz.y, pm.y);
                                    acc[2 + K + k] = fma(pn.y, pn.y, fma(pn.x, pn.x, acc[2 + K + k]));
                                }
                                st2(P.p[k] + off, pn);
                            } else if (K > 1 && ((rbmask >> k) & 1)) {
                                // roll back the speculative last update of the previous pass (K = 1: the
                                // call ends at that decision -> final rollback pass instead)
                                const double2 pv = sg(L::PP + (t * K + k) * 32 + lane);
                                st2(P.p[k] + off, make_double2(fma(-rbd[k], yprev.x, pv.x),
                                                               fma(-rbd[k], yprev.y, pv.y)));
                            }
                        }
                    }
                }
            }
            // advance the windows by RT rows
#pragma unroll
            for (int q = 0; q < 4; q++) aw[q] = aw[RT + q];
#pragma unroll
            for (int q = 0; q < 3; q++) yw[q] = yw[RT + q];
#pragma unroll
            for (int q = 0; q < 2; q++) uw[q] = uw[RT + q];
        }
    }
    cp_async_wait<0>();
    if (SLAB) {
        // boundary rows 0..3 / n-2, n-1 of y_{m+1} this strip wrote -> the neighbours' ghost blocks (peer
        // stores of rows this warp just stored itself: L2 hits), then a system-scope fence so they are
        // visible before this CTA's barrier arrival (outside the streaming loop: no per-row branches there)
        const int b = cbeg / nc;
        const int r0 = (cbeg - b * nc) * RT, r1 = min(n, (cend - b * nc) * RT);
        const int jraw = b * kBand2 - 2 + 2 * lane;
        const bool outl = lane >= 1 && lane <= 30 && jraw < n1 && jraw < b * kBand2 + kBand2;
        bool halo = false;
        for (int r = r0; r < r1; r++) {
            if (r >= 4 && r < n - 2) {
                r = n - 3;   // skip to the last two rows
                continue;
            }
            if (outl) {
                const double2 v = ld2(T.dst + (size_t)r * n1 + jraw);
                st2((r < 4 ? T.hup + (size_t)(2 + r) * n1 : T.hdn + (size_t)(r - n + 2) * n1) + jraw, v);
            }
            halo = true;
        }
        if (halo) __threadfence_system();
    }
}

// the four (first pass, two iterations) instantiations of strip2d_tb2
template <int K, bool DIAG, bool SLAB>
__device__ __forceinline__ void tb2_strip(const LejaParams& P, bool first, bool two, const Tb2Pass& T, int c_b,
                                          int c_e, int lane, double alpha, double b1, double b2, const double* d0,
                                          const double* da, const double* db, int active, int rbmask,
                                          const double* rbd, double (&acc)[2 * (1 + K)], double2* __restrict__ ring) {
    if (first) {
        if (two) strip2d_tb2<K, DIAG, true, true, SLAB>(P, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active,
                                                       rbmask, rbd, acc, ring);
        else strip2d_tb2<K, DIAG, true, false, SLAB>(P, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active,
                                                     rbmask, rbd, acc, ring);
    } else {
        if (two) strip2d_tb2<K, DIAG, false, true, SLAB>(P, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active,
                                                        rbmask, rbd, acc, ring);
        else strip2d_tb2<K, DIAG, false, false, SLAB>(P, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active,
                                                      rbmask, rbd, acc, ring);
    }
}

// Final rollback pass: p_k -= rbd[k] * y (y = the last written y_{m+1}) on the strip's output points.
template <int K, int RT>
__device__ __forceinline__ void strip2d_tb2_rollback(const LejaParams& P, const double* y, int cbeg, int cend,
                                                     int lane, int rbmask, const double* rbd) {
    const int n1 = P.n1, n = P.n_loc, nc = P.nrb;
    for (int ci = cbeg; ci < cend; ci++) {
        const int b = ci / nc, ic = ci - b * nc;
        const int c0 = b * kBand2;
        const int jraw = c0 - 2 + 2 * lane;
        if (!(lane >= 1 && lane <= 30 && jraw < n1 && jraw < c0 + kBand2)) continue;
        const int i0 = ic * RT;
        const int nout = min(RT, n - i0);
        for (int t = 0; t < nout; t++) {
            const size_t off = (size_t)(i0 + t) * n1 + jraw;
            const double2 yy = ld2(y + off);
#pragma unroll
            for (int k = 0; k < K; k++) {
                if ((rbmask >> k) & 1) {
                    const double2 pp = ld2(P.p[k] + off);
                    st2(P.p[k] + off, make_double2(fma(-rbd[k], yy.x, pp.x), fma(-rbd[k], yy.y, pp.y)));
                }
            }
        }
    }
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

// grid barrier + decisions of iterations m (and m+1): flags[1] done, [2] active, [3] rollback mask.
// g = generation offset of this barrier within the call (waiters release at gen0 + g).
template <int K, bool SLAB>
__device__ __forceinline__ void barrier_decide_tb2(const LejaParams& P, int m, int g, bool two, unsigned gen0,
                                                   const double* da, const double* db, int active,
                                                   double (*s_red)[kSlot], int* s_flags) {
    constexpr int NV = 2 * (1 + K);
    const int tid = threadIdx.x;
    Ctrl* ctrl = P.ctrl;
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
        for (int gi = tid; gi < P.ngrp; gi += kThreads) {
#pragma unroll
            for (int i = 0; i < NV; i++) acc[i] += __ldcg(P.grp_part + (size_t)gi * NV + i);
        }
        block_reduce<NV>(acc, s_red);
        if (tid == 0) {
            int act = active, done = 0, status = 0;
            if (SLAB && m == 0) {   // the call's first barrier: ghost rows of v (and u) are in place
                status = xrank_sum<0>(P, acc);
                done = status != 0;
            } else {
                if (SLAB) status = xrank_sum<NV>(P, acc);
                if (status) {
                    done = 1;
                } else {
                    leja_decide<K>(P, m, acc, da, act, done, status, P.rec);
                }
            }
            if (status == 10) atomicExch(&P.rec->status, 10);
            const int rb = (m > 0) ? (active & ~act) : 0;   // converged at the first iteration of a pass -> roll back
            if (m > 0 && !done && two) leja_decide<K>(P, m + 1, acc + 1 + K, db, act, done, status, P.rec);
            ctrl->arrive = 0u;
            if (m > 0) {
                const int pass = (m - 1) >> 1;
                ctrl->work[(pass + 1) & 1] = 0u;     // segment counter of the next pass
                if (done) ctrl->work[pass & 1] = 0u;  // ... and of this one for the next call
            } else if (done) {
                ctrl->work[0] = 0u;
            }
            const unsigned long long w = ((unsigned long long)(gen0 + (unsigned)g) << 32) |
                                         ((unsigned long long)(status & 0xff) << 16) |
                                         ((unsigned long long)(rb & 0xf) << 12) |
                                         ((unsigned long long)(done & 0xf) << 8) | (unsigned long long)(act & 0xff);
            st_release64(&ctrl->word, w);
            s_flags[1] = done;
            s_flags[2] = act;
            s_flags[3] = two ? rb : 0;
        }
    } else if (tid == 0) {
        // waiters: time-based watchdog, longer than the last arriver's cross-rank limit (SLAB)
        const unsigned long long limit = (SLAB ? P.timeout_ns : 0ull) + 10000000000ull;
        const unsigned long long t0 = globaltimer_ns();
        unsigned long long w = ld_relaxed64(&ctrl->word);
        int spins = 0;
        while ((int)((unsigned)(w >> 32) - gen0) < g) {
            if (++spins > 4096) {
                __nanosleep(32);
                if ((spins & 1023) == 0 && globaltimer_ns() - t0 > limit) {
                    atomicExch(&P.rec->status, 10);
                    w = (1ull << 8);
                    break;
                }
            }
            w = ld_relaxed64(&ctrl->word);
        }
        fence_acquire();
        s_flags[1] = (int)((w >> 8) & 0xf);
        s_flags[2] = (int)(w & 0xff);
        s_flags[3] = two ? (int)((w >> 12) & 0xf) : 0;
    }
    __syncthreads();
}

template <int K>
__device__ __forceinline__ void coef_first5(const LejaParams& P, int k, double* d) {
    // d_0..d_4 of accumulator k by lane 0 of the warp (column form, explicitly rounded), broadcast
    const int M = P.max_nodes;
    double e[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int jj = 0; jj < 5; jj++) {
            if (jj < M) {
                double v = coef_h(P, k, jj);
#pragma unroll
                for (int i = 0; i < jj; i++) v = dd_step(v, e[i], P.R[(size_t)i * M + jj]);
                e[jj] = v;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 5; i++) d[i] = __shfl_sync(0xffffffffu, e[i], 0);
}

// Two Leja iterations per HBM pass.  SLAB = the slab-decomposed variant:
// one persistent kernel per Leja call and rank; the halo rows travel through peer memory from inside
// the pass (tb2 strip), the norm partials through the exchange headers at the grid barrier
// (xrank_sum); no host round trip, no NCCL call and no extra launch per iteration.
template <int K, bool DIAG, bool SLAB>
__global__ void __launch_bounds__(kThreads, 2) k_leja2d_tb2(const __grid_constant__ LejaParams P) {
    __shared__ double s_red[kWarps][kSlot];
    extern __shared__ double2 tb2_ring[];
    __shared__ int s_flags[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool cwarp = (blockIdx.x == 0 && warp == 0);
    const int gw = blockIdx.x * kWarps + warp - 1;
    const int W = gridDim.x * kWarps - 1;
    constexpr int RT = tb2_rt(K);
    constexpr int NV = 2 * (1 + K);
    double2* ring = tb2_ring + (size_t)warp * Tb2Stage<K, DIAG>::WARP;
    const int cbeg = cwarp ? 0 : (int)((long long)gw * P.nunits / W);
    const int cend = cwarp ? 0 : (int)((long long)(gw + 1) * P.nunits / W);
    unsigned gen0 = 0;
    if (tid == 0) gen0 = (unsigned)(ld_acquire64(&P.ctrl->word) >> 32);
    int active = P.active0, rbmask = 0;
    const int M = P.max_nodes;
    const double alpha = P_alpha(P);
    const int n = P.n_loc, n1 = P.n1;
    if (SLAB) {
        // halo rows of v (and u) into the neighbours' ghost blocks, then the call's first cross-rank barrier
        const long long tot = 6LL * n1;
        for (long long x = (long long)blockIdx.x * kThreads + tid; x < tot; x += (long long)gridDim.x * kThreads) {
            const int r = (int)(x / n1), j = (int)(x - (long long)r * n1);
            const int sr = r < 4 ? r : n - 6 + r;                // rows 0..3 -> rank-1, rows n-2, n-1 -> rank+1
            double* gv = r < 4 ? P.hup_v + (size_t)(2 + r) * n1 : P.hdn_v + (size_t)(r - 4) * n1;
            gv[j] = P.v.base[(size_t)sr * n1 + j];
            if (DIAG) {
                double* gu = r < 4 ? P.hup_u + (size_t)(2 + r) * n1 : P.hdn_u + (size_t)(r - 4) * n1;
                gu[j] = P.u[(size_t)sr * n1 + j];
            }
        }
        __threadfence_system();
        barrier_decide_tb2<K, true>(P, 0, 1, false, gen0, nullptr, nullptr, active, s_red, s_flags);
        if (s_flags[1]) return;   // peer timeout
    }
    double dd[K][5];
#pragma unroll
    for (int k = 0; k < K; k++) coef_first5<K>(P, k, dd[k]);
    if (cwarp && P.coef_gen) {
        for (int r = 0; r < 5 && r < M; r++) {
            double row[K];
#pragma unroll
            for (int k = 0; k < K; k++) row[k] = dd[k][r];
            coef_write_row<K>(P, r, lane, active, row);
        }
    }
    double d0[K], da[K], db[K], rbd[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        d0[k] = dd[k][0];
        da[k] = dd[k][1];
        db[k] = dd[k][2];
        rbd[k] = 0.0;
    }
    double na[K], nb[K];   // rows m+2, m+3 (rows 3, 4 from the prologue for the first pass)
#pragma unroll
    for (int k = 0; k < K; k++) {
        na[k] = dd[k][3];
        nb[k] = dd[k][4];
    }
    int m = 1;
    double nb1 = coef_beta(P, 1), nb2 = (2 < M) ? coef_beta(P, 2) : 0.0;
    for (; m < M; m += 2) {
        const bool two = (m + 1 < M);
        const double b1 = nb1, b2 = two ? nb2 : 0.0;
        // next pass's shifts (constant inputs): loaded now, off the post-barrier critical path
        nb1 = (m + 2 < M) ? coef_beta(P, m + 2) : 0.0;
        nb2 = (m + 3 < M) ? coef_beta(P, m + 3) : 0.0;
        const int pass = (m - 1) >> 1;
        double acc[NV];
#pragma unroll
        for (int i = 0; i < NV; i++) acc[i] = 0.0;
        if (cwarp) {
            if (P.coef_gen) {
                if (m + 4 < M) coef_write_row<K>(P, m + 4, lane, active, nullptr);
                if (m + 5 < M) coef_write_row<K>(P, m + 5, lane, active, nullptr);
            }
        } else {
            Tb2Pass T;
            T.src = (m == 1) ? P.v.base : P.ydst[(pass & 1) ^ 1];
            T.gsrc = (m == 1) ? P.gv : P.gy[(pass & 1) ^ 1];
            T.gu = P.gu;
            T.dst = P.ydst[pass & 1];
            T.hup = P.hup[pass & 1];
            T.hdn = P.hdn[pass & 1];
            // dynamic segments of P.seg chunks, band fastest (adjacent bands of the same rows run together;
            // the dynamic schedule balances the end-of-pass tail).  The norm partials stay deterministic:
            // each segment's sums are formed by one warp in a fixed order and stored by segment index; the
            // last finisher of each group of 32 segments sums the group in index order (fixed butterfly);
            // the barrier sums the groups in order.
            unsigned* ctr = &P.ctrl->work[pass & 1];
#pragma unroll 1
            for (;;) {
                int sg = 0;
                if (lane == 0) sg = (int)atomicAdd(ctr, 1u);
                sg = __shfl_sync(FULL_MASK, sg, 0);
                if (sg >= P.nseg) break;
                const int rs = sg / P.nb, b = sg - rs * P.nb;
                const int c_b = b * P.nrb + rs * P.seg;
                const int c_e = b * P.nrb + min(P.nrb, rs * P.seg + P.seg);
#pragma unroll
                for (int i = 0; i < NV; i++) acc[i] = 0.0;
                tb2_strip<K, DIAG, SLAB>(P, m == 1, two, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active, rbmask,
                                         rbd, acc, ring);
                double sacc[NV];
#pragma unroll
                for (int i = 0; i < NV; i++) sacc[i] = acc[i];
                warp_sum<NV>(sacc);
                int last = 0;
                const int g = sg >> 5;
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < NV; i++) P.seg_part[(size_t)sg * NV + i] = sacc[i];
                    __threadfence();
                    const unsigned t = atomicAdd(&P.grp_cnt[g], 1u);
                    last = (int)(t == (unsigned)(min(32, P.nseg - g * 32) - 1));
                }
                last = __shfl_sync(FULL_MASK, last, 0);
                if (last) {
                    __threadfence();
                    const int s2 = g * 32 + lane;
                    double gv[NV];
#pragma unroll
                    for (int i = 0; i < NV; i++) gv[i] = (s2 < P.nseg) ? __ldcg(P.seg_part + (size_t)s2 * NV + i) : 0.0;
                    warp_sum<NV>(gv);
                    if (lane == 0) {
#pragma unroll
                        for (int i = 0; i < NV; i++) P.grp_part[(size_t)g * NV + i] = gv[i];
                        P.grp_cnt[g] = 0u;
                    }
                }
            }
        }
        barrier_decide_tb2<K, SLAB>(P, m, SLAB ? m + 1 : m, two, gen0, da, db, active, s_red, s_flags);
        active = s_flags[2];
        rbmask = s_flags[3];
#pragma unroll
        for (int k = 0; k < K; k++) {
            rbd[k] = db[k];
            da[k] = na[k];
            db[k] = nb[k];
            // rows m+4, m+5 (written by the coefficient warp during pass m-2... visible after this barrier)
            na[k] = (m + 4 < M) ? P.table[(size_t)(m + 4) * (1 + K) + 1 + k] : 0.0;
            nb[k] = (m + 5 < M) ? P.table[(size_t)(m + 5) * (1 + K) + 1 + k] : 0.0;
        }
        if (s_flags[1]) break;
    }
    // the call ended on the first iteration of a pass for some accumulators: final rollback
    if (rbmask && !cwarp && m < M) strip2d_tb2_rollback<K, RT>(P, P.ydst[((m - 1) >> 1) & 1], cbeg, cend, lane, rbmask, rbd);
}

static void* leja_tb2_ptr(int K, bool diag, bool slab) {
#define LX_TB2_CASE(KK)                                                                                         \
    case KK:                                                                                                   \
        return slab ? (diag ? (void*)k_leja2d_tb2<KK, true, true> : (void*)k_leja2d_tb2<KK, false, true>)      \
                    : (diag ? (void*)k_leja2d_tb2<KK, true, false> : (void*)k_leja2d_tb2<KK, false, false>);
    switch (K) {
        LX_TB2_CASE(1)
        LX_TB2_CASE(2)
        LX_TB2_CASE(3)
        LX_TB2_CASE(4)
    }
#undef LX_TB2_CASE
    return nullptr;
}

static int tb2_prepare(int device, int K, bool diag) {
    // dynamic shared memory opt-in (once per kernel) + co-resident CTAs with that smem, cached
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    const int key = K * 2 + (diag ? 1 : 0);
    auto it = cache.find({device, key});
    if (it != cache.end()) return it->second;
    const int smem = tb2_smem_bytes(K, diag);
    int per = 1 << 30;
    for (int sl = 0; sl < 2; sl++) {
        const void* kern = leja_tb2_ptr(K, diag, sl != 0);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int p = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, kern, kThreads, smem);
        if (p < per) per = p;
    }
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    if (per < 1) per = 1;
    cache[{device, key}] = nsm * per;
    return nsm * per;
}

int leja_tb2_grid_size(int device, int K, bool diag, int nunits) {
    long long g = tb2_prepare(device, K, diag);
    long long need = (nunits + kWarps - 1) / kWarps + 1;
    if (g > need) g = need;
    return (int)g;
}

cudaError_t launch_leja_tb2(const LejaParams& P, cudaStream_t s, bool diag, bool slab) {
    void* kern = leja_tb2_ptr(P.K, diag, slab);
    if (!kern) return cudaErrorInvalidValue;
    void* args[] = {(void*)&P};
    return cudaLaunchCooperativeKernel(kern, dim3(P.grid), dim3(kThreads), args, tb2_smem_bytes(P.K, diag), s);
}

cudaError_t preload_tb2() {
    for (int K = 1; K <= kMaxK; K++)
        for (int d = 0; d < 4; d++) {
            cudaFuncAttributes a;
            if (cudaFuncGetAttributes(&a, leja_tb2_ptr(K, d & 1, d >> 1)) != cudaSuccess) return cudaGetLastError();
        }
    return cudaSuccess;
}

}  // namespace lx
