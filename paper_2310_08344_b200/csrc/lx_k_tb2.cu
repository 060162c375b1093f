// lx_k_tb2.cu -- the two-iterations-per-pass Leja kernel (k_leja2d_tb2) and its
// slab-decomposed instantiation over peer memory (SLAB).
#include "lx_dev.cuh"

namespace lx {

// ===========================================================================
// Temporal blocking: TWO Leja iterations per HBM pass.
//   pass q = iterations (m, m+1) = (2q+1, 2q+2): read y_{m-1}, p_{m-1}; y_m is formed
//   in registers on a widened halo (rows i0-1 .. i0+RT+1, columns j0-2 .. j0+61 of a
//   64-column warp window whose 60 inner columns are outputs); y_{m+1} and p_{m+1}
//   are written -> 32 B/pt per TWO iterations.  Both iterations' norms are reduced
//   and the stopping rule of P:155 is applied to m and then m+1 exactly as in the
//   one-step kernel (same decisions, same iteration counts).
//
// Pipelined passes (no grid barrier between passes).  Work = (pass, 32-row x 60-column
// segment) tickets taken in order from one counter.  A segment of pass q starts when
//   * pass q-1 has finished on its 3 x 3 neighbour segments (per-segment completion
//     counters; in a slab, the neighbouring rank's boundary segments signal through
//     per-band flags in this rank's exchange block after storing their halo rows into
//     its ghost block), and
//   * the stopping decision of pass q-2 is known (the decision is LAGGED by one pass:
//     pass q+1 runs speculatively while pass q is decided; if pass q ends the call,
//     pass q+1 is discarded -- p ping-pongs between the caller's output and a
//     scratch vector, so the accepted p_q is never overwritten).
// The last finisher of a pass sums its per-segment partials in fixed order (and, in a
// slab, exchanges the per-rank sums through every rank's exchange header) and publishes
// the decision.  An accumulator that converges on the FIRST iteration of its pass is
// rolled back, p_m = p_{m+1} - d_{m+1} y_{m+1} (<= 1 ulp from the one-step value),
// by the pass two later (before it overwrites y_{m+1}) or by the end-of-call fix-up,
// which also copies results that ended in the scratch half of the ping-pong.
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
// EDGE = false: a segment row away from the slab / periodic boundary (rows always in [0, n)).
template <bool SLAB, bool EDGE = true>
__device__ __forceinline__ const double* tb2_row(const double* base, const double* g, int r, int n, int n1) {
    if (!EDGE) return base + (size_t)r * n1;
    if (SLAB && (unsigned)r >= (unsigned)n) return g + (size_t)(r < 0 ? r + 2 : r - n + 2) * n1;
    return base + (size_t)(r < 0 ? r + n : (r >= n ? r - n : r)) * n1;
}

// Per-pass sources / destinations of the two-step kernel
struct Tb2Pass {
    const double* src;            // y_{m-1} (v on the first pass)
    const double* gsrc;           // its ghost block (SLAB)
    const double* gu;             // ghost block of u (SLAB, DIAG)
    double* dst;                  // y_{m+1}
    const double* pin[kMaxK];     // p_{m-1}^(k) (ping-pong half (q-1) & 1)
    double* pout[kMaxK];          // p_{m+1}^(k) (half q & 1)
};

// stage the global rows of chunk ci into ring stage st (every lane: its own 16-byte pieces)
template <int K, bool DIAG, bool FIRST, bool SLAB, bool EDGE>
__device__ __forceinline__ void tb2_issue(const LejaParams& P, const Tb2Pass& T, double2* __restrict__ ring, int ci,
                                          int st, int lane, int active) {
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
        cp_async16(sg + L::Y + q * 32 + lane, tb2_row<SLAB, EDGE>(T.src, T.gsrc, i0 + 4 + q, n, n1) + j);
        if (lane == 31)
            cp_async16(sg + L::H + q, tb2_row<SLAB, EDGE>(T.src, T.gsrc, i0 + 2 + q, n, n1) + colw(jraw + 2));
        if (DIAG) cp_async16(sg + L::U + q * 32 + lane, tb2_row<SLAB, EDGE>(P.u, T.gu, i0 + 2 + q, n, n1) + j);
    }
    if (!FIRST) {
#pragma unroll
        for (int t = 0; t < RT; t++) {
#pragma unroll
            for (int k = 0; k < KK; k++)
                if ((active >> k) & 1)
                    cp_async16(sg + L::PP + (t * K + k) * 32 + lane,
                               T.pin[k] + (size_t)(EDGE ? wrap(i0 + t) : i0 + t) * n1 + j);
        }
    }
}

// Temporally blocked pass over a contiguous range [cbeg, cend) of (band, chunk) work items of ONE band
// (chunk = RT rows of a 60-column band).  A warp marches down its rows with register windows:
// y_{m-1} rows [i0, i0+RT+4), y_m rows [i0-1, i0+RT+2), u rows [i0, i0+RT+2); per chunk it consumes RT
// new rows of y_{m-1} (and p, u) staged DEPTH-1 chunks ahead by cp.async, forms RT new rows of y_m
// (the 3-row halo recomputation happens only at a strip start) and writes RT rows of y_{m+1} and
// p_{m+1}.  Lanes 1..30 own the band's 60 output columns; lanes 0 and 31 carry halo columns.
// Requires n_loc >= 16, n1 >= 64 (host-checked).
template <int K, bool DIAG, bool FIRST, bool TWO, bool SLAB, bool EDGE>
__device__ __forceinline__ void strip2d_tb2(const LejaParams& P, const Tb2Pass& T, int cbeg, int cend, int lane,
                                            double alpha, double b1, double b2, const double* d0, const double* da,
                                            const double* db, int active, double (&acc)[2 * (1 + K)],
                                            double2* __restrict__ ring) {
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
        if (cbeg + d < cend) tb2_issue<K, DIAG, FIRST, SLAB, EDGE>(P, T, ring, cbeg + d, d, lane, active);
        cp_async_commit();
    }
    int ci = cbeg, st = 0;
    const int b = ci / nc;
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
        for (int q = 0; q < 6; q++) t6[q] = ld2(tb2_row<SLAB, EDGE>(T.src, T.gsrc, i0 - 2 + q, n, n1) + j);
#pragma unroll
        for (int q = 0; q < 3; q++) {
            h3[q] = (lane == 31) ? ld2(tb2_row<SLAB, EDGE>(T.src, T.gsrc, i0 - 1 + q, n, n1) + jh) : z2;
            u3[q] = DIAG ? ldg2(tb2_row<SLAB, EDGE>(P.u, T.gu, i0 - 1 + q, n, n1) + j) : z2;
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
    for (int i0 = (ci - b * nc) * RT; ci < cend; ci++, i0 += RT) {
        // keep D-1 chunks in flight: stage chunk ci+D-1, then wait for chunk ci's group
        {
            int sn = st + D - 1;
            if (sn >= D) sn -= D;
            if (ci + D - 1 < cend) tb2_issue<K, DIAG, FIRST, SLAB, EDGE>(P, T, ring, ci + D - 1, sn, lane, active);
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
                            st2(T.pout[k] + off, pn);
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
    cp_async_wait<0>();
}

// the eight (first pass, two iterations, boundary segment row) instantiations of strip2d_tb2
template <int K, bool DIAG, bool SLAB, bool FIRST, bool TWO>
__device__ __forceinline__ void tb2_strip_e(const LejaParams& P, bool edge, const Tb2Pass& T, int c_b, int c_e,
                                            int lane, double alpha, double b1, double b2, const double* d0,
                                            const double* da, const double* db, int active,
                                            double (&acc)[2 * (1 + K)], double2* __restrict__ ring) {
    if (edge) strip2d_tb2<K, DIAG, FIRST, TWO, SLAB, true>(P, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active, acc, ring);
    else strip2d_tb2<K, DIAG, FIRST, TWO, SLAB, false>(P, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active, acc, ring);
}
template <int K, bool DIAG, bool SLAB>
__device__ __forceinline__ void tb2_strip(const LejaParams& P, bool first, bool two, bool edge, const Tb2Pass& T,
                                          int c_b, int c_e, int lane, double alpha, double b1, double b2,
                                          const double* d0, const double* da, const double* db, int active,
                                          double (&acc)[2 * (1 + K)], double2* __restrict__ ring) {
    if (first) {
        if (two) tb2_strip_e<K, DIAG, SLAB, true, true>(P, edge, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active, acc, ring);
        else tb2_strip_e<K, DIAG, SLAB, true, false>(P, edge, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active, acc, ring);
    } else {
        if (two) tb2_strip_e<K, DIAG, SLAB, false, true>(P, edge, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active, acc, ring);
        else tb2_strip_e<K, DIAG, SLAB, false, false>(P, edge, T, c_b, c_e, lane, alpha, b1, b2, d0, da, db, active, acc, ring);
    }
}

// Output columns of band b owned by this lane (lanes 1..30, two columns each), or -1.
__device__ __forceinline__ int tb2_col(int b, int lane, int n1) {
    const int jraw = b * kBand2 - 2 + 2 * lane;
    return (lane >= 1 && lane <= 30 && jraw < n1 && jraw < b * kBand2 + kBand2) ? jraw : -1;
}

// SLAB halo delivery: rows [r0, r0 + nr) of x, band b -> ghost rows [g0, g0 + nr) of a neighbour's ghost
// block, then (all lanes) a system-scope fence and (lane 0) the release of the neighbour's band flag.
__device__ __forceinline__ void tb2_deliver(const double* x, int r0, int nr, double* g, int g0, int b, int lane,
                                            int n1, unsigned* flag, unsigned value, const double* x2, double* g2) {
    const int j = tb2_col(b, lane, n1);
    if (j >= 0) {
        for (int r = 0; r < nr; r++) {
            st2(g + (size_t)(g0 + r) * n1 + j, ld2(x + (size_t)(r0 + r) * n1 + j));
            if (x2) st2(g2 + (size_t)(g0 + r) * n1 + j, ldg2(x2 + (size_t)(r0 + r) * n1 + j));
        }
    }
    __threadfence_system();
    __syncwarp();
    if (lane == 0) st_release_sys32(flag, value);
}

// Decision word of pass q: [63:32] tag (pbase + q), [31:24] status, [19:16] rollback mask (accumulators
// that converged on the first iteration of the pass), [15:8] done, [7:0] active mask after the pass.
__device__ __forceinline__ unsigned dec_tag(unsigned long long w) { return (unsigned)(w >> 32); }
__device__ __forceinline__ int dec_done(unsigned long long w) { return (int)((w >> 8) & 0xff); }
__device__ __forceinline__ int dec_act(unsigned long long w) { return (int)(w & 0xff); }
__device__ __forceinline__ int dec_rb(unsigned long long w) { return (int)((w >> 16) & 0xf); }
__device__ __forceinline__ int dec_status(unsigned long long w) { return (int)((w >> 24) & 0xff); }

// wrap-safe "counter has reached target" for 32-bit tags
__device__ __forceinline__ bool tag_ge(unsigned a, unsigned b) { return (int)(a - b) >= 0; }

// The call has ended at a pass < q (its final decision is published or about to be): pass q is
// beyond the speculative pass and its decision will never come.
__device__ __forceinline__ bool tb2_ended_before(const LejaParams& P, unsigned pbase, int q) {
    const unsigned ft = ld_acquire(&P.tc->final_tag);
    return tag_ge(ft, pbase) && (int)(ft - pbase) < q;
}

constexpr unsigned long long kDecStop = 1ull;   // tb2_wait_dec: the call ended earlier (tag 0: never a real word)

// Spin (one thread) until the decision of pass q is published.  Returns the word, kDecStop if the call
// ended before pass q, 0 on watchdog / abort.
__device__ __forceinline__ unsigned long long tb2_wait_dec(const LejaParams& P, unsigned pbase, int q) {
    Tb2Ctl* tc = P.tc;
    const unsigned tag = pbase + (unsigned)q;
    unsigned long long w = ld_acquire64(&tc->dec[q & 1]);
    if (dec_tag(w) == tag) return w;
    const unsigned long long t0 = globaltimer_ns();
    for (int spins = 0;; spins++) {
        // back off (64 ns .. 512 ns): idle waiters leave issue slots and L2 to the warps still working
        __nanosleep(spins < 8 ? 64 : 512);
        w = ld_acquire64(&tc->dec[q & 1]);
        if (dec_tag(w) == tag) return w;
        if ((spins & 15) == 15 && tb2_ended_before(P, pbase, q)) return kDecStop;
        if ((spins & 255) == 255 && (ld_acquire(&tc->abort) || globaltimer_ns() - t0 > P.timeout_ns)) {
            atomicExch(&tc->abort, 1u);
            atomicExch(&P.rec->status, 10);
            return 0ull;
        }
    }
}

// Spin (one thread) until *c >= target.  Returns 1; 2 if `q >= 0` and the call ended before pass q
// (a speculative pass stops quietly); 0 on watchdog / abort.
__device__ __forceinline__ int tb2_wait_ge(const LejaParams& P, const unsigned* c, unsigned target, bool sys,
                                           unsigned pbase, int q) {
    if (tag_ge(sys ? ld_acquire_sys32(c) : ld_acquire(c), target)) return 1;
    const unsigned long long t0 = globaltimer_ns();
    for (int spins = 0;; spins++) {
        __nanosleep(32);
        if (tag_ge(sys ? ld_acquire_sys32(c) : ld_acquire(c), target)) return 1;
        if (q >= 0 && (spins & 15) == 15 && tb2_ended_before(P, pbase, q)) return 2;
        if ((spins & 255) == 255 && (ld_acquire(&P.tc->abort) || globaltimer_ns() - t0 > P.timeout_ns)) {
            atomicExch(&P.tc->abort, 1u);
            atomicExch(&P.rec->status, 10);
            return 0;
        }
    }
}

// Decision of pass q (lane 0 of the warp that finished its last segment group): wait for the decision of
// pass q-1; if that ended the call, pass q was speculative -> published as done without a decision
// (and without a cross-rank exchange: every rank decides the same passes).  Else the fixed-order group
// sums (and in a slab the rank-ordered cross-rank sums) enter the P:155 test for iterations 2q+1 and 2q+2.
template <int K, bool SLAB>
__device__ __forceinline__ void tb2_decide(const LejaParams& P, unsigned pbase, int q, bool two, const double* sums_in,
                                           const double* da, const double* db) {
    constexpr int NV = 2 * (1 + K);
    Tb2Ctl* tc = P.tc;
    int act = P.active0, status = 0;
    if (q >= 1) {
        const unsigned long long wp = tb2_wait_dec(P, pbase, q - 1);
        if (wp <= kDecStop) return;
        if (dec_done(wp)) {
            const unsigned long long w = ((unsigned long long)(pbase + (unsigned)q) << 32) |
                                         ((unsigned long long)(dec_status(wp) & 0xff) << 24) | (1ull << 8) |
                                         (unsigned long long)(dec_act(wp) & 0xff);
            tc->gdone[q & 1] = 0u;
            st_release64(&tc->dec[q & 1], w);
            return;
        }
        act = dec_act(wp);
    }
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) acc[i] = sums_in[i];
    if (SLAB) {
        status = xrank_sum<NV>(P, acc);
        if (status) {
            atomicExch(&tc->abort, 1u);
            atomicExch(&P.rec->status, 10);
            return;
        }
    }
    const int act0 = act;
    int done = 0;
    leja_decide<K>(P, 2 * q + 1, acc, da, act, done, status, P.rec);
    const int rb = two ? (act0 & ~act) : 0;     // converged on the first iteration: p_{m+1} holds one term too many
    const int act1 = act;
    if (!done && two) leja_decide<K>(P, 2 * q + 2, acc + 1 + K, db, act, done, status, P.rec);
    for (int k = 0; k < K; k++) {
        if (((act0 >> k) & 1) && !((act >> k) & 1)) {   // frozen in this pass
            tc->frtag[k] = pbase + (unsigned)q;
            tc->frrb[k] = (rb >> k) & 1;
            tc->frd[k] = db[k];
        }
    }
    (void)act1;
    if (done) tc->final_tag = pbase + (unsigned)q;
    tc->gdone[q & 1] = 0u;                          // reused by pass q+2 (which starts after this decision)
    const unsigned long long w = ((unsigned long long)(pbase + (unsigned)q) << 32) |
                                 ((unsigned long long)(status & 0xff) << 24) | ((unsigned long long)(rb & 0xf) << 16) |
                                 ((unsigned long long)(done & 0xff) << 8) | (unsigned long long)(act & 0xff);
    st_release64(&tc->dec[q & 1], w);
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


// Two Leja iterations per HBM pass, passes pipelined (see the header comment).  SLAB = the
// slab-decomposed variant: one persistent kernel per Leja call and rank; halo rows and
// norm partials travel through peer memory from inside the kernel; no host round trip, no NCCL call and
// no extra launch per iteration.
template <int K, bool DIAG, bool SLAB>
__global__ void __launch_bounds__(kThreads, 2) k_leja2d_tb2(const __grid_constant__ LejaParams P) {
    extern __shared__ double2 tb2_ring[];
    __shared__ int s_flag;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool cwarp = (blockIdx.x == 0 && warp == 0);
    constexpr int NV = 2 * (1 + K);
    constexpr int RT = tb2_rt(K);
    double2* ring = tb2_ring + (size_t)warp * Tb2Stage<K, DIAG>::WARP;
    Tb2Ctl* tc = P.tc;
    const unsigned pbase = tc->pbase;             // written by the previous call's leader (kernel boundary)
    // p ping-pong parity: pass q writes half (q + poff) & 1 (half 0 = the caller's output).  poff is the
    // final-pass parity of the last call with the same parameters (a small table written by each call's
    // leader): repeated calls then end in the caller's buffer and the fix-up copies nothing
    const unsigned long long key = tb2_call_key<K>(P);
    int poff = 0, pslot = -1, fpred = -2;
    for (int i = 0; i < kTb2Pred; i++)
        if (tc->pkey[i] == key) {
            poff = (int)(tc->pfin[i] & 1u);
            fpred = (int)tc->pfin[i];
            pslot = i;
        }
    unsigned rel0 = 0;
    if (tid == 0) rel0 = ld_acquire(&tc->release);
    const int M = P.max_nodes;
    const int qmax = (M - 2) / 2;                 // last pass: first iteration 2q+1 <= M-1
    const int nb = P.nb, nseg = P.nseg, nsr = nseg / nb, n = P.n_loc, n1 = P.n1;
    const double alpha = P_alpha(P);
    if (SLAB) {
        // this rank's boundary rows of v (and u) into the neighbours' ghost blocks, one band per CTA (rows
        // 0..3 -> rank-1's rows n..n+3, rows n-2, n-1 -> rank+1's rows -2, -1), then the band flags (tag
        // pbase: "pass -1 delivered"); done first so that no pass-0 segment waits for a late delivery
        for (int b = blockIdx.x; b < nb; b += gridDim.x) {
            const int pr = tid / 30, lp = tid - pr * 30;   // 6 rows x 30 column pairs
            if (pr < 6) {
                const int j = b * kBand2 + 2 * lp;
                if (j < n1) {
                    const int src = pr < 4 ? pr : n - 6 + pr;
                    double* gv = pr < 4 ? P.hup_v + (size_t)(2 + pr) * n1 : P.hdn_v + (size_t)(pr - 4) * n1;
                    st2(gv + j, ld2(P.v.base + (size_t)src * n1 + j));
                    if (DIAG) {
                        double* gu = pr < 4 ? P.hup_u + (size_t)(2 + pr) * n1 : P.hdn_u + (size_t)(pr - 4) * n1;
                        st2(gu + j, ldg2(P.u + (size_t)src * n1 + j));
                    }
                }
            }
            __threadfence_system();
            __syncthreads();
            if (tid == 0) {
                st_release_sys32(P.fl_dn_up + b, pbase);
                st_release_sys32(P.fl_up_dn + b, pbase);
            }
        }
    }
    double dd[K][5];
#pragma unroll
    for (int k = 0; k < K; k++) coef_first5<K>(P, k, dd[k]);
    if (cwarp) {
        // coefficient warp: rows 0..4 now, then d_j (lane k = accumulator k) ahead of the issued passes
        if (!P.coef_gen && lane == 0) st_release(&tc->crow, (unsigned)M);   // prebuilt table
        if (P.coef_gen) {
            for (int r = 0; r < 5 && r < M; r++) {
                double row[K];
#pragma unroll
                for (int k = 0; k < K; k++) row[k] = dd[k][r];
                coef_write_row<K>(P, r, lane, P.active0, row);
            }
            __syncwarp();
            __threadfence();
            if (lane == 0) st_release(&tc->crow, 5u);
            int j = 5;
            while (j < M) {
                unsigned t = 0, stop = 0;
                if (lane == 0) {
                    t = ld_acquire(&tc->ticket);
                    stop = ld_acquire(&tc->abort) || tag_ge(ld_acquire(&tc->final_tag), pbase);
                }
                t = __shfl_sync(FULL_MASK, t, 0);
                if (__shfl_sync(FULL_MASK, stop, 0)) break;
                const int want = min(M - 1, 2 * (int)(t / (unsigned)nseg) + 8);
                if (j > want) {
                    __nanosleep(256);
                    continue;
                }
                coef_write_row<K>(P, j, lane, (1 << K) - 1, nullptr);
                __syncwarp();
                __threadfence();
                if (lane == 0) st_release(&tc->crow, (unsigned)(j + 1));
                j++;
            }
        }
    } else {
        for (;;) {
            unsigned tk = 0;
            if (lane == 0) tk = atomicAdd(&tc->ticket, 1u);
            tk = __shfl_sync(FULL_MASK, tk, 0);
            const int q = (int)(tk / (unsigned)nseg);
            if (q > qmax) break;
            // pass q visits the segment rows starting at row q mod nsr (band fastest): its first segments
            // depend on the rows pass q-1 visited FIRST, so consecutive passes overlap instead of pass q
            // waiting for the previous pass's last (periodically adjacent) rows
            const int ti = (int)(tk - (unsigned)q * (unsigned)nseg);
            const int rsi = ti / nb;
            const int s = ((rsi + q) % nsr) * nb + (ti - rsi * nb);
            // lagged decision: pass q needs the decision of pass q-2
            int act = P.active0, rbm = 0, stop = 0;
            if (lane == 0) {
                if (q >= 2) {
                    const unsigned long long w = tb2_wait_dec(P, pbase, q - 2);
                    if (w <= kDecStop || dec_done(w)) stop = 1;
                    else {
                        act = dec_act(w);
                        rbm = dec_rb(w);
                    }
                }
                if (!stop && q >= 1) {   // pass q-1 already known to end the call: nothing left to do
                    const unsigned long long w1 = ld_acquire64(&tc->dec[(q - 1) & 1]);
                    if (dec_tag(w1) == pbase + (unsigned)(q - 1) && dec_done(w1)) stop = 1;
                }
                if (!stop && q == fpred + 1) {
                    // the last call with these parameters ended at pass q-1: rather than running pass q
                    // speculatively (a pass of wasted HBM traffic when the prediction holds), wait for the
                    // decision of pass q-1
                    const unsigned long long w1 = tb2_wait_dec(P, pbase, q - 1);
                    if (w1 <= kDecStop || dec_done(w1)) stop = 1;
                }
            }
            if (__shfl_sync(FULL_MASK, stop, 0)) break;
            act = __shfl_sync(FULL_MASK, act, 0);
            rbm = __shfl_sync(FULL_MASK, rbm, 0);
            const bool two = (2 * q + 2 < M);
            // Newton coefficients of iterations 2q+1, 2q+2 (rows 0..4 from the prologue)
            double d0[K], da[K], db[K];
            if (q >= 2) {
                if (lane == 0 && tb2_wait_ge(P, &tc->crow, (unsigned)min(2 * q + 3, M), false, pbase, q) != 1) stop = 1;
                if (__shfl_sync(FULL_MASK, stop, 0)) break;
                __syncwarp();
            }
#pragma unroll
            for (int k = 0; k < K; k++) {
                d0[k] = dd[k][0];
                da[k] = q == 0 ? dd[k][1] : (q == 1 ? dd[k][3] : __ldcg(P.table + (size_t)(2 * q + 1) * (1 + K) + 1 + k));
                db[k] = !two ? 0.0 : (q == 0 ? dd[k][2] : (q == 1 ? dd[k][4] : __ldcg(P.table + (size_t)(2 * q + 2) * (1 + K) + 1 + k)));
            }
            const double b1 = coef_beta(P, 2 * q + 1), b2 = two ? coef_beta(P, 2 * q + 2) : 0.0;
            const int rs = s / nb, b = s - rs * nb;
            const bool top = SLAB && rs == 0, bot = SLAB && rs == nsr - 1;
            // dependencies: pass q-1 done on the 3 x 3 neighbour segments (slab edges: the neighbour
            // rank's boundary segments, signalled by band flags after their halo rows landed here)
            if (lane < 9) {
                const int dr = lane / 3 - 1, dbn = lane % 3 - 1;
                const int bb = (b + dbn + nb) % nb;
                const int rr = rs + dr;
                if (SLAB && rr < 0) stop = tb2_wait_ge(P, P.fl_up + bb, pbase + (unsigned)q, true, pbase, q) != 1;
                else if (SLAB && rr >= nsr) stop = tb2_wait_ge(P, P.fl_dn + bb, pbase + (unsigned)q, true, pbase, q) != 1;
                else if (q >= 1)
                    stop = tb2_wait_ge(P, P.scnt + ((rr + nsr) % nsr) * nb + bb, pbase + (unsigned)q, false, pbase, q) != 1;
            }
            if (__any_sync(FULL_MASK, stop)) break;
            __syncwarp();
            // segment rows of P.seg chunks; the last one also takes the remainder (>= 4 rows: a segment's
            // stencil halo, rows -2 .. +3, then reaches only the adjacent segment rows / ghost rows)
            const int c_b = b * P.nrb + rs * P.seg;
            const int c_e = b * P.nrb + (rs == nsr - 1 ? P.nrb : rs * P.seg + P.seg);
            const int r0 = rs * P.seg * RT, r1 = (rs == nsr - 1) ? n : (rs * P.seg + P.seg) * RT;
            // accumulators that converged on the first iteration of pass q-2: p_m = p_{m+1} - d_{m+1} y_{m+1},
            // in place in their final ping-pong half, before this pass overwrites y_{m+1}
            if (rbm) {
                const int j = tb2_col(b, lane, n1);
                const double* y = P.ydst[q & 1];
#pragma unroll
                for (int k = 0; k < K; k++) {
                    if (!((rbm >> k) & 1) || j < 0) continue;
                    double* pk = P.pp[k][(q + poff) & 1];
                    const double dk = __ldcg(&tc->frd[k]);
                    for (int r = r0; r < r1; r++) {
                        const size_t off = (size_t)r * n1 + j;
                        const double2 yy = ld2(y + off), pv = ld2(pk + off);
                        st2(pk + off, make_double2(fma(-dk, yy.x, pv.x), fma(-dk, yy.y, pv.y)));
                    }
                }
            }
            Tb2Pass T;
            T.src = (q == 0) ? P.v.base : P.ydst[(q - 1) & 1];
            T.gsrc = (q == 0) ? P.gv : P.gy[(q - 1) & 1];
            T.gu = P.gu;
            T.dst = P.ydst[q & 1];
#pragma unroll
            for (int k = 0; k < kMaxK; k++) {
                T.pin[k] = P.pp[k][(q - 1 + poff) & 1];
                T.pout[k] = P.pp[k][(q + poff) & 1];
            }
            double acc[NV];
#pragma unroll
            for (int i = 0; i < NV; i++) acc[i] = 0.0;
            // boundary segment rows (the first and the last: their stencil halo reaches the periodic image or
            // the ghost rows) take the checked row addressing, all others the direct one
            tb2_strip<K, DIAG, SLAB>(P, q == 0, two, rs == 0 || rs == nsr - 1, T, c_b, c_e, lane, alpha, b1, b2, d0,
                                     da, db, act, acc, ring);
            // SLAB: this pass's boundary rows of y into the neighbours' ghost blocks (+ their band flags)
            // (the rows / ghost slots of lx_slab_halo_plan mode 1)
            if (top) tb2_deliver(T.dst, 0, kTb2UpRows, P.hup[q & 1], 2, b, lane, n1, P.fl_dn_up + b,
                                 pbase + (unsigned)q + 1, nullptr, nullptr);
            if (bot) tb2_deliver(T.dst, n - kTb2DnRows, kTb2DnRows, P.hdn[q & 1], 0, b, lane, n1, P.fl_up_dn + b,
                                 pbase + (unsigned)q + 1, nullptr, nullptr);
            // the segment is done with pass q: its norm partials, then ONE fence (ordering this warp's y / p
            // stores and the partials) before the completion tag and the group counter
            warp_sum<NV>(acc);
            double* segp = P.seg_part + ((size_t)(q & 1) * P.nseg + s) * NV;
            const int g = s >> 5;
            int last = 0;
            if (lane == 0) {
#pragma unroll
                for (int i = 0; i < NV; i++) segp[i] = acc[i];
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                st_relaxed32(P.scnt + s, pbase + (unsigned)q + 1);
                const unsigned t = atomicAdd(&P.grp_cnt[(q & 1) * P.ngrp + g], 1u);
                last = (int)(t == (unsigned)(min(32, nseg - g * 32) - 1));
            }
            last = __shfl_sync(FULL_MASK, last, 0);
            if (last) {
                __threadfence();
                const int s2 = g * 32 + lane;
                double gv[NV];
#pragma unroll
                for (int i = 0; i < NV; i++)
                    gv[i] = (s2 < nseg) ? __ldcg(P.seg_part + ((size_t)(q & 1) * P.nseg + s2) * NV + i) : 0.0;
                warp_sum<NV>(gv);
                int lastg = 0;
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < NV; i++) P.grp_part[((size_t)(q & 1) * P.ngrp + g) * NV + i] = gv[i];
                    P.grp_cnt[(q & 1) * P.ngrp + g] = 0u;
                    __threadfence();
                    lastg = (int)(atomicAdd(&tc->gdone[q & 1], 1u) == (unsigned)(P.ngrp - 1));
                }
                lastg = __shfl_sync(FULL_MASK, lastg, 0);
                if (lastg) {
                    // the pass is complete: fixed-order sum over its groups (lane-strided, then butterfly)
                    __threadfence();
                    double sv[NV];
#pragma unroll
                    for (int i = 0; i < NV; i++) sv[i] = 0.0;
                    for (int g2 = lane; g2 < P.ngrp; g2 += 32) {
#pragma unroll
                        for (int i = 0; i < NV; i++) sv[i] += __ldcg(P.grp_part + ((size_t)(q & 1) * P.ngrp + g2) * NV + i);
                    }
                    warp_sum<NV>(sv);
                    if (lane == 0) tb2_decide<K, SLAB>(P, pbase, q, two, sv, da, db);
                    __syncwarp();
                }
            }
        }
    }
    // ---- end of the call: every warp has stopped (one grid barrier per call), then the fix-up
    __syncthreads();
    if (tid == 0) {
        const unsigned t = atom_add_acq_rel(&tc->arrive, 1u);
        s_flag = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_flag) {
        if (tid == 0) {
            // leader: snapshot the call's outcome for the fix-up, reset the per-call counters (nobody uses
            // them after this barrier), advance the pass tags above every tag of this call (speculative
            // pass f + 1 included), then release
            const unsigned ft = ld_acquire(&tc->final_tag);
            const unsigned ab = ld_acquire(&tc->abort);
            const unsigned fl = tag_ge(ft, pbase) ? ft - pbase : 0u;
            tc->snap_final = fl;
            tc->snap_abort = ab;
            if (!ab) {   // remember this call's final pass for the next call with the same parameters
                const int slot = pslot >= 0 ? pslot : (int)(tc->pnext++ % (unsigned)kTb2Pred);
                tc->pkey[slot] = key;
                tc->pfin[slot] = fl;
            }
            tc->ticket = 0u;
            tc->crow = 0u;
            tc->abort = 0u;
            tc->pbase = pbase + fl + 3u + (ab ? (unsigned)qmax + 3u : 0u);
            tc->arrive = 0u;
            st_release(&tc->release, rel0 + 1u);
        }
    } else if (tid == 0) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire(&tc->release) == rel0) {
            __nanosleep(64);
            if (globaltimer_ns() - t0 > P.timeout_ns + 10000000000ull) {
                atomicExch(&P.rec->status, 10);
                break;
            }
        }
    }
    __syncthreads();
    const bool aborted = __ldcg(&tc->snap_abort) != 0u;
    const int f = (int)__ldcg(&tc->snap_final);
    // fix-up: each accumulator's final value is p of its freeze pass f_k (ping-pong half f_k & 1), minus
    // d y_{m+1} if it converged on the first iteration of that pass and pass f_k + 2 (which rolls back in
    // place) did not run on the segment; results in the scratch half are copied to the caller's output
    if (!aborted) {
        int fk[K], rbk[K];
        double dk[K];
        bool any = false;
#pragma unroll
        for (int k = 0; k < K; k++) {
            const unsigned tg = __ldcg(&tc->frtag[k]);
            const bool frozen = tag_ge(tg, pbase) && ((P.active0 >> k) & 1);
            fk[k] = frozen ? (int)(tg - pbase) : f;
            rbk[k] = frozen ? (int)__ldcg(&tc->frrb[k]) : 0;
            dk[k] = __ldcg(&tc->frd[k]);
            any = any || rbk[k] || ((fk[k] + poff) & 1);
        }
        if (any) {
            const int gw = blockIdx.x * kWarps + warp, W = gridDim.x * kWarps;
            for (int s = gw; s < nseg; s += W) {
                const int rs = s / nb, b = s - rs * nb;
                const int j = tb2_col(b, lane, n1);
                if (j < 0) continue;
                const int r0 = rs * P.seg * RT, r1 = (rs == nsr - 1) ? n : (rs * P.seg + P.seg) * RT;
                const unsigned done_s = ld_acquire(P.scnt + s);
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const bool pend = rbk[k] && !tag_ge(done_s, pbase + (unsigned)fk[k] + 3u);
                    if (!pend && !((fk[k] + poff) & 1)) continue;
                    const double* src = P.pp[k][(fk[k] + poff) & 1];
                    const double* y = P.ydst[fk[k] & 1];
                    double* out = P.pp[k][0];
                    for (int r = r0; r < r1; r++) {
                        const size_t off = (size_t)r * n1 + j;
                        double2 pv = ld2(src + off);
                        if (pend) {
                            const double2 yy = ld2(y + off);
                            pv = make_double2(fma(-dk[k], yy.x, pv.x), fma(-dk[k], yy.y, pv.y));
                        }
                        st2(out + off, pv);
                    }
                }
            }
        }
    }
    // the speculative pass (and an aborted call) may leave group counters partly counted: clear them for the
    // next call (nobody counts after the barrier)
    for (int i = blockIdx.x * kThreads + tid; i < 2 * P.ngrp; i += gridDim.x * kThreads) P.grp_cnt[i] = 0u;
    if (blockIdx.x == 0 && tid < 2) tc->gdone[tid] = 0u;
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
