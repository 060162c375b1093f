// lx_internal.h -- structures shared by the host runtime and the sm_100a kernels.
// Not part of the public ABI (include/lexint.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef LX_KRT3
#define LX_KRT3 2
#endif
namespace lx {

constexpr int kThreads = 256;     // threads per CTA (8 warps)
constexpr int kWarps = kThreads / 32;
constexpr int kRT = 4;            // rows per warp work unit (2D)
// rows per warp work unit of the flux-form (Burgers) 2D tile: two, so the kernel fits two CTAs per SM
// (measured at 4096^2: phi_1 0.60 -> 0.72 of the copy peak vs four rows at one CTA per SM)
constexpr int kRTF = 2;
// black-box Leja: iterations enqueued ahead of the decision the host reads (<= 3).  Measured (4096^2 FD / linear):
// 2 or 3 in flight are 2-4 % slower than 1 -- the extra f evaluations after convergence cost more than the
// host's wake-up latency they hide.
constexpr int kBbLag = 1;
constexpr int kRT3 = LX_KRT3;         // planes per warp work unit (3D)
// two-step (temporally blocked) kernel: rows per chunk, bytes of one staged chunk, ring depth
// (chunks per warp ring; 8 warps x depth x stage <= 110 KB so that two CTAs fit on an SM)
__host__ __device__ constexpr int tb2_rt(int K) { return K == 1 ? 4 : 2; }
__host__ __device__ constexpr int tb2_stage_bytes(int K, bool diag) {
    return 16 * (tb2_rt(K) * 32 * (1 + K + (diag ? 1 : 0)) + tb2_rt(K));
}
__host__ __device__ constexpr int tb2_depth(int K, bool diag) { return tb2_stage_bytes(K, diag) * 24 <= 112640 ? 3 : 2; }
__host__ __device__ constexpr int tb2_smem_bytes(int K, bool diag) { return 8 * tb2_depth(K, diag) * tb2_stage_bytes(K, diag); }
constexpr int kBand2 = 60;        // output columns per warp band of the two-step kernel (64 loaded)
constexpr int kMaxK = 4;          // vertical accumulators
// Slab halos (the +x-biased upwind stencil reaches rows i-1, i+1, i+2, reading R10):
//   step protocol (one iteration per exchange): rows 0, 1 -> rank-1 (its rows n, n+1), row n-1 -> rank+1 (its row -1)
//   two-step slab kernel (two iterations per exchange): rows 0..3 -> rank-1 (its rows n..n+3), rows n-2, n-1 ->
//   rank+1 (its rows -2, -1); ghost blocks of 3 and 6 rows respectively (comm_halo_plan, lx_slab_halo_plan)
constexpr int kStepUpRows = 2, kStepDnRows = 1;
constexpr int kTb2UpRows = 4, kTb2DnRows = 2;
constexpr int kSlot = 12;         // doubles per CTA partial slot (2 (1 + K) <= 10 for two-step passes)

// Per-call record, written on the device, read by the host once per call/step.
struct Record {
    int iters;            // total Leja iterations accumulated by this record
    int status;           // first non-OK status (lx_status numbering)
    int iters_k[kMaxK];   // iteration at which accumulator k converged (last Leja call)
    int ncalls;           // number of Leja calls accumulated
    int pad;
    double margin_accept; // min thr/err at acceptance (inf if err == 0)
    double margin_reject; // min err/thr over rejected checks
    double err;           // embedded error estimate (steps)
    double est;           // spectrum estimate / bound
};

// Device control block of a persistent kernel (grid barrier + decision).
struct Ctrl {
    unsigned int arrive;  // barrier arrivals (reset by the last arriver)
    unsigned int gen;     // barrier generation (monotone, release flag)
    int done;             // decision: stop after this iteration
    int active;           // decision: bit k = accumulator k still accumulating
    int status;           // decision: status so far
    int m;                // last decided iteration
    int pad0, pad1;
    double scale;         // power iteration: 1/||w_m|| for the next application
    double est;           // power iteration: latest estimate
    unsigned int ticket;  // last-block ticket for non-persistent reductions
    unsigned int pad2;
    unsigned long long umax;  // max reduction (bit pattern of a non-negative double)
    int hist[2];          // step mode: active mask after iteration j stored at hist[j & 1]
    // persistent kernels: packed decision word released by the barrier's last arriver
    // [63:32] generation (gen0 + m), [31:16] status, [15:8] done, [7:0] active mask
    unsigned long long word;
    unsigned int work[2];  // two-step kernel: dynamic segment counters of even / odd passes
    unsigned int pad3[2];
};

// Rows of a slab: rows [0, n_loc) at base, row r in {-1, n_loc, n_loc+1}
// either from `ghost` (3 rows: -1, n_loc, n_loc+1) or by periodic wrap.
struct RowSrc {
    const double* base;
    const double* ghost;
    long long stride;     // doubles per row (n1 in 2D, n1*n2 in 3D)
    int n_loc;
    int pad;
};

// Constant-coefficient stencil of A (diff*lap + nu*sum_d D_d) per dimension:
// offsets -1, 0, +1, +2 (third-order upwind +x-biased).
struct Stencil {
    double c0;            // centre (summed over dimensions)
    double m1[3], p1[3], p2[3];
    double qa, qb;        // diagonal of J: qa + qb * u^2   (react*(1 - 3u^2))
    double react;         // g(u) = react*(u - u^3)
    // flux form (Burgers, Problem III): diffusion and upwind coefficients kept separate
    double flux, nu;      // beta, nu:  J y = diff lap y + sum_d D_d((nu + beta u) y)
    double dd0, dm1[3], dp1[3];             // diff*lap: centre, -1, +1
    double a0[3], am1[3], ap1[3], ap2[3];   // D_d: centre, -1, +1, +2
};

// Exchange header of the peer-memory slab transport (one per rank, in IPC-shareable device memory;
// every rank writes into every rank's header).  flag[q] = last epoch rank q published here;
// part[e & 1][q] = rank q's partial sums of epoch e.  `epoch` is this rank's own counter.
constexpr int kMaxRanks = 8;
constexpr int kXNV = 2 * (1 + kMaxK);
struct XHdr {
    unsigned long long flag[kMaxRanks];
    unsigned long long epoch;
    unsigned long long pad[7];
    double part[2][kMaxRanks][kXNV + 2];
};

// Per-context state of the pipelined two-step kernel (k_leja2d_tb2).  Pass tags are pbase + pass and
// grow across calls (the leader of each call advances pbase past every tag it used), so no per-call
// reset of completion counters, flags or decision words is needed.
struct Tb2Ctl {
    unsigned ticket;              // next (pass, segment) work item of this call
    unsigned pbase;               // pass-tag base of the current call (starts at 1)
    unsigned gdone[2];            // segment groups finished, by pass parity
    unsigned long long dec[2];    // decision words of the last two passes (tag, status, rb, done, active)
    unsigned crow;                // Newton-coefficient rows ready (rows < crow)
    unsigned abort;               // a watchdog fired in this call
    unsigned arrive, release;     // end-of-call grid barrier
    unsigned final_tag;           // pbase + the pass whose decision ended the call
    unsigned snap_final, snap_abort;   // the leader's snapshot for the fix-up
    unsigned frtag[kMaxK];        // pbase + the pass in which accumulator k froze
    unsigned frrb[kMaxK];         // ... on the first iteration of that pass (rollback pending)
    double frd[kMaxK];            // its rollback coefficient d_{m+1}
    unsigned long long pkey[8];   // ping-pong parity prediction: parameter keys of recent calls ...
    unsigned pfin[8];             // ... and their final passes
    unsigned pnext;
};
constexpr int kTb2Pred = 8;

struct LejaParams {
    int ndim;
    int n_loc;            // local rows (dim 0)
    int n1, n2;           // dims 1, 2 (n2 = 1 in 2D)
    int nb;               // column bands of 64 along the contiguous dimension
    int nrow;             // rows of the CTA-tile index (2D: n_loc row blocks; 3D: n1 rows)
    int nrb;              // row blocks of kRT along dim 0
    int nunits;           // warp work units per iteration
    int K;
    int max_nodes;
    int active0;          // initial active mask
    int power_iters;      // POWER mode: number of applications
    double N_glob;
    double alpha;         // 1/gamma
    double rtol, atol;
    Stencil st;
    const double* coef;   // [max_nodes][1+K]: beta_m, d_m^(k)
    RowSrc v;             // input vector (iteration 1)
    RowSrc ysrc[2];       // y ping-pong read views
    double* ydst[2];      // y ping-pong write pointers (== ysrc[i].base)
    double* p[kMaxK];
    const double* u;      // linearisation state (diag), unpadded local
    double* partials;     // [2][grid][kSlot]
    Ctrl* ctrl;
    Record* rec;
    int grid;
    int timeout_spins;
    // step (multi-rank) mode: per-rank partial and the gathered [nranks][kSlot] partials
    double* rank_part;
    const double* gathered;
    int nranks;
    // In-kernel coefficients: the kernel fills `table` ([max_nodes][1+K]: beta_m,
    // d_m^(k)) itself, two iterations ahead, on a dedicated coefficient warp (CTA 0, warp 0).
    int coef_gen;
    int l;
    int lk[kMaxK];        // phi index of accumulator k (= l, or per accumulator: lx_real_leja_phi_multi)
    double cdt, cc, cgamma;
    double ak[kMaxK];
    const double* xi;     // [max_nodes] Leja points
    const double* R;      // [max_nodes][max_nodes]: 1/(xi_j - xi_i), j > i
    double* table;        // == coef
    // device-resident (c, gamma) (lx_integrate: spectrum recomputed on the device every step);
    // nullptr -> cc / cgamma / alpha from the host
    const double* cg_dev;
    const double* source;  // optional source S added by the f(u) (M_RHS) tiles (Problem II)
    // two-step kernel: dynamic segments of `seg` chunks (band fastest); per-segment norm partials,
    // reduced in fixed order per group of 32 segments by the group's last finisher, then over groups
    int seg;
    int nseg, ngrp;
    double* seg_part;     // [nseg][2(1+K)]
    double* grp_part;     // [ngrp][2(1+K)]
    unsigned* grp_cnt;    // [ngrp] finished segments of the group (reset by its last finisher)
    // peer-memory slab mode (k_leja2d_tb2<K, DIAG, true>): ghost blocks hold rows
    // -2, -1, n, n+1, n+2, n+3 of the local slab
    XHdr* xh[kMaxRanks];  // every rank's exchange header (peer pointers; xh[xrank] is this rank's)
    int xrank, xranks;
    const double* gy[2];  // this rank's ghost blocks of Y[0], Y[1]
    const double* gv;     // ... of the iteration-1 input v
    const double* gu;     // ... of the linearisation state u (DIAG)
    double* hup[2];       // ghost blocks of Y[i] on rank-1 (receive rows 0..3) ...
    double* hdn[2];       // ... and on rank+1 (receive rows n-2, n-1)
    double* hup_v; double* hdn_v; double* hup_u; double* hdn_u;
    unsigned long long timeout_ns;   // wait limit of the persistent kernels' watchdogs (LX_ERR_TIMEOUT)
    // pipelined two-step kernel: control block, per-segment completion tags, p ping-pong halves
    // (pp[k][0] = the caller's output, pp[k][1] = context scratch), slab band flags (pbase + pass after
    // the halo rows of that pass landed): fl_up / fl_dn this rank's (deliveries from rank-1 / rank+1),
    // fl_up_dn = rank+1's fl_up, fl_dn_up = rank-1's fl_dn (this rank signals into them)
    Tb2Ctl* tc;
    unsigned* scnt;
    double* pp[kMaxK][2];
    unsigned* fl_up;
    unsigned* fl_dn;
    unsigned* fl_up_dn;
    unsigned* fl_dn_up;
};

// launchers (lx_kernels.cu)
cudaError_t launch_leja_persistent(const LejaParams& P, cudaStream_t s, bool diag);
cudaError_t launch_power_persistent(const LejaParams& P, cudaStream_t s, bool diag);
int leja_grid_size(int device, int K, bool diag, int ndim, int nunits);
// 3D marching kernel with shared-memory plane tiles (single GPU, n1 % 8 == 0, n2 % 64 == 0, prebuilt
// coefficient table); ncu = CTA units (8 j-rows x 64 k x 64 planes)
int leja3d_smem_grid_size(int device, int K, bool diag, int ncu);
int leja3d_smem_units(int n0, int n1, int n2);
cudaError_t launch_leja3d_smem(const LejaParams& P, cudaStream_t s, bool diag);
// 3D two-step kernel (2.5D temporal blocking); slab = the peer-memory slab instantiation (ghost planes
// -2, -1, n .. n+3 in the exchange block, norm partials exchanged at each pass barrier)
int leja3d_tb2_grid_size(int device, int K, int ncu, bool slab = false);
cudaError_t launch_leja3d_tb2(const LejaParams& P, cudaStream_t s, bool slab = false);
// temporally blocked 2D kernel: two Leja iterations per HBM pass (single GPU, constant coefficients + diag)
int leja_tb2_grid_size(int device, int K, bool diag, int nunits);
cudaError_t launch_leja_tb2(const LejaParams& P, cudaStream_t s, bool diag, bool slab = false);

struct StageArgs {
    int ndim, n_loc, n1, n2, nb, nrb, nunits;
    double N_glob;
    Stencil st;
    RowSrc src;           // stencil input
    const double* u;      // state
    const double* x0; const double* x1; const double* x2; const double* x3;
    double* y0; double* y1;
    double a0, a1, a2, a3, a4, a5;
    double dt;
    double* partials;     // [grid][kSlot]
    Ctrl* ctrl;
    Record* rec;
    int grid;
    double* rank_part;    // multi-rank: norm partial goes here instead of rec->err
};

enum StageOp {
    ST_RHS_SCALED = 0,    // y0 = a0 * f(src)                       (stencil)
    ST_AXPBY = 1,         // y0 = a0*x0 + a1*x1
    ST_REMAINDER_DIFF,    // y0 = dt*F(x0) - dt*F(u)   F(x)=g(x)-g'(u)x      (R18)
    ST_STAGE_REMAINDER,   // s = x0 + a0*x1 + a1*x2 ; y0 = a2*(dt*F(s) - dt*F(u))  (s not stored)
    ST_EXPRB32_A,         // y1 = x0 + x1 (a) ; y0 = dt*F(a) - dt*F(u)
    ST_COMBINE2,          // y0 = a0*x0 + a1*x1 ; y1 = a2*x0 + a3*x1
    ST_FINAL4,            // y0 = x0 + x1 + x2 (u3) ; y1 = y0 + x3 (u4) ; err = ||y1 - y0||
    ST_FINAL_EXPRB32,     // y0 = x0 + 2 x1 ; err = ||2 x1||
    ST_MAXSQ,             // ctrl->umax = max x0^2
    ST_SUM3,              // y0 = x0 + x1 + x2
    ST_LIN3,              // y0 = x0 + a0*x1 + a1*x2
    ST_LIN4,              // y0 = x0 + a0*x1 + a1*x2 + a2*x3
    ST_LIN4_ERR,          // y0 = x0 + a0*x1 + a1*x2 + a2*x3 ; err = ||y0 - y1|| (y1 read: the embedded solution)
    ST_REM2_W34,          // D_a = dt F(u + a0 x1) - dt F(u), D_b = dt F(u + a1 x2) - dt F(u) (not stored);
                          // y0 = a2 D_a + a3 D_b, y1 = a4 D_a + a5 D_b  (two-stage EPIRK final-stage inputs)
    ST_REMB_W34,          // D_b = dt F(u + a0 x1 + a1 x2) - dt F(u) (not stored), D_a = x3;
                          // y0 = a2 D_a + a3 D_b, y1 = a4 D_a + a5 D_b  (EXPRB43 final-stage inputs)
};
cudaError_t launch_stage(int op, const StageArgs& A, cudaStream_t s);
cudaError_t launch_rhs(const LejaParams& P, double scale, cudaStream_t s);
// f(u) dt on 3D grids with the smem kernel's plane tiles (single domain, n1 % 16 == 0, n2 % 64 == 0)
cudaError_t launch_rhs3d_smem(const LejaParams& P, double scale, cudaStream_t s, int device);
// Burgers remainder difference (stencil): y = a2 * (dt F(x) - dt F(u)), x = P.v (with halo), u = P.u
cudaError_t launch_rem_flux(const LejaParams& P, double dt, double a2, double* out, cudaStream_t s);
cudaError_t launch_fill_start(double* v, long long n, bool add_e0, cudaStream_t s);
// step mode (one launch per iteration; decision for m-1 in the prologue from P.gathered)
cudaError_t launch_leja_step(const LejaParams& P, int m, cudaStream_t s, bool diag);
cudaError_t launch_power_step(const LejaParams& P, int m, cudaStream_t s, bool diag);
int step_grid_size(int device, int nunits);
cudaError_t launch_finalize_err(const double* gathered, int nranks, double N, Record* rec, cudaStream_t s);
cudaError_t launch_max_u64(const unsigned long long* vals, int n, unsigned long long* out, cudaStream_t s);
// (c, gamma) on the device from the spectrum bound of J(u): sum_d (4 diff/h^2 + 4 vmax/(3h)),
// vmax = |nu| + |beta| max|u|, + react*max(0, 3 max u^2 - 1)  (readings R9, R16, R23)
struct ShiftArgs {
    int ndim;
    double h[3];
    double diff, nu, flux, react;
};
cudaError_t launch_shift_scale(const unsigned long long* umax, const ShiftArgs& a, double* cg_out, cudaStream_t s);
int stage_grid_size(int device, int op);
// device coefficient table: [M][1+K] = {beta_m, d_m^(k)}; a[K] device array of vertical coefficients
struct CoefJob {
    double* table;   // [M][1+K]
    double a;        // vertical coefficient of accumulator k
    int l, K, k;
};
struct CoefJobs {
    CoefJob j[16];
    int n;
};
// R[i*M + j] = 1/(xi_j - xi_i) for j > i (per-context table)
cudaError_t launch_coef_tables(const double* xi, const double* R, int M, const CoefJobs& jobs, double dt, double c,
                               double gamma, const double* cg_dev, int* status, cudaStream_t s);

// ---------------------------------------------------------------- black-box RHS path (lx_blackbox.cu)
// Control block of the callback-driven Leja loop: decision + FD scaling state.
struct BbCtrl {
    int done;                          // decision: stop (kernels of later iterations return at entry)
    int active;                        // bit k = accumulator k still accumulating
    int status;
    int m;                             // last decided iteration
    unsigned int ticket;               // last-CTA ticket
    unsigned int pad;
    unsigned long long maxbits[3];     // max|y| of y_{m} at [m & 1]; [2]: remainder direction (bit patterns)
    unsigned long long umaxbits;       // max|u| (FD scaling, R25)
};
struct BbArgs {
    long long N;                       // local points
    double N_glob;
    int K, mode;                       // mode 1 = FD Jacobian, 2 = linear operator (J y = f(y))
    int max_nodes, grid;
    double alpha, rtol, atol;
    const double* table;               // [max_nodes][1+K]: beta_m, d_m^(k) (k_coef_tables)
    const double* u;                   // linearisation state (FD)
    const double* fu;                  // f(u) (FD)
    const double* y_in;                // y_{m-1} (v at m = 1)
    double* y_out;                     // y_m
    double* w;                         // perturbed state u + eps y_{m-1}
    const double* fw;                  // f(w) (FD) or f(y_{m-1}) (linear)
    double* p[kMaxK];
    double* partials;                  // [grid][1+K]
    BbCtrl* ctrl;
    Record* rec;
    int* done_host;                    // mapped pinned word: iteration at which the loop stopped
};
struct BbLin {
    long long N;
    double N_glob;
    int grid;
    const double* x0; const double* x1; const double* x2; const double* x3;
    double a0, a1, a2, a3;
    double* y0;
    const double* u;
    const double* fu;
    double* partials;
    BbCtrl* ctrl;
    Record* rec;
};
// literal, contraction-free f(u) of the built-in problems (lx_builtin_rhs; single domain)
struct RhsLit {
    int ndim;
    long long n[3];                    // points per dimension (n[2] = 1 in 2D)
    double dx[3];
    double diff, nu, react, flux;
    const double* src;                 // optional source S
    const double* in;
    double* out;
};
cudaError_t launch_rhs_literal(const RhsLit& R, int grid, cudaStream_t s);
// load every kernel now (CUDA lazy loading): required before virtual ranks run spinning persistent kernels
cudaError_t preload_kernels();
cudaError_t preload_bb_kernels();
int bb_grid(int nsm);
cudaError_t launch_bb_init(const BbArgs& A, cudaStream_t s);
cudaError_t launch_bb_perturb(const BbArgs& A, int m, cudaStream_t s);
cudaError_t launch_bb_update(const BbArgs& A, int m, cudaStream_t s);
cudaError_t launch_bb_maxabs(const double* x, long long N, BbCtrl* c, int grid, cudaStream_t s);
cudaError_t launch_bb_fdpiece(const BbLin& L, int op, cudaStream_t s);   // 0: u + eps x0 ; 1: x0 - (x1 - fu)/eps
cudaError_t launch_bb_lincomb(const BbLin& L, cudaStream_t s);
cudaError_t launch_bb_norm(const BbLin& L, cudaStream_t s);

}  // namespace lx
