// lx_host.cpp -- host runtime and C ABI of the B200-native LeXInt hot path.
//
// Owns the context (scratch buffers allocated once, P:307 / P:359-407), builds
// the per-call coefficient tables (beta_m = -c/gamma - xi_{m-1}, d_m^(k)),
// launches the persistent Leja kernel / stage kernels on the context stream
// and reads back one small record per call or step.  See include/lexint.h.
#include "../../include/lexint.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lx_hostmath.h"
#include "lx_internal.h"
#include "lx_comm.h"

using namespace lx;

static thread_local std::string g_err;

static lx_status fail(lx_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CUDA_TRY(x)                                                                       \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) return fail(LX_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

#define LX_TRY(x)                     \
    do {                              \
        lx_status s_ = (x);           \
        if (s_ != LX_OK) return s_;   \
    } while (0)

static constexpr int kCoefSlots = 32;
static constexpr int kStage = 10;  // integrator scratch vectors (4 stages + 3 states for lx_integrate + 1 EPIRK5P1
                                   // + 2 EXPRB54s4)
static constexpr int kHost = 6;    // host-pointer staging vectors
static constexpr int kBb = 11;     // black-box path vectors
// Auto policy of the two-step kernel (measured round 1): its per-pass latency chain (~27 us)
// loses to the one-pass kernel below ~1700^2 points (Leja calls and Allen-Cahn EXPRB43 alike).
static constexpr int64_t kTb2MinPoints = 3 << 20;
static constexpr int64_t kTb3MinPoints = 1 << 20;   // 3D two-step kernel from this many points on

struct lx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int ndim = 2;
    int64_t n[3] = {1, 1, 1};
    int64_t i_begin = 0, i_end = 0;
    int n_loc = 0;
    int64_t row = 0;          // doubles per row (n1*n2)
    int64_t N_loc = 0;
    double N_glob = 0;
    int max_nodes = 300;
    int nsm = 0;
    // device memory
    double* Y[2] = {nullptr, nullptr};
    double* Yg[2] = {nullptr, nullptr};   // ghost rows (comm mode)
    double* vg = nullptr;                 // ghost rows of the iteration-1 input
    double* S[kStage] = {};
    double* H[kHost] = {};
    double* partials = nullptr;
    int max_grid = 0;
    Ctrl* ctrl = nullptr;
    Record* rec_dev = nullptr;            // [2]: 0 sync, 1 async
    Record* rec_host = nullptr;           // pinned [2]
    Record* rec_init = nullptr;           // pinned template
    unsigned long long* umax_host = nullptr;
    double* coef_dev = nullptr;
    double* coef_host = nullptr;
    size_t coef_stride = 0;
    cudaEvent_t coef_ev[kCoefSlots] = {};
    int coef_next = 0;
    unsigned long long slot_key[kCoefSlots] = {};   // key of the prebuilt table in each ring slot (0: none)
    int64_t launches = 0;
    std::vector<double> xi;
    double* xi_dev = nullptr;             // Leja points on the device
    double* rcp_dev = nullptr;            // [M][M]: 1/(xi_j - xi_i), j > i (divided-difference recurrence)
    Comm* comm = nullptr;                 // slab decomposition (lx_comm.cpp)
    int tblock = 0;                       // 2D single-GPU: Leja iterations per HBM pass (lx_ctx_set_kernel:
                                          // 1 or 2; 0 = auto: two-step from kTb2MinPoints local points on)
    int tb2_cap = 0;                      // segments the buffers below can hold
    Tb2Ctl* tb2_ctl = nullptr;            // pipelined two-step kernel control block (pbase starts at 1)
    unsigned* tb2_scnt = nullptr;         // [cap] per-segment completion tags
    double* tb2_pscr[kMaxK] = {};         // p ping-pong scratch halves (one N-vector per accumulator)
    double* tb2_seg_part = nullptr;       // [2 pass parities][cap][2(1+kMaxK)]
    double* tb2_grp_part = nullptr;       // [2][cap/32+1][2(1+kMaxK)]
    unsigned* tb2_grp_cnt = nullptr;      // [2][cap/32+1]
    void* ipc_blk = nullptr;              // exchange block handed out by lx_ctx_ipc_handle (before set_comm_ipc)
    bool bb_literal = true;               // lx_builtin_rhs: literal formula order (FD mode) or fused stencil
    // pipelined host-buffer staging of Leja calls (pinned host memory): two slots, copy-in / copy-out streams
    cudaStream_t s_in = nullptr, s_out = nullptr;
    double* pin_in[2] = {};
    double* pin_out[2][kMaxK] = {};
    cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
    int pipe_next = 0;
    const void* pin_key = nullptr;        // host input staged in pin_in[pin_key_slot], valid until the next
    int pin_key_slot = 0;                 // synchronisation point (the caller may not modify it before)
    int k3d = 0;                          // 3D single-GPU Leja kernel: 0 = smem marching when n1 % 16 == 0 and
                                          // n2 % 64 == 0 (else warp tiles), 1 = warp tiles (lx_ctx_set_kernel)
    double* cg_dev = nullptr;             // device (c, gamma, bound) of lx_integrate
    const double* cg_active = nullptr;    // when set, Leja kernels take (c, gamma) from here
    // black-box RHS path (lx_real_leja_phi_cb / lx_step_cb)
    BbCtrl* bb = nullptr;                 // device control block
    int* bb_done_host = nullptr;          // mapped pinned word written by the deciding CTA
    int* bb_done_dev = nullptr;           // its device alias
    cudaEvent_t bb_ev[4] = {};
    double* B[kBb] = {};                  // black-box vectors: f(u), f_u dt, t1..t7, w, f(w)
};

// ------------------------------------------------------------------ helpers
static bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static bool is_pinned_host_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

static Stencil make_stencil(const lx_problem* pb) {
    Stencil st;
    std::memset(&st, 0, sizeof st);
    double c0 = 0.0;
    for (int d = 0; d < pb->ndim; d++) {
        const double h = pb->dx[d], ih2 = 1.0 / (h * h);
        // diff*(u[+1] - 2u + u[-1])/h^2 + nu*(-u[+2] + 6u[+1] - 3u - 2u[-1])/(6h)
        st.m1[d] = pb->diff * ih2 - pb->nu / (3.0 * h);
        st.p1[d] = pb->diff * ih2 + pb->nu / h;
        st.p2[d] = -pb->nu / (6.0 * h);
        c0 += -2.0 * pb->diff * ih2 - pb->nu / (2.0 * h);
    }
    st.c0 = c0;
    st.react = pb->react;
    st.qa = pb->react;          // J_ii = react*(1 - 3u^2)
    st.qb = -3.0 * pb->react;
    // flux form (Burgers): diffusion and upwind kept apart, velocity field nu + beta*u
    st.flux = pb->flux;
    st.nu = pb->nu;
    for (int d = 0; d < pb->ndim; d++) {
        const double h = pb->dx[d], ih2 = 1.0 / (h * h);
        st.dm1[d] = pb->diff * ih2;
        st.dp1[d] = pb->diff * ih2;
        st.dd0 += -2.0 * pb->diff * ih2;
        st.am1[d] = -2.0 / (6.0 * h);
        st.a0[d] = -3.0 / (6.0 * h);
        st.ap1[d] = 6.0 / (6.0 * h);
        st.ap2[d] = -1.0 / (6.0 * h);
    }
    return st;
}

static lx_status check_problem(const lx_ctx* ctx, const lx_problem* pb) {
    if (!pb) return fail(LX_ERR_ARG, "problem is NULL");
    if (pb->ndim != ctx->ndim) return fail(LX_ERR_DIM, "problem ndim %d != context ndim %d", pb->ndim, ctx->ndim);
    for (int d = 0; d < pb->ndim; d++)
        if (pb->n[d] != ctx->n[d]) return fail(LX_ERR_DIM, "problem n[%d] differs from the context grid", d);
    for (int d = 0; d < pb->ndim; d++)
        if (!(pb->dx[d] > 0.0)) return fail(LX_ERR_ARG, "dx[%d] must be > 0", d);
    if (pb->flux != 0.0 && (pb->ndim != 2 || ctx->comm))
        return fail(LX_ERR_UNSUPPORTED, "flux (Burgers) problems: 2D single-GPU contexts only");
    return LX_OK;
}

static double* stage_buf(lx_ctx* ctx, int i) {
    if (!ctx->H[i]) {
        if (cudaMalloc(&ctx->H[i], ctx->N_loc * sizeof(double)) != cudaSuccess) return nullptr;
    }
    return ctx->H[i];
}

static double* scratch(lx_ctx* ctx, int i) {
    if (!ctx->S[i]) {
        if (cudaMalloc(&ctx->S[i], ctx->N_loc * sizeof(double)) != cudaSuccess) return nullptr;
    }
    return ctx->S[i];
}

// Host<->device staging of one call's vectors.
struct Staging {
    lx_ctx* ctx;
    int next = 0;
    struct Out { double* host; double* dev; };
    std::vector<Out> outs;
    bool any_host = false;
    explicit Staging(lx_ctx* c) : ctx(c) {}
    lx_status in(const double* p, const double** dev) {
        if (!p) { *dev = nullptr; return LX_OK; }
        if (is_device_ptr(p)) { *dev = p; return LX_OK; }
        any_host = true;
        double* b = stage_buf(ctx, next++);
        if (!b) return fail(LX_ERR_CUDA, "staging allocation failed");
        CUDA_TRY(cudaMemcpyAsync(b, p, ctx->N_loc * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        *dev = b;
        return LX_OK;
    }
    lx_status out(double* p, double** dev) {
        if (!p) { *dev = nullptr; return LX_OK; }
        if (is_device_ptr(p)) { *dev = p; return LX_OK; }
        any_host = true;
        double* b = stage_buf(ctx, next++);
        if (!b) return fail(LX_ERR_CUDA, "staging allocation failed");
        outs.push_back({p, b});
        *dev = b;
        return LX_OK;
    }
    lx_status finish() {
        for (auto& o : outs)
            CUDA_TRY(cudaMemcpyAsync(o.host, o.dev, ctx->N_loc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        return LX_OK;
    }
};

static lx_status reset_record(lx_ctx* ctx, int r) {
    CUDA_TRY(cudaMemcpyAsync(ctx->rec_dev + r, ctx->rec_init, sizeof(Record), cudaMemcpyHostToDevice, ctx->stream));
    return LX_OK;
}

static lx_status read_record(lx_ctx* ctx, int r, Record* out) {
    CUDA_TRY(cudaMemcpyAsync(ctx->rec_host + r, ctx->rec_dev + r, sizeof(Record), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    *out = ctx->rec_host[r];
    return LX_OK;
}

static lx_status status_of(const Record& r) {
    switch (r.status) {
        case 0: return LX_OK;
        case 5: return fail(LX_ERR_NOCONV, "Leja interpolation did not converge within the node cap (iters %d)", r.iters);
        case 6: return fail(LX_ERR_NONFINITE, "non-finite norm in the Leja iteration (spectrum not enclosed?)");
        case 10: return fail(LX_ERR_TIMEOUT, "device barrier watchdog fired");
        default: return fail(LX_ERR_CUDA, "device status %d", r.status);
    }
}

// Coefficient tables ({beta_m, d_m^(k)}, m < max_nodes) of one or several Leja calls, built ON THE
// DEVICE by one k_coef_tables launch (one CTA per accumulator) on the context stream: no host
// arithmetic, no H2D copy.  Ring slots keep tables of in-flight calls apart (stream order makes
// reuse safe).
struct TableSpec {
    int l;
    int K;
    const double* coeffs;
};

// Leja iterations per HBM pass of this context's 2D single-GPU Leja calls (1 or 2).
static bool tb3_shape(const lx_ctx* ctx) {
    return ctx->ndim == 3 && ctx->k3d != 1 && ctx->n[1] % 16 == 0 && ctx->n[2] % 64 == 0;
}

static int ctx_tblock(const lx_ctx* ctx) {
    if (ctx->comm) return ((ctx->ndim == 2 || tb3_shape(ctx)) && comm_peer_ready(ctx->comm)) ? 2 : 1;
    if (ctx->ndim == 3) {
        if (!tb3_shape(ctx) || ctx->tblock == 1) return 1;
        return (ctx->tblock == 2 || ctx->N_loc >= kTb3MinPoints) ? 2 : 1;
    }
    if (ctx->ndim != 2 || ctx->n_loc < 16 || ctx->n[1] < 64) return 1;
    if (ctx->tblock == 1) return 1;
    if (ctx->tblock == 2) return 2;
    return ctx->N_loc >= kTb2MinPoints ? 2 : 1;
}

static lx_status build_tables(lx_ctx* ctx, const TableSpec* specs, int n, double dt, double c, double gamma, int rec,
                              const double** tables_out) {
    CoefJobs jobs;
    std::memset(&jobs, 0, sizeof jobs);
    for (int t = 0; t < n; t++) {
        const int slot = ctx->coef_next;
        ctx->coef_next = (slot + 1) % kCoefSlots;
        ctx->slot_key[slot] = 0;
        double* dev = ctx->coef_dev + slot * ctx->coef_stride;
        tables_out[t] = dev;
        for (int k = 0; k < specs[t].K; k++) {
            if (jobs.n >= 16) return fail(LX_ERR_ARG, "too many coefficient tables in one batch");
            jobs.j[jobs.n++] = CoefJob{dev, specs[t].coeffs[k], specs[t].l, specs[t].K, k};
        }
    }
    CUDA_TRY(launch_coef_tables(ctx->xi_dev, ctx->rcp_dev, ctx->max_nodes, jobs, dt, c, gamma, nullptr,
                                &ctx->rec_dev[rec].status, ctx->stream));
    ctx->launches++;
    return LX_OK;
}

static LejaParams base_params(lx_ctx* ctx, const lx_problem* pb) {
    LejaParams P;
    std::memset(&P, 0, sizeof P);
    P.ndim = ctx->ndim;
    P.n_loc = ctx->n_loc;
    P.n1 = (int)ctx->n[1];
    P.n2 = (int)ctx->n[2];
    P.nrb = (P.n_loc + kRT - 1) / kRT;
    if (ctx->ndim == 3) {
        P.nrb = (P.n_loc + kRT3 - 1) / kRT3;
        P.nb = (P.n2 + 63) / 64;                 // 64-wide bands along the contiguous dim 2
        P.nunits = P.nb * P.n1 * P.nrb;          // u = (plane_block*nb + band)*n1 + j
    } else {
        P.nb = (P.n1 + 63) / 64;
        P.nunits = P.nb * P.nrb;                 // u = row_block*nb + band
    }
    P.N_glob = ctx->N_glob;
    P.st = make_stencil(pb);
    if (pb->flux != 0.0) {
        P.ndim = 4;   // flux-form (Burgers) tile variant of the 2D kernels
        P.nrb = (P.n_loc + kRTF - 1) / kRTF;
        P.nunits = P.nb * P.nrb;
    }
    P.ctrl = ctx->ctrl;
    P.partials = ctx->partials;
    P.timeout_spins = 1 << 24;
    for (int i = 0; i < 2; i++) {
        P.ysrc[i] = RowSrc{ctx->Y[i], ctx->comm ? ctx->Yg[i] : nullptr, ctx->row, ctx->n_loc, 0};
        P.ydst[i] = ctx->Y[i];
    }
    return P;
}

// Core Leja call on device pointers (no staging, no sync).
// Work decomposition of the two-step kernel (single domain and slab): items = (60-column band,
// RT-row chunk); 32-row segments handed out dynamically, band fastest; per-segment / per-group partials.
// Control block of the two-step kernels (2D: pipelined-pass state + prediction table; 3D: the table of
// final iterations of recent calls).
static lx_status tb2_ctl_alloc(lx_ctx* ctx) {
    if (!ctx->tb2_ctl) {
        CUDA_TRY(cudaMalloc(&ctx->tb2_ctl, sizeof(Tb2Ctl)));
        Tb2Ctl init;
        std::memset(&init, 0, sizeof init);
        init.pbase = 1u;   // tags >= 1: the zeroed counters, flags and decision words never match
        CUDA_TRY(cudaMemcpy(ctx->tb2_ctl, &init, sizeof init, cudaMemcpyHostToDevice));
    }
    return LX_OK;
}

static lx_status tb2_buffers(lx_ctx* ctx, int nseg, int K) {
    LX_TRY(tb2_ctl_alloc(ctx));
    if (nseg > ctx->tb2_cap) {
        cudaFree(ctx->tb2_seg_part);
        cudaFree(ctx->tb2_grp_part);
        cudaFree(ctx->tb2_grp_cnt);
        cudaFree(ctx->tb2_scnt);
        ctx->tb2_seg_part = nullptr;
        ctx->tb2_grp_part = nullptr;
        ctx->tb2_grp_cnt = nullptr;
        ctx->tb2_scnt = nullptr;
        ctx->tb2_cap = 0;
        const size_t nv = 2 * (1 + kMaxK), ngrp = (size_t)(nseg + 31) / 32;
        CUDA_TRY(cudaMalloc(&ctx->tb2_seg_part, 2 * (size_t)nseg * nv * sizeof(double)));
        CUDA_TRY(cudaMalloc(&ctx->tb2_grp_part, 2 * ngrp * nv * sizeof(double)));
        CUDA_TRY(cudaMalloc(&ctx->tb2_grp_cnt, 2 * ngrp * sizeof(unsigned)));
        CUDA_TRY(cudaMalloc(&ctx->tb2_scnt, (size_t)nseg * sizeof(unsigned)));
        CUDA_TRY(cudaMemsetAsync(ctx->tb2_grp_cnt, 0, 2 * ngrp * sizeof(unsigned), ctx->stream));
        CUDA_TRY(cudaMemsetAsync(ctx->tb2_scnt, 0, (size_t)nseg * sizeof(unsigned), ctx->stream));
        ctx->tb2_cap = nseg;
    }
    for (int k = 0; k < K; k++)
        if (!ctx->tb2_pscr[k]) CUDA_TRY(cudaMalloc(&ctx->tb2_pscr[k], ctx->N_loc * sizeof(double)));
    return LX_OK;
}

// Work decomposition of the two-step kernel (single domain and slab): items = (60-column band,
// RT-row chunk); 32-row segments handed out in (pass, segment) order, band fastest; per-segment /
// per-group partials by pass parity; p ping-pong between the caller's output and context scratch.
static lx_status tb2_setup(lx_ctx* ctx, LejaParams& P, int K, bool diag) {
    P.nb = (P.n1 + kBand2 - 1) / kBand2;
    P.nrb = (P.n_loc + tb2_rt(K) - 1) / tb2_rt(K);
    P.nunits = P.nb * P.nrb;
    P.grid = leja_tb2_grid_size(ctx->device, K, diag, P.nunits);
    if (ctx->comm) P.grid = comm_grid_cap(ctx->comm, P.grid);
    P.seg = 32 / tb2_rt(K);   // 32-row segments (measured: 64 rows are 5% slower at 4096^2)
    // segment rows of 32 rows; a short remainder (< 4 rows) joins the last full one, so that every
    // segment row has >= 4 rows (the kernel's dependency sets assume it)
    int nsr = (P.nrb + P.seg - 1) / P.seg;
    if (nsr > 1 && P.n_loc - (nsr - 1) * P.seg * tb2_rt(K) < 4) nsr--;
    P.nseg = P.nb * nsr;
    P.ngrp = (P.nseg + 31) / 32;
    LX_TRY(tb2_buffers(ctx, P.nseg, K));
    P.seg_part = ctx->tb2_seg_part;
    P.grp_part = ctx->tb2_grp_part;
    P.grp_cnt = ctx->tb2_grp_cnt;
    P.tc = ctx->tb2_ctl;
    P.scnt = ctx->tb2_scnt;
    for (int k = 0; k < kMaxK; k++) {
        P.pp[k][0] = k < K ? P.p[k] : nullptr;
        P.pp[k][1] = k < K ? ctx->tb2_pscr[k] : nullptr;
    }
    if (!P.timeout_ns) P.timeout_ns = 60ull * 1000000000ull;
    return LX_OK;
}

// The 3D kernels read the Newton coefficients from a table built by one k_coef_tables launch.
static lx_status leja3d_table(lx_ctx* ctx, LejaParams& P, int K, int l, const double* coeffs, double dt, double c,
                              double gamma, int rec) {
    (void)l;
    if (!P.coef_gen) return LX_OK;
    // a table depends only on (K, l_k, a_k, dt, c, gamma): a repeated call (fixed dt and spectrum: every step
    // of a linear problem) reuses the ring slot that still holds it instead of rebuilding it (host-known
    // (c, gamma) only; lx_integrate's device-side (c, gamma) always rebuild)
    unsigned long long key = 0;
    if (!ctx->cg_active) {
        unsigned long long h = 1469598103934665603ull;
        auto mix = [&h](unsigned long long x) {
            h ^= x;
            h *= 1099511628211ull;
        };
        auto bits = [](double x) {
            unsigned long long b;
            std::memcpy(&b, &x, sizeof b);
            return b;
        };
        mix((unsigned long long)K | ((unsigned long long)ctx->max_nodes << 8));
        for (int k = 0; k < K; k++) {
            mix((unsigned long long)P.lk[k]);
            mix(bits(coeffs[k]));
        }
        mix(bits(dt));
        mix(bits(c));
        mix(bits(gamma));
        key = h | 1ull;
        for (int sl = 0; sl < kCoefSlots; sl++)
            if (ctx->slot_key[sl] == key) {
                P.table = ctx->coef_dev + sl * ctx->coef_stride;
                P.coef = P.table;
                P.coef_gen = 0;
                return LX_OK;
            }
    }
    CoefJobs jobs;
    std::memset(&jobs, 0, sizeof jobs);
    for (int k = 0; k < K; k++) jobs.j[jobs.n++] = CoefJob{P.table, coeffs[k], P.lk[k], K, k};
    CUDA_TRY(launch_coef_tables(ctx->xi_dev, ctx->rcp_dev, ctx->max_nodes, jobs, dt, c, gamma, ctx->cg_active,
                                &ctx->rec_dev[rec].status, ctx->stream));
    ctx->launches++;
    if (key) ctx->slot_key[(P.table - ctx->coef_dev) / ctx->coef_stride] = key;
    P.coef_gen = 0;
    return LX_OK;
}

static lx_status leja_device(lx_ctx* ctx, const lx_problem* pb, const double* u, const double* v, double* const* outs,
                             const double* coeffs, int K, double dt, double c, double gamma, int l, double rtol,
                             double atol, int rec, const double* table = nullptr, const int* ls = nullptr) {
    const double* coef = table;
    LejaParams P = base_params(ctx, pb);
    const bool diag = pb->react != 0.0;
    // coefficient description (read by the prologue of every Leja kernel); ls: one phi index per accumulator
    P.l = l;
    for (int k = 0; k < kMaxK; k++) P.lk[k] = (ls && k < K) ? ls[k] : l;
    P.cdt = dt;
    P.cc = c;
    P.cgamma = gamma;
    for (int k = 0; k < kMaxK; k++) P.ak[k] = k < K ? coeffs[k] : 1.0;
    P.xi = ctx->xi_dev;
    P.R = ctx->rcp_dev;
    P.table = const_cast<double*>(coef);
    P.cg_dev = ctx->cg_active;
    if (!coef) {
        // the Leja kernels compute their own Newton coefficients (coefficient warp) into a ring slot
        const int slot = ctx->coef_next;
        ctx->coef_next = (slot + 1) % kCoefSlots;
        ctx->slot_key[slot] = 0;
        double* tab = ctx->coef_dev + slot * ctx->coef_stride;
        P.coef_gen = 1;
        P.table = tab;
        coef = tab;
    }
    P.K = K;
    P.max_nodes = ctx->max_nodes;
    P.active0 = (1 << K) - 1;
    P.alpha = (dt == 0.0) ? 0.0 : 1.0 / gamma;
    P.rtol = rtol;
    P.atol = atol;
    P.coef = coef;
    P.v = RowSrc{v, nullptr, ctx->row, ctx->n_loc, 0};
    for (int k = 0; k < K; k++) P.p[k] = outs[k];
    P.u = u;
    P.rec = ctx->rec_dev + rec;
    if (ctx->comm) {
        // slab decomposition: the persistent two-step slab kernel over peer memory when the transport
        // provides it (2D constant-coefficient / Allen-Cahn operators), else the per-iteration protocol
        if (P.ndim == 2 && comm_peer_ready(ctx->comm) && P.n_loc >= 16 && P.n1 >= 64) {
            LX_TRY(tb2_setup(ctx, P, K, diag));
            comm_peer_params(ctx->comm, P, diag);
            CUDA_TRY(launch_leja_tb2(P, ctx->stream, diag, true));
            ctx->launches++;
            return LX_OK;
        }
        if (P.ndim == 3 && !diag && comm_peer_ready(ctx->comm) && tb3_shape(ctx)) {
            // 3D: the two-step plane-sweep kernel over peer memory (ghost planes, global barrier per pass)
            LX_TRY(leja3d_table(ctx, P, K, l, coeffs, dt, c, gamma, rec));
            LX_TRY(tb2_ctl_alloc(ctx));
            P.tc = ctx->tb2_ctl;
            P.grid = comm_grid_cap(ctx->comm, leja3d_tb2_grid_size(ctx->device, K, leja3d_smem_units(P.n_loc, P.n1, P.n2), true));
            comm_peer_params(ctx->comm, P, diag);
            CUDA_TRY(launch_leja3d_tb2(P, ctx->stream, true));
            ctx->launches++;
            return LX_OK;
        }
        return comm_leja(ctx->comm, P, diag, ctx->stream, &ctx->launches);
    }
    if (P.ndim == 2 && ctx_tblock(ctx) == 2) {
        LX_TRY(tb2_setup(ctx, P, K, diag));
        CUDA_TRY(launch_leja_tb2(P, ctx->stream, diag));
        ctx->launches++;
        return LX_OK;
    }
    if (P.ndim == 3 && ctx->k3d != 1 && P.n1 % 16 == 0 && P.n2 % 64 == 0) {
        // 3D marching kernel with shared-memory plane tiles: Newton coefficients from a prebuilt table
        LX_TRY(leja3d_table(ctx, P, K, l, coeffs, dt, c, gamma, rec));
        const int ncu = leja3d_smem_units(P.n_loc, P.n1, P.n2);
        if (!diag && ctx_tblock(ctx) == 2) {
            // two Leja iterations per HBM pass (2.5D temporal blocking)
            LX_TRY(tb2_ctl_alloc(ctx));
            P.tc = ctx->tb2_ctl;
            P.grid = leja3d_tb2_grid_size(ctx->device, K, ncu);
            CUDA_TRY(launch_leja3d_tb2(P, ctx->stream));
            ctx->launches++;
            return LX_OK;
        }
        P.grid = leja3d_smem_grid_size(ctx->device, K, diag, ncu);
        CUDA_TRY(launch_leja3d_smem(P, ctx->stream, diag));
        ctx->launches++;
        return LX_OK;
    }
    P.grid = leja_grid_size(ctx->device, K, diag, P.ndim, P.nunits);
    CUDA_TRY(launch_leja_persistent(P, ctx->stream, diag));
    ctx->launches++;
    return LX_OK;
}

static lx_status validate_leja(const lx_problem* pb, const double* u, const double* v, double* const* outs,
                               const double* coeffs, int K, double dt, double gamma, int l, const int* ls = nullptr) {
    if (!v || !outs || !coeffs) return fail(LX_ERR_ARG, "NULL argument");
    if (K < 1 || K > kMaxK) return fail(LX_ERR_UNSUPPORTED, "K = %d not in [1, 4]", K);
    for (int k = 0; k < (ls ? K : 1); k++) {
        const int lk = ls ? ls[k] : l;
        if (lk < 0 || lk > 4) return fail(LX_ERR_UNSUPPORTED, "phi_%d not supported (l <= 4)", lk);
    }
    if (!(gamma > 0.0) && dt != 0.0) return fail(LX_ERR_ARG, "gamma must be > 0 (got %g)", gamma);
    if (!std::isfinite(dt)) return fail(LX_ERR_ARG, "dt not finite");
    for (int k = 0; k < K; k++) {
        if (!(coeffs[k] > 0.0 && coeffs[k] <= 1.0)) return fail(LX_ERR_ARG, "coeffs[%d] not in (0, 1]", k);
        if (!ls && k > 0 && !(coeffs[k] > coeffs[k - 1])) return fail(LX_ERR_ARG, "coeffs not strictly increasing");
        for (int j = 0; ls && j < k; j++)
            if (ls[j] == ls[k] && coeffs[j] == coeffs[k]) return fail(LX_ERR_ARG, "(l, coeff) pairs must be distinct");
        if (!outs[k]) return fail(LX_ERR_ARG, "outs[%d] is NULL", k);
        if (outs[k] == v || (u && outs[k] == u)) return fail(LX_ERR_ALIAS, "out must not alias v or u_lin");
        for (int j = 0; j < k; j++)
            if (outs[j] == outs[k]) return fail(LX_ERR_ALIAS, "outs must be distinct");
    }
    if ((pb->react != 0.0 || pb->flux != 0.0) && !u) return fail(LX_ERR_ARG, "u_lin required when react/flux != 0");
    return LX_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

const char* lx_last_error(void) { return g_err.c_str(); }
const char* lx_version(void) { return "lexint-b200 0.1 (sm_100a, fp64)"; }

lx_status lx_leja_points(int count, double* xi_out) {
    if (lx::leja_points(count, xi_out)) return fail(LX_ERR_ARG, "count must be in [1, 4096]");
    return LX_OK;
}

lx_status lx_phi_scalar(int l, double z, double* out) {
    if (!out) return fail(LX_ERR_ARG, "out is NULL");
    if (l < 0 || l > 4) return fail(LX_ERR_UNSUPPORTED, "phi_%d not supported (l <= 4)", l);
    *out = lx::phi(l, z);
    return LX_OK;
}

lx_status lx_divided_differences(int l, const double* xi, int m, double dt, double c, double gamma, double a,
                                 double* d_out) {
    const int s = lx::divided_differences(l, xi, m, dt, c, gamma, a, d_out);
    if (s == 1) return fail(LX_ERR_ARG, "bad arguments");
    if (s == 4) return fail(LX_ERR_UNSUPPORTED, "phi_%d not supported", l);
    if (s == 6) return fail(LX_ERR_NONFINITE, "divided differences overflow");
    return LX_OK;
}

int lx_slab_halo_plan(int rank, int nranks, int64_t n_loc, int mode, int* ops, int max_ops) {
    if (!ops) return -1;
    return comm_halo_plan(rank, nranks, (int)n_loc, mode, ops, max_ops);
}

lx_status lx_slab_range(int64_t n0, int rank, int nranks, int64_t* i_begin, int64_t* i_end) {
    if (nranks < 1 || rank < 0 || rank >= nranks || n0 < 1 || !i_begin || !i_end)
        return fail(LX_ERR_ARG, "bad slab arguments");
    *i_begin = (n0 * rank) / nranks;
    *i_end = (n0 * (rank + 1)) / nranks;
    return LX_OK;
}

lx_status lx_shift_scale(double lambda_abs, double* c_out, double* gamma_out) {
    if (!(lambda_abs >= 0.0) || !c_out || !gamma_out) return fail(LX_ERR_ARG, "lambda_abs must be >= 0");
    const double eig = -1.05 * lambda_abs;
    *c_out = eig / 2.0;
    *gamma_out = -eig / 4.0;
    return LX_OK;
}

static void free_ctx(lx_ctx* ctx) {
    if (!ctx) return;
    if (ctx->comm) comm_destroy(ctx->comm);
    for (double* p : ctx->Y) cudaFree(p);
    for (double* p : ctx->Yg) cudaFree(p);
    cudaFree(ctx->vg);
    for (double* p : ctx->S) cudaFree(p);
    for (double* p : ctx->H) cudaFree(p);
    for (int i = 0; i < 2; i++) {
        cudaFree(ctx->pin_in[i]);
        for (double* p : ctx->pin_out[i]) cudaFree(p);
        for (cudaEvent_t e : {ctx->ev_in[i], ctx->ev_comp[i], ctx->ev_out[i]})
            if (e) cudaEventDestroy(e);
    }
    if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
    if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
    cudaFree(ctx->partials);
    cudaFree(ctx->tb2_seg_part);
    cudaFree(ctx->tb2_grp_part);
    cudaFree(ctx->tb2_grp_cnt);
    cudaFree(ctx->ctrl);
    cudaFree(ctx->rec_dev);
    cudaFree(ctx->coef_dev);
    cudaFree(ctx->xi_dev);
    cudaFree(ctx->rcp_dev);
    cudaFree(ctx->cg_dev);
    cudaFreeHost(ctx->rec_host);
    cudaFreeHost(ctx->rec_init);
    cudaFreeHost(ctx->umax_host);
    cudaFreeHost(ctx->coef_host);
    for (auto& e : ctx->coef_ev)
        if (e) cudaEventDestroy(e);
    for (double* p : ctx->B) cudaFree(p);
    cudaFree(ctx->bb);
    cudaFreeHost(ctx->bb_done_host);
    for (auto& e : ctx->bb_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

static lx_status alloc_local(lx_ctx* ctx) {
    const size_t bytes = ctx->N_loc * sizeof(double);
    for (int i = 0; i < 2; i++) {
        if (ctx->Y[i]) cudaFree(ctx->Y[i]);
        CUDA_TRY(cudaMalloc(&ctx->Y[i], bytes));
        CUDA_TRY(cudaMemsetAsync(ctx->Y[i], 0, bytes, ctx->stream));
    }
    for (int i = 0; i < kStage; i++) {
        cudaFree(ctx->S[i]);
        ctx->S[i] = nullptr;
    }
    for (int i = 0; i < kHost; i++) {
        cudaFree(ctx->H[i]);
        ctx->H[i] = nullptr;
    }
    return LX_OK;
}

lx_status lx_ctx_create(const lx_problem* pb, int max_nodes, int device, void* cuda_stream, lx_ctx** out) {
    if (!pb || !out) return fail(LX_ERR_ARG, "NULL argument");
    *out = nullptr;
    if (pb->ndim != 2 && pb->ndim != 3) return fail(LX_ERR_UNSUPPORTED, "ndim must be 2 or 3");
    for (int d = 0; d < pb->ndim; d++)
        if (pb->n[d] < 4) return fail(LX_ERR_DIM, "n[%d] = %lld < 4", d, (long long)pb->n[d]);
    if (pb->n[pb->ndim - 1] % 2) return fail(LX_ERR_DIM, "the contiguous dimension must be even (double2 access)");
    if (pb->n[0] > (1 << 30) || pb->n[1] > (1 << 30) || (pb->ndim == 3 && pb->n[2] > (1 << 30)))
        return fail(LX_ERR_DIM, "grid too large");
    if (pb->ndim == 3 && (double)pb->n[1] * (double)((pb->n[2] + 63) / 64) * (double)((pb->n[0] + 1) / 2) > 2e9)
        return fail(LX_ERR_DIM, "grid too large for the 32-bit work-unit index");
    if (max_nodes == 0) max_nodes = 300;
    if (max_nodes < 2 || max_nodes > 1024) return fail(LX_ERR_ARG, "max_nodes must be in [2, 1024]");
    lx_ctx* ctx = new lx_ctx();
    if (device < 0) cudaGetDevice(&device);
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) { delete ctx; return fail(LX_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e)); }
    if (cuda_stream) {
        ctx->stream = (cudaStream_t)cuda_stream;
    } else {
        e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) { delete ctx; return fail(LX_ERR_CUDA, "stream: %s", cudaGetErrorString(e)); }
        ctx->own_stream = true;
    }
    ctx->ndim = pb->ndim;
    for (int d = 0; d < 3; d++) ctx->n[d] = d < pb->ndim ? pb->n[d] : 1;
    ctx->i_begin = 0;
    ctx->i_end = ctx->n[0];
    ctx->n_loc = (int)ctx->n[0];
    ctx->row = ctx->n[1] * ctx->n[2];
    ctx->N_loc = (int64_t)ctx->n_loc * ctx->row;
    ctx->N_glob = (double)ctx->n[0] * (double)ctx->row;
    ctx->max_nodes = max_nodes;
    cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, device);
    ctx->max_grid = ctx->nsm * 8;
    ctx->xi.resize(max_nodes);
    lx::leja_points(max_nodes, ctx->xi.data());
    lx_status s = LX_OK;
#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) { s = fail(LX_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); goto bad; } \
    } while (0)
    CK(cudaMalloc(&ctx->partials, (size_t)2 * ctx->max_grid * kSlot * sizeof(double)));
    CK(cudaMalloc(&ctx->ctrl, sizeof(Ctrl)));
    CK(cudaMemsetAsync(ctx->ctrl, 0, sizeof(Ctrl), ctx->stream));
    CK(cudaMalloc(&ctx->rec_dev, 2 * sizeof(Record)));
    CK(cudaMallocHost(&ctx->rec_host, 2 * sizeof(Record)));
    CK(cudaMallocHost(&ctx->rec_init, sizeof(Record)));
    CK(cudaMallocHost(&ctx->umax_host, sizeof(unsigned long long)));
    std::memset(ctx->rec_init, 0, sizeof(Record));
    ctx->rec_init->margin_accept = INFINITY;
    ctx->rec_init->margin_reject = INFINITY;
    ctx->coef_stride = (size_t)max_nodes * (1 + kMaxK);
    CK(cudaMalloc(&ctx->coef_dev, kCoefSlots * ctx->coef_stride * sizeof(double)));
    CK(cudaMallocHost(&ctx->coef_host, kCoefSlots * ctx->coef_stride * sizeof(double)));
    for (auto& ev : ctx->coef_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaMalloc(&ctx->cg_dev, 4 * sizeof(double)));
    CK(cudaMalloc(&ctx->xi_dev, max_nodes * sizeof(double)));
    // stream-ordered uploads: the context's stream may be non-blocking, and a pageable cudaMemcpy
    // may return before its DMA lands
    CK(cudaMemcpyAsync(ctx->xi_dev, ctx->xi.data(), max_nodes * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    {
        std::vector<double> R((size_t)max_nodes * max_nodes, 0.0);
        for (int i = 0; i < max_nodes; i++)
            for (int j = i + 1; j < max_nodes; j++) R[(size_t)i * max_nodes + j] = 1.0 / (ctx->xi[j] - ctx->xi[i]);
        CK(cudaMalloc(&ctx->rcp_dev, R.size() * sizeof(double)));
        CK(cudaMemcpyAsync(ctx->rcp_dev, R.data(), R.size() * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));   // R is a local buffer
    }
#undef CK
    s = alloc_local(ctx);
    if (s != LX_OK) goto bad;
    for (int r = 0; r < 2; r++) {
        s = reset_record(ctx, r);
        if (s != LX_OK) goto bad;
    }
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) { s = fail(LX_ERR_CUDA, "sync: %s", cudaGetErrorString(e)); goto bad; }
    *out = ctx;
    return LX_OK;
bad:
    free_ctx(ctx);
    return s;
}

lx_status lx_ctx_destroy(lx_ctx* ctx) {
    if (!ctx) return LX_OK;
    cudaStreamSynchronize(ctx->stream);
    free_ctx(ctx);
    return LX_OK;
}

lx_status lx_nccl_unique_id(void* out128) {
    if (!out128) return fail(LX_ERR_ARG, "NULL");
    return comm_unique_id(out128) ? fail(LX_ERR_NCCL, "ncclGetUniqueId failed: %s", comm_error()) : LX_OK;
}

static lx_status check_slabs(lx_ctx* ctx, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LX_ERR_ARG, "bad rank/nranks");
    for (int r = 0; r < nranks; r++) {
        int64_t bb, ee;
        lx_slab_range(ctx->n[0], r, nranks, &bb, &ee);
        if (ee - bb < 2) return fail(LX_ERR_DIM, "slab of rank %d has < 2 rows", r);
    }
    return LX_OK;
}

// Re-shape the context to the local slab of `rank` and bind the communicator.
static lx_status attach_comm(lx_ctx* ctx, Comm* c, int rank, int nranks) {
    int64_t b, e;
    lx_slab_range(ctx->n[0], rank, nranks, &b, &e);
    if (ctx->comm) comm_destroy(ctx->comm);
    ctx->comm = c;
    ctx->i_begin = b;
    ctx->i_end = e;
    ctx->n_loc = (int)(e - b);
    ctx->N_loc = (int64_t)ctx->n_loc * ctx->row;
    LX_TRY(alloc_local(ctx));
    if (ctx->comm) {
        for (int i = 0; i < 2; i++) {
            cudaFree(ctx->Yg[i]);
            ctx->Yg[i] = nullptr;
            CUDA_TRY(cudaMalloc(&ctx->Yg[i], 3 * ctx->row * sizeof(double)));
        }
        cudaFree(ctx->vg);
        ctx->vg = nullptr;
        CUDA_TRY(cudaMalloc(&ctx->vg, 3 * ctx->row * sizeof(double)));
        comm_bind(ctx->comm, ctx->Y, ctx->Yg, ctx->vg, ctx->n_loc, rank, nranks);
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return LX_OK;
}

// Peer-memory slab contexts: every buffer a later call could allocate is allocated now.  A rank's
// persistent slab kernel spins until all ranks' kernels arrive; a cudaMalloc / cudaFree on another rank
// in between may wait for the device to idle (virtual ranks share one context) -> deadlock until the
// watchdog.  Scratch vectors, and the two-step segment buffers for the largest segment count (RT = 2).
static lx_status prealloc_slab(lx_ctx* ctx) {
    LX_TRY(tb2_ctl_alloc(ctx));
    for (int i = 0; i < kStage; i++)
        if (!scratch(ctx, i)) return fail(LX_ERR_CUDA, "scratch allocation failed");
    const int nb = ((int)ctx->n[1] + kBand2 - 1) / kBand2, nrb = (ctx->n_loc + 1) / 2, seg = 16;
    LX_TRY(tb2_buffers(ctx, nb * ((nrb + seg - 1) / seg), kMaxK));   // the largest segment count (RT = 2)
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return LX_OK;
}

// The persistent slab kernels over peer memory need a 2D grid with >= 16 rows per rank and >= 64
// columns, or a 3D grid of the two-step kernel's shape (n1 % 16 == 0, n2 % 64 == 0) with >= 4 planes per
// rank (the same condition on every rank: all ranks take the same path).
static bool peer_eligible(const lx_ctx* ctx, int nranks, int flags) {
    if ((flags & LX_COMM_NO_PEER) || nranks > 8) return false;
    if (ctx->ndim == 3) return ctx->n[1] % 16 == 0 && ctx->n[2] % 64 == 0 && ctx->n[0] / nranks >= 4;
    return ctx->ndim == 2 && ctx->n[0] / nranks >= 16 && ctx->n[1] >= 64;
}

static lx_status detach_comm(lx_ctx* ctx) {
    if (ctx->comm) comm_destroy(ctx->comm);
    ctx->comm = nullptr;
    return attach_comm(ctx, nullptr, 0, 1);
}

lx_status lx_ctx_set_comm_ex(lx_ctx* ctx, const void* uid, int rank, int nranks, int flags) {
    if (!ctx || !uid) return fail(LX_ERR_ARG, "NULL");
    LX_TRY(check_slabs(ctx, rank, nranks));
    cudaStreamSynchronize(ctx->stream);
    if (nranks == 1 && !(flags & LX_COMM_FORCE)) return detach_comm(ctx);   // one rank = the single domain
    Comm* c = nullptr;
    if (comm_create(uid, rank, nranks, ctx->device, ctx->row, ctx->nsm * 8, &c))
        return fail(LX_ERR_NCCL, "NCCL communicator: %s", comm_error());
    LX_TRY(attach_comm(ctx, c, rank, nranks));
    if (peer_eligible(ctx, nranks, flags)) {
        if (comm_peer_enable(c, ctx->row)) return fail(LX_ERR_NCCL, "peer-memory transport: %s", comm_error());
        LX_TRY(prealloc_slab(ctx));
    }
    return LX_OK;
}

lx_status lx_ctx_set_comm(lx_ctx* ctx, const void* uid, int rank, int nranks) {
    return lx_ctx_set_comm_ex(ctx, uid, rank, nranks, 0);
}

lx_status lx_ctx_ipc_handle(lx_ctx* ctx, void* out64) {
    if (!ctx || !out64) return fail(LX_ERR_ARG, "NULL");
    const bool ok = ctx->ndim == 2 ? ctx->n[1] >= 64 : (ctx->n[1] % 16 == 0 && ctx->n[2] % 64 == 0);
    if (!ok) return fail(LX_ERR_UNSUPPORTED, "peer transport: 2D grids with n1 >= 64, 3D with n1 % 16 == 0, n2 % 64 == 0");
    if (!ctx->ipc_blk) {
        const size_t bytes = comm_block_bytes(ctx->row);
        CUDA_TRY(cudaMalloc(&ctx->ipc_blk, bytes));
        CUDA_TRY(cudaMemset(ctx->ipc_blk, 0, bytes));
        CUDA_TRY(cudaDeviceSynchronize());
    }
    CUDA_TRY(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)out64, ctx->ipc_blk));
    return LX_OK;
}

lx_status lx_ctx_set_comm_ipc(lx_ctx* ctx, int rank, int nranks, const void* handles) {
    if (!ctx || !handles) return fail(LX_ERR_ARG, "NULL");
    if (!ctx->ipc_blk) return fail(LX_ERR_ARG, "call lx_ctx_ipc_handle first");
    if (nranks < 1 || nranks > 8) return fail(LX_ERR_ARG, "IPC communicator: 1..8 ranks");
    LX_TRY(check_slabs(ctx, rank, nranks));
    if (!peer_eligible(ctx, nranks, 0)) return fail(LX_ERR_DIM, "IPC communicator: needs >= 16 rows per rank");
    cudaStreamSynchronize(ctx->stream);
    Comm* c = nullptr;
    void* blk = ctx->ipc_blk;
    ctx->ipc_blk = nullptr;   // owned by the communicator from here on
    if (comm_create_ipc(rank, nranks, ctx->device, ctx->row, handles, blk, &c))
        return fail(LX_ERR_NCCL, "IPC communicator: %s", comm_error());
    LX_TRY(attach_comm(ctx, c, rank, nranks));
    return prealloc_slab(ctx);
}

struct lx_local_group {
    LocalGroup* g;
    int nranks;
};

lx_status lx_local_group_create(int nranks, lx_local_group** out) {
    if (nranks < 1 || nranks > 64 || !out) return fail(LX_ERR_ARG, "bad nranks");
    *out = new lx_local_group{local_group_create(nranks), nranks};
    return LX_OK;
}

lx_status lx_local_group_destroy(lx_local_group* g) {
    if (g) {
        local_group_destroy(g->g);
        delete g;
    }
    return LX_OK;
}

lx_status lx_ctx_set_comm_local_ex(lx_ctx* ctx, lx_local_group* g, int rank, int flags) {
    if (!ctx || !g) return fail(LX_ERR_ARG, "NULL");
    LX_TRY(check_slabs(ctx, rank, g->nranks));
    cudaStreamSynchronize(ctx->stream);
    if (g->nranks == 1 && !(flags & LX_COMM_FORCE)) return detach_comm(ctx);
    Comm* c = nullptr;
    // virtual ranks share this CUDA context: load every kernel before any of them spins on another
    // (a lazy module load needs the context to idle -> deadlock with a spinning persistent kernel)
    CUDA_TRY(preload_kernels());
    CUDA_TRY(preload_bb_kernels());
    if (comm_create_local(g->g, rank, ctx->device, ctx->row, &c))
        return fail(LX_ERR_NCCL, "local communicator: %s", comm_error());
    LX_TRY(attach_comm(ctx, c, rank, g->nranks));
    if (peer_eligible(ctx, g->nranks, flags)) {
        comm_set_grid_div(c, g->nranks);   // the virtual ranks' persistent grids share one GPU
        if (comm_peer_enable(c, ctx->row)) return fail(LX_ERR_NCCL, "peer-memory transport: %s", comm_error());
        LX_TRY(prealloc_slab(ctx));
    }
    return LX_OK;
}

lx_status lx_ctx_set_comm_local(lx_ctx* ctx, lx_local_group* g, int rank) {
    return lx_ctx_set_comm_local_ex(ctx, g, rank, 0);
}

lx_status lx_ctx_local(const lx_ctx* ctx, int64_t* i_begin, int64_t* i_end, int64_t* n_local) {
    if (!ctx) return fail(LX_ERR_ARG, "NULL");
    if (i_begin) *i_begin = ctx->i_begin;
    if (i_end) *i_end = ctx->i_end;
    if (n_local) *n_local = ctx->N_loc;
    return LX_OK;
}

lx_status lx_ctx_synchronize(lx_ctx* ctx, int* iters_total, double* err_last) {
    if (!ctx) return fail(LX_ERR_ARG, "NULL");
    Record r;
    LX_TRY(read_record(ctx, 1, &r));
    LX_TRY(reset_record(ctx, 1));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (ctx->s_out) CUDA_TRY(cudaStreamSynchronize(ctx->s_out));   // pipelined host outputs landed
    ctx->pin_key = nullptr;                                         // host inputs may change from here on
    if (iters_total) *iters_total = r.iters;
    if (err_last) *err_last = r.err;
    return status_of(r);
}

int64_t lx_ctx_launch_count(const lx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int lx_ctx_iterations_per_pass(const lx_ctx* ctx) { return ctx ? ctx_tblock(ctx) : 0; }

lx_status lx_ctx_set_kernel(lx_ctx* ctx, int iterations_per_pass, int kernel3d) {
    if (!ctx) return fail(LX_ERR_ARG, "NULL");
    if (iterations_per_pass < 0 || iterations_per_pass > 2) return fail(LX_ERR_ARG, "iterations_per_pass in {0, 1, 2}");
    if (kernel3d < 0 || kernel3d > 1) return fail(LX_ERR_ARG, "kernel3d in {0, 1}");
    ctx->tblock = iterations_per_pass;
    ctx->k3d = kernel3d;
    return LX_OK;
}

// ---------------------------------------------------------------- Leja
// Pipelined host staging of Leja calls (pinned host buffers): slot i & 1 of a two-slot ring.
//   copy-in stream : wait "kernel of call i-2 done with slot" -> H2D v -> event in[slot]
//   context stream : wait in[slot], wait "D2H of call i-2 done" -> Leja kernel(s) -> event comp[slot]
//   copy-out stream: wait comp[slot] -> D2H outputs -> event out[slot]
// so consecutive calls overlap their copies with each other's kernels (H2D and D2H use separate copy
// engines).  A call with iters_out waits for its own outputs; an asynchronous call (iters_out NULL)
// returns at once -- the caller must not touch its host buffers before lx_ctx_synchronize.
static lx_status leja_pipelined(lx_ctx* ctx, const lx_problem* pb, const double* ud, const double* v,
                                double* const* outs, const double* coeffs, int K, double dt, double c, double gamma,
                                int l, double rtol, double atol, int* iters_out, const int* ls = nullptr) {
    const size_t bytes = ctx->N_loc * sizeof(double);
    if (!ctx->s_in) {
        CUDA_TRY(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
        for (int i = 0; i < 2; i++) {
            CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_in[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_comp[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_out[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventRecord(ctx->ev_comp[i], ctx->stream));
            CUDA_TRY(cudaEventRecord(ctx->ev_out[i], ctx->s_out));
        }
    }
    const int sl = ctx->pipe_next;
    ctx->pipe_next ^= 1;
    const bool vhost = !is_device_ptr(v);
    const double* vd = v;
    if (vhost && ctx->pin_key == v) {
        // the same host input as an earlier asynchronous call since the last synchronisation point: the
        // caller may not modify it before lx_ctx_synchronize (lexint.h), so its staged copy is reused
        const int ks = ctx->pin_key_slot;
        CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[ks], 0));
        vd = ctx->pin_in[ks];
    } else if (vhost) {
        int is = sl;
        if (ctx->pin_key && ctx->pin_key_slot == is) is ^= 1;   // keep a cached input in place
        if (!ctx->pin_in[is]) CUDA_TRY(cudaMalloc(&ctx->pin_in[is], bytes));
        CUDA_TRY(cudaStreamWaitEvent(ctx->s_in, ctx->ev_comp[is], 0));
        CUDA_TRY(cudaMemcpyAsync(ctx->pin_in[is], v, bytes, cudaMemcpyHostToDevice, ctx->s_in));
        CUDA_TRY(cudaEventRecord(ctx->ev_in[is], ctx->s_in));
        CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[is], 0));
        vd = ctx->pin_in[is];
        ctx->pin_key = v;
        ctx->pin_key_slot = is;
    }
    double* od[kMaxK];
    bool ohost[kMaxK];
    for (int k = 0; k < K; k++) {
        ohost[k] = !is_device_ptr(outs[k]);
        od[k] = outs[k];
        if (ohost[k]) {
            if (!ctx->pin_out[sl][k]) CUDA_TRY(cudaMalloc(&ctx->pin_out[sl][k], bytes));
            od[k] = ctx->pin_out[sl][k];
        }
    }
    CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_out[sl], 0));
    const bool sync = iters_out != nullptr;
    const int rec = sync ? 0 : 1;
    if (sync) LX_TRY(reset_record(ctx, 0));
    LX_TRY(leja_device(ctx, pb, ud, vd, od, coeffs, K, dt, c, gamma, l, rtol, atol, rec, nullptr, ls));
    CUDA_TRY(cudaEventRecord(ctx->ev_comp[sl], ctx->stream));
    if (vhost) CUDA_TRY(cudaEventRecord(ctx->ev_comp[ctx->pin_key_slot], ctx->stream));   // input slot in use
    CUDA_TRY(cudaStreamWaitEvent(ctx->s_out, ctx->ev_comp[sl], 0));
    for (int k = 0; k < K; k++)
        if (ohost[k]) CUDA_TRY(cudaMemcpyAsync(outs[k], od[k], bytes, cudaMemcpyDeviceToHost, ctx->s_out));
    CUDA_TRY(cudaEventRecord(ctx->ev_out[sl], ctx->s_out));
    if (!sync) return LX_OK;
    ctx->pin_key = nullptr;   // synchronous call: the caller may modify its buffers after it returns
    CUDA_TRY(cudaEventSynchronize(ctx->ev_out[sl]));
    Record r;
    LX_TRY(read_record(ctx, 0, &r));
    *iters_out = r.iters;
    return status_of(r);
}

// Leja call on a validated request: host-buffer pipelining, staging, one device call, record read-back.
// ls: per-accumulator phi index (lx_real_leja_phi_multi) or NULL (every accumulator phi_l).
static lx_status leja_api(lx_ctx* ctx, const lx_problem* pb, const double* u_lin, const double* v, double* const* outs,
                          const double* coeffs, int K, double dt, double c, double gamma, int l, double rtol,
                          double atol, int* iters_out, const int* ls) {
    if (pb->react == 0.0 && pb->flux == 0.0) u_lin = nullptr;
    {
        // host buffers in PINNED memory (v and/or outputs; u_lin on the device): pipelined staging --
        // the H2D of this call, the kernels of the previous one and the D2H of the one before overlap
        bool host = !is_device_ptr(v), pinned = !host || is_pinned_host_ptr(v);
        for (int k = 0; k < K; k++) {
            const bool h = !is_device_ptr(outs[k]);
            host = host || h;
            pinned = pinned && (!h || is_pinned_host_ptr(outs[k]));
        }
        if (host && pinned && (!u_lin || is_device_ptr(u_lin)))
            return leja_pipelined(ctx, pb, u_lin, v, outs, coeffs, K, dt, c, gamma, l, rtol, atol, iters_out, ls);
    }
    Staging sg(ctx);
    const double *vd, *ud;
    double* od[kMaxK];
    LX_TRY(sg.in(v, &vd));
    LX_TRY(sg.in(u_lin, &ud));
    for (int k = 0; k < K; k++) LX_TRY(sg.out(outs[k], &od[k]));
    const bool sync = iters_out != nullptr || sg.any_host;
    const int rec = sync ? 0 : 1;
    if (sync) LX_TRY(reset_record(ctx, 0));
    LX_TRY(leja_device(ctx, pb, ud, vd, od, coeffs, K, dt, c, gamma, l, rtol, atol, rec, nullptr, ls));
    LX_TRY(sg.finish());
    if (!sync) return LX_OK;
    Record r;
    LX_TRY(read_record(ctx, 0, &r));
    if (iters_out) *iters_out = r.iters;
    return status_of(r);
}

lx_status lx_real_leja_phi_vertical(lx_ctx* ctx, const lx_problem* pb, const double* u_lin, const double* v,
                                    double* const* outs, const double* coeffs, int K, double dt, double c,
                                    double gamma, int l, double rtol, double atol, int* iters_out) {
    if (!ctx) return fail(LX_ERR_ARG, "ctx is NULL");
    LX_TRY(check_problem(ctx, pb));
    LX_TRY(validate_leja(pb, u_lin, v, outs, coeffs, K, dt, gamma, l));
    return leja_api(ctx, pb, u_lin, v, outs, coeffs, K, dt, c, gamma, l, rtol, atol, iters_out, nullptr);
}

lx_status lx_real_leja_phi_multi(lx_ctx* ctx, const lx_problem* pb, const double* u_lin, const double* v,
                                 double* const* outs, const int* ls, const double* coeffs, int K, double dt, double c,
                                 double gamma, double rtol, double atol, int* iters_out) {
    if (!ctx || !ls) return fail(LX_ERR_ARG, "NULL argument");
    LX_TRY(check_problem(ctx, pb));
    LX_TRY(validate_leja(pb, u_lin, v, outs, coeffs, K, dt, gamma, ls[0], ls));
    return leja_api(ctx, pb, u_lin, v, outs, coeffs, K, dt, c, gamma, ls[0], rtol, atol, iters_out, ls);
}

lx_status lx_real_leja_phi(lx_ctx* ctx, const lx_problem* pb, const double* u_lin, const double* v, double* out,
                           double dt, double c, double gamma, int l, double rtol, double atol, int* iters_out) {
    const double one = 1.0;
    double* outs[1] = {out};
    return lx_real_leja_phi_vertical(ctx, pb, u_lin, v, outs, &one, 1, dt, c, gamma, l, rtol, atol, iters_out);
}

// ---------------------------------------------------------------- spectrum
lx_status lx_spectrum_bound(lx_ctx* ctx, const lx_problem* pb, const double* u, double* lambda_abs_out) {
    if (!ctx || !lambda_abs_out) return fail(LX_ERR_ARG, "NULL argument");
    LX_TRY(check_problem(ctx, pb));
    double m2 = 0.0;   // max u^2 (Gershgorin shift / Burgers speed)
    if (pb->react != 0.0 || pb->flux != 0.0) {
        if (!u) return fail(LX_ERR_ARG, "u required when react/flux != 0");
        Staging sg(ctx);
        const double* ud;
        LX_TRY(sg.in(u, &ud));
        CUDA_TRY(cudaMemsetAsync(&ctx->ctrl->umax, 0, sizeof(unsigned long long), ctx->stream));
        StageArgs A;
        std::memset(&A, 0, sizeof A);
        A.n_loc = ctx->n_loc;
        A.n1 = (int)ctx->n[1];
        A.n2 = (int)ctx->n[2];
        A.x0 = ud;
        A.ctrl = ctx->ctrl;
        A.grid = stage_grid_size(ctx->device, ST_MAXSQ);
        CUDA_TRY(launch_stage(ST_MAXSQ, A, ctx->stream));
        ctx->launches++;
        if (ctx->comm) LX_TRY(comm_allreduce_max_u64(ctx->comm, &ctx->ctrl->umax, ctx->stream) ? fail(LX_ERR_NCCL, "allreduce max: %s", comm_error()) : LX_OK);
        CUDA_TRY(cudaMemcpyAsync(ctx->umax_host, &ctx->ctrl->umax, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        std::memcpy(&m2, ctx->umax_host, sizeof m2);
    }
    // closed form (Fourier symbol at theta = pi), frozen-coefficient speed for Burgers (R9, R23)
    double vmax = std::fabs(pb->nu);
    if (pb->flux != 0.0) vmax = std::fabs(pb->nu) + std::fabs(pb->flux) * std::sqrt(m2);
    double b = 0.0;
    for (int d = 0; d < pb->ndim; d++) {
        const double h = pb->dx[d];
        b += 4.0 * pb->diff / (h * h) + 4.0 * vmax / (3.0 * h);
    }
    if (pb->react != 0.0) {   // Gershgorin shift of the reaction (R16)
        const double sft = 3.0 * m2 - 1.0;
        if (sft > 0.0) b += pb->react * sft;
    }
    *lambda_abs_out = b;
    return LX_OK;
}

lx_status lx_spectrum_estimate(lx_ctx* ctx, const lx_problem* pb, const double* u, int iters, double* lambda_abs_out) {
    if (!ctx || !lambda_abs_out) return fail(LX_ERR_ARG, "NULL argument");
    LX_TRY(check_problem(ctx, pb));
    if (iters < 1 || iters > 100000) return fail(LX_ERR_ARG, "iters must be in [1, 100000]");
    if ((pb->react != 0.0 || pb->flux != 0.0) && !u) return fail(LX_ERR_ARG, "u required when react/flux != 0");
    Staging sg(ctx);
    const double* ud = nullptr;
    if (pb->react != 0.0 || pb->flux != 0.0) LX_TRY(sg.in(u, &ud));
    LX_TRY(reset_record(ctx, 0));
    CUDA_TRY(launch_fill_start(ctx->Y[0], ctx->N_loc, ctx->i_begin == 0, ctx->stream));
    ctx->launches++;
    LejaParams P = base_params(ctx, pb);
    P.K = 0;
    P.power_iters = iters;
    P.max_nodes = iters + 1;
    P.v = P.ysrc[0];
    P.u = ud;
    P.rec = ctx->rec_dev;
    const bool diag = pb->react != 0.0;
    if (ctx->comm) {
        LX_TRY(comm_power(ctx->comm, P, diag, ctx->stream, &ctx->launches));
    } else {
        P.grid = leja_grid_size(ctx->device, 1, diag, P.ndim, P.nunits);
        CUDA_TRY(launch_power_persistent(P, ctx->stream, diag));
        ctx->launches++;
    }
    Record r;
    LX_TRY(read_record(ctx, 0, &r));
    *lambda_abs_out = r.est;
    return status_of(r);
}

// ---------------------------------------------------------------- stages
static StageArgs stage_args(lx_ctx* ctx, const lx_problem* pb, int rec) {
    StageArgs A;
    std::memset(&A, 0, sizeof A);
    A.ndim = ctx->ndim;
    A.n_loc = ctx->n_loc;
    A.n1 = (int)ctx->n[1];
    A.n2 = (int)ctx->n[2];
    A.N_glob = ctx->N_glob;
    A.st = make_stencil(pb);
    A.partials = ctx->partials;
    A.ctrl = ctx->ctrl;
    A.rec = ctx->rec_dev + rec;
    A.grid = 0;   // chosen per op in run_stage
    return A;
}

static lx_status run_stage(lx_ctx* ctx, int op, const StageArgs& A0) {
    StageArgs A = A0;
    A.grid = stage_grid_size(ctx->device, op);
    if (A.grid > ctx->max_grid) A.grid = ctx->max_grid;
    if (ctx->comm && (op == ST_FINAL4 || op == ST_FINAL_EXPRB32 || op == ST_LIN4_ERR))
        return comm_stage_norm(ctx->comm, op, A, ctx->stream, &ctx->launches) ? fail(LX_ERR_NCCL, "stage norm: %s", comm_error()) : LX_OK;
    CUDA_TRY(launch_stage(op, A, ctx->stream));
    ctx->launches++;
    return LX_OK;
}

static lx_status rhs_device(lx_ctx* ctx, const lx_problem* pb, const double* u, double scale, double* f) {
    LejaParams P = base_params(ctx, pb);
    P.source = pb->source;   // device pointer (staged by the caller)
    P.u = u;
    P.v = RowSrc{u, nullptr, ctx->row, ctx->n_loc, 0};
    P.ydst[0] = f;
    if (ctx->comm) return comm_rhs(ctx->comm, P, scale, ctx->stream, &ctx->launches) ? fail(LX_ERR_NCCL, "rhs halo: %s", comm_error()) : LX_OK;
    if (P.ndim == 3 && ctx->k3d != 1 && P.n1 % 16 == 0 && P.n2 % 64 == 0) {
        CUDA_TRY(launch_rhs3d_smem(P, scale, ctx->stream, ctx->device));
        ctx->launches++;
        return LX_OK;
    }
    P.grid = (P.nunits + kWarps - 1) / kWarps;
    if (P.grid > ctx->nsm * 3) P.grid = ctx->nsm * 3;   // one wave at 3 CTAs per SM (k_rhs2d's launch bounds)
    CUDA_TRY(launch_rhs(P, scale, ctx->stream));
    ctx->launches++;
    return LX_OK;
}

lx_status lx_rhs(lx_ctx* ctx, const lx_problem* pb0, const double* u, double scale, double* f_out) {
    if (!ctx || !u || !f_out) return fail(LX_ERR_ARG, "NULL argument");
    LX_TRY(check_problem(ctx, pb0));
    if (u == f_out) return fail(LX_ERR_ALIAS, "f_out must not alias u");
    Staging sg(ctx);
    lx_problem pbs = *pb0;
    const lx_problem* pb = &pbs;
    LX_TRY(sg.in(pb0->source, &pbs.source));
    const double* ud;
    double* fd;
    LX_TRY(sg.in(u, &ud));
    LX_TRY(sg.out(f_out, &fd));
    LX_TRY(rhs_device(ctx, pb, ud, scale, fd));
    LX_TRY(sg.finish());
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return LX_OK;
}

// Remainder difference y0 = a2 * (dt F(s) - dt F(u)), s = x0 + a0 x1 + a1 x2.  Pointwise problems use
// one fused kernel; flux (Burgers) problems materialise s into `tmp` and apply the stencil remainder.
static lx_status stage_remainder(lx_ctx* ctx, const lx_problem* pb, int rec, const double* u, const double* x0,
                           const double* x1, double a0, const double* x2, double a1, double a2, double dt,
                           double* y0, double* tmp) {
    StageArgs A = stage_args(ctx, pb, rec);
    A.dt = dt;
    A.u = u;
    if (pb->flux == 0.0) {
        A.x0 = x0; A.x1 = x1; A.x2 = x2; A.a0 = a0; A.a1 = a1; A.a2 = a2; A.y0 = y0;
        return run_stage(ctx, ST_STAGE_REMAINDER, A);
    }
    const double* sfield = x0;
    if (x1 || x2) {
        A.x0 = x0; A.x1 = x1; A.x2 = x2; A.a0 = a0; A.a1 = x2 ? a1 : 0.0; A.y0 = tmp;
        LX_TRY(run_stage(ctx, ST_LIN3, A));
        sfield = tmp;
    }
    LejaParams P = base_params(ctx, pb);
    P.v = RowSrc{sfield, nullptr, ctx->row, ctx->n_loc, 0};
    P.u = u;
    P.grid = (P.nunits + kWarps - 1) / kWarps;
    if (P.grid > ctx->nsm * 2) P.grid = ctx->nsm * 2;
    CUDA_TRY(launch_rem_flux(P, dt, a2, y0, ctx->stream));
    ctx->launches++;
    return LX_OK;
}

// Non-embedded methods: err = 0, u_low optional (a copy of u_high).
static bool nonembedded(lx_method m) { return m == LX_ROSENBROCK_EULER || m == LX_EXPRB42; }

// EPIRK5P1 tableau (reading R26; Tokman, Loffeld & Tranquilli 2012, cited at P:83)
namespace epirk5 {
constexpr double a11 = 0.35129592695058193092, a21 = 0.84405472011657126298, a22 = 1.6905891609568963624;
constexpr double b1 = 1.0, b2 = 1.2727127317356892397, b3 = 2.2714599265422622275;
constexpr double g11 = 0.35129592695058193092, g21 = 0.84405472011657126298, g22 = 1.0;
constexpr double g31 = 1.0, g32 = 0.71111095364366870359, g33 = 0.62378111953371494809;
}  // namespace epirk5

static lx_status step_device(lx_ctx* ctx, lx_method method, const lx_problem* pb, const double* u, double* lo,
                             double* hi, double dt, double c, double gamma, double rtol, double atol, int rec) {
    const bool diag = pb->react != 0.0;
    const bool flux = pb->flux != 0.0;
    const double* ul = (diag || flux) ? u : nullptr;
    double* S0 = scratch(ctx, 0);
    if (!S0) return fail(LX_ERR_CUDA, "scratch allocation failed");
    const double one = 1.0;
    // all coefficient tables of the step in one device launch
    static const double c1[1] = {1.0}, c2[2] = {0.5, 1.0}, c3[3] = {0.5, 2.0 / 3.0, 1.0}, c42[2] = {0.75, 1.0};
    // f_u = RHS(u) * dt   (alg:Ros_Eu P:468-469)
    LX_TRY(rhs_device(ctx, pb, u, dt, S0));
    StageArgs A = stage_args(ctx, pb, rec);
    A.dt = dt;
    A.u = u;
    if (method == LX_ROSENBROCK_EULER) {
        double* o[1] = {hi};
        LX_TRY(leja_device(ctx, pb, ul, S0, o, &one, 1, dt, c, gamma, 1, rtol, atol, rec));
        A.x0 = u; A.x1 = hi; A.y0 = hi; A.a0 = 1.0; A.a1 = 1.0;  // u_exprb2 = u + phi_1(J dt) f dt
        LX_TRY(run_stage(ctx, ST_AXPBY, A));
        if (lo && lo != hi) CUDA_TRY(cudaMemcpyAsync(lo, hi, ctx->N_loc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        return LX_OK;
    }
    if (method == LX_EXPRB32) {
        // P:414-418, alg:exprb32: u_flux (in hi) -> a (lo), R_a (S0) -> u_nl_3 (hi) -> u_3 = a + 2 u_nl_3
        double* o[1] = {hi};
        LX_TRY(leja_device(ctx, pb, ul, S0, o, &one, 1, dt, c, gamma, 1, rtol, atol, rec));
        if (!flux) {
            A.x0 = u; A.x1 = hi; A.y1 = lo; A.y0 = S0;
            LX_TRY(run_stage(ctx, ST_EXPRB32_A, A));
        } else {   // a = u + u_flux -> lo ; R_a = dt F(a) - dt F(u) (stencil remainder)
            A.x0 = u; A.x1 = hi; A.a0 = 1.0; A.a1 = 1.0; A.y0 = lo;
            LX_TRY(run_stage(ctx, ST_AXPBY, A));
            LX_TRY(stage_remainder(ctx, pb, rec, u, lo, nullptr, 0.0, nullptr, 0.0, 1.0, dt, S0, nullptr));
        }
        LX_TRY(leja_device(ctx, pb, ul, S0, o, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);
        A.x0 = lo; A.x1 = hi; A.y0 = hi;
        return run_stage(ctx, ST_FINAL_EXPRB32, A);
    }
    if (method == LX_EXPRB42) {
        // EXPRB42 (reading R22): a = u + 3/4 p_34 ; u+ = u + p_1 + phi_3(hJ) (32/9 D_a)
        double* S1 = scratch(ctx, 1);
        double* S2 = scratch(ctx, 2);
        if (!S1 || !S2) return fail(LX_ERR_CUDA, "scratch allocation failed");
        double* pv[2] = {S1, S2};
        LX_TRY(leja_device(ctx, pb, ul, S0, pv, c42, 2, dt, c, gamma, 1, rtol, atol, rec));
        LX_TRY(stage_remainder(ctx, pb, rec, u, u, S1, 0.75, nullptr, 0.0, 32.0 / 9.0, dt, S0, hi));
        double* o3[1] = {S1};
        LX_TRY(leja_device(ctx, pb, ul, S0, o3, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);
        A.x0 = u; A.x1 = S2; A.x2 = S1; A.y0 = hi;
        LX_TRY(run_stage(ctx, ST_SUM3, A));
        if (lo && lo != hi) CUDA_TRY(cudaMemcpyAsync(lo, hi, ctx->N_loc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        return LX_OK;
    }
    if (method == LX_EXPRB54S4) {
        // reading R31: c2 = 1/4, c3 = 1/2, c4 = 9/10, D_x = dt (F(x) - F(u)); 8 Leja calls
        double* S1 = scratch(ctx, 1);
        double* S2 = scratch(ctx, 2);
        double* S3 = scratch(ctx, 3);
        double* S4 = scratch(ctx, 8);    // (scratch 4..6 hold lx_integrate's states)
        double* S5 = scratch(ctx, 9);
        if (!S1 || !S2 || !S3 || !S4 || !S5) return fail(LX_ERR_CUDA, "scratch allocation failed");
        const double e4[4] = {0.25, 0.5, 0.9, 1.0}, half = 0.5, c4 = 0.9;
        double* pv[4] = {S1, S2, S3, S4};                    // phi_1(c hJ) hf, c = 1/4, 1/2, 9/10, 1
        LX_TRY(leja_device(ctx, pb, ul, S0, pv, e4, 4, dt, c, gamma, 1, rtol, atol, rec));
        LX_TRY(stage_remainder(ctx, pb, rec, u, u, S1, 0.25, nullptr, 0.0, 1.0, dt, S0, hi));   // D2 -> S0
        double* q1[1] = {S1};
        LX_TRY(leja_device(ctx, pb, ul, S0, q1, &half, 1, dt, c, gamma, 3, rtol, atol, rec));    // phi_3(hJ/2) D2
        A = stage_args(ctx, pb, rec);                        // U3 = u + 1/2 P05 + 4 Q -> S5
        A.x0 = u; A.x1 = S2; A.x2 = S1; A.a0 = 0.5; A.a1 = 4.0; A.y0 = S5;
        LX_TRY(run_stage(ctx, ST_LIN3, A));
        LX_TRY(stage_remainder(ctx, pb, rec, u, S5, nullptr, 0.0, nullptr, 0.0, 1.0, dt, S2, nullptr));  // D3 -> S2
        A = stage_args(ctx, pb, rec);                        // U4 stage combinations of D2, D3 -> S1, S5
        A.x0 = S0; A.x1 = S2; A.y0 = S1; A.y1 = S5;
        A.a0 = 5832.0 / 125.0; A.a1 = -729.0 / 125.0; A.a2 = -157464.0 / 625.0; A.a3 = 39366.0 / 625.0;
        LX_TRY(run_stage(ctx, ST_COMBINE2, A));
        double* o3a[1] = {lo};
        LX_TRY(leja_device(ctx, pb, ul, S1, o3a, &c4, 1, dt, c, gamma, 3, rtol, atol, rec));
        double* o4a[1] = {hi};
        LX_TRY(leja_device(ctx, pb, ul, S5, o4a, &c4, 1, dt, c, gamma, 4, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);                        // U4 = u + 9/10 P09 + lo + hi -> S1
        A.x0 = u; A.x1 = S3; A.x2 = lo; A.x3 = hi; A.a0 = 0.9; A.a1 = 1.0; A.a2 = 1.0; A.y0 = S1;
        LX_TRY(run_stage(ctx, ST_LIN4, A));
        LX_TRY(stage_remainder(ctx, pb, rec, u, S1, nullptr, 0.0, nullptr, 0.0, 1.0, dt, S3, nullptr));  // D4 -> S3
        A = stage_args(ctx, pb, rec);                        // embedded: 64 D2 - 8 D3 -> S1, -384 D2 + 96 D3 -> S5
        A.x0 = S0; A.x1 = S2; A.y0 = S1; A.y1 = S5;
        A.a0 = 64.0; A.a1 = -8.0; A.a2 = -384.0; A.a3 = 96.0;
        LX_TRY(run_stage(ctx, ST_COMBINE2, A));
        LX_TRY(leja_device(ctx, pb, ul, S1, o3a, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
        LX_TRY(leja_device(ctx, pb, ul, S5, o4a, &one, 1, dt, c, gamma, 4, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);                        // E = lo + hi -> S0
        A.x0 = lo; A.x1 = hi; A.a0 = 1.0; A.a1 = 1.0; A.y0 = S0;
        LX_TRY(run_stage(ctx, ST_AXPBY, A));
        A = stage_args(ctx, pb, rec);                        // 18 D3 - 250/81 D4 -> S1, -60 D3 + 500/27 D4 -> S5
        A.x0 = S2; A.x1 = S3; A.y0 = S1; A.y1 = S5;
        A.a0 = 18.0; A.a1 = -250.0 / 81.0; A.a2 = -60.0; A.a3 = 500.0 / 27.0;
        LX_TRY(run_stage(ctx, ST_COMBINE2, A));
        LX_TRY(leja_device(ctx, pb, ul, S1, o3a, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
        LX_TRY(leja_device(ctx, pb, ul, S5, o4a, &one, 1, dt, c, gamma, 4, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);                        // d = lo + hi - E -> S2
        A.x0 = lo; A.x1 = hi; A.x2 = S0; A.a0 = 1.0; A.a1 = -1.0; A.y0 = S2;
        LX_TRY(run_stage(ctx, ST_LIN3, A));
        A = stage_args(ctx, pb, rec);                        // u4 = u + P1 + E ; u5 = u4 + d ; err = ||d||
        A.x0 = u; A.x1 = S4; A.x2 = S0; A.x3 = S2; A.y0 = lo; A.y1 = hi;
        return run_stage(ctx, ST_FINAL4, A);
    }
    if (method == LX_EXPRB53S3) {
        // reading R27: c2 = 1/2, c3 = 9/10, D_x = dt (F(x) - F(u))
        double* S1 = scratch(ctx, 1);
        double* S2 = scratch(ctx, 2);
        double* S3 = scratch(ctx, 3);
        double* S7 = scratch(ctx, 7);
        if (!S1 || !S2 || !S3 || !S7) return fail(LX_ERR_CUDA, "scratch allocation failed");
        const double e3[3] = {0.5, 0.9, 1.0};
        double* pv[3] = {S1, S2, S3};                        // phi_1(c hJ) hf, c = 1/2, 9/10, 1
        LX_TRY(leja_device(ctx, pb, ul, S0, pv, e3, 3, dt, c, gamma, 1, rtol, atol, rec));
        LX_TRY(stage_remainder(ctx, pb, rec, u, u, S1, 0.5, nullptr, 0.0, 1.0, dt, S0, hi));   // D2 -> S0
        double* qv[3] = {S1, hi, lo};                        // phi_3(c hJ) D2, c = 1/2, 9/10, 1
        LX_TRY(leja_device(ctx, pb, ul, S0, qv, e3, 3, dt, c, gamma, 3, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);                        // U3 = u + c3 P09 + 27/25 Q05 + 729/125 Q09
        A.x0 = u; A.x1 = S2; A.x2 = S1; A.x3 = hi; A.a0 = 0.9; A.a1 = 27.0 / 25.0; A.a2 = 729.0 / 125.0; A.y0 = S7;
        LX_TRY(run_stage(ctx, ST_LIN4, A));
        LX_TRY(stage_remainder(ctx, pb, rec, u, S7, nullptr, 0.0, nullptr, 0.0, 1.0, dt, S2, nullptr));  // D3 -> S2
        A = stage_args(ctx, pb, rec);                        // w3 -> S1, w4 -> S7
        A.x0 = S0; A.x1 = S2; A.y0 = S1; A.y1 = S7;
        A.a0 = 18.0; A.a1 = -250.0 / 81.0; A.a2 = -60.0; A.a3 = 500.0 / 27.0;
        LX_TRY(run_stage(ctx, ST_COMBINE2, A));
        double* o3[1] = {hi};
        LX_TRY(leja_device(ctx, pb, ul, S1, o3, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
        double* o4[1] = {S0};
        LX_TRY(leja_device(ctx, pb, ul, S7, o4, &one, 1, dt, c, gamma, 4, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);                        // d = Z3 + Z4 - 8 Q1 -> S2
        A.x0 = hi; A.x1 = S0; A.x2 = lo; A.a0 = 1.0; A.a1 = -8.0; A.y0 = S2;
        LX_TRY(run_stage(ctx, ST_LIN3, A));
        A = stage_args(ctx, pb, rec);                        // q8 = 8 Q1 (in place)
        A.x0 = lo; A.a0 = 8.0; A.y0 = lo;
        LX_TRY(run_stage(ctx, ST_AXPBY, A));
        A = stage_args(ctx, pb, rec);                        // u3 = u + P1 + q8 ; u5 = u3 + d ; err = ||d||
        A.x0 = u; A.x1 = S3; A.x2 = lo; A.x3 = S2; A.y0 = lo; A.y1 = hi;
        return run_stage(ctx, ST_FINAL4, A);
    }
    if (method == LX_EPIRK5P1) {
        // reading R26: R(x) = dt (F(x) - F(u)); vertical phi_1 {g11, g21, 1} on f dt, vertical phi_1
        // {1/2, g32, 1} on R(Y1), vertical phi_3 {g33, 1} on R(Y2) - 2 R(Y1); the 1/2 and the second phi_3
        // accumulator make the embedded fourth-order solution (reading R33)
        using namespace epirk5;
        double* S1 = scratch(ctx, 1);
        double* S2 = scratch(ctx, 2);
        double* S3 = scratch(ctx, 3);
        double* S7 = scratch(ctx, 7);
        double* S8 = scratch(ctx, 8);    // (scratch 4..6 hold lx_integrate's states; 8, 9 are free here)
        double* S9 = scratch(ctx, 9);
        double* u4 = lo ? lo : scratch(ctx, 6);
        if (!S1 || !S2 || !S3 || !S7 || !S8 || !S9 || !u4) return fail(LX_ERR_CUDA, "scratch allocation failed");
        const double e3[3] = {g11, g21, g31}, e2[3] = {0.5, g32, g22}, e1[2] = {g33, 1.0};
        double* pv[3] = {S1, S2, S3};
        LX_TRY(leja_device(ctx, pb, ul, S0, pv, e3, 3, dt, c, gamma, 1, rtol, atol, rec));
        // R1 = dt F(u + a11 P1) - dt F(u) -> S0 (f dt consumed)
        LX_TRY(stage_remainder(ctx, pb, rec, u, u, S1, a11, nullptr, 0.0, 1.0, dt, S0, hi));
        // Qh = phi_1(hJ/2) R1 (embedded), Q1 = phi_1(g32 hJ) R1, Q2 = phi_1(hJ) R1
        double* qv[3] = {S8, S1, hi};
        LX_TRY(leja_device(ctx, pb, ul, S0, qv, e2, 3, dt, c, gamma, 1, rtol, atol, rec));
        // R2 = dt F(u + a21 P2 + a22 Q2) - dt F(u) -> S2
        LX_TRY(stage_remainder(ctx, pb, rec, u, u, S2, a21, hi, a22, 1.0, dt, S7, S2));
        A = stage_args(ctx, pb, rec);
        A.x0 = S7; A.x1 = S0; A.a0 = 1.0; A.a1 = -2.0; A.y0 = S0;  // R2 - 2 R1
        LX_TRY(run_stage(ctx, ST_AXPBY, A));
        double* o3[2] = {S2, S9};                            // phi_3(g33 hJ), phi_3(hJ) (embedded)
        LX_TRY(leja_device(ctx, pb, ul, S0, o3, e1, 2, dt, c, gamma, 3, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);                        // u4 (embedded)
        A.x0 = u; A.x1 = S3; A.x2 = S8; A.x3 = S9; A.a0 = b1; A.a1 = b2; A.a2 = b3; A.y0 = u4;
        LX_TRY(run_stage(ctx, ST_LIN4, A));
        A = stage_args(ctx, pb, rec);                        // u5 ; err = ||u5 - u4||
        A.x0 = u; A.x1 = S3; A.x2 = S1; A.x3 = S2; A.a0 = b1; A.a1 = b2; A.a2 = b3; A.y0 = hi; A.y1 = u4;
        return run_stage(ctx, ST_LIN4_ERR, A);
    }
    // EXPRB43 / EPIRK4s3A (reading R17) / EPIRK4s3B (reading R34) / EPIRK4s3 (reading R35)
    const bool epb = method == LX_EPIRK4S3B;
    const bool e4s3 = method == LX_EPIRK4S3;
    const bool epirk = method == LX_EPIRK4S3A || epb || e4s3;   // two independent stages a, b
    double* S1 = scratch(ctx, 1);
    double* S2 = scratch(ctx, 2);
    double* S3 = epirk ? scratch(ctx, 3) : nullptr;
    if (!S1 || !S2 || (epirk && !S3)) return fail(LX_ERR_CUDA, "scratch allocation failed");
    const double cf2[2] = {0.5, 1.0}, cf3[3] = {0.5, 2.0 / 3.0, 1.0}, cfb[2] = {0.5, 0.75};
    const double cf9[3] = {1.0 / 9.0, 1.0 / 8.0, 1.0};
    // EPIRK4s3: stage a uses the 1/8 output, stage b the 1/9 output (vertical coefficients increase)
    double* pv[3] = {e4s3 ? S2 : S1, e4s3 ? S1 : S2, S3};
    if (epb) {
        // phi_2(hJ/2) f dt, phi_2(3hJ/4) f dt (vertical), phi_1(hJ) f dt
        LX_TRY(leja_device(ctx, pb, ul, S0, pv, cfb, 2, dt, c, gamma, 2, rtol, atol, rec));
        double* o1[1] = {S3};
        LX_TRY(leja_device(ctx, pb, ul, S0, o1, &one, 1, dt, c, gamma, 1, rtol, atol, rec));
    } else {
        LX_TRY(leja_device(ctx, pb, ul, S0, pv, e4s3 ? cf9 : epirk ? cf3 : cf2, epirk ? 3 : 2, dt, c, gamma, 1, rtol,
                           atol, rec));
    }
    double* p_one = epirk ? S3 : S2;
    const double wa = epb ? 2.0 / 3.0 : e4s3 ? 0.125 : 0.5, wb = epb ? 1.0 : e4s3 ? 1.0 / 9.0 : 2.0 / 3.0;
    const double c3a = epb ? 54.0 : e4s3 ? -1024.0 : epirk ? 32.0 : 16.0;
    const double c3b = epb ? -16.0 : e4s3 ? 1458.0 : epirk ? -13.5 : -2.0;
    const double c4a = epb ? -324.0 : e4s3 ? 27648.0 : epirk ? -144.0 : -48.0;
    const double c4b = epb ? 144.0 : e4s3 ? -34992.0 : epirk ? 81.0 : 12.0;
    if (epirk && pb->flux == 0.0) {
        // independent stages a, b: both remainders and the final stage's two combinations in ONE pointwise
        // kernel (D_a, D_b stay in registers): w3 -> S0 (f dt consumed), w4 -> hi
        A = stage_args(ctx, pb, rec);
        A.dt = dt;
        A.u = u;
        A.x1 = S1; A.x2 = S2; A.a0 = wa; A.a1 = wb;
        A.a2 = c3a; A.a3 = c3b; A.a4 = c4a; A.a5 = c4b;
        A.y0 = S0; A.y1 = hi;
        LX_TRY(run_stage(ctx, ST_REM2_W34, A));
        double* o3[1] = {S1};   // q3 (p_a consumed)
        LX_TRY(leja_device(ctx, pb, ul, S0, o3, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
        double* o4[1] = {S2};   // q4 (p_b consumed)
        LX_TRY(leja_device(ctx, pb, ul, hi, o4, &one, 1, dt, c, gamma, 4, rtol, atol, rec));
        A = stage_args(ctx, pb, rec);   // u3 = u + p_one + q3 -> lo ; u4 = u3 + q4 -> hi ; err = ||u4 - u3||
        A.x0 = u; A.x1 = p_one; A.x2 = S1; A.x3 = S2; A.y0 = lo; A.y1 = hi;
        return run_stage(ctx, ST_FINAL4, A);
    }
    // D_a = dt F(u + w_a p_a) - dt F(u)  -> S0   (w_a = 1/2; EPIRK4s3B: 2/3 on the phi_2 vector; EPIRK4s3: 1/8)
    LX_TRY(stage_remainder(ctx, pb, rec, u, u, S1, wa, nullptr, 0.0, 1.0, dt, S0, hi));
    double* Db;
    if (epirk) {
        // D_b = dt F(u + w_b p_b) - dt F(u) -> S1   (w_b = 2/3; EPIRK4s3B: 1; EPIRK4s3: 1/9)
        LX_TRY(stage_remainder(ctx, pb, rec, u, u, S2, wb, nullptr, 0.0, 1.0, dt, S1, hi));
        Db = S1;
    } else {
        // phi_1(hJ) D_a -> S1 ; b = u + p_one + S1 ; D_b -> lo
        double* o[1] = {S1};
        LX_TRY(leja_device(ctx, pb, ul, S0, o, &one, 1, dt, c, gamma, 1, rtol, atol, rec));
        if (pb->flux == 0.0) {
            // D_b and the final stage's two combinations in one pointwise kernel: w3 -> S1, w4 -> hi
            A = stage_args(ctx, pb, rec);
            A.dt = dt;
            A.u = u;
            A.x1 = p_one; A.x2 = S1; A.x3 = S0; A.a0 = 1.0; A.a1 = 1.0;
            A.a2 = c3a; A.a3 = c3b; A.a4 = c4a; A.a5 = c4b;
            A.y0 = S1; A.y1 = hi;
            LX_TRY(run_stage(ctx, ST_REMB_W34, A));
            double* o3[1] = {S0};   // q3 (D_a consumed)
            LX_TRY(leja_device(ctx, pb, ul, S1, o3, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
            double* o4[1] = {lo};   // q4
            LX_TRY(leja_device(ctx, pb, ul, hi, o4, &one, 1, dt, c, gamma, 4, rtol, atol, rec));
            A = stage_args(ctx, pb, rec);   // u3 = u + p_one + q3 -> lo ; u4 = u3 + q4 -> hi ; err
            A.x0 = u; A.x1 = p_one; A.x2 = S0; A.x3 = lo; A.y0 = lo; A.y1 = hi;
            return run_stage(ctx, ST_FINAL4, A);
        }
        LX_TRY(stage_remainder(ctx, pb, rec, u, u, p_one, 1.0, S1, 1.0, 1.0, dt, lo, hi));
        Db = lo;
    }
    // w3 = a3 D_a + b3 D_b, w4 = a4 D_a + b4 D_b
    double* w3 = epirk ? S2 : S1;
    A = stage_args(ctx, pb, rec);
    A.x0 = S0; A.x1 = Db; A.y0 = w3; A.y1 = hi;
    A.a0 = c3a; A.a1 = c3b; A.a2 = c4a; A.a3 = c4b;
    LX_TRY(run_stage(ctx, ST_COMBINE2, A));
    // q3 -> S0 (D_a consumed); q4 -> S1 (EPIRK: D_b consumed) / lo (EXPRB43: D_b consumed)
    double* q3 = S0;
    double* q4 = epirk ? S1 : lo;
    double* o3[1] = {q3};
    LX_TRY(leja_device(ctx, pb, ul, w3, o3, &one, 1, dt, c, gamma, 3, rtol, atol, rec));
    double* o4[1] = {q4};
    LX_TRY(leja_device(ctx, pb, ul, hi, o4, &one, 1, dt, c, gamma, 4, rtol, atol, rec));
    // u3 = u + p_one + q3 -> lo ; u4 = u3 + q4 -> hi ; err = ||u4 - u3||
    A = stage_args(ctx, pb, rec);
    A.x0 = u; A.x1 = p_one; A.x2 = q3; A.x3 = q4; A.y0 = lo; A.y1 = hi;
    return run_stage(ctx, ST_FINAL4, A);
}

lx_status lx_step(lx_ctx* ctx, lx_method method, const lx_problem* pb0, const double* u, double* u_low, double* u_high,
                  double* err_out, double dt, double c, double gamma, double rtol, double atol, int* iters_out) {
    if (!pb0) return fail(LX_ERR_ARG, "problem is NULL");
    lx_problem pbs = *pb0;
    const lx_problem* pb = &pbs;
    if (!ctx) return fail(LX_ERR_ARG, "ctx is NULL");
    LX_TRY(check_problem(ctx, pb));
    if ((int)method < 0 || (int)method > 9) return fail(LX_ERR_UNKNOWN_INTEGRATOR, "unknown integrator %d", (int)method);
    if (!u || !u_high) return fail(LX_ERR_ARG, "NULL argument");
    if (!nonembedded(method) && method != LX_EPIRK5P1 && !u_low)   // EPIRK5P1: u_low optional (R33)
        return fail(LX_ERR_ARG, "u_low required for embedded methods");
    if (u_low == u || u_high == u) return fail(LX_ERR_ALIAS, "outputs must not alias u");
    if (u_low && u_low == u_high) return fail(LX_ERR_ALIAS, "u_low must differ from u_high");
    if (!(gamma > 0.0) && dt != 0.0) return fail(LX_ERR_ARG, "gamma must be > 0");
    Staging sg(ctx);
    LX_TRY(sg.in(pb0->source, &pbs.source));
    const double* ud;
    double *lo = nullptr, *hi;
    LX_TRY(sg.in(u, &ud));
    LX_TRY(sg.out(u_high, &hi));
    if (u_low) LX_TRY(sg.out(u_low, &lo));
    const bool sync = iters_out || err_out || sg.any_host;
    const int rec = sync ? 0 : 1;
    if (sync) LX_TRY(reset_record(ctx, 0));
    LX_TRY(step_device(ctx, method, pb, ud, lo, hi, dt, c, gamma, rtol, atol, rec));
    LX_TRY(sg.finish());
    if (!sync) return LX_OK;
    Record r;
    LX_TRY(read_record(ctx, 0, &r));
    if (iters_out) *iters_out = r.iters;
    if (err_out) *err_out = nonembedded(method) ? 0.0 : r.err;
    return status_of(r);
}

// Embedded-error step-size control ("may be used to control the step sizes"; reading R32): accept iff
// err <= tol; next step h min(5, max(0.2, 0.9 (tol/err)^(1/(q+1)))) (err = 0 -> 5), q = order of the embedded
// solution; the last step clipped to land on t_end; a step whose Leja calls fail (NOCONV / NONFINITE) is a
// rejection with factor 0.2.  (c, gamma) from the spectrum bound of the current state.  One host
// round trip per attempted step (the decision needs err).
static int embedded_order(lx_method m) {
    switch (m) {
        case LX_EXPRB32: return 2;
        case LX_EXPRB43: return 3;
        case LX_EPIRK4S3A: return 3;
        case LX_EXPRB53S3: return 3;
        case LX_EPIRK5P1: return 4;   // reading R33
        case LX_EPIRK4S3B: return 3;  // reading R34
        case LX_EPIRK4S3: return 3;   // reading R35
        case LX_EXPRB54S4: return 4;
        default: return 0;
    }
}

lx_status lx_integrate_adaptive(lx_ctx* ctx, lx_method method, const lx_problem* pb0, double* u, double t_end,
                                double dt0, double tol, double rtol, double atol, int max_steps, int* accepted,
                                int* rejected, double* log_dt, double* log_err, int* iters_out) {
    if (!ctx || !u || !pb0) return fail(LX_ERR_ARG, "NULL argument");
    LX_TRY(check_problem(ctx, pb0));
    const int q = embedded_order(method);
    if (q == 0) return fail(LX_ERR_ARG, "step-size control needs an embedded method (EXPRB32/43/53s3/54s4, EPIRK4s3A)");
    if (!(dt0 > 0.0) || !(tol > 0.0) || !(t_end > 0.0) || max_steps < 1) return fail(LX_ERR_ARG, "bad t_end / dt0 / tol");
    if (!is_device_ptr(u)) return fail(LX_ERR_ARG, "u must be a device pointer");
    lx_problem pbs = *pb0;
    const lx_problem* pb = &pbs;
    Staging sg(ctx);
    LX_TRY(sg.in(pb0->source, &pbs.source));
    double* lo = scratch(ctx, 6);   // (scratch 6 is lx_integrate's discarded lower-order solution)
    double* hi = scratch(ctx, 4);
    if (!lo || !hi) return fail(LX_ERR_CUDA, "scratch allocation failed");
    double t = 0.0, h = dt0;
    int acc = 0, rej = 0, total = 0;
    lx_status st = LX_OK;
    for (int k = 0; k < max_steps && t < t_end; k++) {
        if (h > t_end - t) h = t_end - t;
        double bound = 0.0, c = 0.0, gamma = 0.0;
        LX_TRY(lx_spectrum_bound(ctx, pb, u, &bound));
        LX_TRY(lx_shift_scale(bound, &c, &gamma));
        LX_TRY(reset_record(ctx, 0));
        LX_TRY(step_device(ctx, method, pb, u, lo, hi, h, c, gamma, rtol, atol, 0));
        Record r;
        LX_TRY(read_record(ctx, 0, &r));
        total += r.iters;
        double err = r.err;
        if (r.status == 5 || r.status == 6) err = INFINITY;   // failed step: rejected
        else if (r.status != 0) {
            st = status_of(r);
            break;
        }
        const bool ok = err <= tol;
        if (log_dt) log_dt[k] = h;
        if (log_err) log_err[k] = err;
        double fac = err > 0.0 ? 0.9 * std::pow(tol / err, 1.0 / (q + 1)) : 5.0;
        fac = std::min(5.0, std::max(0.2, fac));
        if (ok) {
            CUDA_TRY(cudaMemcpyAsync(u, hi, ctx->N_loc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
            t = (h == t_end - t) ? t_end : t + h;
            acc++;
        } else {
            rej++;
        }
        h = h * fac;
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (accepted) *accepted = acc;
    if (rejected) *rejected = rej;
    if (iters_out) *iters_out = total;
    if (st == LX_OK && t < t_end) return fail(LX_ERR_NOCONV, "step budget exhausted at t = %g of %g", t, t_end);
    return st;
}

// The paper's time loop (listing alg:lexint) on the device: every step recomputes the
// spectrum bound (Gershgorin / closed form, x1.05, c = eig/2, gamma = -eig/4) with a
// device max-reduction + k_shift_scale, so the whole run is enqueued without host round trips.
lx_status lx_integrate(lx_ctx* ctx, lx_method method, const lx_problem* pb0, double* u, double dt, int nsteps,
                       double rtol, double atol, int* iters_out, double* err_out) {
    if (!ctx || !u || !pb0) return fail(LX_ERR_ARG, "NULL argument");
    lx_problem pbs = *pb0;
    const lx_problem* pb = &pbs;
    LX_TRY(check_problem(ctx, pb));
    if ((int)method < 0 || (int)method > 9) return fail(LX_ERR_UNKNOWN_INTEGRATOR, "unknown integrator %d", (int)method);
    if (nsteps < 0) return fail(LX_ERR_ARG, "nsteps < 0");
    if (!std::isfinite(dt)) return fail(LX_ERR_ARG, "dt not finite");
    Staging sg(ctx);
    LX_TRY(sg.in(pb0->source, &pbs.source));
    const double* uin;
    double* ud;
    LX_TRY(sg.in(u, &uin));
    ud = const_cast<double*>(uin);
    double* st[2] = {scratch(ctx, 4), scratch(ctx, 5)};
    double* lo = scratch(ctx, 6);   // lower-order solution (discarded)
    if (!st[0] || !st[1] || !lo) return fail(LX_ERR_CUDA, "scratch allocation failed");
    ShiftArgs sa;
    std::memset(&sa, 0, sizeof sa);
    sa.ndim = pb->ndim;
    for (int d = 0; d < pb->ndim; d++) sa.h[d] = pb->dx[d];
    sa.diff = pb->diff;
    sa.nu = pb->nu;
    sa.flux = pb->flux;
    sa.react = pb->react;
    const bool sync = iters_out || err_out || sg.any_host;
    const int rec = sync ? 0 : 1;
    if (sync) LX_TRY(reset_record(ctx, 0));
    StageArgs A = stage_args(ctx, pb, rec);
    A.ctrl = ctx->ctrl;
    double* cur = ud;
    ctx->cg_active = ctx->cg_dev;
    lx_status status = LX_OK;
    for (int n = 0; n < nsteps && status == LX_OK; n++) {
        // spectrum of J(u_n) on the device
        if (pb->react != 0.0 || pb->flux != 0.0) {
            if (cudaMemsetAsync(&ctx->ctrl->umax, 0, sizeof(unsigned long long), ctx->stream) != cudaSuccess) {
                status = fail(LX_ERR_CUDA, "memset");
                break;
            }
            StageArgs B = A;
            B.x0 = cur;
            B.grid = stage_grid_size(ctx->device, ST_MAXSQ);
            if (launch_stage(ST_MAXSQ, B, ctx->stream) != cudaSuccess) { status = fail(LX_ERR_CUDA, "maxsq"); break; }
            ctx->launches++;
            if (ctx->comm && comm_allreduce_max_u64(ctx->comm, &ctx->ctrl->umax, ctx->stream)) {
                status = fail(LX_ERR_NCCL, "allreduce max: %s", comm_error());
                break;
            }
        }
        if (launch_shift_scale(&ctx->ctrl->umax, sa, ctx->cg_dev, ctx->stream) != cudaSuccess) {
            status = fail(LX_ERR_CUDA, "shift_scale");
            break;
        }
        ctx->launches++;
        double* hi = (cur == st[0]) ? st[1] : st[0];
        status = step_device(ctx, method, pb, cur, lo, hi, dt, 0.0, 1.0, rtol, atol, rec);
        cur = hi;
    }
    ctx->cg_active = nullptr;
    if (status != LX_OK) return status;
    if (cur != ud) CUDA_TRY(cudaMemcpyAsync(ud, cur, ctx->N_loc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    if (sg.any_host) CUDA_TRY(cudaMemcpyAsync(u, ud, ctx->N_loc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (!sync) return LX_OK;
    Record r;
    LX_TRY(read_record(ctx, 0, &r));
    if (iters_out) *iters_out = r.iters;
    if (err_out) *err_out = nonembedded(method) ? 0.0 : r.err;
    return status_of(r);
}

lx_status lx_step_exprb42(lx_ctx* ctx, const lx_problem* pb, const double* u, double* u_out, double dt, double c,
                          double gamma, double rtol, double atol, int* iters_out) {
    return lx_step(ctx, LX_EXPRB42, pb, u, nullptr, u_out, nullptr, dt, c, gamma, rtol, atol, iters_out);
}

lx_status lx_step_epirk5p1(lx_ctx* ctx, const lx_problem* pb, const double* u, double* u_out, double dt, double c,
                           double gamma, double rtol, double atol, int* iters_out) {
    return lx_step(ctx, LX_EPIRK5P1, pb, u, nullptr, u_out, nullptr, dt, c, gamma, rtol, atol, iters_out);
}

lx_status lx_step_rosenbrock_euler(lx_ctx* ctx, const lx_problem* pb, const double* u, double* u_out, double dt,
                                   double c, double gamma, double rtol, double atol, int* iters_out) {
    return lx_step(ctx, LX_ROSENBROCK_EULER, pb, u, nullptr, u_out, nullptr, dt, c, gamma, rtol, atol, iters_out);
}
lx_status lx_step_exprb32(lx_ctx* ctx, const lx_problem* pb, const double* u, double* u_low, double* u_high,
                          double* err_out, double dt, double c, double gamma, double rtol, double atol, int* iters_out) {
    return lx_step(ctx, LX_EXPRB32, pb, u, u_low, u_high, err_out, dt, c, gamma, rtol, atol, iters_out);
}
lx_status lx_step_exprb43(lx_ctx* ctx, const lx_problem* pb, const double* u, double* u_low, double* u_high,
                          double* err_out, double dt, double c, double gamma, double rtol, double atol, int* iters_out) {
    return lx_step(ctx, LX_EXPRB43, pb, u, u_low, u_high, err_out, dt, c, gamma, rtol, atol, iters_out);
}
lx_status lx_step_epirk4s3a(lx_ctx* ctx, const lx_problem* pb, const double* u, double* u_low, double* u_high,
                            double* err_out, double dt, double c, double gamma, double rtol, double atol,
                            int* iters_out) {
    return lx_step(ctx, LX_EPIRK4S3A, pb, u, u_low, u_high, err_out, dt, c, gamma, rtol, atol, iters_out);
}


// ============================================================== black-box right-hand side
// (P:120-133 listing alg:RHS; P:416 finite-difference Jacobian; reading R25)
}  // extern "C"

static lx_status bb_ensure(lx_ctx* ctx) {
    if (ctx->comm) return fail(LX_ERR_UNSUPPORTED, "black-box RHS path: single-GPU contexts only");
    if (!ctx->bb) {
        CUDA_TRY(cudaMalloc(&ctx->bb, sizeof(BbCtrl)));
        CUDA_TRY(cudaHostAlloc(&ctx->bb_done_host, sizeof(int), cudaHostAllocMapped));
        CUDA_TRY(cudaHostGetDevicePointer((void**)&ctx->bb_done_dev, ctx->bb_done_host, 0));
        for (auto& e : ctx->bb_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return LX_OK;
}

static double* bb_vec(lx_ctx* ctx, int i) {
    if (!ctx->B[i]) {
        if (cudaMalloc(&ctx->B[i], ctx->N_loc * sizeof(double)) != cudaSuccess) return nullptr;
    }
    return ctx->B[i];
}

namespace {
enum { BB_FU = 0, BB_FDT = 1, BB_T1 = 2, BB_W = 9, BB_FW = 10 };

struct BbRun {
    lx_ctx* ctx;
    lx_rhs_fn f;
    void* user;
    const double* u;     // linearisation state (FD) or nullptr (linear operator)
    const double* fu;    // f(u) (FD)
    int rec;

    lx_status call_f(const double* in, double* out) {
        f(in, out, user, (void*)ctx->stream);
        CUDA_TRY(cudaGetLastError());
        return LX_OK;
    }
    BbLin lin() const {
        BbLin L;
        std::memset(&L, 0, sizeof L);
        L.N = ctx->N_loc;
        L.N_glob = ctx->N_glob;
        L.grid = bb_grid(ctx->nsm);
        L.u = u;
        L.fu = fu;
        L.partials = ctx->partials;
        L.ctrl = ctx->bb;
        L.rec = ctx->rec_dev + rec;
        return L;
    }
    // y = a0 x0 + a1 x1 + a2 x2 + a3 x3
    lx_status comb(double* y, double a0, const double* x0, double a1 = 0.0, const double* x1 = nullptr,
                   double a2 = 0.0, const double* x2 = nullptr, double a3 = 0.0, const double* x3 = nullptr) {
        BbLin L = lin();
        L.y0 = y;
        L.x0 = x0; L.x1 = x1; L.x2 = x2; L.x3 = x3;
        L.a0 = a0; L.a1 = a1; L.a2 = a2; L.a3 = a3;
        CUDA_TRY(launch_bb_lincomb(L, ctx->stream));
        ctx->launches++;
        return LX_OK;
    }
    // F(x) = f(x) - J_FD(u) x -> out (the listing's Nonlinear_remainder, alg:exprb32)
    lx_status remainder(const double* x, double* out) {
        double* w = bb_vec(ctx, BB_W);
        double* fw = bb_vec(ctx, BB_FW);
        if (!w || !fw) return fail(LX_ERR_CUDA, "black-box buffer allocation failed");
        LX_TRY(call_f(x, out));
        CUDA_TRY(cudaMemsetAsync(&ctx->bb->maxbits[2], 0, sizeof(unsigned long long), ctx->stream));
        CUDA_TRY(launch_bb_maxabs(x, ctx->N_loc, ctx->bb, bb_grid(ctx->nsm), ctx->stream));
        BbLin L = lin();
        L.x0 = x;
        L.y0 = w;
        CUDA_TRY(launch_bb_fdpiece(L, 0, ctx->stream));
        LX_TRY(call_f(w, fw));
        L = lin();
        L.x0 = out;
        L.x1 = fw;
        L.y0 = out;
        CUDA_TRY(launch_bb_fdpiece(L, 1, ctx->stream));
        ctx->launches += 3;
        return LX_OK;
    }
    // phi_l(a_k dt J) v -> outs[k]  (Eq. (2), stopping rule P:155)
    lx_status leja(const double* v, double* const* outs, const double* coeffs, int K, double dt, double c,
                   double gamma, int l, double rtol, double atol) {
        double* w = bb_vec(ctx, BB_W);
        double* fw = bb_vec(ctx, BB_FW);
        if (!w || !fw) return fail(LX_ERR_CUDA, "black-box buffer allocation failed");
        TableSpec spec{l, K, coeffs};
        const double* tab = nullptr;
        LX_TRY(build_tables(ctx, &spec, 1, dt, c, gamma, rec, &tab));
        BbArgs A;
        std::memset(&A, 0, sizeof A);
        A.N = ctx->N_loc;
        A.N_glob = ctx->N_glob;
        A.K = K;
        A.mode = u ? 1 : 2;
        A.max_nodes = ctx->max_nodes;
        A.grid = bb_grid(ctx->nsm);
        A.alpha = (dt == 0.0) ? 0.0 : 1.0 / gamma;
        A.rtol = rtol;
        A.atol = atol;
        A.table = tab;
        A.u = u;
        A.fu = fu;
        A.w = w;
        A.fw = fw;
        for (int k = 0; k < K; k++) A.p[k] = outs[k];
        A.partials = ctx->partials;
        A.ctrl = ctx->bb;
        A.rec = ctx->rec_dev + rec;
        A.done_host = ctx->bb_done_dev;
        // decision state: everything but max|u| (kept for the remainders of a step)
        CUDA_TRY(cudaMemsetAsync(ctx->bb, 0, offsetof(BbCtrl, umaxbits), ctx->stream));
        const int act0 = (1 << K) - 1;
        CUDA_TRY(cudaMemcpyAsync(&ctx->bb->active, &act0, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));   // host word reset below must not race the previous call
        *(volatile int*)ctx->bb_done_host = 0;
        A.y_in = v;
        CUDA_TRY(launch_bb_init(A, ctx->stream));
        ctx->launches++;
        for (int m = 1; m < ctx->max_nodes; m++) {
            A.y_in = (m == 1) ? v : ctx->Y[(m - 1) & 1];
            A.y_out = ctx->Y[m & 1];
            if (u) {
                CUDA_TRY(launch_bb_perturb(A, m, ctx->stream));
                LX_TRY(call_f(w, fw));
            } else {
                LX_TRY(call_f(A.y_in, fw));
            }
            CUDA_TRY(launch_bb_update(A, m, ctx->stream));
            ctx->launches += u ? 2 : 1;
            CUDA_TRY(cudaEventRecord(ctx->bb_ev[m & 3], ctx->stream));
            // kBbLag iterations in flight: wait for the decision of m - kBbLag while the later ones run
            // (their kernels return at entry once the decision says done; f still runs on an unchanged w)
            if (m > kBbLag) {
                CUDA_TRY(cudaEventSynchronize(ctx->bb_ev[(m - kBbLag) & 3]));
                if (*(volatile int*)ctx->bb_done_host) break;
            }
        }
        return LX_OK;
    }
};
}  // namespace

static lx_status bb_setup(lx_ctx* ctx, BbRun& R, lx_rhs_fn f, void* user, const double* u) {
    LX_TRY(bb_ensure(ctx));
    R.ctx = ctx;
    R.f = f;
    R.user = user;
    R.u = u;
    R.fu = nullptr;
    R.rec = 0;
    // FD Jacobians (u given) divide f's rounding differences by eps: the built-in f then runs in the literal,
    // contraction-free formula order (R30); a linear black-box operator uses the fused stencil
    ctx->bb_literal = u != nullptr;
    CUDA_TRY(cudaMemsetAsync(ctx->bb, 0, sizeof(BbCtrl), ctx->stream));
    if (u) {
        double* fu = bb_vec(ctx, BB_FU);
        if (!fu) return fail(LX_ERR_CUDA, "black-box buffer allocation failed");
        LX_TRY(R.call_f(u, fu));                      // f(u), unscaled (FD base point)
        R.fu = fu;
        // max|u| (FD scaling, R25) -> umaxbits
        CUDA_TRY(launch_bb_maxabs(u, ctx->N_loc, ctx->bb, bb_grid(ctx->nsm), ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(&ctx->bb->umaxbits, &ctx->bb->maxbits[2], sizeof(unsigned long long),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        ctx->launches++;
    }
    return LX_OK;
}

static lx_status bb_step(BbRun& R, lx_method method, const double* u, double* lo, double* hi, double dt, double c,
                         double gamma, double rtol, double atol) {
    lx_ctx* ctx = R.ctx;
    double* t[8];
    for (int i = 1; i <= 7; i++) {
        t[i] = bb_vec(ctx, BB_T1 + i - 1);
        if (!t[i]) return fail(LX_ERR_CUDA, "black-box buffer allocation failed");
    }
    double* f_u = bb_vec(ctx, BB_FDT);
    if (!f_u) return fail(LX_ERR_CUDA, "black-box buffer allocation failed");
    const double one = 1.0;
    LX_TRY(R.comb(f_u, dt, R.fu));                    // f_u = RHS(u) dt  (alg:Ros_Eu P:468-469)
    if (method == LX_ROSENBROCK_EULER) {
        double* o[1] = {t[1]};
        LX_TRY(R.leja(f_u, o, &one, 1, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.comb(hi, 1.0, u, 1.0, t[1]));        // u + phi_1(J dt) f_u
        if (lo && lo != hi) LX_TRY(R.comb(lo, 1.0, hi));
        return LX_OK;
    }
    if (method == LX_EXPRB32) {                        // P:414-418, alg:exprb32
        double* o[1] = {t[1]};
        LX_TRY(R.leja(f_u, o, &one, 1, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.comb(lo, 1.0, u, 1.0, t[1]));        // a = u_exprb2
        LX_TRY(R.remainder(u, t[2]));                 // NL_u
        LX_TRY(R.remainder(lo, t[3]));                // NL_a
        LX_TRY(R.comb(t[4], dt, t[3], -dt, t[2]));    // R_a = (NL_a - NL_u) dt
        double* o3[1] = {t[5]};
        LX_TRY(R.leja(t[4], o3, &one, 1, dt, c, gamma, 3, rtol, atol));
        LX_TRY(R.comb(hi, 1.0, lo, 2.0, t[5]));       // u_exprb3 = a + 2 u_nl_3
        BbLin L = R.lin();
        L.x0 = t[5];
        L.a0 = 2.0;
        CUDA_TRY(launch_bb_norm(L, ctx->stream));     // error = ||2 u_nl_3||
        ctx->launches++;
        return LX_OK;
    }
    if (method == LX_EXPRB42) {                        // reading R22
        const double cf[2] = {0.75, 1.0};
        double* pv[2] = {t[1], t[2]};
        LX_TRY(R.leja(f_u, pv, cf, 2, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.comb(t[3], 1.0, u, 0.75, t[1]));     // a
        LX_TRY(R.remainder(u, t[4]));
        LX_TRY(R.remainder(t[3], t[5]));
        LX_TRY(R.comb(t[6], dt, t[5], -dt, t[4]));    // D_a
        LX_TRY(R.comb(t[6], 32.0 / 9.0, t[6]));
        double* o3[1] = {t[7]};
        LX_TRY(R.leja(t[6], o3, &one, 1, dt, c, gamma, 3, rtol, atol));
        LX_TRY(R.comb(hi, 1.0, u, 1.0, t[2], 1.0, t[7]));
        if (lo && lo != hi) LX_TRY(R.comb(lo, 1.0, hi));
        return LX_OK;
    }
    if (method == LX_EXPRB54S4) {                      // reading R31
        const double e4[4] = {0.25, 0.5, 0.9, 1.0}, half = 0.5, c4 = 0.9;
        double* pv[4] = {t[1], t[2], t[3], t[7]};
        LX_TRY(R.leja(f_u, pv, e4, 4, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.remainder(u, t[4]));                 // NL_u
        LX_TRY(R.comb(t[5], 1.0, u, 0.25, t[1]));     // U2
        LX_TRY(R.remainder(t[5], t[6]));
        LX_TRY(R.comb(t[5], dt, t[6], -dt, t[4]));    // D2
        double* q1[1] = {t[1]};
        LX_TRY(R.leja(t[5], q1, &half, 1, dt, c, gamma, 3, rtol, atol));
        LX_TRY(R.comb(t[6], 1.0, u, 0.5, t[2], 4.0, t[1]));   // U3
        LX_TRY(R.remainder(t[6], lo));
        LX_TRY(R.comb(t[6], dt, lo, -dt, t[4]));      // D3
        LX_TRY(R.comb(t[1], 5832.0 / 125.0, t[5], -729.0 / 125.0, t[6]));
        LX_TRY(R.comb(t[2], -157464.0 / 625.0, t[5], 39366.0 / 625.0, t[6]));
        double* ol[1] = {lo};
        double* oh[1] = {hi};
        LX_TRY(R.leja(t[1], ol, &c4, 1, dt, c, gamma, 3, rtol, atol));
        LX_TRY(R.leja(t[2], oh, &c4, 1, dt, c, gamma, 4, rtol, atol));
        LX_TRY(R.comb(t[1], 1.0, u, 0.9, t[3], 1.0, lo, 1.0, hi));   // U4
        LX_TRY(R.remainder(t[1], t[2]));
        LX_TRY(R.comb(t[3], dt, t[2], -dt, t[4]));    // D4
        LX_TRY(R.comb(t[1], 64.0, t[5], -8.0, t[6]));
        LX_TRY(R.comb(t[2], -384.0, t[5], 96.0, t[6]));
        double* o4[1] = {t[4]};
        LX_TRY(R.leja(t[1], o4, &one, 1, dt, c, gamma, 3, rtol, atol));
        double* o5[1] = {lo};
        LX_TRY(R.leja(t[2], o5, &one, 1, dt, c, gamma, 4, rtol, atol));
        LX_TRY(R.comb(lo, 1.0, u, 1.0, t[7], 1.0, t[4], 1.0, lo));   // u4
        LX_TRY(R.comb(t[1], 18.0, t[6], -250.0 / 81.0, t[3]));
        LX_TRY(R.comb(t[2], -60.0, t[6], 500.0 / 27.0, t[3]));
        LX_TRY(R.leja(t[1], o4, &one, 1, dt, c, gamma, 3, rtol, atol));
        double* o6[1] = {t[5]};
        LX_TRY(R.leja(t[2], o6, &one, 1, dt, c, gamma, 4, rtol, atol));
        LX_TRY(R.comb(hi, 1.0, u, 1.0, t[7], 1.0, t[4], 1.0, t[5]));  // u5
        BbLin L = R.lin();
        L.x0 = hi;
        L.a0 = 1.0;
        L.x1 = lo;
        L.a1 = -1.0;
        CUDA_TRY(launch_bb_norm(L, ctx->stream));
        ctx->launches++;
        return LX_OK;
    }
    if (method == LX_EXPRB53S3) {                      // reading R27
        const double e3[3] = {0.5, 0.9, 1.0};
        double* pv[3] = {t[1], t[2], t[3]};
        LX_TRY(R.leja(f_u, pv, e3, 3, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.remainder(u, t[4]));                 // NL_u
        LX_TRY(R.comb(t[5], 1.0, u, 0.5, t[1]));      // U2
        LX_TRY(R.remainder(t[5], t[6]));
        LX_TRY(R.comb(t[5], dt, t[6], -dt, t[4]));    // D2
        double* qv[3] = {t[1], t[6], t[7]};
        LX_TRY(R.leja(t[5], qv, e3, 3, dt, c, gamma, 3, rtol, atol));
        LX_TRY(R.comb(t[1], 1.0, u, 0.9, t[2], 27.0 / 25.0, t[1], 729.0 / 125.0, t[6]));   // U3
        LX_TRY(R.remainder(t[1], t[2]));
        LX_TRY(R.comb(t[6], dt, t[2], -dt, t[4]));    // D3
        LX_TRY(R.comb(t[1], 18.0, t[5], -250.0 / 81.0, t[6]));   // w3
        LX_TRY(R.comb(t[2], -60.0, t[5], 500.0 / 27.0, t[6]));   // w4
        double* o3[1] = {t[4]};
        LX_TRY(R.leja(t[1], o3, &one, 1, dt, c, gamma, 3, rtol, atol));
        double* o4[1] = {t[5]};
        LX_TRY(R.leja(t[2], o4, &one, 1, dt, c, gamma, 4, rtol, atol));
        LX_TRY(R.comb(hi, 1.0, u, 1.0, t[3], 1.0, t[4], 1.0, t[5]));   // u5
        LX_TRY(R.comb(lo, 1.0, u, 1.0, t[3], 8.0, t[7]));              // u3
        BbLin L = R.lin();
        L.x0 = hi;
        L.a0 = 1.0;
        L.x1 = lo;
        L.a1 = -1.0;
        CUDA_TRY(launch_bb_norm(L, ctx->stream));
        ctx->launches++;
        return LX_OK;
    }
    if (method == LX_EPIRK5P1) {                       // reading R26
        using namespace epirk5;
        const double e3[3] = {g11, g21, g31}, e2[3] = {0.5, g32, g22}, e1[2] = {g33, 1.0};
        double* pv[3] = {t[1], t[2], t[3]};
        LX_TRY(R.leja(f_u, pv, e3, 3, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.remainder(u, t[4]));                 // NL_u
        LX_TRY(R.comb(t[5], 1.0, u, a11, t[1]));      // Y1
        LX_TRY(R.remainder(t[5], t[6]));
        LX_TRY(R.comb(t[5], dt, t[6], -dt, t[4]));    // R1
        double* qv[3] = {t[1], t[6], t[7]};           // phi_1 {1/2 (embedded, R33), g32, 1} on R1
        LX_TRY(R.leja(t[5], qv, e2, 3, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.comb(t[2], 1.0, u, a21, t[2], a22, t[7]));   // Y2 (in place)
        LX_TRY(R.remainder(t[2], t[7]));
        LX_TRY(R.comb(t[2], dt, t[7], -dt, t[4]));    // R2
        LX_TRY(R.comb(t[2], 1.0, t[2], -2.0, t[5]));  // R2 - 2 R1
        double* o3[2] = {t[7], t[5]};                 // phi_3 {g33, 1 (embedded)}
        LX_TRY(R.leja(t[2], o3, e1, 2, dt, c, gamma, 3, rtol, atol));
        LX_TRY(R.comb(hi, 1.0, u, b1, t[3], b2, t[6], b3, t[7]));   // u5
        double* u4 = lo ? lo : t[4];
        LX_TRY(R.comb(u4, 1.0, u, b1, t[3], b2, t[1], b3, t[5]));   // u4
        BbLin L = R.lin();
        L.x0 = hi;
        L.a0 = 1.0;
        L.x1 = u4;
        L.a1 = -1.0;
        CUDA_TRY(launch_bb_norm(L, ctx->stream));
        ctx->launches++;
        return LX_OK;
    }
    // EXPRB43 / EPIRK4s3A (reading R17) / EPIRK4s3B (reading R34) / EPIRK4s3 (reading R35)
    const bool epb = method == LX_EPIRK4S3B;
    const bool e4s3 = method == LX_EPIRK4S3;
    const bool epirk = method == LX_EPIRK4S3A || epb || e4s3;
    const double cf2[2] = {0.5, 1.0}, cf3[3] = {0.5, 2.0 / 3.0, 1.0}, cfb[2] = {0.5, 0.75};
    const double cf9[3] = {1.0 / 9.0, 1.0 / 8.0, 1.0};
    double* pv[3] = {e4s3 ? t[2] : t[1], e4s3 ? t[1] : t[2], t[3]};   // EPIRK4s3: t1 <- 1/8, t2 <- 1/9
    if (epb) {
        LX_TRY(R.leja(f_u, pv, cfb, 2, dt, c, gamma, 2, rtol, atol));   // phi_2 {1/2, 3/4}
        double* o1[1] = {t[3]};
        LX_TRY(R.leja(f_u, o1, &one, 1, dt, c, gamma, 1, rtol, atol));
    } else {
        LX_TRY(R.leja(f_u, pv, e4s3 ? cf9 : epirk ? cf3 : cf2, epirk ? 3 : 2, dt, c, gamma, 1, rtol, atol));
    }
    double* p_half = t[1];
    double* p_one = epirk ? t[3] : t[2];
    double *NLu = t[4], *Da = t[5], *Db = t[6], *tmp = t[7];
    LX_TRY(R.remainder(u, NLu));
    LX_TRY(R.comb(lo, 1.0, u, epb ? 2.0 / 3.0 : e4s3 ? 0.125 : 0.5, p_half));   // a
    LX_TRY(R.remainder(lo, tmp));
    LX_TRY(R.comb(Da, dt, tmp, -dt, NLu));
    if (epirk) {
        LX_TRY(R.comb(lo, 1.0, u, epb ? 1.0 : e4s3 ? 1.0 / 9.0 : 2.0 / 3.0, t[2]));  // b
    } else {
        double* o[1] = {hi};
        LX_TRY(R.leja(Da, o, &one, 1, dt, c, gamma, 1, rtol, atol));
        LX_TRY(R.comb(lo, 1.0, u, 1.0, p_one, 1.0, hi));   // b = u + p_one + phi_1 D_a
    }
    LX_TRY(R.remainder(lo, tmp));
    LX_TRY(R.comb(Db, dt, tmp, -dt, NLu));
    const double a3 = epb ? 54.0 : e4s3 ? -1024.0 : epirk ? 32.0 : 16.0;
    const double b3 = epb ? -16.0 : e4s3 ? 1458.0 : epirk ? -13.5 : -2.0;
    const double a4 = epb ? -324.0 : e4s3 ? 27648.0 : epirk ? -144.0 : -48.0;
    const double b4 = epb ? 144.0 : e4s3 ? -34992.0 : epirk ? 81.0 : 12.0;
    LX_TRY(R.comb(tmp, a3, Da, b3, Db));              // w3
    LX_TRY(R.comb(NLu, a4, Da, b4, Db));              // w4
    double* o3[1] = {Da};
    LX_TRY(R.leja(tmp, o3, &one, 1, dt, c, gamma, 3, rtol, atol));
    double* o4[1] = {Db};
    LX_TRY(R.leja(NLu, o4, &one, 1, dt, c, gamma, 4, rtol, atol));
    LX_TRY(R.comb(lo, 1.0, u, 1.0, p_one, 1.0, Da));  // u3
    LX_TRY(R.comb(hi, 1.0, lo, 1.0, Db));             // u4
    BbLin L = R.lin();
    L.x0 = hi;
    L.a0 = 1.0;
    L.x1 = lo;
    L.a1 = -1.0;
    CUDA_TRY(launch_bb_norm(L, ctx->stream));         // err = ||u4 - u3||
    ctx->launches++;
    return LX_OK;
}

extern "C" {

void lx_builtin_rhs(const double* in, double* out, void* user, void* cuda_stream) {
    (void)cuda_stream;
    const lx_builtin_rhs_user* b = (const lx_builtin_rhs_user*)user;
    if (!b || !b->ctx || !b->pb) return;
    lx_ctx* ctx = b->ctx;
    if (ctx->comm || !ctx->bb_literal) {   // slab contexts / a linear black-box operator: the fused stencil
        rhs_device(ctx, b->pb, in, 1.0, out);
        return;
    }
    RhsLit R;
    R.ndim = ctx->ndim;
    for (int d = 0; d < 3; d++) {
        R.n[d] = d < ctx->ndim ? ctx->n[d] : 1;
        R.dx[d] = b->pb->dx[d];
    }
    R.diff = b->pb->diff;
    R.nu = b->pb->nu;
    R.react = b->pb->react;
    R.flux = b->pb->flux;
    R.src = b->pb->source;
    R.in = in;
    R.out = out;
    if (launch_rhs_literal(R, ctx->nsm * 4, ctx->stream) == cudaSuccess) ctx->launches++;
}

lx_status lx_real_leja_phi_cb(lx_ctx* ctx, lx_rhs_fn f, void* user, const double* u, const double* v,
                              double* const* outs, const double* coeffs, int K, double dt, double c, double gamma,
                              int l, double rtol, double atol, int* iters_out) {
    if (!ctx || !f) return fail(LX_ERR_ARG, "NULL argument");
    lx_problem pb;
    std::memset(&pb, 0, sizeof pb);
    LX_TRY(validate_leja(&pb, u, v, outs, coeffs, K, dt, gamma, l));
    Staging sg(ctx);
    const double *vd, *ud;
    double* od[kMaxK];
    LX_TRY(sg.in(v, &vd));
    LX_TRY(sg.in(u, &ud));
    for (int k = 0; k < K; k++) LX_TRY(sg.out(outs[k], &od[k]));
    BbRun R;
    LX_TRY(bb_setup(ctx, R, f, user, ud));
    LX_TRY(reset_record(ctx, 0));
    LX_TRY(R.leja(vd, od, coeffs, K, dt, c, gamma, l, rtol, atol));
    LX_TRY(sg.finish());
    Record r;
    LX_TRY(read_record(ctx, 0, &r));
    if (iters_out) *iters_out = r.iters;
    return status_of(r);
}

lx_status lx_step_cb(lx_ctx* ctx, lx_method method, lx_rhs_fn f, void* user, const double* u, double* u_low,
                     double* u_high, double* err_out, double dt, double c, double gamma, double rtol, double atol,
                     int* iters_out) {
    if (!ctx || !f || !u || !u_high) return fail(LX_ERR_ARG, "NULL argument");
    if ((int)method < 0 || (int)method > 9) return fail(LX_ERR_UNKNOWN_INTEGRATOR, "unknown integrator %d", (int)method);
    if (!nonembedded(method) && method != LX_EPIRK5P1 && !u_low)   // EPIRK5P1: u_low optional (R33)
        return fail(LX_ERR_ARG, "u_low required for embedded methods");
    if (u_low == u || u_high == u) return fail(LX_ERR_ALIAS, "outputs must not alias u");
    if (u_low && u_low == u_high) return fail(LX_ERR_ALIAS, "u_low must differ from u_high");
    if (!(gamma > 0.0) && dt != 0.0) return fail(LX_ERR_ARG, "gamma must be > 0 (got %g)", gamma);
    Staging sg(ctx);
    const double* ud;
    double *lo, *hi;
    LX_TRY(sg.in(u, &ud));
    LX_TRY(sg.out(u_low, &lo));
    LX_TRY(sg.out(u_high, &hi));
    BbRun R;
    LX_TRY(bb_setup(ctx, R, f, user, ud));
    LX_TRY(reset_record(ctx, 0));
    LX_TRY(bb_step(R, method, ud, lo, hi, dt, c, gamma, rtol, atol));
    LX_TRY(sg.finish());
    Record r;
    LX_TRY(read_record(ctx, 0, &r));
    if (iters_out) *iters_out = r.iters;
    if (err_out) *err_out = nonembedded(method) ? 0.0 : r.err;
    return status_of(r);
}

}  // extern "C"
