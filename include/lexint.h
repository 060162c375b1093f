/*
 * lexint.h -- C ABI of the B200-native LeXInt hot path (arxiv 2310.08344).
 *
 * Library: paper_2310_08344_b200/liblexint_b200.so (sm_100a, fp64).
 * Citations: P:<line> = PAPER.md line (section / equation / listing).
 *
 * Conventions (apply to every call below)
 * ---------------------------------------
 *  - Scalars and all vector data are IEEE fp64.  Vectors are contiguous,
 *    row-major, dimension 0 slowest (index = (i*n1 + j)*n2 + k), unpadded,
 *    and hold the caller's LOCAL slab: rows [i_begin, i_end) of dimension 0
 *    (the whole grid when the context has no communicator).  P:155 "data ...
 *    have to lie contiguous in memory".
 *  - Pointers may be DEVICE pointers (cudaMalloc / torch CUDA tensors, on the
 *    context's device, 16-byte aligned) or HOST pointers (pageable or pinned).
 *    Host data is staged through context-owned device buffers (the
 *    host<->device copies are part of the call).  Mixing host and device
 *    pointers in one call is allowed.  Leja calls (lx_real_leja_phi*) whose
 *    host vectors are all PINNED (cudaHostAlloc / cudaHostRegister / torch
 *    pin_memory) and whose u_lin is on the device are PIPELINED: H2D on a
 *    copy-in stream, the kernels on the context stream, D2H on a copy-out
 *    stream, two staging slots, so consecutive calls overlap their copies
 *    with each other's kernels; such calls may also be asynchronous (all
 *    out-pointers NULL) -- the host outputs are valid after
 *    lx_ctx_synchronize.  Other host-pointer calls are synchronous.
 *  - Ownership: the caller allocates and owns every input and output vector
 *    ("the user has to assign the required amount of memory for
 *    the output vector").  The context owns all scratch (P:307, P:359-407:
 *    "allocated only once - when an object of this class is created"); it is
 *    freed by lx_ctx_destroy.
 *  - Stream ordering: all device work is enqueued on the context stream.
 *    Calls taking an `int* iters_out` (or `double* err_out`) return after one
 *    small device->host read of the call's record (one host synchronisation
 *    per call/step, never per Leja iteration).  Passing NULL for every such
 *    out-pointer makes the call ASYNCHRONOUS (device pointers only): results
 *    accumulate in the context record and are read by lx_ctx_synchronize.
 *  - Errors: every call returns an lx_status; lx_last_error() returns a
 *    thread-local message for the last non-OK status.  On LX_ERR_NOCONV the
 *    output holds the last polynomial and *iters_out the node cap - 1.
 *  - Concurrency: a context is not thread-safe; use one per host thread /
 *    stream.  Distinct contexts may run concurrently.  No global mutable state
 *    except the thread-local error string and the (immutable once built)
 *    Leja-point table.
 */
#ifndef LEXINT_H
#define LEXINT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LX_OK = 0,
    LX_ERR_ARG = 1,           /* invalid argument (NULL, gamma <= 0 with dt != 0, bad coeffs, ...) */
    LX_ERR_DIM = 2,           /* grid shape unsupported (n < 4, odd n_last, slab too thin)        */
    LX_ERR_ALIAS = 3,         /* an output aliases an input it must not alias                     */
    LX_ERR_UNSUPPORTED = 4,   /* l > 4, K > 4, ndim not 2/3, ...                                  */
    LX_ERR_NOCONV = 5,        /* node cap reached without meeting the tolerance          */
    LX_ERR_NONFINITE = 6,     /* NaN/Inf in a norm (spectrum not enclosed / bad input)            */
    LX_ERR_UNKNOWN_INTEGRATOR = 7,
    LX_ERR_CUDA = 8,
    LX_ERR_NCCL = 9,
    LX_ERR_TIMEOUT = 10       /* device-side barrier watchdog fired                               */
} lx_status;

const char *lx_last_error(void);
const char *lx_version(void);

/* ------------------------------------------------------------------------ */
/* Host math (no device work)                                                */
/* ------------------------------------------------------------------------ */

/* Real Leja points on [-2, 2] (§2.1): xi_0 = +2 (|z_0| = max|z|),
 * xi_j = argmax_z prod_{k<j} |z - xi_k|, ties to the larger z.
 * count in [1, 4096]; xi_out[count] written.  Errors: LX_ERR_ARG. */
lx_status lx_leja_points(int count, double *xi_out);

/* phi_l(z): phi_0 = exp, phi_{l+1}(z) = (phi_l(z) - 1/l!)/z.
 * l in [0, 4] (else LX_ERR_UNSUPPORTED).  Relative accuracy ~1e-15. */
lx_status lx_phi_scalar(int l, double z, double *out);

/* Newton divided differences d_0..d_{m-1} of h(xi) = phi_l(a*dt*(c + gamma*xi))
 * at xi[0..m-1] (interpolate phi_l(c + gamma xi) on the Leja
 * points; a = vertical coefficient, 1.0 for a plain call).
 * Errors: LX_ERR_ARG (m < 1, NULL), LX_ERR_UNSUPPORTED (l > 4),
 * LX_ERR_NONFINITE (overflow). */
lx_status lx_divided_differences(int l, const double *xi, int m, double dt, double c,
                                 double gamma, double a, double *d_out);

/* Rows [i_begin, i_end) of dimension 0 owned by `rank` of `nranks` slabs. */
lx_status lx_slab_range(int64_t n0, int rank, int nranks, int64_t *i_begin, int64_t *i_end);

/* Halo exchange plan of one rank (host only, no device): the +x-biased upwind stencil reaches rows i-1,
 * i+1, i+2 (reading R10).  Writes up to max_ops ops of 5 ints {kind (0 = send, 1 = recv), peer,
 * first local row (send; 0 for recv), row count, first ghost slot (at the peer for a send, at this rank for
 * a recv)} in issue order and returns their number (-1 on bad arguments; max_ops >= 4).
 *   mode 0: the step protocol, one Leja iteration per exchange: rows 0, 1 -> rank-1 (its rows n, n+1), row
 *           n-1 -> rank+1 (its row -1); 3-row ghost block, slot 0 = row -1, slots 1, 2 = rows n, n+1.
 *   mode 1: the two-step slab kernel, two iterations per exchange: rows 0..3 -> rank-1 (its rows n..n+3),
 *           rows n-2, n-1 -> rank+1 (its rows -2, -1); 6-row ghost block, slots 0, 1 = rows -2, -1, slots
 *           2..5 = rows n..n+3.
 * The NCCL step protocol issues exactly these ops; the slab kernel's peer stores follow mode 1. */
int lx_slab_halo_plan(int rank, int nranks, int64_t n_loc, int mode, int *ops, int max_ops);

/* ------------------------------------------------------------------------ */
/* Problem: du/dt = f(u) = A u + g(u)   (Eq. (1))                   */
/*   A u  = diff * lap(u) + nu * sum_d D_d u                                */
/*          lap: second-order centred; D_d: third-order upwind, +x-biased   */
/*          (stencil (-u[i+2] + 6u[i+1] - 3u[i] - 2u[i-1])/(6 dx))   */
/*   g(u) = react * (u - u^3)   (Allen-Cahn; react = 0 for Problems I/II)   */
/*        + (flux/2) sum_d D_d(u^2)   (viscous Burgers, Problem III)          */
/*   + S   (optional source, Problem II)                                     */
/*   J(u) v = A v + react * (1 - 3u^2) v + flux sum_d D_d(u v)  (exact J)     */
/* Periodic on every dimension.                                              */
/* ------------------------------------------------------------------------ */
typedef struct {
    int ndim;         /* 2 or 3                                               */
    int64_t n[3];     /* GLOBAL points per dimension (n[2] = 1 when ndim = 2) */
    double dx[3];     /* grid spacing per dimension                           */
    double diff;      /* diffusion coefficient                                */
    double nu;        /* advection velocity                           */
    double react;     /* reaction weight (0 or 1)                             */
    double flux;      /* Burgers flux weight beta (Problem III): f += (beta/2) sum_d D_d(u^2),
                         J(u) v += beta sum_d D_d(u v); 2D single-GPU contexts only               */
    const double *source; /* optional time-independent source S added to f (Problem II,
                             P:583-586: f(u) = A u + S); caller's local slab, device or host
                             pointer; NULL -> no source.  S does not enter J(u) and cancels in
                             every nonlinear-remainder difference F(x) - F(u) (reading R21). */
} lx_problem;

typedef struct lx_ctx lx_ctx;

/* Create a context for problems on the grid of `pb` (only pb->ndim, pb->n
 * are used here).  max_nodes = Leja node cap (0 -> 300; <= 1024).
 * device = CUDA device ordinal (-1 -> current).  cuda_stream = cudaStream_t
 * to enqueue on (NULL -> a non-blocking stream owned by the context; pass
 * cudaStreamLegacy = (void*)1 for the legacy default stream).
 * Allocates: 2 y buffers + 3-row ghosts each, 7 stage vectors, partial-sum
 * slots, control block, coefficient-table ring, host staging (lazily).
 * Errors: LX_ERR_ARG, LX_ERR_DIM, LX_ERR_UNSUPPORTED, LX_ERR_CUDA. */
lx_status lx_ctx_create(const lx_problem *pb, int max_nodes, int device, void *cuda_stream,
                        lx_ctx **out);
lx_status lx_ctx_destroy(lx_ctx *ctx);

/* Attach a communicator for slab decomposition over nranks GPUs (one process
 * per GPU; SURVEY 8(e) -- the paper has no multi-GPU path).
 * nccl_unique_id: 128 bytes from lx_nccl_unique_id on rank 0, broadcast by the
 * caller (e.g. torch.distributed).  After this call every vector argument is
 * the caller's local slab (lx_slab_range).  Collective: every rank must call it
 * with the same flags.
 * Leja calls on 2D grids with >= 16 rows per rank and >= 64 columns run ONE
 * persistent kernel per call and rank (two Leja iterations per HBM pass): halo
 * rows are stored into the neighbours' ghost rows through peer memory (CUDA IPC
 * mappings of every rank's exchange block, handles gathered over NCCL) from
 * inside the pass, and the per-rank norm partials meet at the pass barrier in
 * every rank's exchange header (summed in rank order: identical decisions on
 * every rank).  No NCCL call, no launch and no host round trip per iteration;
 * a peer that does not arrive within 60 s ends the call with LX_ERR_TIMEOUT.
 * Leja calls on 3D grids with n1 % 16 == 0, n2 % 64 == 0 and >= 4 planes per
 * rank (constant-coefficient operators) do the same with ghost PLANES (the 3D
 * two-step kernel: two iterations per plane sweep, one global barrier per pass).
 * Other operations (3D Allen-Cahn, Burgers, power iteration, stage kernels) use
 * one step kernel + one NCCL group (1+2 halo rows, allgather of partials) per
 * iteration.
 * flags: LX_COMM_FORCE  -- build the communicator even for nranks == 1 (the slab
 *                          protocol with itself; by default one rank = the
 *                          single-domain context);
 *        LX_COMM_NO_PEER -- never use the peer-memory slab kernel.
 * Errors: LX_ERR_NCCL, LX_ERR_DIM (slab < 2 rows), LX_ERR_ARG. */
#define LX_COMM_FORCE 1
#define LX_COMM_NO_PEER 2
lx_status lx_nccl_unique_id(void *out128);
lx_status lx_ctx_set_comm(lx_ctx *ctx, const void *nccl_unique_id, int rank, int nranks);
lx_status lx_ctx_set_comm_ex(lx_ctx *ctx, const void *nccl_unique_id, int rank, int nranks, int flags);

/* In-process slab decomposition over `nranks` VIRTUAL ranks (host threads of
 * one process, all on the context's device).  Runs exactly the multi-rank
 * protocols of lx_ctx_set_comm -- the peer-memory slab kernel (each virtual
 * rank's persistent grid gets 1/nranks of the GPU) and the per-iteration step
 * protocol with device-to-device copies and host barriers as the transport;
 * used to validate the slab path on one GPU.  Each rank's calls must be issued
 * from its own host thread, all ranks making the same sequence of calls.
 * flags as for lx_ctx_set_comm_ex. */
typedef struct lx_local_group lx_local_group;
lx_status lx_local_group_create(int nranks, lx_local_group **out);
lx_status lx_local_group_destroy(lx_local_group *group);
lx_status lx_ctx_set_comm_local(lx_ctx *ctx, lx_local_group *group, int rank);
lx_status lx_ctx_set_comm_local_ex(lx_ctx *ctx, lx_local_group *group, int rank, int flags);

/* Peer-memory communicator whose handles the CALLER exchanges (e.g. over a
 * torch.distributed gloo group): lx_ctx_ipc_handle allocates this context's
 * exchange block and writes its 64-byte CUDA IPC handle to out64; after every
 * rank gathered all handles (rank order, nranks x 64 bytes),
 * lx_ctx_set_comm_ipc maps the peers' blocks.  Only Leja calls (the slab
 * kernel) are available on such a context: operations that need a collective
 * outside the kernel return LX_ERR_NCCL.  Ranks may share one GPU (processes
 * time-slice it).  1..8 ranks; 2D: >= 16 rows per rank, n1 >= 64; 3D: >= 4 planes per rank,
 * n1 % 16 == 0, n2 % 64 == 0.
 * Errors: LX_ERR_UNSUPPORTED, LX_ERR_DIM, LX_ERR_ARG, LX_ERR_NCCL, LX_ERR_CUDA. */
lx_status lx_ctx_ipc_handle(lx_ctx *ctx, void *out64);
lx_status lx_ctx_set_comm_ipc(lx_ctx *ctx, int rank, int nranks, const void *handles);

/* Local slab of this context: rows [*i_begin, *i_end), *n_local points. */
lx_status lx_ctx_local(const lx_ctx *ctx, int64_t *i_begin, int64_t *i_end, int64_t *n_local);

/* Wait for all enqueued work; report the iterations / status accumulated by
 * asynchronous calls since the last synchronize, then reset that record. */
lx_status lx_ctx_synchronize(lx_ctx *ctx, int *iters_total, double *err_last);

/* Number of kernel launches this context has issued (for bench accounting). */
int64_t lx_ctx_launch_count(const lx_ctx *ctx);
/* Leja iterations per HBM pass of this context's Leja calls on its constant-coefficient / Allen-Cahn
 * problems: 2 = the temporally blocked kernels (2D single domain with >= 3*2^20
 * local points, 3D (n1 % 16 == 0, n2 % 64 == 0) with >= 2^20, or lx_ctx_set_kernel(ctx, 2, .), and
 * the peer-memory slab kernels), 1 = one pass per iteration.  Burgers (flux) problems, and Allen-Cahn
 * problems in 3D, always run one pass per iteration.  Determines the algorithmic bytes of a call
 * (DESIGN.md §5).  0 for a NULL context. */
int lx_ctx_iterations_per_pass(const lx_ctx *ctx);
/* Kernel choice of this context (default 0 = automatic):
 * iterations_per_pass -- 2D single-domain Leja calls: 1 = one Leja iteration per HBM pass
 *                        (k_leja2d), 2 = two (k_leja2d_tb2, needs >= 16 rows and >= 64
 *                        columns), 0 = two from 3*2^20 points on (measured crossover);
 * kernel3d            -- 3D: 0 = shared-memory plane tiles when n1 % 16 == 0 and
 *                        n2 % 64 == 0 (else warp tiles), 1 = warp tiles.
 * All variants compute the same iterations (bitwise-equal fields except after a
 * two-step rollback, which is within one rounding).  Errors: LX_ERR_ARG. */
lx_status lx_ctx_set_kernel(lx_ctx *ctx, int iterations_per_pass, int kernel3d);

/* ------------------------------------------------------------------------ */
/* Spectrum (P:91, P:274-278 listing alg:lexint)                             */
/* ------------------------------------------------------------------------ */

/* Power iteration on J(u): v_0 = 1 + e_0, `iters` applications,
 * estimate ||J v|| / ||v||.  u may be NULL when pb->react == 0.
 * One fused stencil + norm pass per iteration on the device. */
lx_status lx_spectrum_estimate(lx_ctx *ctx, const lx_problem *pb, const double *u, int iters,
                               double *lambda_abs_out);

/* Closed-form bound of |lambda_max(J(u))|: sum_d (4 diff/dx_d^2 + 4|nu|/(3dx_d))
 * (Fourier symbol at theta = pi) + react * max(0, 3 max_i u_i^2 - 1)
 * (Gershgorin; device max-reduction, bitwise deterministic).  Synchronous. */
lx_status lx_spectrum_bound(lx_ctx *ctx, const lx_problem *pb, const double *u,
                            double *lambda_abs_out);

/* Listing alg:lexint P:277-278: eig = -1.05*|lambda|; c = eig/2; gamma = -eig/4. */
lx_status lx_shift_scale(double lambda_abs, double *c_out, double *gamma_out);

/* ------------------------------------------------------------------------ */
/* Real Leja interpolation (Eq. (2); P:155 stopping rule;          */
/* listings alg:leja_exp_ext, alg:leja_phi_nl_ext, alg:leja_phi)             */
/*   out ~= phi_l(dt J(u)) v, with (c, gamma) enclosing the spectrum of J(u) */
/*   (NOT of dt J):  y_m = y_{m-1} ((J - c)/gamma - xi_{m-1}),               */
/*   p_m = p_{m-1} + d_m y_m, stop at the first m >= 1 with                  */
/*   |d_m| ||y_m|| <= rtol ||p_m|| + atol (norms l2 / sqrt(N_global)).       */
/*   *iters_out = m (number of operator applications).                       */
/* Each Leja iteration is ONE fused HBM pass (stencil of y_{m-1}, Newton     */
/* update, polynomial accumulate, both norm partial sums) and the stopping   */
/* decision is taken on the device (no host round trip per iteration).       */
/* u_lin: linearisation state for J(u) (NULL when pb->react == 0).           */
/* out must not alias v or u_lin (LX_ERR_ALIAS).                             */
/* ------------------------------------------------------------------------ */
lx_status lx_real_leja_phi(lx_ctx *ctx, const lx_problem *pb, const double *u_lin,
                           const double *v, double *out, double dt, double c, double gamma,
                           int l, double rtol, double atol, int *iters_out);

/* Vertical interpolation (Tokman16): outs[k] ~= phi_l(coeffs[k] dt J(u)) v
 * for K coefficients 0 < coeffs[0] < ... < coeffs[K-1] <= 1 sharing one
 * y-recurrence; converged accumulators are frozen; *iters_out = recurrence
 * steps until all K converged.  K in [1, 4]. */
lx_status lx_real_leja_phi_vertical(lx_ctx *ctx, const lx_problem *pb, const double *u_lin,
                                    const double *v, double *const *outs, const double *coeffs,
                                    int K, double dt, double c, double gamma, int l, double rtol,
                                    double atol, int *iters_out);

/* Several phi functions of one vector in one interpolation: outs[k] ~= phi_{ls[k]}(coeffs[k] dt J(u)) v.
 * The Newton basis y_m ((J - cI)/gamma - xi_m I applied to v, Eq. (2)) does not depend on l,
 * so K accumulators with their own divided differences (h(xi) = phi_{l_k}(a_k dt (c +
 * gamma xi))) share it, exactly as the vertical interpolation shares it across coefficients: each
 * accumulator stops at the iteration P:155 gives it, bitwise the output and iteration count of its own
 * lx_real_leja_phi / _vertical call; *iters_out = steps until all K converged.  Typical use: phi_0 .. phi_3
 * of the same v, or an EPIRK stage's phi_2 {1/2, 3/4} and phi_1 {1} on the same f (R34).
 * ls[k] in [0, 4], coeffs[k] in (0, 1], (ls[k], coeffs[k]) pairs distinct, K in [1, 4]; otherwise as
 * lx_real_leja_phi_vertical (host buffers staged, NULL iters_out = asynchronous).
 * Errors: LX_ERR_ARG, LX_ERR_UNSUPPORTED, LX_ERR_ALIAS, LX_ERR_NOCONV, LX_ERR_NONFINITE, LX_ERR_CUDA. */
lx_status lx_real_leja_phi_multi(lx_ctx *ctx, const lx_problem *pb, const double *u_lin, const double *v,
                                 double *const *outs, const int *ls, const double *coeffs, int K, double dt,
                                 double c, double gamma, double rtol, double atol, int *iters_out);

/* ------------------------------------------------------------------------ */
/* Exponential integrator steps (listings alg:Ros_Eu, alg:exprb32; */
/* EXPRB43 / EPIRK4s3A tableaux from the papers cited at P:83).              */
/*   u: state u^n; u_low / u_high: lower / higher order u^{n+1};             */
/*   *err_out = ||u_high - u_low|| / sqrt(N) (EXPRB32: ||2 u_nl_3||). */
/*   *iters_out = total Leja iterations of the step.                         */
/* Outputs must not alias u; u_low != u_high.                                */
/* ------------------------------------------------------------------------ */
typedef enum {
    LX_ROSENBROCK_EULER = 0,
    LX_EXPRB32 = 1,
    LX_EXPRB43 = 2,
    LX_EPIRK4S3A = 3,
    LX_EXPRB42 = 4,       /* Luan 2017 (cited at P:83), 4th order, non-embedded (err = 0) */
    LX_EPIRK5P1 = 5,      /* Tokman et al. 2012 (cited at P:83, Table 2), 5th order, embedded 4th (R26, R33) */
    LX_EXPRB53S3 = 6,     /* Luan & Ostermann 2014 (cited at P:83), 5th order, embedded 3rd (R27)      */
    LX_EXPRB54S4 = 7,     /* Luan & Ostermann 2014 (cited at P:83), 5th order, embedded 4th (R31)      */
    LX_EPIRK4S3B = 8,     /* Rainwater & Tokman 2016 (cited at P:83), 4th order, embedded 3rd (R34):
                             a = u + 2/3 hphi_2(hJ/2) f, b = u + hphi_2(3hJ/4) f, u3 = u + hphi_1(hJ) f +
                             phi_3(hJ)(54 D_a - 16 D_b), u4 = u3 + phi_4(hJ)(-324 D_a + 144 D_b)          */
    LX_EPIRK4S3 = 9       /* cited at P:83, 4th order, embedded 3rd (R35): a = u + 1/8 hphi_1(hJ/8) f,
                             b = u + 1/9 hphi_1(hJ/9) f, u3 = u + hphi_1(hJ) f + phi_3(hJ)(-1024 D_a + 1458 D_b),
                             u4 = u3 + phi_4(hJ)(27648 D_a - 34992 D_b)                                    */
} lx_method;

/* Rosenbrock-Euler: u_out = u + phi_1(dt J(u)) f(u) dt (alg:Ros_Eu). */
lx_status lx_step_rosenbrock_euler(lx_ctx *ctx, const lx_problem *pb, const double *u,
                                   double *u_out, double dt, double c, double gamma,
                                   double rtol, double atol, int *iters_out);
lx_status lx_step_exprb32(lx_ctx *ctx, const lx_problem *pb, const double *u, double *u_low,
                          double *u_high, double *err_out, double dt, double c, double gamma,
                          double rtol, double atol, int *iters_out);
lx_status lx_step_exprb43(lx_ctx *ctx, const lx_problem *pb, const double *u, double *u_low,
                          double *u_high, double *err_out, double dt, double c, double gamma,
                          double rtol, double atol, int *iters_out);
lx_status lx_step_epirk4s3a(lx_ctx *ctx, const lx_problem *pb, const double *u, double *u_low,
                            double *u_high, double *err_out, double dt, double c, double gamma,
                            double rtol, double atol, int *iters_out);
/* EXPRB42 (reading R22): a = u + 3/4 hphi_1(3/4 hJ) f; u_out = u + hphi_1(hJ) f + 32/9 hphi_3(hJ) D_a. */
lx_status lx_step_exprb42(lx_ctx *ctx, const lx_problem *pb, const double *u, double *u_out, double dt,
                          double c, double gamma, double rtol, double atol, int *iters_out);
/* EPIRK5P1 (reading R26): Y1 = u + a11 hphi_1(g11 hJ) f; Y2 = u + a21 hphi_1(g21 hJ) f + a22 phi_1(hJ) R(Y1);
 * u_out = u + hphi_1(hJ) f + b2 phi_1(g32 hJ) R(Y1) + b3 phi_3(g33 hJ)(R(Y2) - 2R(Y1)), R(x) = h(F(x) - F(u)).
 * lx_step(LX_EPIRK5P1, ...) also returns the embedded fourth-order solution u_low (g32 -> 1/2, g33 -> 1,
 * reading R33; u_low may be NULL) and err = ||u_high - u_low|| / sqrt(N). */
lx_status lx_step_epirk5p1(lx_ctx *ctx, const lx_problem *pb, const double *u, double *u_out, double dt,
                           double c, double gamma, double rtol, double atol, int *iters_out);
/* Dispatch by method (the paper's exp_int / embed_exp_int). */
lx_status lx_step(lx_ctx *ctx, lx_method method, const lx_problem *pb, const double *u,
                  double *u_low, double *u_high, double *err_out, double dt, double c,
                  double gamma, double rtol, double atol, int *iters_out);

/* Embedded-error step-size control (the embedded error "may be used to control the step sizes";
 * reading R32).  Integrates u (device pointer, in place) from 0 to t_end with an embedded method
 * (EXPRB32, EXPRB43, EPIRK4s3A, EXPRB53S3, EXPRB54S4): per attempted step the spectrum bound of the
 * current state gives (c, gamma), the step gives err = ||u_high - u_low|| / sqrt(N); accept
 * iff err <= tol; next step h * min(5, max(0.2, 0.9 (tol/err)^(1/(q+1)))) with q the embedded order
 * (2, 3, 3, 3, 4); the last step is clipped to land on t_end; a step whose Leja calls fail (NOCONV /
 * NONFINITE) is rejected with factor 0.2.  Optional logs (max_steps entries): every attempted step size
 * and its error.  One host round trip per attempted step.  Errors: LX_ERR_ARG (non-embedded method, bad
 * t_end / dt0 / tol, host u), LX_ERR_NOCONV (max_steps attempts did not reach t_end), device errors. */
lx_status lx_integrate_adaptive(lx_ctx *ctx, lx_method method, const lx_problem *pb, double *u, double t_end,
                                double dt0, double tol, double rtol, double atol, int max_steps, int *accepted,
                                int *rejected, double *log_dt, double *log_err, int *iters_out);

/* The paper's time loop (listing alg:lexint) run on the device: nsteps steps of
 * `method` from the state in u (overwritten with u^{n+nsteps}).  Before every step the spectrum
 * bound of J(u^n) is recomputed ON THE DEVICE (closed form + Gershgorin max-reduction,
 * eig = -1.05 |lambda|, c = eig/2, gamma = -eig/4) and the Leja kernels read (c, gamma)
 * from device memory, so the whole run is enqueued without host round trips.  *iters_out = total
 * Leja iterations, *err_out = embedded error of the last step.  NULL out-pointers -> asynchronous
 * (device u only).  Uses 3 extra context state vectors. */
lx_status lx_integrate(lx_ctx *ctx, lx_method method, const lx_problem *pb, double *u, double dt, int nsteps,
                       double rtol, double atol, int *iters_out, double *err_out);

/* f(u) * dt (alg:Ros_Eu P:468-469) as a standalone fused stencil pass. */
lx_status lx_rhs(lx_ctx *ctx, const lx_problem *pb, const double *u, double scale, double *f_out);

/* ------------------------------------------------------------------------ */
/* Black-box right-hand side.                              */
/* The paper's interface: the user supplies only f (listing       */
/* alg:RHS: a functor taking an input and an output pointer to contiguous    */
/* data) and the Jacobian action is "computed numerically using finite       */
/* differences".  Reading R25:                           */
/*   J(u) y = (f(u + eps y) - f(u)) / eps,                                   */
/*   eps = 2^-26 (1 + ||u||_inf) / ||y||_inf,  J(u) 0 = 0;                    */
/*   nonlinear remainder F(x) = f(x) - J(u) x literally (alg:exprb32).        */
/* ------------------------------------------------------------------------ */
/* f(in) -> out on the device: in / out are N_loc contiguous doubles on the
 * context's device (in read-only; out never aliases in).  f must enqueue its
 * work on cuda_stream (the context stream) or complete it before returning;
 * it must not call back into the same context except through lx_builtin_rhs. */
typedef void (*lx_rhs_fn)(const double *in, double *out, void *user, void *cuda_stream);

/* phi_l(a_k dt J) v for a black-box operator (P:175-191 real_Leja_phi_nl(RHS, ...),
 * P:421-443 real_Leja_phi; recurrence P:142-147 Eq. (2); stopping rule P:155):
 *   u != NULL: J = J(u) by finite differences of f (R25);
 *   u == NULL: J y = f(y) -- f must then be LINEAR (Problem I's RHS = A).
 * Same argument meaning, layout, ownership and errors as lx_real_leja_phi_vertical.
 * Per Leja iteration: one f call (plus one for f(u)), a perturbation kernel (FD) and one
 * fused update kernel (Newton update + K accumulators + norms + device decision); the host
 * waits for the decision of iteration m-1 while iteration m runs (one extra f call at the
 * end, whose kernels return at entry).  Single-GPU contexts only (LX_ERR_UNSUPPORTED). */
lx_status lx_real_leja_phi_cb(lx_ctx *ctx, lx_rhs_fn f, void *user, const double *u, const double *v,
                              double *const *outs, const double *coeffs, int K, double dt, double c,
                              double gamma, int l, double rtol, double atol, int *iters_out);

/* One integrator step with a black-box f (the paper's exp_int / embed_exp_int on a user
 * RHS; listings alg:Ros_Eu, alg:exprb32; R17, R22 tableaux), Jacobian actions and
 * nonlinear remainders by finite differences (R25).  Arguments and errors as lx_step. */
lx_status lx_step_cb(lx_ctx *ctx, lx_method method, lx_rhs_fn f, void *user, const double *u,
                     double *u_low, double *u_high, double *err_out, double dt, double c, double gamma,
                     double rtol, double atol, int *iters_out);

/* The built-in stencil f of a problem packaged as an lx_rhs_fn (user points to this struct;
 * pb->source, if any, must be a device pointer).  Lets the black-box path be checked against
 * the same operator the fused kernels apply. */
typedef struct {
    lx_ctx *ctx;
    const lx_problem *pb;
} lx_builtin_rhs_user;
void lx_builtin_rhs(const double *in, double *out, void *user, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* LEXINT_H */
