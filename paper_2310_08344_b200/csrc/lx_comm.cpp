// lx_comm.cpp -- slab decomposition of the Leja path over several ranks.
//
// Protocol per Leja iteration m (identical for every transport):
//   1. k_leja2d_step(m): decision of m-1 from the gathered per-rank partials
//      (summed in rank order -> the same decision on every rank), tiles of m,
//      per-rank partial {S_y, S_p^(k)} by a fixed-order last-block reduction;
//   2. halo: the 1 last row goes to rank r+1 (its ghost row -1) and the 2 first
//      rows go to rank r-1 (its ghost rows n, n+1) -- the +x-biased upwind
//      stencil reaches i-1, i+1, i+2 (reading R10); periodic in rank;
//   3. allgather of the per-rank partials (1+K doubles).
// The host enqueues iterations in chunks and polls the device `done` flag once
// per chunk (launches after convergence exit at entry), so every rank issues the
// same sequence of collectives.
//
// Transports: NCCL (one process per GPU, NVLink/NVSwitch) and LOCAL (virtual
// ranks = host threads of one process sharing one GPU; D2D copies + host
// barriers).  LOCAL runs the same protocol and kernels, so the multi-rank path is
// validated on a single B200 against the single-domain result.
#include "lx_comm.h"

#include <chrono>
#include <condition_variable>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#ifdef LX_HAVE_NCCL
#include <nccl.h>
#endif

namespace lx {

static thread_local std::string g_comm_err;
const char* comm_error() { return g_comm_err.c_str(); }
static int cerr(const std::string& m) {
    g_comm_err = m;
    return 1;
}
#define CU(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) return cerr(std::string(#x ": ") + cudaGetErrorString(e_));  \
    } while (0)

// The halo exchange plan of one rank: ops of 5 ints {kind (0 send, 1 recv), peer, first local row
// (send) / 0, row count, first ghost slot (at the peer for a send, here for a recv)}, in the order the
// transport issues them ("up" then "down", so that with two ranks -- both neighbours the same peer -- the
// messages still match one to one).  mode 0: the step protocol (3-row ghost block: slot 0 = row -1, slots 1, 2
// = rows n, n+1); mode 1: the two-step slab kernel's deliveries (6-row ghost block: slots 0, 1 = rows -2, -1,
// slots 2..5 = rows n..n+3).
int comm_halo_plan(int rank, int nranks, int n_loc, int mode, int* ops, int max_ops) {
    if (nranks < 1 || rank < 0 || rank >= nranks || max_ops < 4 || (mode != 0 && mode != 1)) return -1;
    const int up = (rank - 1 + nranks) % nranks, dn = (rank + 1) % nranks;
    const int nu = mode ? kTb2UpRows : kStepUpRows, nd = mode ? kTb2DnRows : kStepDnRows;
    const int gup = mode ? 2 : 1, gdn = 0;   // ghost slot of the first row received from below / above
    const int o[4][5] = {{0, up, 0, nu, gup},            // my first rows -> rank-1's rows n..
                         {1, dn, 0, nu, gup},            // rank+1's first rows -> my rows n..
                         {0, dn, n_loc - nd, nd, gdn},   // my last rows -> rank+1's rows -nd..-1
                         {1, up, 0, nd, gdn}};           // rank-1's last rows -> my rows -nd..-1
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 5; j++) ops[5 * i + j] = o[i][j];
    return 4;
}

struct Transport {
    int rank = 0, nranks = 1;
    virtual ~Transport() {}
    // make this rank's later writes safe against peers' still-pending reads of its buffers (the in-process
    // transport's D2D pulls run on the peers' streams); NCCL orders send/recv itself
    virtual int settle(cudaStream_t s) {
        (void)s;
        return 0;
    }
    // asynchronous transport error (NCCL: ncclCommGetAsyncError); abort() tears the communicator down so
    // that no rank blocks forever on a peer that failed
    virtual int async_error() { return 0; }
    virtual void abort() {}
    virtual int exchange_rows(const double* base, double* ghost, int n_loc, long long row, cudaStream_t s) = 0;
    virtual int allgather(const double* send, double* recv, int count, cudaStream_t s) = 0;
    virtual int allreduce_max_u64(unsigned long long* buf, cudaStream_t s) = 0;
    // peer-memory slab transport: make every rank's exchange block addressable from this process;
    // all[q] = rank q's block (all[rank] = mine).  Collective.
    virtual int exchange_blocks(void* mine, void** all) = 0;
    virtual void close_blocks(void** all) { (void)all; }
    // the per-iteration exchange: halo rows of y_m and the allgather of the per-rank partials
    virtual int exchange_and_gather(const double* base, double* ghost, int n_loc, long long row, const double* send,
                                    double* recv, int count, cudaStream_t s) {
        if (exchange_rows(base, ghost, n_loc, row, s)) return 1;
        return allgather(send, recv, count, s);
    }
};

// ------------------------------------------------------------------ NCCL
#ifdef LX_HAVE_NCCL
#define NC(x)                                                                                   \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) return cerr(std::string(#x ": ") + ncclGetErrorString(r_));      \
    } while (0)

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) ncclCommDestroy(comm);
    }
    // the step protocol's halo (comm_halo_plan mode 0) as one NCCL group
    int issue_halo(const double* base, double* ghost, int n_loc, long long row, cudaStream_t s) {
        int ops[20];
        const int nop = comm_halo_plan(rank, nranks, n_loc, 0, ops, 4);
        for (int i = 0; i < nop; i++) {
            const int* o = ops + 5 * i;
            if (o[0] == 0) NC(ncclSend(base + (long long)o[2] * row, (size_t)o[3] * row, ncclDouble, o[1], comm, s));
            else NC(ncclRecv(ghost + (long long)o[4] * row, (size_t)o[3] * row, ncclDouble, o[1], comm, s));
        }
        return 0;
    }
    int exchange_rows(const double* base, double* ghost, int n_loc, long long row, cudaStream_t s) override {
        NC(ncclGroupStart());
        if (issue_halo(base, ghost, n_loc, row, s)) return 1;
        NC(ncclGroupEnd());
        return 0;
    }
    int allgather(const double* send, double* recv, int count, cudaStream_t s) override {
        NC(ncclAllGather(send, recv, count, ncclDouble, comm, s));
        return 0;
    }
    int allreduce_max_u64(unsigned long long* buf, cudaStream_t s) override {
        NC(ncclAllReduce(buf, buf, 1, ncclUint64, ncclMax, comm, s));
        return 0;
    }
    // ONE NCCL group per Leja iteration: the 1+2-row halo send/recv and the partials allgather are
    // aggregated into a single launch (halves the per-iteration NCCL launches of the slab protocol)
    int exchange_and_gather(const double* base, double* ghost, int n_loc, long long row, const double* send,
                            double* recv, int count, cudaStream_t s) override {
        NC(ncclGroupStart());
        if (issue_halo(base, ghost, n_loc, row, s)) return 1;
        NC(ncclAllGather(send, recv, count, ncclDouble, comm, s));
        NC(ncclGroupEnd());
        return 0;
    }
    int fused = 1;
    int async_error() override {
        ncclResult_t st = ncclSuccess;
        if (ncclCommGetAsyncError(comm, &st) != ncclSuccess || (st != ncclSuccess && st != ncclInProgress))
            return cerr(std::string("NCCL async error: ") + ncclGetErrorString(st));
        return 0;
    }
    void abort() override {
        if (comm) ncclCommAbort(comm);
        comm = nullptr;
    }
    int exchange_blocks(void* mine, void** all) override {
        cudaIpcMemHandle_t h;
        CU(cudaIpcGetMemHandle(&h, mine));
        char* buf = nullptr;
        CU(cudaMalloc(&buf, (size_t)(nranks + 1) * sizeof h));
        int rc = 0;
        std::vector<cudaIpcMemHandle_t> hs(nranks);
        if (cudaMemcpy(buf + (size_t)nranks * sizeof h, &h, sizeof h, cudaMemcpyHostToDevice) != cudaSuccess) {
            rc = cerr("handle upload failed");
        } else {
            ncclResult_t r = ncclAllGather(buf + (size_t)nranks * sizeof h, buf, sizeof h, ncclChar, comm, 0);
            if (r != ncclSuccess) rc = cerr(std::string("ncclAllGather(handles): ") + ncclGetErrorString(r));
            else if (cudaStreamSynchronize(0) != cudaSuccess ||
                     cudaMemcpy(hs.data(), buf, (size_t)nranks * sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess)
                rc = cerr("handle download failed");
        }
        cudaFree(buf);
        for (int q = 0; q < nranks && !rc; q++) {
            if (q == rank) {
                all[q] = mine;
                continue;
            }
            if (cudaIpcOpenMemHandle(&all[q], hs[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
                rc = cerr("cudaIpcOpenMemHandle of rank " + std::to_string(q) + " failed");
        }
        return rc;
    }
    void close_blocks(void** all) override {
        for (int q = 0; q < nranks; q++)
            if (q != rank && all[q]) cudaIpcCloseMemHandle(all[q]);
    }
};
#endif

int comm_unique_id(void* out128) {
#ifdef LX_HAVE_NCCL
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return cerr(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out128, &id, 128);
    return 0;
#else
    (void)out128;
    return cerr("built without NCCL");
#endif
}

// ------------------------------------------------------------------ LOCAL
struct LocalGroup {
    int nranks;
    std::mutex mu;
    std::condition_variable cv;
    int count = 0;
    long long gen = 0;
    std::vector<const void*> ptr;
    std::vector<int> nloc;
    std::vector<cudaEvent_t> ev;
    std::vector<void*> blk;    // peer-memory exchange blocks (same process: plain device pointers)
    explicit LocalGroup(int n) : nranks(n), ptr(n, nullptr), nloc(n, 0), ev(n, nullptr), blk(n, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long long g = gen;
        if (++count == nranks) {
            count = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

LocalGroup* local_group_create(int nranks) { return new LocalGroup(nranks); }
void local_group_destroy(LocalGroup* g) { delete g; }

struct LocalTransport : Transport {
    LocalGroup* g = nullptr;
    cudaEvent_t ev = nullptr;
    unsigned long long* tmp = nullptr;  // device [nranks]
    ~LocalTransport() override {
        if (ev) cudaEventDestroy(ev);
        cudaFree(tmp);
    }
    int publish(const void* p, int n_loc, cudaStream_t s) {
        CU(cudaEventRecord(ev, s));
        g->ptr[rank] = p;
        g->nloc[rank] = n_loc;
        g->ev[rank] = ev;
        g->barrier();
        return 0;
    }
    int exchange_rows(const double* base, double* ghost, int n_loc, long long row, cudaStream_t s) override {
        if (publish(base, n_loc, s)) return 1;
        const int up = (rank - 1 + nranks) % nranks, down = (rank + 1) % nranks;
        int rc = 0;
        if (cudaStreamWaitEvent(s, g->ev[up], 0) != cudaSuccess || cudaStreamWaitEvent(s, g->ev[down], 0) != cudaSuccess)
            rc = cerr("cudaStreamWaitEvent failed");
        const double* ub = (const double*)g->ptr[up];
        const double* db = (const double*)g->ptr[down];
        if (!rc && cudaMemcpyAsync(ghost, ub + (long long)(g->nloc[up] - 1) * row, row * sizeof(double),
                                   cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            rc = cerr("halo copy (up) failed");
        if (!rc && cudaMemcpyAsync(ghost + row, db, 2 * row * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            rc = cerr("halo copy (down) failed");
        g->barrier();  // everybody enqueued their pulls before pointers are republished
        return rc;
    }
    // Make every rank's stream wait until all peers finished the copies they just
    // enqueued (so a rank cannot overwrite a buffer a peer has not read yet).
    int settle(cudaStream_t s) override {
        if (publish(nullptr, 0, s)) return 1;
        int rc = 0;
        for (int r = 0; r < nranks; r++)
            if (cudaStreamWaitEvent(s, g->ev[r], 0) != cudaSuccess) rc = cerr("cudaStreamWaitEvent failed");
        g->barrier();
        return rc;
    }
    int allgather(const double* send, double* recv, int count, cudaStream_t s) override {
        if (publish(send, 0, s)) return 1;
        int rc = 0;
        for (int r = 0; r < nranks && !rc; r++) {
            if (cudaStreamWaitEvent(s, g->ev[r], 0) != cudaSuccess ||
                cudaMemcpyAsync(recv + (long long)r * count, g->ptr[r], count * sizeof(double), cudaMemcpyDeviceToDevice,
                                s) != cudaSuccess)
                rc = cerr("allgather copy failed");
        }
        g->barrier();
        if (settle(s)) return 1;
        return rc;
    }
    int exchange_blocks(void* mine, void** all) override {
        g->blk[rank] = mine;
        g->barrier();
        for (int q = 0; q < nranks; q++) all[q] = g->blk[q];
        g->barrier();
        return 0;
    }
    int allreduce_max_u64(unsigned long long* buf, cudaStream_t s) override {
        if (publish(buf, 0, s)) return 1;
        int rc = 0;
        for (int r = 0; r < nranks && !rc; r++) {
            if (cudaStreamWaitEvent(s, g->ev[r], 0) != cudaSuccess ||
                cudaMemcpyAsync(tmp + r, g->ptr[r], sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                rc = cerr("allreduce copy failed");
        }
        g->barrier();
        if (settle(s)) return 1;   // all peers have read every buf before anyone overwrites its own
        if (!rc && launch_max_u64(tmp, nranks, buf, s) != cudaSuccess) rc = cerr("max kernel failed");
        return rc;
    }
};

// ------------------------------------------------------------------ IPC only
// Peer-memory transport whose handles were exchanged by the caller (lx_ctx_set_comm_ipc): the Leja
// calls run the slab kernel over peer memory; operations that need a collective outside that kernel
// (stage halos, norms, spectrum bounds) are not available in this mode.
struct IpcTransport : Transport {
    std::vector<cudaIpcMemHandle_t> hs;
    int exchange_rows(const double*, double*, int, long long, cudaStream_t) override { return nocoll(); }
    int allgather(const double*, double*, int, cudaStream_t) override { return nocoll(); }
    int allreduce_max_u64(unsigned long long*, cudaStream_t) override { return nocoll(); }
    static int nocoll() { return cerr("IPC-only communicator: only Leja calls (slab kernel) are supported"); }
    int exchange_blocks(void* mine, void** all) override {
        for (int q = 0; q < nranks; q++) {
            if (q == rank) {
                all[q] = mine;
                continue;
            }
            if (cudaIpcOpenMemHandle(&all[q], hs[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
                return cerr("cudaIpcOpenMemHandle of rank " + std::to_string(q) + " failed");
        }
        return 0;
    }
    void close_blocks(void** all) override {
        for (int q = 0; q < nranks; q++)
            if (q != rank && all[q]) cudaIpcCloseMemHandle(all[q]);
    }
};

// ------------------------------------------------------------------ Comm
struct Comm {
    Transport* tr = nullptr;
    int rank = 0, nranks = 1, device = 0;
    long long row = 0;
    int n_loc = 0;
    double* Y[2] = {nullptr, nullptr};
    double* Yg[2] = {nullptr, nullptr};
    double* vg = nullptr;
    double* rank_part = nullptr;   // device [kSlot]
    double* gathered = nullptr;    // device [nranks][kSlot]
    int* done_host = nullptr;      // pinned [2]
    Ctrl* ctrl_init = nullptr;     // pinned [kMaxK + 1] templates (hist[0] = active0)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int chunk = 4;
    // peer-memory slab transport (k_leja2d_tb2<K, DIAG, true>)
    bool peer = false;
    char* blk = nullptr;           // this rank's exchange block: XHdr | ghost Y[0] | ghost Y[1] | ghost v | ghost u
    void* blks[kMaxRanks] = {};    // every rank's block (peer pointers)
    int grid_div = 1;              // virtual ranks share one GPU: each persistent grid gets 1/nranks of it
    unsigned long long timeout_ns = 60ull * 1000000000ull;
};

static constexpr size_t kXHdrBytes = 4096;
static_assert(sizeof(XHdr) <= kXHdrBytes, "exchange header");

// exchange block: XHdr | ghost blocks (6 rows each) of Y[0], Y[1], v, u | band flags fl_up[nbmax], fl_dn[nbmax]
static size_t blk_nbmax(long long row) { return (size_t)(row / kBand2 + 2); }
static size_t blk_bytes(long long row) {
    return kXHdrBytes + 4 * 6 * (size_t)row * sizeof(double) + 2 * blk_nbmax(row) * sizeof(unsigned);
}
static double* blk_ghost(void* b, long long row, int which) {   // 0, 1: Y[i]; 2: v; 3: u
    return (double*)((char*)b + kXHdrBytes) + (size_t)which * 6 * row;
}
static unsigned* blk_flags(void* b, long long row, int dir) {   // 0: fl_up, 1: fl_dn
    return (unsigned*)((char*)b + kXHdrBytes + 4 * 6 * (size_t)row * sizeof(double)) + (size_t)dir * blk_nbmax(row);
}

static int comm_alloc(Comm* c) {
    CU(cudaMalloc(&c->rank_part, kSlot * sizeof(double)));
    CU(cudaMalloc(&c->gathered, (size_t)c->nranks * kSlot * sizeof(double)));
    CU(cudaMemset(c->rank_part, 0, kSlot * sizeof(double)));
    CU(cudaMemset(c->gathered, 0, (size_t)c->nranks * kSlot * sizeof(double)));
    CU(cudaMallocHost(&c->done_host, 2 * sizeof(int)));
    CU(cudaMallocHost(&c->ctrl_init, (kMaxK + 1) * sizeof(Ctrl)));
    std::memset(c->ctrl_init, 0, (kMaxK + 1) * sizeof(Ctrl));
    for (int k = 0; k <= kMaxK; k++) c->ctrl_init[k].hist[0] = c->ctrl_init[k].hist[1] = (1 << k) - 1;
    for (auto& e : c->ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return 0;
}

int comm_create(const void* uid, int rank, int nranks, int device, long long row, int max_grid, Comm** out) {
    (void)max_grid;
#ifdef LX_HAVE_NCCL
    CU(cudaSetDevice(device));
    Comm* c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    c->row = row;
    auto* t = new NcclTransport();
    t->rank = rank;
    t->nranks = nranks;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclResult_t r = ncclCommInitRank(&t->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete t;
        delete c;
        return cerr(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    c->tr = t;
    if (comm_alloc(c)) {
        comm_destroy(c);
        return 1;
    }
    *out = c;
    return 0;
#else
    (void)uid; (void)rank; (void)nranks; (void)device; (void)row; (void)out;
    return cerr("built without NCCL");
#endif
}

int comm_create_local(LocalGroup* g, int rank, int device, long long row, Comm** out) {
    CU(cudaSetDevice(device));
    Comm* c = new Comm();
    c->rank = rank;
    c->nranks = g->nranks;
    c->device = device;
    c->row = row;
    auto* t = new LocalTransport();
    t->rank = rank;
    t->nranks = g->nranks;
    t->g = g;
    c->tr = t;
    if (cudaEventCreateWithFlags(&t->ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&t->tmp, g->nranks * sizeof(unsigned long long)) != cudaSuccess || comm_alloc(c)) {
        comm_destroy(c);
        return cerr("local transport allocation failed");
    }
    *out = c;
    return 0;
}

void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->peer) c->tr->close_blocks(c->blks);
    cudaFree(c->blk);
    delete c->tr;
    cudaFree(c->rank_part);
    cudaFree(c->gathered);
    cudaFreeHost(c->done_host);
    cudaFreeHost(c->ctrl_init);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    delete c;
}

void comm_bind(Comm* c, double* const Y[2], double* const Yg[2], double* vg, int n_loc, int rank, int nranks) {
    (void)rank; (void)nranks;
    for (int i = 0; i < 2; i++) {
        c->Y[i] = Y[i];
        c->Yg[i] = Yg[i];
    }
    c->vg = vg;
    c->n_loc = n_loc;
}

int comm_exchange(Comm* c, const double* base, double* ghost, cudaStream_t s) {
    return c->tr->exchange_rows(base, ghost, c->n_loc, c->row, s);
}

// Enqueue iterations 1..last in chunks; poll `done` once per chunk (one chunk behind).
template <typename Launch>
static lx_status run_chunked(Comm* c, Ctrl* ctrl, int last, Launch launch, cudaStream_t s) {
    int chunk = 0;
    for (int m = 1; m <= last; m++) {
        if (launch(m)) return LX_ERR_NCCL;
        if (m % c->chunk == 0 || m == last) {
            if (cudaMemcpyAsync(&c->done_host[chunk & 1], &ctrl->done, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaEventRecord(c->ev[chunk & 1], s) != cudaSuccess)
                return LX_ERR_CUDA;
            if (chunk >= 1) {
                // poll instead of blocking: a failed peer (NCCL async error) or a stall beyond the watchdog
                // aborts the communicator rather than hanging this rank forever
                const auto t0 = std::chrono::steady_clock::now();
                for (;;) {
                    const cudaError_t q = cudaEventQuery(c->ev[(chunk - 1) & 1]);
                    if (q == cudaSuccess) break;
                    if (q != cudaErrorNotReady) return LX_ERR_CUDA;
                    if (c->tr->async_error() ||
                        std::chrono::steady_clock::now() - t0 > std::chrono::seconds(c->timeout_ns / 1000000000ull)) {
                        if (!c->tr->async_error()) cerr("slab protocol: no progress within the watchdog limit");
                        c->tr->abort();
                        return LX_ERR_NCCL;
                    }
                    std::this_thread::sleep_for(std::chrono::microseconds(20));
                }
                if (c->done_host[(chunk - 1) & 1]) break;
            }
            chunk++;
        }
    }
    return LX_OK;
}

lx_status comm_leja(Comm* c, LejaParams& P, bool diag, cudaStream_t s, int64_t* launches) {
    P.nranks = c->nranks;
    P.rank_part = c->rank_part;
    P.gathered = c->gathered;
    P.grid = step_grid_size(c->device, P.nunits);
    P.v.ghost = c->vg;
    if (cudaMemcpyAsync(P.ctrl, &c->ctrl_init[P.K], sizeof(Ctrl), cudaMemcpyHostToDevice, s) != cudaSuccess)
        return LX_ERR_CUDA;
    if (comm_exchange(c, P.v.base, c->vg, s) || c->tr->settle(s)) return LX_ERR_NCCL;
    const int M = P.max_nodes;
    auto launch = [&](int m) -> int {
        if (launch_leja_step(P, m, s, diag) != cudaSuccess) return cerr("step kernel launch failed");
        (*launches)++;
        if (m < M && c->tr->exchange_and_gather(c->Y[m & 1], c->Yg[m & 1], c->n_loc, c->row, c->rank_part,
                                                       c->gathered, kSlot, s)) {
            return 1;
        }
        return 0;
    };
    return run_chunked(c, P.ctrl, M, launch, s);
}

lx_status comm_power(Comm* c, LejaParams& P, bool diag, cudaStream_t s, int64_t* launches) {
    P.nranks = c->nranks;
    P.rank_part = c->rank_part;
    P.gathered = c->gathered;
    P.grid = step_grid_size(c->device, P.nunits);
    if (cudaMemcpyAsync(P.ctrl, &c->ctrl_init[0], sizeof(Ctrl), cudaMemcpyHostToDevice, s) != cudaSuccess)
        return LX_ERR_CUDA;
    if (comm_exchange(c, c->Y[0], c->Yg[0], s)) return LX_ERR_NCCL;
    const int last = P.power_iters + 1;
    auto launch = [&](int m) -> int {
        if (launch_power_step(P, m, s, diag) != cudaSuccess) return cerr("power step launch failed");
        (*launches)++;
        if (m < last) {
            if (comm_exchange(c, c->Y[m & 1], c->Yg[m & 1], s)) return 1;
            if (c->tr->allgather(c->rank_part, c->gathered, kSlot, s)) return 1;
        }
        return 0;
    };
    return run_chunked(c, P.ctrl, last, launch, s);
}

int comm_allreduce_max_u64(Comm* c, unsigned long long* dev, cudaStream_t s) {
    return c->tr->allreduce_max_u64(dev, s);
}

int comm_stage_norm(Comm* c, int op, const StageArgs& A0, cudaStream_t s, int64_t* launches) {
    StageArgs A = A0;
    A.rank_part = c->rank_part;
    CU(launch_stage(op, A, s));
    (*launches)++;
    if (c->tr->allgather(c->rank_part, c->gathered, kSlot, s)) return 1;
    CU(launch_finalize_err(c->gathered, c->nranks, A.N_glob, A.rec, s));
    (*launches)++;
    return 0;
}

int comm_rhs(Comm* c, LejaParams& P, double scale, cudaStream_t s, int64_t* launches) {
    if (comm_exchange(c, P.v.base, c->vg, s)) return 1;
    if (c->tr->settle(s)) return 1;   // peers' pulls of this rank's rows done before the caller may overwrite u
    P.v.ghost = c->vg;
    P.grid = step_grid_size(c->device, P.nunits);
    CU(launch_rhs(P, scale, s));
    (*launches)++;
    return 0;
}

// ------------------------------------------------------------------ peer-memory slab transport
int comm_peer_enable(Comm* c, long long row) {
    if (c->nranks > kMaxRanks) return cerr("peer transport: at most 8 ranks");
    CU(cudaMalloc(&c->blk, blk_bytes(row)));
    CU(cudaMemset(c->blk, 0, blk_bytes(row)));
    CU(cudaDeviceSynchronize());   // zeroed flags before any peer can write them
    if (c->tr->exchange_blocks(c->blk, c->blks)) return 1;
    c->peer = true;
    return 0;
}

size_t comm_block_bytes(long long row) { return blk_bytes(row); }

int comm_create_ipc(int rank, int nranks, int device, long long row, const void* handles, void* blk, Comm** out) {
    CU(cudaSetDevice(device));
    if (nranks > kMaxRanks) return cerr("peer transport: at most 8 ranks");
    Comm* c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    c->row = row;
    c->blk = (char*)blk;   // owned from here on
    auto* t = new IpcTransport();
    t->rank = rank;
    t->nranks = nranks;
    t->hs.resize(nranks);
    std::memcpy(t->hs.data(), handles, (size_t)nranks * sizeof(cudaIpcMemHandle_t));
    c->tr = t;
    if (comm_alloc(c) || c->tr->exchange_blocks(c->blk, c->blks)) {
        comm_destroy(c);
        return 1;
    }
    c->peer = true;
    *out = c;
    return 0;
}

void comm_set_grid_div(Comm* c, int div) { c->grid_div = div < 1 ? 1 : div; }
bool comm_peer_ready(const Comm* c) { return c && c->peer; }
int comm_grid_cap(const Comm* c, int grid) {
    const int g = grid / c->grid_div;
    return g < 1 ? 1 : g;
}

void comm_peer_params(const Comm* c, LejaParams& P, bool diag) {
    (void)diag;
    const int up = (c->rank - 1 + c->nranks) % c->nranks, dn = (c->rank + 1) % c->nranks;
    P.xrank = c->rank;
    P.xranks = c->nranks;
    for (int q = 0; q < kMaxRanks; q++) P.xh[q] = q < c->nranks ? (XHdr*)c->blks[q] : nullptr;
    for (int i = 0; i < 2; i++) {
        P.gy[i] = blk_ghost(c->blk, c->row, i);
        P.hup[i] = blk_ghost(c->blks[up], c->row, i);
        P.hdn[i] = blk_ghost(c->blks[dn], c->row, i);
    }
    P.gv = blk_ghost(c->blk, c->row, 2);
    P.gu = blk_ghost(c->blk, c->row, 3);
    P.hup_v = blk_ghost(c->blks[up], c->row, 2);
    P.hdn_v = blk_ghost(c->blks[dn], c->row, 2);
    P.hup_u = blk_ghost(c->blks[up], c->row, 3);
    P.hdn_u = blk_ghost(c->blks[dn], c->row, 3);
    P.fl_up = blk_flags(c->blk, c->row, 0);
    P.fl_dn = blk_flags(c->blk, c->row, 1);
    P.fl_up_dn = blk_flags(c->blks[dn], c->row, 0);
    P.fl_dn_up = blk_flags(c->blks[up], c->row, 1);
    P.timeout_ns = c->timeout_ns;
}

}  // namespace lx
