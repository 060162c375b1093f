// lx_comm.h -- slab decomposition over NCCL (one process per GPU).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/lexint.h"
#include "lx_internal.h"

namespace lx {
struct Comm;
const char* comm_error();
int comm_unique_id(void* out128);
int comm_halo_plan(int rank, int nranks, int n_loc, int mode, int* ops, int max_ops);
int comm_create(const void* uid, int rank, int nranks, int device, long long row, int max_grid, Comm** out);
struct LocalGroup;
LocalGroup* local_group_create(int nranks);
void local_group_destroy(LocalGroup* g);
int comm_create_local(LocalGroup* g, int rank, int device, long long row, Comm** out);
void comm_destroy(Comm* c);
void comm_bind(Comm* c, double* const Y[2], double* const Yg[2], double* vg, int n_loc, int rank, int nranks);
lx_status comm_leja(Comm* c, LejaParams& P, bool diag, cudaStream_t s, int64_t* launches);
lx_status comm_power(Comm* c, LejaParams& P, bool diag, cudaStream_t s, int64_t* launches);
int comm_allreduce_max_u64(Comm* c, unsigned long long* dev, cudaStream_t s);
int comm_stage_norm(Comm* c, int op, const StageArgs& A, cudaStream_t s, int64_t* launches);
int comm_rhs(Comm* c, LejaParams& P, double scale, cudaStream_t s, int64_t* launches);
// peer-memory slab transport (2D Leja calls: one persistent k_leja2d_tb2<K, DIAG, true> per call)
int comm_peer_enable(Comm* c, long long row);                       // collective
size_t comm_block_bytes(long long row);                            // exchange block of one rank
// IPC-only communicator: blk = this rank's exchange block (cudaMalloc'd, zeroed; ownership passes to
// the communicator), handles = every rank's cudaIpcMemHandle_t of its block (64 bytes each)
int comm_create_ipc(int rank, int nranks, int device, long long row, const void* handles, void* blk, Comm** out);
void comm_set_grid_div(Comm* c, int div);
bool comm_peer_ready(const Comm* c);
int comm_grid_cap(const Comm* c, int grid);
void comm_peer_params(const Comm* c, LejaParams& P, bool diag);
}  // namespace lx
