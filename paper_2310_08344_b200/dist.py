"""Multi-process plumbing of the slab decomposition (one process per GPU).

torch.distributed is used only for bootstrap and timing: the NCCL unique id of
the library's own communicator is broadcast with ``broadcast_object_list``,
timings are reduced with MAX.  The per-iteration halo exchange and the partial
gather run inside liblexint_b200.so (csrc/lx_comm.cpp) on the context stream.

The exchange plan itself is the library's (``lx_slab_halo_plan``); the CPU gloo
tests drive an oracle-based emulation of both slab protocols with it.
"""
from __future__ import annotations

import os
from . import Context, lx_nccl_unique_id, lx_slab_range


def env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def share_unique_id() -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    import torch.distributed as dist
    obj = [lx_nccl_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def attach(ctx: Context, flags: int = 0) -> tuple:
    """Attach the context to an NCCL communicator spanning the process group (lx_ctx_set_comm_ex;
    flags: LX_COMM_FORCE, LX_COMM_NO_PEER).  Returns this rank's slab (i_begin, i_end)."""
    import torch.distributed as dist
    uid = share_unique_id()
    ctx.set_comm(uid, dist.get_rank(), dist.get_world_size(), flags)
    b, e, _ = ctx.local()
    return b, e


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def slabs(n0: int, world: int) -> list:
    return [lx_slab_range(n0, r, world) for r in range(world)]
