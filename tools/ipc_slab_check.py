#!/usr/bin/env python
"""Two PROCESSES, one GPU, the peer-memory slab kernel through real CUDA IPC mappings.

Each process owns a context on cuda:0 and one slab of a 2D (or, with "shape" of length 3, 3D) advection-diffusion
grid; the 64-byte IPC
handles of the exchange blocks are gathered by the parent and handed back (lx_ctx_ipc_handle /
lx_ctx_set_comm_ipc -- the caller-side handle exchange the ABI offers), then every process runs
lx_real_leja_phi on its slab.  The processes time-slice the GPU, so each cross-rank barrier waits for
the other process's time slice: this checks cross-process visibility of the halo rows and partials
(system-scope fences / acquire-release flags), not speed.  Prints one JSON line with the gathered
result; the caller (tests/test_gpu_slab.py) compares it with the oracle and the single-domain kernel.
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(rank, nranks, conn, shape, dt, c, g, ls, tol):
    import numpy as np
    import torch
    import paper_2310_08344_b200 as lx
    import workloads as W
    torch.cuda.set_device(0)
    pb = lx.Problem(shape, tuple(2.0 / n for n in shape), 1.0, 10.0, 0.0)
    ctx = lx.Context(pb)
    conn.send(ctx.ipc_handle())
    ctx.set_comm_ipc(rank, conn.recv())
    b, e, _ = ctx.local()
    v = torch.from_numpy(np.ascontiguousarray(W.ic_random(shape, seed=51, amp=0.2)[b:e])).cuda()
    res = []
    t0 = time.time()
    for l in ls:
        out = torch.empty_like(v)
        it = lx.lx_real_leja_phi(ctx, v, out, dt, c, g, l, tol, tol)
        res.append((it, out.cpu().numpy().tolist()))
    conn.send({"rank": rank, "b": b, "e": e, "res": res, "ipp": ctx.iterations_per_pass,
               "wall_s": time.time() - t0})
    ctx.close()


def main():
    args = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
    shape = tuple(args.get("shape", (96, 128)))
    nranks = 2
    dt, c, g, ls, tol = args["dt"], args["c"], args["g"], args["ls"], args["tol"]
    ctx = mp.get_context("spawn")
    pipes = [ctx.Pipe() for _ in range(nranks)]
    procs = [ctx.Process(target=child, args=(r, nranks, pipes[r][1], shape, dt, c, g, ls, tol)) for r in range(nranks)]
    for p in procs:
        p.start()
    handles = [pipes[r][0].recv() for r in range(nranks)]
    for r in range(nranks):
        pipes[r][0].send(handles)
    out = [pipes[r][0].recv() for r in range(nranks)]
    for p in procs:
        p.join(timeout=300)
    print(json.dumps({"shape": shape, "ranks": out}), flush=True)


if __name__ == "__main__":
    main()
