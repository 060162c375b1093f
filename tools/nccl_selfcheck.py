#!/usr/bin/env python
"""Exercise the NCCL-created slab communicator on ONE GPU: a world of size 1 over torch.distributed/NCCL with
LX_COMM_FORCE (the library's own communicator with itself as both neighbours).  Mode "nccl": Leja calls run
the peer-memory slab kernel (exchange block handles gathered over NCCL), stage operations the NCCL step
protocol; mode "nccl_nopeer" (LX_COMM_NO_PEER): every Leja iteration through step kernels + NCCL groups.
Compares a Leja call, an EXPRB43 step and the Gershgorin bound with the single-domain path (and, on a 3D grid,
a vertical Leja call and an EPIRK4s3A step through the 3D slab kernel): identical iteration counts, fields
equal to 1e-13 (only the norm summation order differs).  --time: per-iteration
cost of the three paths at 4096^2 (config 1 shape).  Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2310_08344_b200 as lx  # noqa: E402
import paper_2310_08344_b200.dist as lxd  # noqa: E402
import workloads as W  # noqa: E402


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29631")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    out = {}
    n = 256
    pb = lx.Problem((n, n), (2 / n, 2 / n), 1e-4, 0.0, 1.0)
    u = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
    v = torch.from_numpy(W.ic_random((n, n), seed=3, amp=0.2)).cuda()
    res = {}
    modes = {"single": None, "nccl": lx.LX_COMM_FORCE, "nccl_nopeer": lx.LX_COMM_FORCE | lx.LX_COMM_NO_PEER}
    for mode, flags in modes.items():
        ctx = lx.Context(pb)
        if flags is not None:
            lxd.attach(ctx, flags)
        out["ipp_" + mode] = ctx.iterations_per_pass
        bound = lx.lx_spectrum_bound(ctx, u)
        c, g = lx.lx_shift_scale(bound)
        o = torch.empty_like(u)
        it = lx.lx_real_leja_phi(ctx, v, o, 0.01, c, g, 1, 1e-10, 1e-10, u_lin=u)
        lo, hi = torch.empty_like(u), torch.empty_like(u)
        its, err = lx.lx_step(ctx, "exprb43", u, lo, hi, 0.01, c, g, 1e-10, 1e-10)
        res[mode] = (bound, it, o.cpu().numpy(), its, err, hi.cpu().numpy())
        ctx.close()
    a = res["single"]
    ok = out["ipp_nccl"] == 2 and out["ipp_nccl_nopeer"] == 1
    for mode in ("nccl", "nccl_nopeer"):
        b = res[mode]
        out[mode] = {"bound_equal": a[0] == b[0], "leja_iters": [a[1], b[1]],
                     "leja_maxrel": float(np.abs(a[2] - b[2]).max() / np.abs(a[2]).max()),
                     "step_iters": [a[3], b[3]], "step_err": [a[4], b[4]],
                     "step_maxrel": float(np.abs(a[5] - b[5]).max() / np.abs(a[5]).max())}
        r = out[mode]
        ok = ok and bool(r["bound_equal"] and a[1] == b[1] and a[3] == b[3] and r["leja_maxrel"] <= 1e-13
                         and r["step_maxrel"] <= 1e-13)
    # 3D (the 3D two-step peer-memory slab kernel with itself as neighbour: ghost planes through the
    # NCCL-gathered exchange block) -- a vertical Leja call and an EPIRK4s3A step
    shape = (32, 16, 64)
    pb3 = lx.Problem(shape, tuple(2.0 / m for m in shape), 1.0, 10.0, 0.0)
    v3 = torch.from_numpy(W.ic_random(shape, seed=5, amp=0.2)).cuda()
    dt3 = 5 * min(W.dt_cfl(m, 10.0, 3) for m in shape)
    res3 = {}
    for mode, flags in modes.items():
        ctx = lx.Context(pb3)
        if flags is not None:
            lxd.attach(ctx, flags)
        else:
            ctx.set_kernel(2)
        out["ipp3_" + mode] = ctx.iterations_per_pass
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        outs = [torch.empty_like(v3) for _ in range(2)]
        it = lx.lx_real_leja_phi_vertical(ctx, v3, outs, (0.5, 1.0), dt3, c, g, 1, 1e-10, 1e-10)
        lo, hi = torch.empty_like(v3), torch.empty_like(v3)
        its, err = lx.lx_step(ctx, "epirk4s3a", v3, lo, hi, dt3, c, g, 1e-10, 1e-10)
        res3[mode] = (it, [o.cpu().numpy() for o in outs], its, hi.cpu().numpy())
        ctx.close()
    a = res3["single"]
    ok = ok and out["ipp3_single"] == 2 and out["ipp3_nccl"] == 2 and out["ipp3_nccl_nopeer"] == 1
    for mode in ("nccl", "nccl_nopeer"):
        b = res3[mode]
        r = {"leja_iters": [a[0], b[0]], "step_iters": [a[2], b[2]],
             "leja_maxrel": max(float(np.abs(x - y).max() / np.abs(x).max()) for x, y in zip(a[1], b[1])),
             "step_maxrel": float(np.abs(a[3] - b[3]).max() / np.abs(a[3]).max())}
        out[mode + "_3d"] = r
        ok = ok and a[0] == b[0] and a[2] == b[2] and r["leja_maxrel"] <= 1e-13 and r["step_maxrel"] <= 1e-13
    out["ok"] = ok
    if "--time" in sys.argv:
        # per-iteration cost of the slab protocol (step kernels + NCCL halo/allgather, here to itself) vs the
        # single-domain persistent kernel, 4096^2 phi_0 (config 1 shape)
        wl = W.config(1)
        pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
        u0 = torch.from_numpy(W.ic_problem1_2d(4096)).cuda()
        for mode, flags in modes.items():
            ctx = lx.Context(pb)
            if flags is not None:
                lxd.attach(ctx, flags)
            c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
            o = torch.empty_like(u0)
            it = lx.lx_real_leja_phi(ctx, u0, o, wl.dt, c, g, 0, wl.rtol, wl.atol)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s0.record()
            for _ in range(5):
                lx.lx_real_leja_phi(ctx, u0, o, wl.dt, c, g, 0, wl.rtol, wl.atol)
            s1.record()
            torch.cuda.synchronize()
            kern = {"single": "two-step persistent (single domain)",
                    "nccl": "two-step persistent slab kernel, peer-memory halos (itself as neighbour)",
                    "nccl_nopeer": "step kernels + NCCL group per iteration"}[mode]
            out["t_" + mode] = {"iters": it, "us_per_iter": s0.elapsed_time(s1) * 1e3 / (5 * it), "kernel": kern}
            ctx.close()
    print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
