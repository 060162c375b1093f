#!/usr/bin/env python
"""Per-iteration cost of the slab paths on ONE GPU (device-timed, CUDA events on each rank's stream).

* single: one context, the whole grid (two-step kernel);
* peer P: P virtual ranks (host threads, one stream each) with the persistent peer-memory slab kernel,
  each rank's grid capped to 1/P of the GPU -- the same bytes as "single" on the same GPU, so the ratio
  t_peer / t_single isolates the slab protocol's overhead (ghost-row stores, cross-rank barrier);
* step P: the same with LX_COMM_NO_PEER (step kernel + D2D halo copies + host barriers per iteration).
Grid: n0 x n1 = (rows per rank x P) x n1, phi_0 of the Problem-I Gaussian at 10 x CFL; with a third argument
n2, the 3D grid (planes per rank x P) x n1 x n2 (random input, 5 x CFL; the 3D two-step kernel and its
peer-memory slab instantiation).  Prints JSON lines.
"""
import json
import os
import sys
import threading

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2310_08344_b200 as lx  # noqa: E402
import workloads as W  # noqa: E402


def run(shape, P, flags, reps=5):
    pb = lx.Problem(shape, tuple(2.0 / s for s in shape), 1.0, 10.0, 0.0)
    u0 = W.ic_problem1_2d(*shape) if len(shape) == 2 and shape[0] == shape[1] else W.ic_random(shape, seed=3, amp=0.2)
    dt = (10 if len(shape) == 2 else 5) * W.dt_cfl(max(shape), 10.0, len(shape))
    c, g = lx.lx_shift_scale(sum(4.0 / (h * h) + 40.0 / (3.0 * h) for h in (2.0 / s for s in shape)))   # R9
    out = [None] * P
    errs = []
    group = lx.LocalGroup(P) if P else None

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = lx.Context(pb, stream=s)
                if P:
                    ctx.set_comm_local(group, r, flags)
                b, e, _ = ctx.local()
                v = torch.from_numpy(u0[b:e].copy()).cuda()
                o = torch.empty_like(v)
                it = lx.lx_real_leja_phi(ctx, v, o, dt, c, g, 0, 1e-10, 1e-10)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.synchronize()
                e0.record(s)
                for _ in range(reps):
                    lx.lx_real_leja_phi(ctx, v, o, dt, c, g, 0, 1e-10, 1e-10, sync=False)
                e1.record(s)
                s.synchronize()
                out[r] = (it, e0.elapsed_time(e1) / reps, ctx.iterations_per_pass)
                ctx.close()
        except BaseException as ex:  # noqa: BLE001
            errs.append(ex)

    if P == 0:
        out = [None]
        worker(0)
    else:
        th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
        [t.start() for t in th]
        [t.join() for t in th]
    if errs:
        raise errs[0]
    it = out[0][0]
    ms = max(o[1] for o in out)
    return {"shape": list(shape), "P": P, "flags": flags, "iters": it, "ms_per_call": ms,
            "us_per_iter": ms * 1e3 / it, "iterations_per_pass": out[0][2]}


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    n1 = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    rest = (int(sys.argv[3]),) if len(sys.argv) > 3 else ()
    for P in ((1, 2, 4, 8) if rest else (1, 2, 4)):
        shape = (rows * max(P, 1), n1) + rest
        base = run(shape, 0, 0)
        print(json.dumps(dict(base, mode="single")), flush=True)
        for mode, flags in (("peer", lx.LX_COMM_FORCE), ("step", lx.LX_COMM_FORCE | lx.LX_COMM_NO_PEER)):
            r = run(shape, P, flags)
            r["mode"] = mode
            r["ratio_vs_single"] = r["ms_per_call"] / base["ms_per_call"]
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
