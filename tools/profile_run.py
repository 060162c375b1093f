#!/usr/bin/env python
"""Small driver for ncu captures: runs one workload a few times (first call = warm-up).

  python tools/profile_run.py leja2d 4096 0      # phi_0 Leja call, 2D
  python tools/profile_run.py leja3d 512 0       # phi_0 Leja call, 3D
  python tools/profile_run.py vert3d 512 1       # config 5's dominant call: vertical phi_1 {1/2, 2/3, 1} on f(u) dt
  python tools/profile_run.py ac 2048 2          # Allen-Cahn EXPRB43, 2 steps
  python tools/profile_run.py step 4096 0        # bench step (phi_0..phi_3), warm-up + 1
  python tools/profile_run.py aci 2048 2         # the same through lx_integrate
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_08344_b200 as lx  # noqa: E402
import workloads as W  # noqa: E402


def main():
    what, n, arg = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    torch.cuda.set_device(0)
    if what in ("leja2d", "leja3d"):
        if what == "leja2d":
            wl = W.config(1, n=n)
            u = torch.from_numpy(W.ic_problem1_2d(n)).cuda()
        else:
            wl = W.config(4, n=n)
            c1 = W.coords(n)
            u = torch.empty(wl.shape, dtype=torch.float64, device="cuda")
            y, z = np.meshgrid(c1, c1, indexing="ij")
            for i in range(n):
                u[i] = torch.from_numpy(1.0 + np.exp(-((c1[i] + .5) ** 2 + (y + .5) ** 2 + (z + .5) ** 2) / 0.01))
        pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
        ctx = lx.Context(pb)
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        out = torch.empty_like(u)
        for _ in range(reps):
            it = lx.lx_real_leja_phi(ctx, u, out, wl.dt, c, g, arg, wl.rtol, wl.atol)
        print("iters", it)
    elif what == "vert3d":   # bench config 5's dominant kernel (the EPIRK4s3A step's K = 3 call)
        wl = W.config(4, n=n)
        pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
        ctx = lx.Context(pb)
        u = torch.from_numpy(W.ic_gaussian_3d(n)).cuda()
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        fdt = torch.empty_like(u)
        lx.lx_rhs(ctx, u, fdt, wl.dt)
        coeffs = (0.5, 2.0 / 3.0, 1.0)
        outs = [torch.empty_like(u) for _ in coeffs]
        m_k = [lx.lx_real_leja_phi(ctx, fdt, outs[0], wl.dt * a, c, g, arg, wl.rtol, wl.atol) for a in coeffs]
        for _ in range(reps):
            it = lx.lx_real_leja_phi_vertical(ctx, fdt, outs, coeffs, wl.dt, c, g, arg, wl.rtol, wl.atol)
        print("iters", it, "accumulators", ":".join(str(m) for m in m_k))
    elif what == "ac":
        wl = W.config(2, n=n)
        pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
        ctx = lx.Context(pb)
        u = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
        lo, hi = torch.empty_like(u), torch.empty_like(u)
        for _ in range(arg):
            c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, u))
            it, err = lx.lx_step(ctx, "exprb43", u, lo, hi, wl.dt, c, g, wl.rtol, wl.atol)
            u, hi = hi, u
            print("iters", it, "err", err)
    elif what == "step":   # one bench step after a warm-up step: phi_0..phi_3 at n^2 (config 1)
        wl = W.config(1, n=n)
        u = torch.from_numpy(W.ic_problem1_2d(n)).cuda()
        pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
        ctx = lx.Context(pb)
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        outs = [torch.empty_like(u) for _ in range(4)]
        for _ in range(reps):
            its = [lx.lx_real_leja_phi(ctx, u, outs[l], wl.dt, c, g, l, wl.rtol, wl.atol) for l in range(4)]
        print("iters", its)
    elif what == "aci":   # the same through lx_integrate (device-side spectrum)
        wl = W.config(2, n=n)
        pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
        ctx = lx.Context(pb)
        u = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
        it, err = lx.lx_integrate(ctx, "exprb43", u, wl.dt, arg, wl.rtol, wl.atol)
        print("iters", it, "err", err)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
