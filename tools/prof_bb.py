"""Black-box RHS Leja calls: FD Jacobian of the built-in Allen-Cahn f at n0 and linear operator
(builtin stencil) at 4096^2, device-timed; prints iterations and ms per call."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import workloads as W  # noqa: E402
import paper_2310_08344_b200 as lx  # noqa: E402


def timed(stream, fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        r = fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, r


s = torch.cuda.Stream()
res = {"tag": os.environ.get("TAG", "")}
for n in (() if os.environ.get("PROF_BB_ONLY") == "linear" else (2048, 4096)):
    wl = W.config(2, n=n)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=s)
    u = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
    out = torch.empty_like(u)
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, u))
    f = torch.empty_like(u)
    lx.lx_rhs(ctx, u, f, wl.dt)
    rhs = lx.Rhs.builtin(ctx)
    ms, it = timed(s, lambda: lx.lx_real_leja_phi_cb(ctx, rhs, f, [out], [1.0], wl.dt, c, g, 1, wl.rtol, wl.atol,
                                                      u=u), 5)
    res[f"fd_{n}"] = {"iters": it, "ms": ms, "frac": u.numel() * 88 * it / ms / 1e6 / 6528.7}
    ctx.close()
wl = W.config(1, n=4096)
pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
ctx = lx.Context(pb, stream=s)
u = torch.from_numpy(W.ic_problem1_2d(4096)).cuda()
out = torch.empty_like(u)
c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
rhs = lx.Rhs.builtin(ctx)
ms, it = timed(s, lambda: lx.lx_real_leja_phi_cb(ctx, rhs, u, [out], [1.0], wl.dt, c, g, 0, wl.rtol, wl.atol), 5)
res["linear_4096"] = {"iters": it, "ms": ms, "frac": u.numel() * 56 * it / ms / 1e6 / 6528.7}
print(json.dumps(res))
