"""One warm Burgers (Problem III) phi_1 Leja call at 4096^2 (the sweep's row-5 call), for ncu:
`ncu -k regex:k_leja2d -s 1 -c 1 python tools/prof_burgers.py` captures the second (warm) call."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import workloads as W  # noqa: E402
import paper_2310_08344_b200 as lx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
s = torch.cuda.Stream()
pb = lx.Problem((n, n), (2.0 / n, 2.0 / n), 1.0, 0.0, 0.0, None, 10.0)
ctx = lx.Context(pb, stream=s)
u = torch.from_numpy(W.ic_burgers_2d(n)).cuda()
dt = 10.0 * W.dt_cfl(n, 20.0)
c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, u))
f = torch.empty_like(u)
lx.lx_rhs(ctx, u, f, dt)
out = torch.empty_like(u)
for _ in range(2):
    m = lx.lx_real_leja_phi(ctx, f, out, dt, c, g, 1, 1e-10, 1e-10, u_lin=u)
print("iterations", m, "points", u.numel())
ctx.close()
