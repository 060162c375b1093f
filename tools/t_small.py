import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2310_08344_b200 as lx, workloads as W
n = int(sys.argv[1])
wl = W.config(1, n=n)
pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
ctx = lx.Context(pb)
u = torch.from_numpy(W.ic_problem1_2d(n)).cuda()
out = torch.empty_like(u)
c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
print(lx.lx_real_leja_phi(ctx, u, out, wl.dt, c, g, 0, wl.rtol, wl.atol))
