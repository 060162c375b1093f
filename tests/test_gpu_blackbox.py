"""GPU parity of the black-box right-hand-side path vs the oracle.

The user supplies only f; Jacobian actions and nonlinear remainders come from
finite differences (reading R25).  Two callbacks are exercised: the library's own stencil
f (lx_builtin_rhs, native) and a torch implementation of f called through a Python trampoline.

Tolerances.  Linear black-box operator (J y = f(y)): the same 1e-10 / same-iteration bar as the
fused path.  FD mode: the two sides evaluate f with different summation orders; the difference
delta_f ~ eps_mach sum|stencil terms| is divided by the FD step eps ~ 1.5e-8 (1+|u|)/|y|, so every
Jacobian application differs by ~ eps_mach / 1.5e-8 ~ 1e-8 relative to |A| |y| -- the parity bar is
FD_TOL = 1e-8 relative L2 on Leja outputs and iteration counts equal.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2310_08344_b200 as lx  # noqa: E402

TOL = 1e-10
FD_TOL = 1e-8
# Integrator steps.  The built-in black-box f (lx_builtin_rhs) evaluates the stencil formulas literally
# with explicitly rounded operations (no FMA contraction; the order of P:549 / R10 / R24) and the FD
# perturbation w = u + eps y is unfused, so the device's f(w) and f(u) equal the oracle's bit for bit;
# the 1/eps amplification of rounding differences (~1e-8 per Jacobian application) is then gone and the
# remaining differences are ordinary fp64 rounding in the Newton updates.  The steps are held to the f-1
# bar of SURVEY 8(f), 1e-8 relative L2 (AC: 1e-9), with iteration counts equal.  A wrong tableau weight
# moves u by ~|D| ~ 1e-7 and fails it.
STEP_TOL_AC = 1e-9
STEP_TOL_BURGERS = 1e-8


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a.reshape(b.shape) - b) / (nb if nb > 0 else 1.0)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _pair(shape, diff=1.0, nu=10.0, react=0.0, flux=0.0):
    dx = tuple(2.0 / n for n in shape)
    return (lx.Problem(shape, dx, diff, nu, react, None, flux),
            O.Problem(shape, dx, diff, nu, react, None, flux))


@pytest.mark.parametrize("l", [0, 1, 3])
@pytest.mark.parametrize("mult", [1.0, 10.0, 100.0])
def test_linear_blackbox_leja(xi300, l, mult):
    # Problem I through the black-box interface (real_Leja_exp(RHS = A))
    n = 64
    pb, ob = _pair((n, n))
    dt = mult * W.dt_cfl(n, 10.0)
    u0 = W.ic_problem1_2d(n)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it = lx.lx_real_leja_phi_cb(ctx, lx.Rhs.builtin(ctx), _dev(u0), [out], [1.0], dt, c, g, l, TOL, TOL)
        fused = torch.empty_like(out)
        it_f = lx.lx_real_leja_phi(ctx, _dev(u0), fused, dt, c, g, l, TOL, TOL)
    r = O.real_leja_phi(ob, u0, dt, c, g, l, TOL, TOL, xi300, jac="linear_f")
    assert it == r.iters == it_f
    assert _rel(out, r.outs[0]) <= TOL


@pytest.mark.parametrize("coeffs", [(1.0,), (0.5, 1.0), (0.5, 2 / 3, 1.0)])
def test_fd_leja_allen_cahn(xi300, coeffs):
    n = 64
    pb, ob = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    v = 0.01 * O.rhs(ob, u)
    dt = 0.01
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    with lx.Context(pb) as ctx:
        outs = [torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in coeffs]
        it = lx.lx_real_leja_phi_cb(ctx, lx.Rhs.builtin(ctx), _dev(v), outs, coeffs, dt, c, g, 1, TOL, TOL,
                                    u=_dev(u))
    r = O.real_leja_phi(ob, v, dt, c, g, 1, TOL, TOL, xi300, u_lin=u, coeffs=coeffs, jac="fd")
    assert r.status == O.OK
    assert it == r.iters
    for k in range(len(coeffs)):
        assert _rel(outs[k], r.outs[k]) <= FD_TOL, k


def _torch_allen_cahn(n, eps2):
    h = 2.0 / n

    def f(x, out):
        lap = (torch.roll(x, 1, 0) + torch.roll(x, -1, 0) + torch.roll(x, 1, 1) + torch.roll(x, -1, 1) - 4 * x) / (h * h)
        out.copy_(eps2 * lap + x - x * x * x)
    return f


def test_fd_leja_torch_callback(xi300):
    # a genuinely black-box f: torch ops on the library's stream, called through a ctypes trampoline
    n = 48
    pb, ob = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    v = 0.01 * O.rhs(ob, u)
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    rhs = lx.Rhs.from_torch(_torch_allen_cahn(n, 1e-4), (n, n))
    with lx.Context(pb) as ctx:
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it = lx.lx_real_leja_phi_cb(ctx, rhs, _dev(v), [out], [1.0], 0.01, c, g, 1, TOL, TOL, u=_dev(u))
    r = O.real_leja_phi(ob, v, 0.01, c, g, 1, TOL, TOL, xi300, u_lin=u, jac="fd")
    assert it == r.iters
    assert _rel(out, r.outs[0]) <= FD_TOL


@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3", "exprb54s4",
                                    "epirk4s3b", "epirk4s3"])
def test_fd_steps_allen_cahn(xi300, method):
    n = 64
    pb, ob = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    dt = 0.01
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    with lx.Context(pb) as ctx:
        lo = torch.empty((n, n), dtype=torch.float64, device="cuda")
        hi = torch.empty_like(lo)
        it, err = lx.lx_step_cb(ctx, method, lx.Rhs.builtin(ctx), _dev(u), lo, hi, dt, c, g, TOL, TOL)
    r = O.step(ob, method, u, dt, c, g, TOL, TOL, xi300, jac="fd")
    assert r.status == O.OK
    assert it == r.iters
    assert _rel(hi, r.u_high) <= STEP_TOL_AC
    if method not in ("rosenbrock_euler", "exprb42"):
        assert _rel(lo, r.u_low) <= STEP_TOL_AC
        assert err == pytest.approx(r.err, rel=1e-3, abs=1e-12)


@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "epirk4s3a"])
def test_fd_steps_burgers(xi300, method):
    # Problem III as a black box
    n = 48
    pb, ob = _pair((n, n), diff=1.0, nu=0.0, flux=10.0)
    u = W.ic_burgers_2d(n)
    dt = 5 * W.dt_cfl(n, 20.0)
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    with lx.Context(pb) as ctx:
        lo = torch.empty((n, n), dtype=torch.float64, device="cuda")
        hi = torch.empty_like(lo)
        it, err = lx.lx_step_cb(ctx, method, lx.Rhs.builtin(ctx), _dev(u), lo, hi, dt, c, g, TOL, TOL)
    r = O.step(ob, method, u, dt, c, g, TOL, TOL, xi300, jac="fd")
    assert r.status == O.OK
    assert it == r.iters
    assert _rel(hi, r.u_high) <= STEP_TOL_BURGERS


def test_fd_step_matches_exact_jacobian_step(xi300):
    # black-box EXPRB43 vs the fused exact-Jacobian EXPRB43 on the device: equal to FD accuracy
    n = 64
    pb, ob = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    with lx.Context(pb) as ctx:
        lo, hi = (torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in range(2))
        lx.lx_step_cb(ctx, "exprb43", lx.Rhs.builtin(ctx), _dev(u), lo, hi, 0.01, c, g, TOL, TOL)
        lo2, hi2 = torch.empty_like(lo), torch.empty_like(lo)
        lx.lx_step(ctx, "exprb43", _dev(u), lo2, hi2, 0.01, c, g, TOL, TOL)
    assert _rel(hi, hi2.cpu().numpy()) <= 1e-9


def test_blackbox_errors():
    n = 32
    pb, _ = _pair((n, n))
    with lx.Context(pb) as ctx:
        v = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        out = torch.empty_like(v)
        # zero input converges at the first check (R3), for both modes
        assert lx.lx_real_leja_phi_cb(ctx, lx.Rhs.builtin(ctx), v, [out], [1.0], 1e-4, -1.0, 1.0, 1, TOL, TOL) == 1
        assert lx.lx_real_leja_phi_cb(ctx, lx.Rhs.builtin(ctx), v, [out], [1.0], 1e-4, -1.0, 1.0, 1, TOL, TOL,
                                      u=v + 1.0) == 1
        assert torch.all(out == 0)
        with pytest.raises(lx.LxError) as e:
            lx.lx_real_leja_phi_cb(ctx, lx.Rhs.builtin(ctx), v, [v], [1.0], 1e-4, -1.0, 1.0, 1, TOL, TOL)
        assert e.value.status == lx.LX_ERR_ALIAS
        with pytest.raises(lx.LxError) as e:
            lx.lx_step_cb(ctx, 10, lx.Rhs.builtin(ctx), v, out, out, 1e-4, -1.0, 1.0, TOL, TOL)
        assert e.value.status == lx.LX_ERR_UNKNOWN_INTEGRATOR
