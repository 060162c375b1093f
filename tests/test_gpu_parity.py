"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): the SAME number of Leja iterations and
relative L2 error <= 1e-10 in fp64.  Inputs are seeded/synthetic (workloads/).
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2310_08344_b200 as lx  # noqa: E402

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a.reshape(b.shape) - b) / (nb if nb > 0 else 1.0)


def _pair(shape, diff=1.0, nu=10.0, react=0.0):
    dx = tuple(2.0 / n for n in shape)
    return lx.Problem(shape, dx, diff, nu, react), O.Problem(shape, dx, diff, nu, react)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ---------------------------------------------------------------- Leja calls
@pytest.mark.parametrize("l", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("mult", [1.0, 10.0, 100.0])
def test_leja_phi_64(xi300, l, mult):
    n = 64
    pb, ob = _pair((n, n))
    dt = mult * W.dt_cfl(n, 10.0)
    u0 = W.ic_problem1_2d(n)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it = lx.lx_real_leja_phi(ctx, _dev(u0), out, dt, c, g, l, TOL, TOL)
    r = O.real_leja_phi(ob, u0, dt, c, g, l, TOL, TOL, xi300)
    assert it == r.iters
    assert _rel(out, r.outs[0]) <= TOL


@pytest.mark.parametrize("shape", [(50, 70), (37, 130), (64, 128), (130, 66), (8, 4), (5, 6)])
def test_leja_ragged_shapes(xi300, shape):
    # partial column bands (n1 % 64 != 0), partial row blocks (n0 % 4 != 0), tiny grids
    pb, ob = _pair(shape, nu=4.0)
    v = W.ic_random(shape, seed=99, amp=0.2)
    dt = 5 * min(W.dt_cfl(n, 4.0) for n in shape)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        assert (c, g) == O.shift_scale(O.spectrum_bound(ob))
        for l in (0, 1, 3):
            out = torch.empty(shape, dtype=torch.float64, device="cuda")
            it = lx.lx_real_leja_phi(ctx, _dev(v), out, dt, c, g, l, TOL, TOL)
            r = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300)
            assert it == r.iters, (shape, l)
            assert _rel(out, r.outs[0]) <= TOL, (shape, l)


@pytest.mark.parametrize("coeffs", [(0.5, 1.0), (0.5, 2 / 3, 1.0), (0.25, 0.5, 0.75, 1.0)])
def test_leja_vertical(xi300, coeffs):
    n = 96
    pb, ob = _pair((n, n))
    dt = 20 * W.dt_cfl(n, 10.0)
    v = W.ic_problem1_2d(n)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        outs = [torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in coeffs]
        it = lx.lx_real_leja_phi_vertical(ctx, _dev(v), outs, coeffs, dt, c, g, 1, TOL, TOL)
    r = O.real_leja_phi(ob, v, dt, c, g, 1, TOL, TOL, xi300, coeffs=coeffs)
    assert it == r.iters
    for k in range(len(coeffs)):
        assert _rel(outs[k], r.outs[k]) <= TOL, k


def test_leja_allen_cahn_jacobian(xi300):
    n = 128
    pb, ob = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    v = W.random_vector((n, n), seed=5, scale=1e-3)
    with lx.Context(pb) as ctx:
        bound = lx.lx_spectrum_bound(ctx, _dev(u))
        assert bound == pytest.approx(O.spectrum_bound(ob, u), rel=1e-15)
        c, g = lx.lx_shift_scale(bound)
        for l in (1, 3, 4):
            out = torch.empty((n, n), dtype=torch.float64, device="cuda")
            it = lx.lx_real_leja_phi(ctx, _dev(v), out, 0.01, c, g, l, TOL, TOL, u_lin=_dev(u))
            r = O.real_leja_phi(ob, v, 0.01, c, g, l, TOL, TOL, xi300, u_lin=u)
            assert it == r.iters, l
            assert _rel(out, r.outs[0]) <= TOL, l


def test_leja_zero_input_dt_zero_and_noconv(xi300):
    n = 32
    pb, ob = _pair((n, n))
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        z = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        out = torch.full((n, n), 7.0, dtype=torch.float64, device="cuda")
        assert lx.lx_real_leja_phi(ctx, z, out, 1e-3, c, g, 1, TOL, TOL) == 1
        assert torch.all(out == 0)
        v = _dev(W.ic_problem1_2d(n))
        for l in range(5):
            assert lx.lx_real_leja_phi(ctx, v, out, 0.0, c, g, l, TOL, TOL) == 1
            assert torch.equal(out, v * (1.0 / math.factorial(l)))
    with lx.Context(pb, max_nodes=20) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        v0 = W.ic_problem1_2d(n)
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        with pytest.raises(lx.LxError) as e:
            lx.lx_real_leja_phi(ctx, _dev(v0), out, 1000 * W.dt_cfl(n, 10.0), c, g, 0, 1e-14, 0.0)
        assert e.value.status == lx.LX_ERR_NOCONV and e.value.iters == 19
        r = O.real_leja_phi(ob, v0, 1000 * W.dt_cfl(n, 10.0), c, g, 0, 1e-14, 0.0, xi300, max_nodes=20)
        assert r.status == O.ERR_NOCONV and r.iters == 19
        assert _rel(out, r.outs[0]) <= 1e-10


def test_argument_errors():
    n = 16
    pb, _ = _pair((n, n))
    with lx.Context(pb) as ctx:
        v = torch.ones((n, n), dtype=torch.float64, device="cuda")
        with pytest.raises(lx.LxError) as e:
            lx.lx_real_leja_phi(ctx, v, v, 1e-3, -1.0, 1.0, 1, TOL, TOL)
        assert e.value.status == lx.LX_ERR_ALIAS
        with pytest.raises(lx.LxError) as e:
            lx.lx_real_leja_phi(ctx, v, torch.empty_like(v), 1e-3, -1.0, 1.0, 5, TOL, TOL)
        assert e.value.status == lx.LX_ERR_UNSUPPORTED
        with pytest.raises(lx.LxError) as e:
            lx.lx_real_leja_phi(ctx, v, torch.empty_like(v), 1e-3, -1.0, -1.0, 1, TOL, TOL)
        assert e.value.status == lx.LX_ERR_ARG
        with pytest.raises(lx.LxError) as e:
            lx.lx_step(ctx, 10, v, torch.empty_like(v), torch.empty_like(v), 1e-3, -1.0, 1.0, TOL, TOL)
        assert e.value.status == lx.LX_ERR_UNKNOWN_INTEGRATOR
    with pytest.raises(lx.LxError) as e:
        lx.Context(lx.Problem((16, 15), (0.1, 0.1)))
    assert e.value.status == lx.LX_ERR_DIM


def test_host_pointer_path_equals_device_path():
    n = 64
    pb, _ = _pair((n, n))
    u0 = W.ic_problem1_2d(n)
    dt = 10 * W.dt_cfl(n, 10.0)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        out_d = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it_d = lx.lx_real_leja_phi(ctx, _dev(u0), out_d, dt, c, g, 1, TOL, TOL)
        out_h = np.zeros((n, n))
        it_h = lx.lx_real_leja_phi(ctx, u0, out_h, dt, c, g, 1, TOL, TOL)
    assert it_d == it_h
    np.testing.assert_array_equal(out_d.cpu().numpy(), out_h)


def test_async_calls_and_determinism():
    n = 128
    pb, _ = _pair((n, n))
    u0 = _dev(W.ic_problem1_2d(n))
    dt = 10 * W.dt_cfl(n, 10.0)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        outs = [torch.empty_like(u0) for _ in range(4)]
        sync_iters = [lx.lx_real_leja_phi(ctx, u0, outs[l], dt, c, g, l, TOL, TOL) for l in range(4)]
        ref = [o.clone() for o in outs]
        for l in range(4):
            lx.lx_real_leja_phi(ctx, u0, outs[l], dt, c, g, l, TOL, TOL, sync=False)
        total, _ = ctx.synchronize()
        assert total == sum(sync_iters)
        for a, b in zip(outs, ref):
            assert torch.equal(a, b)   # bitwise reproducible (fixed-order reductions)


# ---------------------------------------------------------------- spectrum / rhs
def test_power_iteration_and_rhs(xi300):
    n = 64
    pb, ob = _pair((n, n))
    with lx.Context(pb) as ctx:
        est = lx.lx_spectrum_estimate(ctx, None, 50)
        assert est == pytest.approx(O.power_iteration(ob, None, 50), rel=1e-10)
        u0 = W.ic_problem1_2d(n)
        f = torch.empty((n, n), dtype=torch.float64, device="cuda")
        lx.lx_rhs(ctx, _dev(u0), f, 0.37)
        ref = 0.37 * O.rhs(ob, u0)
        assert np.abs(f.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    pa, oa = _pair((48, 64), diff=1e-3, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(48, 64)
    with lx.Context(pa) as ctx:
        est = lx.lx_spectrum_estimate(ctx, _dev(u), 40)
        assert est == pytest.approx(O.power_iteration(oa, u, 40), rel=1e-10)


# ---------------------------------------------------------------- integrators
@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3", "exprb54s4",
                                    "epirk4s3b", "epirk4s3"])
def test_steps_linear_advdiff(xi300, method):
    n = 64
    pb, ob = _pair((n, n))
    u0 = W.ic_problem1_2d(n)
    dt = 10 * W.dt_cfl(n, 10.0)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        lo = torch.empty((n, n), dtype=torch.float64, device="cuda")
        hi = torch.empty_like(lo)
        it, err = lx.lx_step(ctx, method, _dev(u0), lo, hi, dt, c, g, TOL, TOL)
    r = O.step(ob, method, u0, dt, c, g, TOL, TOL, xi300)
    assert it == r.iters
    assert _rel(hi, r.u_high) <= TOL
    if method not in ("rosenbrock_euler", "exprb42"):
        assert err == r.err == 0.0


@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3", "exprb54s4",
                                    "epirk4s3b", "epirk4s3"])
def test_steps_allen_cahn(xi300, method):
    n = 128
    pb, ob = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    dt = 0.01
    with lx.Context(pb) as ctx:
        ud = _dev(u)
        for step in range(3):
            bound = lx.lx_spectrum_bound(ctx, ud)
            c, g = lx.lx_shift_scale(bound)
            lo = torch.empty_like(ud)
            hi = torch.empty_like(ud)
            it, err = lx.lx_step(ctx, method, ud, lo, hi, dt, c, g, TOL, TOL)
            r = O.step(ob, method, u, dt, c, g, TOL, TOL, xi300)
            assert it == r.iters, (method, step)
            assert _rel(hi, r.u_high) <= TOL, (method, step)
            if method not in ("rosenbrock_euler", "exprb42"):
                assert _rel(lo, r.u_low) <= TOL
                assert err == pytest.approx(r.err, rel=1e-8)
            # continue from the oracle state so both sides see identical inputs
            u = r.u_high
            ud = _dev(u)


# ---------------------------------------------------------------- full size (BASELINE configs)
def test_config0_rosenbrock_euler_64(xi300):
    wl = W.config(0)
    pb, ob = _pair(wl.shape)
    u0 = W.ic_problem1_2d(64)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        out = np.zeros(wl.shape)
        it = lx.lx_step_rosenbrock_euler(ctx, u0, out, wl.dt, c, g, wl.rtol, wl.atol)   # host buffers
    r = O.step(ob, "rosenbrock_euler", u0, wl.dt, c, g, wl.rtol, wl.atol, xi300)
    assert it == r.iters == 23
    assert _rel(out, r.u_high) <= TOL


@pytest.mark.slow
def test_config1_4096_phi0_full_oracle(xi300):
    # BASELINE config 1 at full size, launch configuration of bench.py: phi_0 vs the full oracle.
    wl = W.config(1)
    n = wl.shape[0]
    pb, ob = _pair(wl.shape)
    u0 = W.ic_problem1_2d(n)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        out = torch.empty(wl.shape, dtype=torch.float64, device="cuda")
        it = lx.lx_real_leja_phi(ctx, _dev(u0), out, wl.dt, c, g, 0, wl.rtol, wl.atol)
        got = out.cpu().numpy()
    r = O.real_leja_phi(ob, u0, wl.dt, c, g, 0, wl.rtol, wl.atol, xi300)
    assert it == r.iters
    assert _rel(got, r.outs[0]) <= TOL


# ---------------------------------------------------------------- 3D (config 5 shape family)
@pytest.mark.parametrize("shape", [(16, 24, 32), (20, 12, 66), (9, 10, 130), (32, 32, 64)])
def test_leja_3d(xi300, shape):
    pb, ob = _pair(shape)
    v = W.ic_random(shape, seed=7, amp=0.2)
    dt = 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    with lx.Context(pb) as ctx:
        bound = lx.lx_spectrum_bound(ctx)
        assert bound == O.spectrum_bound(ob)
        c, g = lx.lx_shift_scale(bound)
        for l in (0, 1, 4):
            out = torch.empty(shape, dtype=torch.float64, device="cuda")
            it = lx.lx_real_leja_phi(ctx, _dev(v), out, dt, c, g, l, TOL, TOL)
            r = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300)
            assert it == r.iters, (shape, l)
            assert _rel(out, r.outs[0]) <= TOL, (shape, l)
        f = torch.empty(shape, dtype=torch.float64, device="cuda")
        lx.lx_rhs(ctx, _dev(v), f, 0.5)
        ref = 0.5 * O.rhs(ob, v)
        assert np.abs(f.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
        est = lx.lx_spectrum_estimate(ctx, None, 20)
        assert est == pytest.approx(O.power_iteration(ob, None, 20), rel=1e-10)


@pytest.mark.parametrize("method", ["epirk4s3a", "exprb43", "epirk4s3b", "epirk4s3"])
def test_steps_3d(xi300, method):
    n = 32
    shape = (n, n, n)
    pb, ob = _pair(shape)
    c1 = W.coords(n)
    x, y, z = np.meshgrid(c1, c1, c1, indexing="ij")
    u0 = np.ascontiguousarray(1.0 + np.exp(-((x + .5) ** 2 + (y + .5) ** 2 + (z + .5) ** 2) / 0.05))
    dt = 10 * W.dt_cfl(n, 10.0, 3)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        lo = torch.empty(shape, dtype=torch.float64, device="cuda")
        hi = torch.empty_like(lo)
        it, err = lx.lx_step(ctx, method, _dev(u0), lo, hi, dt, c, g, TOL, TOL)
    r = O.step(ob, method, u0, dt, c, g, TOL, TOL, xi300)
    assert it == r.iters
    assert _rel(hi, r.u_high) <= TOL and _rel(lo, r.u_low) <= TOL
    pa, oa = _pair((16, 16, 32), diff=1e-3, nu=0.0, react=1.0)
    ua = W.ic_random((16, 16, 32), seed=3, amp=0.9) - 1.0
    with lx.Context(pa) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, _dev(ua)))
        lo = torch.empty((16, 16, 32), dtype=torch.float64, device="cuda")
        hi = torch.empty_like(lo)
        it, err = lx.lx_step(ctx, method, _dev(ua), lo, hi, 0.05, c, g, TOL, TOL)
    r = O.step(oa, method, ua, 0.05, c, g, TOL, TOL, xi300)
    assert it == r.iters
    assert _rel(hi, r.u_high) <= TOL and _rel(lo, r.u_low) <= TOL
    assert err == pytest.approx(r.err, rel=1e-8)


@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3", "exprb54s4",
                                    "epirk4s3b", "epirk4s3"])
def test_integrate_device_spectrum(xi300, method):
    # lx_integrate: the paper's time loop with (c, gamma) recomputed ON THE DEVICE every
    # step; the oracle recomputes them from its own state with the same formula (R16).
    n = 96
    pb, ob = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    dt, nsteps = 0.01, 4
    ud = _dev(u)
    with lx.Context(pb) as ctx:
        it, err = lx.lx_integrate(ctx, method, ud, dt, nsteps, TOL, TOL)
    tot = 0
    for _ in range(nsteps):
        c, g = O.shift_scale(O.spectrum_bound(ob, u))
        r = O.step(ob, method, u, dt, c, g, TOL, TOL, xi300)
        tot += r.iters
        u = r.u_high
    assert it == tot
    assert _rel(ud, u) <= TOL
    if method not in ("rosenbrock_euler", "exprb42"):
        assert err == pytest.approx(r.err, rel=1e-8)


@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb43"])
def test_problem2_source(xi300, method):
    # Problem II: f(u) = A u + S, time-independent source
    n = 128
    S = W.source_problem2_2d(n)
    dx = (2 / n, 2 / n)
    ob = O.Problem((n, n), dx, 1.0, 10.0, 0.0, S)
    u0 = W.ic_problem1_2d(n)
    dt = 10 * W.dt_cfl(n, 10.0)
    for src in (_dev(S), S):   # device and host source pointers
        pb = lx.Problem((n, n), dx, 1.0, 10.0, 0.0, src)
        with lx.Context(pb) as ctx:
            c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
            lo = torch.empty((n, n), dtype=torch.float64, device="cuda")
            hi = torch.empty_like(lo)
            it, err = lx.lx_step(ctx, method, _dev(u0), lo, hi, dt, c, g, TOL, TOL)
            r = O.step(ob, method, u0, dt, c, g, TOL, TOL, xi300)
            assert it == r.iters
            assert _rel(hi, r.u_high) <= TOL
            ud = _dev(u0)
            it2, _ = lx.lx_integrate(ctx, method, ud, dt, 2, TOL, TOL)
            u = u0
            tot = 0
            for _ in range(2):
                r = O.step(ob, method, u, dt, c, g, TOL, TOL, xi300)
                tot += r.iters
                u = r.u_high
            assert it2 == tot and _rel(ud, u) <= TOL


# ---------------------------------------------------------------- Problem III: viscous Burgers
def _burgers_pair(n, beta=10.0):
    dx = (2 / n, 2 / n)
    return lx.Problem((n, n), dx, 1.0, 0.0, 0.0, None, beta), O.Problem((n, n), dx, 1.0, 0.0, 0.0, None, beta)


@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3", "exprb54s4",
                                    "epirk4s3b", "epirk4s3"])
def test_burgers_steps(xi300, method):
    n = 128
    pb, ob = _burgers_pair(n)
    u = W.ic_burgers_2d(n)
    dt = 10 * W.dt_cfl(n, 20.0)
    with lx.Context(pb) as ctx:
        ud = _dev(u)
        bound = lx.lx_spectrum_bound(ctx, ud)
        assert bound == pytest.approx(O.spectrum_bound(ob, u), rel=1e-14)
        c, g = O.shift_scale(O.spectrum_bound(ob, u))
        lo = torch.empty_like(ud)
        hi = torch.empty_like(ud)
        it, err = lx.lx_step(ctx, method, ud, lo, hi, dt, c, g, TOL, TOL)
        r = O.step(ob, method, u, dt, c, g, TOL, TOL, xi300)
        assert it == r.iters
        assert _rel(hi, r.u_high) <= TOL
        if method not in ("rosenbrock_euler", "exprb42"):
            assert _rel(lo, r.u_low) <= TOL
            assert err == pytest.approx(r.err, rel=1e-8)


def test_burgers_leja_power_rhs_integrate(xi300):
    n = 96
    pb, ob = _burgers_pair(n)
    u = W.ic_burgers_2d(n)
    v = W.random_vector((n, n), seed=8, scale=0.01)
    dt = 10 * W.dt_cfl(n, 20.0)
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    with lx.Context(pb) as ctx:
        ud = _dev(u)
        outs = [torch.empty_like(ud) for _ in range(2)]
        it = lx.lx_real_leja_phi_vertical(ctx, _dev(v), outs, (0.5, 1.0), dt, c, g, 1, TOL, TOL, u_lin=ud)
        r = O.real_leja_phi(ob, v, dt, c, g, 1, TOL, TOL, xi300, u_lin=u, coeffs=(0.5, 1.0))
        assert it == r.iters
        for k in range(2):
            assert _rel(outs[k], r.outs[k]) <= TOL
        f = torch.empty_like(ud)
        lx.lx_rhs(ctx, ud, f, 0.25)
        ref = 0.25 * O.rhs(ob, u)
        assert np.abs(f.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
        est = lx.lx_spectrum_estimate(ctx, ud, 30)
        assert est == pytest.approx(O.power_iteration(ob, u, 30), rel=1e-10)
        it2, err2 = lx.lx_integrate(ctx, "exprb32", ud, dt, 3, TOL, TOL)
    tot = 0
    for _ in range(3):
        cc, gg = O.shift_scale(O.spectrum_bound(ob, u))
        rr = O.step(ob, "exprb32", u, dt, cc, gg, TOL, TOL, xi300)
        tot += rr.iters
        u = rr.u_high
    assert it2 == tot and _rel(ud, u) <= TOL


@pytest.mark.parametrize("shape", [(67, 90), (33, 130), (5, 64), (7, 62)])
def test_burgers_ragged(xi300, shape):
    # flux-form tile on ragged shapes: 2-row units with an odd row count (a last unit of one row),
    # n1 not a multiple of the 64-column band, the smallest allowed grids; vertical K = 3, f, the spectrum
    # estimate and a two-stage step (its remainders) against the oracle
    n0, n1 = shape
    dx = (2 / n0, 2 / n1)
    pb, ob = lx.Problem(shape, dx, 1.0, 0.0, 0.0, None, 10.0), O.Problem(shape, dx, 1.0, 0.0, 0.0, None, 10.0)
    u = W.ic_burgers_2d(n0, n1)
    v = W.random_vector(shape, seed=31, scale=0.01)
    dt = 10 * W.dt_cfl(max(shape), 20.0)
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    with lx.Context(pb) as ctx:
        ud = _dev(u)
        outs = [torch.empty_like(ud) for _ in range(3)]
        it = lx.lx_real_leja_phi_vertical(ctx, _dev(v), outs, (0.25, 0.5, 1.0), dt, c, g, 1, TOL, TOL, u_lin=ud)
        r = O.real_leja_phi(ob, v, dt, c, g, 1, TOL, TOL, xi300, u_lin=u, coeffs=(0.25, 0.5, 1.0))
        assert it == r.iters
        for k in range(3):
            assert _rel(outs[k], r.outs[k]) <= TOL
        f = torch.empty_like(ud)
        lx.lx_rhs(ctx, ud, f, 0.25)
        ref = 0.25 * O.rhs(ob, u)
        assert np.abs(f.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
        est = lx.lx_spectrum_estimate(ctx, ud, 20)
        assert est == pytest.approx(O.power_iteration(ob, u, 20), rel=1e-10)
        lo = torch.empty_like(ud)
        hi = torch.empty_like(ud)
        its, err = lx.lx_step(ctx, "epirk4s3a", ud, lo, hi, dt, c, g, TOL, TOL)
        rs = O.step(ob, "epirk4s3a", u, dt, c, g, TOL, TOL, xi300)
        assert its == rs.iters
        assert _rel(hi, rs.u_high) <= TOL and _rel(lo, rs.u_low) <= TOL


@pytest.mark.parametrize("shape,K,react,l", [((64, 64), 1, 0.0, 0), ((66, 62), 2, 0.0, 1), ((7, 24), 1, 0.0, 2),
                                             ((130, 122), 3, 1.0, 1), ((131, 182), 4, 0.0, 1),
                                             ((200, 60), 4, 1.0, 3), ((4096, 256), 1, 1.0, 0)])
def test_tblock2_matches_oracle_and_one_step(xi300, shape, K, react, l):
    # two Leja iterations per HBM pass: ragged 60-column bands (n1 = 62, 122,
    # 182, 24 < 64), odd row counts, K = 1..4 (accumulators converging at different m, i.e. on
    # either half of a pass -> rollback), with and without the diagonal term.  Same iteration
    # counts as the oracle and as the one-step kernel; y_m, p_m are bitwise those of the one-step
    # kernel except after a rollback p_m = p_{m+1} - d_{m+1} y_{m+1} (a few ulp).
    diff, nu = (1e-4, 0.0) if react else (1.0, 10.0)
    pb, ob = _pair(shape, diff=diff, nu=nu, react=react)
    u = W.ic_allen_cahn_2d(*shape) if react else None
    v = W.ic_random(shape, seed=23, amp=0.2)
    dt = 0.01 if react else 10 * min(W.dt_cfl(n, 10.0) for n in shape)
    coeffs = (0.25, 0.5, 0.75, 1.0)[-K:]
    res = {}
    for tb in (1, 2):   # one iteration per pass (k_leja2d); two (k_leja2d_tb2; needs >= 16 rows, >= 64 columns)
        with lx.Context(pb) as ctx:
            ctx.set_kernel(tb)
            assert ctx.iterations_per_pass == (tb if shape[0] >= 16 and shape[1] >= 64 else 1)
            ud = _dev(u) if react else None
            c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, ud))
            outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in range(K)]
            it = lx.lx_real_leja_phi_vertical(ctx, _dev(v), outs, coeffs, dt, c, g, l, TOL, TOL, u_lin=ud)
            res[tb] = (it, [o.cpu().numpy() for o in outs])
    r = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300, coeffs=coeffs, u_lin=u)
    assert res[2][0] == res[1][0] == r.iters
    for a, b, ref in zip(res[2][1], res[1][1], r.outs):
        assert np.isfinite(a).all()
        np.testing.assert_allclose(a, b, rtol=0, atol=8 * np.finfo(float).eps * np.abs(b).max())
        assert np.linalg.norm(a - ref) <= TOL * np.linalg.norm(ref)


def test_tblock2_dynamic_segments_reproducible(xi300):
    # dynamic work assignment (atomic segment counter) must not leak into the results: per-segment
    # norm partials are reduced in segment order -> identical iterations and bitwise-equal outputs
    # over repeated calls, at a size with thousands of segments (n = 1536: 26 bands x 384 chunks)
    n = 1536
    pb, _ = _pair((n, n))
    u0 = _dev(W.ic_random((n, n), seed=5, amp=0.3))
    dt = 10 * W.dt_cfl(n, 10.0)
    with lx.Context(pb) as ctx:
        ctx.set_kernel(2)   # below the auto threshold: force the two-step kernel
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        runs = []
        for _ in range(4):
            outs = [torch.empty_like(u0) for _ in range(2)]
            it = lx.lx_real_leja_phi_vertical(ctx, u0, outs, (0.5, 1.0), dt, c, g, 1, TOL, TOL)
            runs.append((it, outs))
    for it, outs in runs[1:]:
        assert it == runs[0][0]
        for a, b in zip(outs, runs[0][1]):
            assert torch.equal(a, b)


def test_tblock_auto_policy():
    # two-step kernel from 3*2^20 local points on (2D single GPU), one-pass below; lx_ctx_set_kernel forces
    for shape, want in (((1536, 1536), 1), ((2048, 2048), 2), ((64, 64), 1)):
        pb, _ = _pair(shape)
        with lx.Context(pb) as ctx:
            assert ctx.iterations_per_pass == want, shape
    with lx.Context(_pair((64, 64))[0]) as ctx:
        ctx.set_kernel(2)
        assert ctx.iterations_per_pass == 2
        with pytest.raises(lx.LxError):
            ctx.set_kernel(3)
    with lx.Context(_pair((8, 8, 64))[0]) as ctx:
        ctx.set_kernel(2)
        assert ctx.iterations_per_pass == 1        # 3D: one pass per iteration


@pytest.mark.parametrize("shape,K,react", [((20, 32, 64), 1, 0.0), ((70, 16, 128), 2, 1.0), ((130, 48, 64), 3, 0.0)])
def test_3d_smem_kernel_bitwise_equals_tiles(xi300, shape, K, react):
    # the shared-memory marching 3D kernel (plane runs of 64, ragged last run) evaluates every point with the
    # warp-tile kernel's operation order: identical iterations and bitwise-equal outputs; oracle parity
    diff, nu = (1e-3, 0.0) if react else (1.0, 10.0)
    pb, ob = _pair(shape, diff=diff, nu=nu, react=react)
    u = W.ic_random(shape, seed=31, amp=0.5) if react else None
    v = W.ic_random(shape, seed=32, amp=0.2)
    dt = 0.01 if react else 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    coeffs = (0.5, 2 / 3, 1.0)[-K:]
    res = {}
    for kern in ("tile", "smem"):
        with lx.Context(pb) as ctx:
            ctx.set_kernel(0, 1 if kern == "tile" else 0)
            ud = _dev(u) if react else None
            c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, ud))
            outs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(K)]
            it = lx.lx_real_leja_phi_vertical(ctx, _dev(v), outs, coeffs, dt, c, g, 1, TOL, TOL, u_lin=ud)
            res[kern] = (it, [o.cpu().numpy() for o in outs])
    r = O.real_leja_phi(ob, v, dt, c, g, 1, TOL, TOL, xi300, coeffs=coeffs, u_lin=u)
    assert res["smem"][0] == res["tile"][0] == r.iters
    for a, b, ref in zip(res["smem"][1], res["tile"][1], r.outs):
        np.testing.assert_array_equal(a, b)
        assert np.linalg.norm(a - ref) <= TOL * np.linalg.norm(ref)


@pytest.mark.parametrize("shape,K,l", [((20, 32, 64), 1, 0), ((70, 16, 128), 2, 1), ((130, 48, 64), 3, 1),
                                       ((7, 16, 64), 4, 2), ((4, 32, 192), 1, 3), ((66, 16, 64), 3, 4)])
def test_3d_tblock2_vs_one_pass(xi300, shape, K, l):
    # 3D two-step kernel (2.5D temporal blocking: two Leja iterations per plane sweep; plane runs of 64 with
    # a ragged last run, runs shorter than the 6-plane halo, accumulators converging on either half of a
    # pass -> rollback) against the one-pass shared-memory kernel and the oracle: same iteration counts;
    # y and p bitwise those of the one-pass kernel except after a rollback (a few ulp)
    pb, ob = _pair(shape)
    v = W.ic_random(shape, seed=41 + K, amp=0.2)
    dt = 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    coeffs = (0.25, 0.5, 2 / 3, 1.0)[-K:]
    res = {}
    for tb in (1, 2):
        with lx.Context(pb) as ctx:
            ctx.set_kernel(tb)
            assert ctx.iterations_per_pass == tb
            c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
            outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in range(K)]
            it = lx.lx_real_leja_phi_vertical(ctx, _dev(v), outs, coeffs, dt, c, g, l, TOL, TOL)
            res[tb] = (it, [o.cpu().numpy() for o in outs])
    r = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300, coeffs=coeffs)
    assert res[2][0] == res[1][0] == r.iters
    for a, b, ref in zip(res[2][1], res[1][1], r.outs):
        assert np.isfinite(a).all()
        np.testing.assert_allclose(a, b, rtol=0, atol=8 * np.finfo(float).eps * np.abs(b).max())
        assert np.linalg.norm(a - ref) <= TOL * np.linalg.norm(ref)


@pytest.mark.parametrize("K", [1, 2])
def test_3d_tblock2_predicted_final_iteration(xi300, K):
    # repeated calls with the same parameters: the 3D two-step kernel predicts the final iteration from the
    # previous call (Tb2Ctl table) and, when it is the FIRST iteration of a pass, performs that iteration
    # alone (no rollback).  Sequence: zero input twice (m = 1: rollback, then predicted), a nonzero input
    # with the stale prediction m = 1 (wrong: the call continues at m = 2 in the next pass), the same input
    # again (right prediction).  Every call against the oracle (iterations, 1e-10) and the one-pass kernel.
    shape = (40, 16, 64)
    pb, ob = _pair(shape)
    v = W.ic_random(shape, seed=77, amp=0.2)
    dt = 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    coeffs = (0.5, 1.0)[-K:]
    zero = np.zeros(shape)
    seq = [zero, zero, v, v, zero, v]
    res = {}
    for tb in (1, 2):
        with lx.Context(pb) as ctx:
            ctx.set_kernel(tb)
            c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
            res[tb] = []
            for x in seq:
                outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in range(K)]
                it = lx.lx_real_leja_phi_vertical(ctx, _dev(x), outs, coeffs, dt, c, g, 1, TOL, TOL)
                res[tb].append((it, [o.cpu().numpy() for o in outs]))
    refs = {id(x): O.real_leja_phi(ob, x, dt, c, g, 1, TOL, TOL, xi300, coeffs=coeffs) for x in (zero, v)}
    assert refs[id(zero)].iters == 1
    for x, (it2, o2), (it1, o1) in zip(seq, res[2], res[1]):
        r = refs[id(x)]
        assert it2 == it1 == r.iters
        for a, b, ref in zip(o2, o1, r.outs):
            if x is zero:
                assert not a.any() and not ref.any()
                continue
            np.testing.assert_allclose(a, b, rtol=0, atol=8 * np.finfo(float).eps * np.abs(b).max())
            assert np.linalg.norm(a - ref) <= TOL * np.linalg.norm(ref)


def test_3d_tblock2_auto_and_limits(xi300):
    # auto policy: two-step from 2^20 points on (n1 % 16 == 0, n2 % 64 == 0), one pass below / for other
    # shapes; the NOCONV limit (R28) and a NONFINITE run end with the same status and m as the oracle
    for shape, want in (((64, 64, 256), 2), ((32, 64, 256), 1), ((64, 72, 256), 1), ((256, 64, 96), 1)):
        with lx.Context(_pair(shape)[0]) as ctx:
            assert ctx.iterations_per_pass == want, shape
    n = 16
    shape = (n, n, 4 * n)
    pb, ob = _pair(shape)
    v = W.ic_random(shape, seed=4, amp=0.5)
    c, g = O.shift_scale(O.spectrum_bound(ob))
    for dt, fac, status in ((20.0 * W.dt_cfl(n, 10.0, 3), 1.0, lx.LX_ERR_NOCONV),   # m = 299: first half, cap
                            (W.dt_cfl(n, 10.0, 3), 1e-4, lx.LX_ERR_NONFINITE)):
        r = O.real_leja_phi(ob, v, dt, c * fac, g * fac, 0, TOL, TOL, xi300)
        assert r.status == {lx.LX_ERR_NOCONV: O.ERR_NOCONV, lx.LX_ERR_NONFINITE: O.ERR_NONFINITE}[status]
        with lx.Context(pb) as ctx:
            ctx.set_kernel(2)
            out = torch.empty(shape, dtype=torch.float64, device="cuda")
            it = _expect_status(lambda: lx.lx_real_leja_phi(ctx, _dev(v), out, dt, c * fac, g * fac, 0, TOL, TOL),
                                status)
        assert it == r.iters


# ---------------------------------------------------------------- non-finite and divergent runs
def _expect_status(fn, status):
    with pytest.raises(lx.LxError) as e:
        fn()
    assert e.value.status == status, e.value
    return e.value.iters


def test_nonfinite_nan_input_and_inf_state(xi300):
    # both sides: LX_ERR_NONFINITE at the iteration whose check saw the non-finite norm (m = 1)
    n = 32
    pb, ob = _pair((n, n))
    v = W.ic_problem1_2d(n)
    v[3, 5] = np.nan
    dt = W.dt_cfl(n, 10.0)
    r = O.real_leja_phi(ob, v, dt, *O.shift_scale(O.spectrum_bound(ob)), 0, TOL, TOL, xi300)
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it = _expect_status(lambda: lx.lx_real_leja_phi(ctx, _dev(v), out, dt, c, g, 0, TOL, TOL),
                            lx.LX_ERR_NONFINITE)
    assert (r.status, r.iters) == (O.ERR_NONFINITE, it) == (O.ERR_NONFINITE, 1)
    pa, oa = _pair((n, n), diff=1e-4, nu=0.0, react=1.0)
    u = W.ic_allen_cahn_2d(n)
    c, g = O.shift_scale(O.spectrum_bound(oa, u))
    u[7, 9] = np.inf
    w = 0.01 * W.ic_problem1_2d(n)
    r = O.real_leja_phi(oa, w, 0.01, c, g, 1, TOL, TOL, xi300, u_lin=u)
    with lx.Context(pa) as ctx:
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it = _expect_status(lambda: lx.lx_real_leja_phi(ctx, _dev(w), out, 0.01, c, g, 1, TOL, TOL, u_lin=_dev(u)),
                            lx.LX_ERR_NONFINITE)
    assert (r.status, r.iters) == (O.ERR_NONFINITE, it) == (O.ERR_NONFINITE, 1)


@pytest.mark.parametrize("n,fac", [(32, 1e-2), (32, 1e-6), (2048, 1e-4)])
def test_nonfinite_unenclosed_spectrum(xi300, n, fac):
    # gamma too small: the Newton basis overflows; both sides stop with NONFINITE at the same m
    # (2048^2, broadband input: the two-iterations-per-pass kernel, NONFINITE at m = 34, the second
    # iteration of a pass)
    pb, ob = _pair((n, n))
    u0 = W.ic_problem1_2d(n) if n < 2048 else W.ic_random((n, n), seed=7, amp=0.2)
    c, g = O.shift_scale(O.spectrum_bound(ob))
    dt = W.dt_cfl(n, 10.0)
    r = O.real_leja_phi(ob, u0, dt, c * fac, g * fac, 0, TOL, TOL, xi300)
    assert r.status == O.ERR_NONFINITE
    with lx.Context(pb) as ctx:
        assert ctx.iterations_per_pass == (2 if n >= 2048 else 1)
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it = _expect_status(lambda: lx.lx_real_leja_phi(ctx, _dev(u0), out, dt, c * fac, g * fac, 0, TOL, TOL),
                            lx.LX_ERR_NONFINITE)
    assert it == r.iters


def test_3d_real_leja_limit_noconv(xi300):
    # 16^3 at 10 x CFL: fp64 divided differences + complex eigenvalues -> NOCONV at the node cap on
    # both sides (reading R28; the oracle side is pinned in test_oracle_leja.py).  The diverged
    # polynomials are amplified rounding noise and are not compared.
    n = 16
    shape = (n, n, n)
    pb, ob = _pair(shape)
    v = W.ic_random(shape, seed=4, amp=0.5)
    dt = 10.0 * W.dt_cfl(n, 10.0, 3)
    c, g = O.shift_scale(O.spectrum_bound(ob))
    r = O.real_leja_phi(ob, v, dt, c, g, 0, TOL, TOL, xi300)
    with lx.Context(pb) as ctx:
        out = torch.empty(shape, dtype=torch.float64, device="cuda")
        it = _expect_status(lambda: lx.lx_real_leja_phi(ctx, _dev(v), out, dt, c, g, 0, TOL, TOL), lx.LX_ERR_NOCONV)
    assert (r.status, r.iters) == (O.ERR_NOCONV, it) == (O.ERR_NOCONV, 299)


def test_pinned_host_pipelined_leja_calls(xi300):
    # lexint.h: Leja calls on PINNED host buffers are pipelined (copy-in / kernel / copy-out streams); async
    # calls reuse a staged input until lx_ctx_synchronize; outputs equal the device-pointer results bitwise
    n = 256
    pb, ob = _pair((n, n))
    dt = 10 * W.dt_cfl(n, 10.0)
    v = torch.from_numpy(W.ic_random((n, n), seed=61, amp=0.3)).pin_memory()
    outs = [torch.full((n, n), float("nan"), dtype=torch.float64).pin_memory() for _ in range(4)]
    with lx.Context(pb) as ctx:
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        ref = []
        for l in range(4):
            o = torch.empty((n, n), dtype=torch.float64, device="cuda")
            ref.append((lx.lx_real_leja_phi(ctx, v.cuda(), o, dt, c, g, l, TOL, TOL), o.cpu()))
        for rnd in range(2):
            for l in range(4):
                lx.lx_real_leja_phi(ctx, v, outs[l], dt, c, g, l, TOL, TOL, sync=False)
            its, _ = ctx.synchronize()
            assert its == sum(r[0] for r in ref)
            for l in range(4):
                assert torch.equal(outs[l], ref[l][1]), (rnd, l)
        v.mul_(0.5)                       # after the synchronize the caller may change v: no stale copy
        it = lx.lx_real_leja_phi(ctx, v, outs[0], dt, c, g, 0, TOL, TOL)
        o = torch.empty((n, n), dtype=torch.float64, device="cuda")
        it2 = lx.lx_real_leja_phi(ctx, v.cuda(), o, dt, c, g, 0, TOL, TOL)
        assert it == it2 and torch.equal(outs[0], o.cpu())
    r = O.real_leja_phi(ob, v.numpy(), dt, c, g, 0, TOL, TOL, xi300)
    assert r.iters == it and _rel(outs[0], r.outs[0]) <= TOL


@pytest.mark.parametrize("method", ["exprb32", "exprb43", "epirk4s3a", "exprb53s3", "exprb54s4", "epirk5p1",
                                    "epirk4s3b", "epirk4s3"])
def test_adaptive_step_size_control(xi300, method):
    # lx_integrate_adaptive vs the oracle's controller (reading R32): the same accept / reject sequence, the
    # same step sizes (they depend on err^(1/(q+1)); err agrees to rounding), the same final state
    n = 32
    pb, ob = _pair((n, n), diff=2e-3, nu=0.0, react=1.0)
    u0 = W.ic_allen_cahn_2d(n)
    t_end, dt0, tol = 0.5, 0.5, 1e-7
    ref = O.integrate_adaptive(ob, method, u0, t_end, dt0, tol, 1e-12, 1e-12, xi300)
    assert ref.status == O.OK and ref.rejected >= 1
    with lx.Context(pb) as ctx:
        u = _dev(u0)
        acc, rej, dts, errs, its = lx.lx_integrate_adaptive(ctx, method, u, t_end, dt0, tol, 1e-12, 1e-12)
    assert (acc, rej) == (ref.accepted, ref.rejected)
    # EPIRK4s3's embedded error is phi_4 of 27648 D_a - 34992 D_b (R35): the cancellation turns rounding-level
    # differences of D into ~1e-7 relative differences of err (~2e-8 of the step sizes, err^(1/4))
    big = method == "epirk4s3"
    np.testing.assert_allclose(dts, ref.dts, rtol=1e-7 if big else 1e-8)
    fin = np.isfinite(ref.errs)
    assert np.array_equal(np.isfinite(errs), fin)
    np.testing.assert_allclose(errs[fin], ref.errs[fin], rtol=1e-5 if big else 1e-6, atol=1e-15)
    assert its == ref.iters
    assert _rel(u, ref.u) <= 1e-9


@pytest.mark.parametrize("shape,kern,ls,coeffs", [((96, 130), 1, (0, 1, 2, 3), (1.0,) * 4),
                                                  ((96, 130), 2, (0, 1, 2, 3), (1.0,) * 4),
                                                  ((128, 128), 2, (2, 2, 1), (0.5, 0.75, 1.0)),
                                                  ((40, 16, 64), 2, (0, 1, 3), (1.0,) * 3),
                                                  ((24, 16, 64), 1, (2, 2, 1), (0.5, 0.75, 1.0))])
def test_multi_phi_shared_basis(xi300, shape, kern, ls, coeffs):
    # lx_real_leja_phi_multi: several phi_l of one vector on one Newton basis (the basis does not depend on l):
    # every output equals its own call (a few ulp: a single-accumulator call may end on a predicted
    # one-iteration pass where the shared call rolls back) and the oracle (1e-10), and the shared call runs
    # until the slowest accumulator converged
    pb, ob = _pair(shape)
    v = W.ic_random(shape, seed=8, amp=0.2)
    dt = (10 if len(shape) == 2 else 5) * min(W.dt_cfl(n, 10.0, len(shape)) for n in shape)
    with lx.Context(pb) as ctx:
        ctx.set_kernel(kern)
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in ls]
        it = lx.lx_real_leja_phi_multi(ctx, _dev(v), outs, ls, coeffs, dt, c, g, TOL, TOL)
        its = []
        for k, (l, a) in enumerate(zip(ls, coeffs)):
            o = torch.empty(shape, dtype=torch.float64, device="cuda")
            its.append(lx.lx_real_leja_phi(ctx, _dev(v), o, a * dt, c, g, l, TOL, TOL))
            np.testing.assert_allclose(outs[k].cpu().numpy(), o.cpu().numpy(), rtol=0,
                                       atol=8 * np.finfo(float).eps * float(o.abs().max()))
            r = O.real_leja_phi(ob, v, a * dt, c, g, l, TOL, TOL, xi300)
            assert its[-1] == r.iters
            assert _rel(outs[k], r.outs[0]) <= TOL
        assert it == max(its)
        with pytest.raises(lx.LxError) as e:
            lx.lx_real_leja_phi_multi(ctx, _dev(v), outs[:2], (1, 1), (1.0, 1.0), dt, c, g, TOL, TOL)
        assert e.value.status == lx.LX_ERR_ARG
        with pytest.raises(lx.LxError) as e:
            lx.lx_real_leja_phi_multi(ctx, _dev(v), outs[:1], (5,), (1.0,), dt, c, g, TOL, TOL)
        assert e.value.status == lx.LX_ERR_UNSUPPORTED


def _fuzz_cases(n, seed):
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        nd = int(rng.integers(2, 4))
        if nd == 2:
            shape = (int(rng.integers(16, 200)), 2 * int(rng.integers(32, 100)))
        else:
            shape = (int(rng.integers(4, 40)), 16 * int(rng.integers(1, 4)), 64 * int(rng.integers(1, 3)))
        K = int(rng.integers(1, 5))
        coeffs = tuple(sorted(rng.choice(np.array([0.125, 0.25, 1 / 3, 0.5, 2 / 3, 0.75, 0.9, 1.0]), K,
                                         replace=False)))
        # 3D at <= 5 x CFL: coarse 3D grids at 10 x CFL reach the real-Leja limit of R28 (NOCONV on both sides)
        cases.append((shape, K, coeffs, int(rng.integers(0, 5)), float(rng.choice([1.0, 5.0, 10.0] if nd == 2 else [1.0, 5.0])),
                      int(rng.integers(0, 3)), int(rng.integers(0, 1 << 30))))
    return cases


@pytest.mark.parametrize("case", _fuzz_cases(40, 2026))
def test_leja_fuzz(xi300, case):
    # seeded random shapes (2D ragged rows / even columns, 3D on and off the two-step kernel's shape), K = 1..4
    # vertical coefficients, phi_0..phi_4, dt = 1 / 5 / 10 x CFL and kernel choice (auto, one pass, two
    # steps): same iteration count as the oracle and 1e-10
    shape, K, coeffs, l, mult, kern, seed = case
    pb, ob = _pair(shape)
    v = W.ic_random(shape, seed=seed % 100000, amp=0.3)
    dt = mult * min(W.dt_cfl(n, 10.0, len(shape)) for n in shape)
    with lx.Context(pb) as ctx:
        ctx.set_kernel(kern)
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in range(K)]
        it = lx.lx_real_leja_phi_vertical(ctx, _dev(v), outs, coeffs, dt, c, g, l, TOL, TOL)
    r = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300, coeffs=coeffs)
    assert it == r.iters, (case, it, r.iters)
    for o, ref in zip(outs, r.outs):
        assert _rel(o, ref) <= TOL, case


_METHODS = ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3", "exprb54s4",
            "epirk4s3b", "epirk4s3"]


@pytest.mark.parametrize("case", [(m, s) for s, m in enumerate(_METHODS)] + [(m, 100 + s) for s, m in enumerate(_METHODS)])
def test_step_fuzz_allen_cahn(xi300, case):
    # every integrator on a seeded random Allen-Cahn grid (ragged rows, even columns) and step size, on the
    # auto kernel choice: same total iterations as the oracle, u_high / u_low / err to 1e-10
    method, seed = case
    rng = np.random.default_rng(seed)
    shape = (int(rng.integers(16, 140)), 2 * int(rng.integers(32, 80)))
    pb, ob = _pair(shape, diff=1e-3, nu=0.0, react=1.0)
    u = W.ic_random(shape, seed=seed, amp=0.8)
    h = float(rng.choice([0.002, 0.005, 0.01]))
    bound = O.spectrum_bound(ob, u)
    c, g = O.shift_scale(bound)
    ref = O.step(ob, method, u, h, c, g, TOL, TOL, xi300)
    assert ref.status == O.OK
    with lx.Context(pb) as ctx:
        lo, hi = torch.empty(shape, dtype=torch.float64, device="cuda"), torch.empty(shape, dtype=torch.float64,
                                                                                        device="cuda")
        it, err = lx.lx_step(ctx, method, _dev(u), lo, hi, h, c, g, TOL, TOL)
    assert it == ref.iters, (case, it, ref.iters)
    assert _rel(hi, ref.u_high) <= TOL
    if method not in ("rosenbrock_euler", "exprb42"):
        assert _rel(lo, ref.u_low) <= TOL
        assert err == pytest.approx(ref.err, rel=1e-6, abs=1e-14)


@pytest.mark.parametrize("shape,react,src", [((24, 16, 64), 0.0, False), ((70, 32, 128), 1.0, False),
                                             ((9, 16, 64), 1.0, True)])
def test_rhs_3d_kernels(xi300, shape, react, src):
    # f(u) dt on 3D grids: the shared-memory plane-tile kernel (default on n1 % 16 == 0, n2 % 64 == 0) and the
    # warp-tile kernel (lx_ctx_set_kernel(., ., 1)) against the oracle's f (runs of 64 planes, a ragged last
    # run, runs shorter than the stencil reach, reaction and source terms)
    dx = tuple(2.0 / m for m in shape)
    diff, nu = (0.01, 0.0) if react else (1.0, 10.0)
    S = W.ic_random(shape, seed=22, amp=0.3) if src else None
    pb = lx.Problem(shape, dx, diff, nu, react, source=_dev(S) if src else None)
    ob = O.Problem(shape, dx, diff, nu, react, source=S)
    u = W.ic_random(shape, seed=21, amp=0.7)
    ref = 0.125 * O.rhs(ob, u)
    outs = []
    for k3d in (0, 1):
        with lx.Context(pb) as ctx:
            ctx.set_kernel(0, k3d)
            f = torch.empty(shape, dtype=torch.float64, device="cuda")
            lx.lx_rhs(ctx, _dev(u), f, 0.125)
            outs.append(f.cpu().numpy())
    for o in outs:
        assert np.abs(o - ref).max() <= 1e-12 * np.abs(ref).max()
    np.testing.assert_array_equal(outs[0], outs[1])   # same FMA order in both kernels


@pytest.mark.parametrize("method", ["epirk4s3a", "exprb43"])
def test_integrate_3d_two_step_kernel(xi300, method):
    # the time loop on a 3D grid through the two-step plane-sweep kernel: repeated calls with the same
    # parameters every step (predicted final iterations, reused coefficient tables) must keep the oracle's
    # iteration counts and results step after step
    shape = (32, 16, 64)
    pb, ob = _pair(shape)
    u = W.ic_random(shape, seed=31, amp=0.3)
    dt, nsteps = 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape), 4
    ud = _dev(u)
    with lx.Context(pb) as ctx:
        ctx.set_kernel(2)
        assert ctx.iterations_per_pass == 2
        it, err = lx.lx_integrate(ctx, method, ud, dt, nsteps, TOL, TOL)
    tot = 0
    for _ in range(nsteps):
        c, g = O.shift_scale(O.spectrum_bound(ob, u))
        r = O.step(ob, method, u, dt, c, g, TOL, TOL, xi300)
        tot += r.iters
        u = r.u_high
    assert it == tot
    assert _rel(ud, u) <= TOL
