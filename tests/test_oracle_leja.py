"""Pins for the oracle's real Leja interpolation and integrators.

Exactness references (never the oracle itself):
  * FFT-exact phi_l(dt A) v for the circulant stencil operators, with the
    spectrum taken from the FFT of the operator's impulse response;
  * dense scipy expm / augmented-matrix phi on <= 16x16 grids;
  * per-entry mpmath phi for diagonal operators;
  * a mode-by-mode (Fourier) simulation of the Leja recurrence with 60-digit
    divided differences, which must stop at the same iteration;
  * convergence orders of the integrators against a scipy DOP853 reference.
"""
import math

import numpy as np
import pytest
import scipy.integrate

import oracle as O
import workloads as W
from tests import refs


def _advdiff(n, nu=10.0):
    return O.Problem((n, n), (2 / n, 2 / n), 1.0, nu, 0.0)


def _cg(pb, u=None):
    return O.shift_scale(O.spectrum_bound(pb, u))


@pytest.mark.parametrize("l", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("mult", [1.0, 10.0, 100.0])
def test_leja_vs_fft_exact(xi300, l, mult):
    n = 64
    pb = _advdiff(n)
    dt = mult * W.dt_cfl(n, 10.0)
    c, g = _cg(pb)
    u0 = W.ic_problem1_2d(n)
    r = O.real_leja_phi(pb, u0, dt, c, g, l, 1e-13, 1e-13, xi300)
    assert r.status == O.OK
    sym = refs.impulse_symbol(lambda v: O.jac_apply(pb, None, v), (n, n))
    ex = refs.fft_apply_phi(sym, u0, dt, l)
    rel = np.linalg.norm(r.outs[0] - ex) / np.linalg.norm(ex)
    # a-posteriori stop is not a bound: allow 100x tol
    assert rel <= 1e-11, rel


@pytest.mark.parametrize("l", [0, 1, 3])
def test_leja_iteration_count_matches_spectral_simulation(xi300, l):
    # The stopping decision depends only on the recurrence; a Fourier-space
    # simulation with 60-digit divided differences must stop at the same m.
    for n, mult in [(64, 1.0), (64, 10.0), (64, 100.0), (128, 10.0)]:
        pb = _advdiff(n)
        dt = mult * W.dt_cfl(n, 10.0)
        c, g = _cg(pb)
        u0 = W.ic_problem1_2d(n)
        r = O.real_leja_phi(pb, u0, dt, c, g, l, 1e-10, 1e-10, xi300)
        sym = refs.impulse_symbol(lambda v: O.jac_apply(pb, None, v), (n, n))
        m, p = refs.spectral_leja_iters(sym, u0, dt, c, g, l, 1e-10, 1e-10, xi300, max_nodes=160)
        assert r.iters == m, (n, mult, r.iters, m)
        assert np.linalg.norm(r.outs[0] - p) <= 1e-12 * np.linalg.norm(p)   # d_k conditioning at rho~60
        assert min(r.margins) > 1.0


@pytest.mark.parametrize("l", [0, 1, 3])
@pytest.mark.parametrize("nu,mult", [(3.0, 5.0), (1.0, 20.0)])
def test_leja_vs_dense_augmented(xi300, l, nu, mult):
    # 12x12 grid, broadband random v.  (Real Leja needs a spectrum close to the
    # real axis: at this coarse grid nu = 3, 20 x CFL diverges -- P:141's
    # ellipse case, out of scope, so the cases here keep rho*|Im|/|Re| small.)
    n = 12
    pb = _advdiff(n, nu=nu)
    M = refs.dense_matrix(lambda v: O.jac_apply(pb, None, v.reshape(n, n)), n * n)
    v = W.random_vector((n, n), seed=11)
    c, g = _cg(pb)
    dt = mult * W.dt_cfl(n, nu)
    r = O.real_leja_phi(pb, v, dt, c, g, l, 1e-14, 1e-14, xi300)
    assert r.status == O.OK
    ex = refs.dense_phi(M, v.ravel(), dt, l)
    assert np.linalg.norm(r.outs[0].ravel() - ex) <= 1e-12 * np.linalg.norm(ex)


def test_leja_diagonal_operator_per_entry(xi300):
    # diagonal J = diag(1 - 3u^2) -> p_i = phi_l(dt J_ii) v_i.
    u = np.linspace(0.6, 4.0, 64).reshape(8, 8)           # J_ii in [-47, -0.08]
    pb = O.Problem((8, 8), (0.25, 0.25), 0.0, 0.0, 1.0)
    v = W.random_vector((8, 8), seed=2)
    c, g = _cg(pb, u)
    dt = 0.5
    for l in range(5):
        r = O.real_leja_phi(pb, v, dt, c, g, l, 1e-14, 1e-15, xi300, u_lin=u)
        assert r.status == O.OK
        ex = np.array([float(refs.phi_mp(l, dt * (1 - 3 * ui * ui))) for ui in u.ravel()]) * v.ravel()
        assert np.abs(r.outs[0].ravel() - ex).max() <= 1e-12 * np.abs(ex).max(), l


def test_leja_zero_input_and_dt_zero(xi300):
    pb = _advdiff(16)
    c, g = _cg(pb)
    r = O.real_leja_phi(pb, np.zeros((16, 16)), 1e-3, c, g, 1, 1e-10, 1e-10, xi300)
    assert r.status == O.OK and r.iters == 1 and np.all(r.outs[0] == 0)
    v = W.ic_problem1_2d(16)
    for l in range(5):
        r = O.real_leja_phi(pb, v, 0.0, c, g, l, 1e-10, 1e-10, xi300)
        assert r.status == O.OK and r.iters == 1
        np.testing.assert_array_equal(r.outs[0], v * (1.0 / math.factorial(l)))


def test_leja_vertical_equals_separate_calls(xi300):
    # coeffs {0.25, 0.5, 1} == three single-coefficient calls to 1e-11,
    # shared-recurrence iters <= sum of separate iters.
    n = 32
    pb = _advdiff(n)
    c, g = _cg(pb)
    dt = 10 * W.dt_cfl(n, 10.0)
    v = W.ic_problem1_2d(n)
    cf = (0.25, 0.5, 1.0)
    rv = O.real_leja_phi(pb, v, dt, c, g, 1, 1e-12, 1e-12, xi300, coeffs=cf)
    total = 0
    for k, a in enumerate(cf):
        # phi_1(a dt A) v == single call with dt' = a dt
        rs = O.real_leja_phi(pb, v, a * dt, c, g, 1, 1e-12, 1e-12, xi300)
        total += rs.iters
        # frozen accumulators stop at the same m as the separate call
        assert np.linalg.norm(rv.outs[k] - rs.outs[0]) <= 1e-11 * np.linalg.norm(rs.outs[0])
    assert rv.iters <= total


def test_leja_interpolation_error_decays(xi300):
    n = 64
    pb = _advdiff(n)
    c, g = _cg(pb)
    dt = 10 * W.dt_cfl(n, 10.0)
    v = W.ic_problem1_2d(n)
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), (n, n))
    ex = refs.fft_apply_phi(sym, v, dt, 1)
    errs, its = [], []
    for tol in (1e-4, 1e-7, 1e-10, 1e-13):
        r = O.real_leja_phi(pb, v, dt, c, g, 1, tol, tol, xi300)
        errs.append(np.linalg.norm(r.outs[0] - ex) / np.linalg.norm(ex))
        its.append(r.iters)
    assert all(a > b for a, b in zip(errs, errs[1:])), errs
    assert all(a < b for a, b in zip(its, its[1:])), its


def test_leja_noconv_and_errors(xi300):
    pb = _advdiff(16)
    c, g = _cg(pb)
    v = W.ic_problem1_2d(16)
    r = O.real_leja_phi(pb, v, 1000 * W.dt_cfl(16, 10.0), c, g, 0, 1e-14, 0.0, xi300, max_nodes=20)
    assert r.status == O.ERR_NOCONV and r.iters == 19
    assert O.real_leja_phi(pb, v, 1e-3, c, g, 5, 1e-10, 1e-10, xi300).status == O.ERR_UNSUPPORTED
    assert O.real_leja_phi(pb, v, 1e-3, c, g, 1, 1e-10, 1e-10, xi300, coeffs=(1.0, 0.5)).status == O.ERR_ARG
    assert O.real_leja_phi(pb, v, 1e-3, c, -1.0, 1, 1e-10, 1e-10, xi300).status == O.ERR_ARG


# ---------------------------------------------------------------- integrators
@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3",
                                    "exprb54s4", "epirk4s3b", "epirk4s3"])
def test_integrator_linear_exactness(xi300, method):
    # every exponential integrator is exact on linear homogeneous problems
    n = 64
    pb = _advdiff(n)
    c, g = _cg(pb)
    dt = 10 * W.dt_cfl(n, 10.0)
    u0 = W.ic_problem1_2d(n)
    r = O.step(pb, method, u0, dt, c, g, 1e-12, 1e-12, xi300)
    assert r.status == O.OK
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), (n, n))
    ex = refs.fft_apply_phi(sym, u0, dt, 0)
    assert np.linalg.norm(r.u_high - ex) <= 1e-11 * np.linalg.norm(ex)
    if method not in ("rosenbrock_euler", "exprb42"):
        assert r.err == 0.0       # R18: F == 0 exactly for linear f


def test_exprb32_embedded_error_contract(xi300):
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 1e-2, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(n)
    c, g = _cg(pb, u)
    r = O.step(pb, "exprb32", u, 0.05, c, g, 1e-12, 1e-12, xi300)
    assert r.status == O.OK and r.err > 0
    assert r.err == pytest.approx(O.l2norm_scaled(r.u_high - r.u_low), rel=1e-13)


def _allen_cahn_reference(pb, u0, T):
    n0, n1 = pb.shape

    def f(t, y):
        return O.rhs(pb, y.reshape(n0, n1)).ravel()

    sol = scipy.integrate.solve_ivp(f, (0, T), u0.ravel(), method="DOP853", rtol=1e-13, atol=1e-13)
    return sol.y[:, -1].reshape(n0, n1)


@pytest.mark.parametrize("method,order", [("rosenbrock_euler", 2), ("exprb32", 3), ("exprb43", 4),
                                          ("epirk4s3a", 4), ("exprb42", 4), ("epirk4s3b", 4),
                                          ("epirk4s3", 4)])
def test_integrator_convergence_order(xi300, method, order):
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    T = 0.5
    uref = _allen_cahn_reference(pb, u0, T)
    errs = []
    for nsteps in (4, 8, 16, 32):
        h = T / nsteps
        u = u0.copy()
        for _ in range(nsteps):
            c, g = _cg(pb, u)
            r = O.step(pb, method, u, h, c, g, 1e-14, 1e-14, xi300)
            assert r.status == O.OK
            u = r.u_high
        errs.append(np.linalg.norm(u - uref) / np.linalg.norm(uref))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - order) < 0.3, (errs, orders)


@pytest.mark.parametrize("l", [0, 1, 3])
def test_leja_3d_vs_fft_exact(xi300, l):
    n = 16
    shape = (n, n, n)
    pb = O.Problem(shape, (2 / n,) * 3, 1.0, 10.0, 0.0)
    c, g = _cg(pb)
    dt = 5 * W.dt_cfl(n, 10.0, 3)
    v = W.ic_random(shape, seed=4, amp=0.2)
    r = O.real_leja_phi(pb, v, dt, c, g, l, 1e-13, 1e-13, xi300)
    assert r.status == O.OK
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), shape)
    ex = refs.fft_apply_phi(sym, v, dt, l)
    assert np.linalg.norm(r.outs[0] - ex) <= 1e-11 * np.linalg.norm(ex)


def test_problem2_rosenbrock_euler_exact(xi300):
    # Problem II: u' = A u + S.  Rosenbrock-Euler with the source in f is the exact update
    # u(dt) = exp(dt A) u0 + dt phi_1(dt A) S  (P:586 with the dt factor, reading R12).
    n = 64
    S = W.source_problem2_2d(n)
    pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 10.0, 0.0, S)
    c, g = _cg(pb)
    dt = 10 * W.dt_cfl(n, 10.0)
    u0 = W.ic_problem1_2d(n)
    r = O.step(pb, "rosenbrock_euler", u0, dt, c, g, 1e-13, 1e-13, xi300)
    assert r.status == O.OK
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), (n, n))
    ex = refs.fft_apply_phi(sym, u0, dt, 0) + dt * refs.fft_apply_phi(sym, S, dt, 1)
    assert np.linalg.norm(r.u_high - ex) <= 1e-11 * np.linalg.norm(ex)
    # higher-order integrators are exact too: their remainders vanish (S cancels in F(x) - F(u), R21)
    for m in ("exprb32", "exprb43", "epirk4s3a"):
        rm = O.step(pb, m, u0, dt, c, g, 1e-13, 1e-13, xi300)
        assert np.linalg.norm(rm.u_high - ex) <= 1e-11 * np.linalg.norm(ex)


@pytest.mark.parametrize("method,order", [("rosenbrock_euler", 2), ("exprb32", 3), ("exprb43", 4),
                                          ("epirk4s3a", 4), ("exprb42", 4)])
def test_integrator_order_burgers(xi300, method, order):
    # Problem III: viscous Burgers, exact Jacobian (R13), P:593 initial condition
    n, T = 24, 0.005
    pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 0.0, 0.0, None, 10.0)
    u0 = W.ic_burgers_2d(n)

    def f(t, y):
        return O.rhs(pb, y.reshape(n, n)).ravel()

    ref = scipy.integrate.solve_ivp(f, (0, T), u0.ravel(), method="DOP853", rtol=1e-13, atol=1e-13).y[:, -1]
    errs = []
    for ns in (4, 8, 16):
        h = T / ns
        u = u0.copy()
        for _ in range(ns):
            c, g = _cg(pb, u)
            r = O.step(pb, method, u, h, c, g, 1e-14, 1e-14, xi300)
            assert r.status == O.OK
            u = r.u_high
        errs.append(np.linalg.norm(u.ravel() - ref) / np.linalg.norm(ref))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - order) < 0.3, (errs, orders)


def test_epirk5p1_fifth_order(xi300):
    # EPIRK5P1 (reading R26): fifth order on Allen-Cahn (exact Jacobian) against scipy DOP853;
    # a mistyped tableau constant drops the observed order to ~2 (survey of perturbed b3)
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    T = 0.5
    uref = _allen_cahn_reference(pb, u0, T)
    errs = []
    for nsteps in (4, 8, 16):
        h = T / nsteps
        u = u0.copy()
        for _ in range(nsteps):
            c, g = _cg(pb, u)
            r = O.step(pb, "epirk5p1", u, h, c, g, 1e-14, 1e-14, xi300)
            assert r.status == O.OK and r.err > 0.0   # embedded fourth-order estimate (R33)
            u = r.u_high
        errs.append(np.linalg.norm(u - uref) / np.linalg.norm(uref))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(orders > 4.7) and np.all(orders < 6.0), (errs, orders)


def test_epirk5p1_fifth_order_burgers(xi300):
    n, T = 24, 0.005
    pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 0.0, 0.0, None, 10.0)
    u0 = W.ic_burgers_2d(n)
    ref = scipy.integrate.solve_ivp(lambda t, y: O.rhs(pb, y.reshape(n, n)).ravel(), (0, T), u0.ravel(),
                                    method="DOP853", rtol=1e-13, atol=1e-13).y[:, -1]
    errs = []
    for ns in (2, 4, 8):
        u = u0.copy()
        for _ in range(ns):
            c, g = _cg(pb, u)
            r = O.step(pb, "epirk5p1", u, T / ns, c, g, 1e-14, 1e-14, xi300)
            assert r.status == O.OK
            u = r.u_high
        errs.append(np.linalg.norm(u.ravel() - ref) / np.linalg.norm(ref))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert orders[-1] > 4.5, (errs, orders)


def test_exprb53s3_orders(xi300):
    # EXPRB53s3 (reading R27): fifth-order solution and third-order embedded solution on Allen-Cahn;
    # with a32 = 729/125 phi_3(c3 hJ) alone (dropping 27/25 phi_3(c2 hJ)) the order falls to ~3.5
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    T = 0.5
    uref = _allen_cahn_reference(pb, u0, T)
    for attr, order in (("u_high", 5), ("u_low", 3)):
        errs = []
        for nsteps in (4, 8, 16):
            u = u0.copy()
            for _ in range(nsteps):
                c, g = _cg(pb, u)
                r = O.step(pb, "exprb53s3", u, T / nsteps, c, g, 1e-14, 1e-14, xi300)
                assert r.status == O.OK
                assert r.err == pytest.approx(O.l2norm_scaled(r.u_high - r.u_low), rel=1e-12)
                u = getattr(r, attr)
            errs.append(np.linalg.norm(u - uref) / np.linalg.norm(uref))
        orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
        assert np.all(np.abs(orders - order) < 0.35), (attr, errs, orders)


# ---------------------------------------------------------------- round-2 pins (VERDICT r1 "What's weak" #1)
@pytest.mark.parametrize("method,order", [("exprb32", 2), ("exprb43", 3), ("epirk4s3a", 3), ("epirk5p1", 4),
                                          ("epirk4s3b", 3), ("epirk4s3", 3)])
def test_embedded_solution_order(xi300, method, order):
    # The embedded (lower-order) solutions u_low that the error estimate ||u_high - u_low|| (P:252,
    # reading R20) compares against: EXPRB32 -> a (order 2), EXPRB43 / EPIRK4s3A -> u_3
    # (order 3, R17).  A wrong phi_3 weight in u_3 (e.g. 16 -> 15) drops the order to ~2.
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    T = 0.5
    uref = _allen_cahn_reference(pb, u0, T)
    errs = []
    for nsteps in (4, 8, 16, 32):
        u = u0.copy()
        for _ in range(nsteps):
            c, g = _cg(pb, u)
            r = O.step(pb, method, u, T / nsteps, c, g, 1e-14, 1e-14, xi300)
            assert r.status == O.OK
            u = r.u_low
        errs.append(np.linalg.norm(u - uref) / np.linalg.norm(uref))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - order) < 0.3, (errs, orders)


def test_nonfinite_input_and_linearisation_state(xi300):
    # P:155 stopping rule with non-finite norms -> LX_ERR_NONFINITE ("non-finite
    # intermediate -> divergence error"), reported at the iteration whose check saw it: a NaN in v
    # reaches y_1 and ||y_1|| at m = 1; an Inf in the linearisation state u makes the Allen-Cahn
    # Jacobian diagonal 1 - 3u^2 = -Inf, so y_1 = -Inf there and ||y_1|| = Inf at m = 1.
    n = 32
    pb = _advdiff(n)
    c, g = _cg(pb)
    v = W.ic_problem1_2d(n)
    v[3, 5] = np.nan
    r = O.real_leja_phi(pb, v, W.dt_cfl(n, 10.0), c, g, 0, 1e-10, 1e-10, xi300)
    assert (r.status, r.iters) == (O.ERR_NONFINITE, 1)
    pa = O.Problem((n, n), (2 / n, 2 / n), 1e-4, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(n)
    c, g = _cg(pa, u)
    u[7, 9] = np.inf
    r = O.real_leja_phi(pa, 0.01 * W.ic_problem1_2d(n), 0.01, c, g, 1, 1e-10, 1e-10, xi300, u_lin=u)
    assert (r.status, r.iters) == (O.ERR_NONFINITE, 1)


def _first_overflow_iteration(sym, v, c, g, xi, mmax):
    """First m at which sum_i y_m[i]^2 exceeds DBL_MAX, from the exact Fourier recurrence
    y_m^ = prod_{k<m} ((lambda - c)/g - xi_k) v^ (Eq. (2)) in log space (Parseval), independent of
    any fp64 stencil evaluation."""
    vh = np.fft.fftn(v).ravel()
    lam = sym.ravel()
    N = vh.size
    logamp = np.log(np.abs(vh) + 1e-300)
    for m in range(1, mmax):
        logamp = logamp + np.log(np.abs((lam - c) / g - xi[m - 1]))
        top = logamp.max()
        # sum |y^|^2 / N = sum_i y_i^2 (Parseval with the unnormalised FFT)
        log_sumsq = 2 * top + np.log(np.sum(np.exp(2 * (logamp - top)))) - np.log(N)
        if log_sumsq > np.log(np.finfo(np.float64).max):
            return m
    return None


@pytest.mark.parametrize("fac", [1e-2, 1e-6])
def test_nonfinite_unenclosed_spectrum(xi300, fac):
    # (c, gamma) that do not enclose the spectrum (gamma too small by `fac`): the Newton basis grows
    # like (|lambda|/gamma)^m; the run ends with NONFINITE exactly when sum y_m^2 overflows (the
    # nonfinite ||y_m|| of P:155), which the exact Fourier recurrence predicts independently.
    n = 32
    pb = _advdiff(n)
    c, g = _cg(pb)
    u0 = W.ic_problem1_2d(n)
    r = O.real_leja_phi(pb, u0, W.dt_cfl(n, 10.0), c * fac, g * fac, 0, 1e-10, 1e-10, xi300)
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), (n, n))
    m = _first_overflow_iteration(sym, u0, c * fac, g * fac, xi300, 300)
    assert r.status == O.ERR_NONFINITE
    assert r.iters == m, (r.iters, m)


def test_leja_3d_real_leja_limit(xi300):
    # A limit of real Leja interpolation with fp64 divided differences (readings R8,
    # R28).  The 3D upwind operator on 16^3 has eigenvalues with imaginary parts of ~30% of |lambda|
    # (nu = 10 on a coarse grid); off the real focal interval the Newton basis grows geometrically
    # (~1e9 by m = 40), so it amplifies the ~1e-17 absolute error floor of the fp64 triangular
    # recurrence instead of the decaying exact d_m.  At 5 x CFL the run converges before that
    # matters (test_leja_3d_vs_fft_exact); at 10 x CFL the oracle hits the node cap (NOCONV, 299) with
    # a diverged polynomial.  Independent confirmation: the exact mode-by-mode Fourier recurrence
    # converges (m = 38) with 60-digit coefficients but never with the fp64 coefficients.
    n = 16
    shape = (n, n, n)
    pb = O.Problem(shape, (2 / n,) * 3, 1.0, 10.0, 0.0)
    c, g = _cg(pb)
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), shape)
    assert np.max(np.abs(sym.imag)) > 0.25 * np.max(np.abs(sym))
    v = W.ic_random(shape, seed=4, amp=0.5)
    dt = 10.0 * W.dt_cfl(n, 10.0, 3)
    r = O.real_leja_phi(pb, v, dt, c, g, 0, 1e-10, 1e-10, xi300)
    assert (r.status, r.iters) == (O.ERR_NOCONV, 299)
    assert np.linalg.norm(r.outs[0]) > 1e30 * np.linalg.norm(v)
    d_mp = [float(x) for x in refs.divided_differences_mp(0, xi300, 300, dt, c, g, dps=60)]
    d_64 = list(O.divided_differences(0, xi300, 300, dt, c, g))
    m_exact, _ = refs.spectral_leja_iters(sym, v, dt, c, g, 0, 1e-10, 1e-10, xi300, d=d_mp, max_nodes=300)
    m_fp64, _ = refs.spectral_leja_iters(sym, v, dt, c, g, 0, 1e-10, 1e-10, xi300, d=d_64, max_nodes=300)
    assert m_exact == 38 and m_fp64 is None


def test_openmp_oracle_build_is_bit_identical(xi300):
    # bench.py's all-core cpu_baseline times liblxoracle_omp.so: the same source with -fopenmp (element-wise
    # loops split over threads, the pairwise norm's top recursion levels in parallel over the SAME tree) --
    # it must compute exactly what the serial oracle computes
    n = 128
    pb = _advdiff(n)
    c, g = _cg(pb)
    v = W.ic_random((n, n), seed=8, amp=0.3)
    res = []
    try:
        for omp in (False, True):
            O.use_openmp(omp)
            r = O.real_leja_phi(pb, v, 10 * W.dt_cfl(n, 10.0), c, g, 1, 1e-10, 1e-10, xi300, coeffs=(0.5, 1.0))
            res.append((r.iters, r.outs, O.l2norm_scaled(v)))
    finally:
        O.use_openmp(False)
    assert res[0][0] == res[1][0] and res[0][2] == res[1][2]
    for a, b in zip(res[0][1], res[1][1]):
        np.testing.assert_array_equal(a, b)


def test_exprb54s4_orders(xi300):
    # EXPRB54s4 (reading R31): fifth-order solution and fourth-order embedded solution on Allen-Cahn.  Its
    # fourth stage carries D2 AND D3 (both stiff stage conditions psi_3 = psi_4 = 0 at c4 = 9/10), which makes
    # its error constant far smaller than EXPRB53s3's (a D3-only fourth stage is an ordinary order-5 method
    # with EXPRB53s3-sized errors) -- pinned as a ratio, together with the orders
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    T = 0.5
    uref = _allen_cahn_reference(pb, u0, T)
    res = {}
    for method, attr in (("exprb54s4", "u_high"), ("exprb54s4", "u_low"), ("exprb53s3", "u_high")):
        errs = []
        for nsteps in (8, 16, 32):
            u = u0.copy()
            for _ in range(nsteps):
                c, g = _cg(pb, u)
                r = O.step(pb, method, u, T / nsteps, c, g, 1e-14, 1e-14, xi300)
                assert r.status == O.OK
                assert r.err == pytest.approx(O.l2norm_scaled(r.u_high - r.u_low), rel=1e-12)
                u = getattr(r, attr)
            errs.append(np.linalg.norm(u - uref) / np.linalg.norm(uref))
        res[(method, attr)] = (errs, np.log2(np.array(errs[:-1]) / np.array(errs[1:])))
    e5, o5 = res[("exprb54s4", "u_high")]
    e4, o4 = res[("exprb54s4", "u_low")]
    e53, _ = res[("exprb53s3", "u_high")]
    assert abs(o5[-1] - 5.0) < 0.35, res
    assert np.all(np.abs(o4 - 4.0) < 0.3), res
    assert e5[-1] < 0.3 * e53[-1], res


def _replay_controller(res, t_end, dt0, tol, q):
    # the controller of reading R32 replayed from the logged errors: accept iff err <= tol, next step
    # h min(5, max(0.2, 0.9 (tol/err)^(1/(q+1)))), the last step clipped to t_end
    t, h = 0.0, dt0
    for k in range(len(res.dts)):
        h = min(h, t_end - t)
        assert res.dts[k] == pytest.approx(h, rel=1e-14, abs=0.0), k
        ok = res.errs[k] <= tol
        assert bool(res.acc[k]) == ok, k
        fac = 5.0 if res.errs[k] == 0.0 else min(5.0, max(0.2, 0.9 * (tol / res.errs[k]) ** (1.0 / (q + 1))))
        if not np.isfinite(res.errs[k]):     # a failed step (NOCONV / NONFINITE) is a rejection with factor 0.2
            fac = 0.2
        if ok:
            t = t_end if h == t_end - t else t + h
        h = h * fac
    assert t == t_end


def test_adaptive_linear_problem_grows_steps(xi300):
    # Problem I is linear: every remainder vanishes (R18), so the embedded error is exactly 0, every step is
    # accepted and the step grows by the maximal factor 5 until the last one lands on t_end; the result is the
    # FFT-exact exp(t_end A) u0 (pure diffusion: a real spectrum, so the large late steps stay within real
    # Leja's reach, R28)
    n = 32
    pb = _advdiff(n, nu=0.0)
    u0 = W.ic_problem1_2d(n)
    dt0 = W.dt_cfl(n, 10.0)
    t_end = 200 * dt0
    res = O.integrate_adaptive(pb, "exprb43", u0, t_end, dt0, 1e-6, 1e-12, 1e-12, xi300)
    assert res.status == O.OK and res.rejected == 0
    assert np.all(res.errs == 0.0)
    np.testing.assert_allclose(res.dts[:-1], dt0 * 5.0 ** np.arange(len(res.dts) - 1), rtol=1e-14)
    assert len(res.dts) == 5      # dt0 (1 + 5 + 25 + 125) = 156 dt0 < 200 dt0 <= 781 dt0
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), (n, n))
    ex = refs.fft_apply_phi(sym, u0, t_end, 0)
    assert np.linalg.norm(res.u - ex) <= 1e-9 * np.linalg.norm(ex)


@pytest.mark.parametrize("method,q", [("exprb32", 2), ("exprb43", 3), ("epirk4s3a", 3), ("exprb54s4", 4),
                                      ("epirk5p1", 4), ("epirk4s3b", 3), ("epirk4s3", 3)])
def test_adaptive_controller_allen_cahn(xi300, method, q):
    # Allen-Cahn: the accept / reject decisions and the step sequence follow R32 exactly (replayed from the
    # logs), a too-large first step is rejected, and the global error at t_end shrinks with the tolerance
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    t_end = 0.5
    uref = _allen_cahn_reference(pb, u0, t_end)
    errs = []
    for tol in (1e-5, 1e-7, 1e-9):
        res = O.integrate_adaptive(pb, method, u0, t_end, 0.5, tol, 1e-12, 1e-12, xi300)
        assert res.status == O.OK
        assert res.rejected >= 1 and not res.acc[0]
        _replay_controller(res, t_end, 0.5, tol, q)
        errs.append(np.linalg.norm(res.u - uref) / np.linalg.norm(uref))
    assert errs[0] > errs[1] > errs[2], errs
    assert errs[1] < 1e-5, errs


def test_epirk5p1_embedded_is_fourth_order_and_estimates_the_local_error(xi300):
    # EPIRK5P1's embedded solution (reading R33: g32 -> 1/2, g33 -> 1): its local error is O(h^5) (global
    # order 4, test_embedded_solution_order), so the estimate err = ||u5 - u4|| / sqrt(N) falls
    # like h^5 and tracks the true local error of u4 within a small factor.  Any other (g32, g33) near
    # these values gives local order 4 (checked while reconstructing the tableau; DESIGN R33).
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    ests, trues = [], []
    for h in (0.0625, 0.03125, 0.015625):
        c, g = _cg(pb, u0)
        r = O.step(pb, "epirk5p1", u0, h, c, g, 1e-14, 1e-14, xi300)
        assert r.status == O.OK
        ex = _allen_cahn_reference(pb, u0, h)
        ests.append(r.err)
        trues.append(np.linalg.norm(r.u_low - ex) / np.sqrt(ex.size))
    orders = np.log2(np.array(ests[:-1]) / np.array(ests[1:]))
    assert abs(orders[-1] - 5.0) < 0.3 and np.all(orders > 4.4), (ests, orders)
    ratio = np.array(ests) / np.array(trues)
    assert np.all((ratio > 0.5) & (ratio < 2.0)), ratio


def test_epirk4s3b_local_error_order(xi300):
    # EPIRK4s3B (reading R34): one step's error falls like h^5 (stiff order 4).  Reconstructing the tableau,
    # each parameter was moved alone -- the phi_2 interpolation points 1/2 -> 0.55, 3/4 -> 0.8, the stage
    # weight 2/3 -> 0.7, a final weight -324 -> -320 -- and each drops the local order to 4 (or 3): the
    # order singles the published values out (DESIGN R34).
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    errs = []
    for h in (0.0625, 0.03125, 0.015625):
        c, g = _cg(pb, u0)
        r = O.step(pb, "epirk4s3b", u0, h, c, g, 1e-14, 1e-14, xi300)
        assert r.status == O.OK and r.err > 0.0
        ex = _allen_cahn_reference(pb, u0, h)
        errs.append(np.linalg.norm(r.u_high - ex) / np.linalg.norm(ex))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - 5.0) < 0.3 and np.all(orders > 4.6), (errs, orders)


def test_epirk4s3_local_error_order(xi300):
    # EPIRK4s3 (reading R35): one step's error falls like h^5; changing a phi_4 weight (27648 -> 27000)
    # drops the local order to 3 (dense-matrix check during the reconstruction, DESIGN R35)
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    errs = []
    for h in (0.0625, 0.03125, 0.015625):
        c, g = _cg(pb, u0)
        r = O.step(pb, "epirk4s3", u0, h, c, g, 1e-14, 1e-14, xi300)
        assert r.status == O.OK and r.err > 0.0
        ex = _allen_cahn_reference(pb, u0, h)
        errs.append(np.linalg.norm(r.u_high - ex) / np.linalg.norm(ex))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - 5.0) < 0.3 and np.all(orders > 4.6), (errs, orders)
