"""Pins for the oracle's black-box RHS mode: finite-difference
Jacobian-vector products ("computed numerically using finite differences"),
the literal nonlinear remainder F(x) = f(x) - J(u)x (alg:exprb32), and the
linear black-box operator (the RHS is A itself, P:161-171 real_Leja_exp(RHS, ...)).

References (never the FD oracle itself):
  * the forward-difference error expansion J_FD y - J y = (eps/2) f''(u)[y, y] + O(eps^2)
    with the exact second derivative written out (Allen-Cahn: -6 u y^2;
    Burgers: beta sum_d D_d(y^2)), eps per reading R25;
  * FFT-exact phi_l(dt A) v and exp(dt A) u for the circulant Problem-I operator;
  * the exact-Jacobian integrators' convergence order against scipy DOP853.
"""
import numpy as np
import pytest
import scipy.integrate

import oracle as O
import workloads as W
from tests import refs

EPS0 = 2.0 ** -26   # sqrt(DBL_EPSILON), reading R25


def _eps(u, y):
    return EPS0 * (1.0 + np.abs(u).max()) / np.abs(y).max()


def _curvature_coefficient(err, second):
    """Least-squares coefficient of the predicted curvature term in the FD error.  At the
    optimal eps the quotient's roundoff is of the same order as the curvature term pointwise,
    but it is unsystematic; projected on the curvature field it averages out (~1/sqrt(N))."""
    return float(np.sum(err * second) / np.sum(second * second))


def test_fd_jvp_error_expansion_allen_cahn():
    # f''(u)[y, y] = -6 u y^2 for f = eps2 lap u + u - u^3 (the stencil part is linear)
    n = 64
    u = W.ic_allen_cahn_2d(n)
    y = W.random_vector((n, n), seed=11)
    e = _eps(u, y)
    second = 0.5 * e * (-6.0 * u * y * y)
    for diff in (0.0, 1e-4):
        pb = O.Problem((n, n), (2 / n, 2 / n), diff, 0.0, 1.0)
        err = O.jac_apply_fd(pb, u, y) - O.jac_apply(pb, u, y)
        k = _curvature_coefficient(err, second)
        assert abs(k - 1.0) < 0.1, (diff, k)     # eps off by 2 -> 2, sign -> -1, no (1+|u|) -> ~0.35


def test_fd_jvp_error_expansion_burgers():
    # pure Burgers flux (beta/2) sum_d D_d(u^2) -> f''(u)[y, y] = beta sum_d D_d(y^2)
    n, beta = 64, 10.0
    pb = O.Problem((n, n), (2 / n, 2 / n), 0.0, 0.0, 0.0, None, beta)
    u = W.ic_burgers_2d(n)
    y = W.random_vector((n, n), seed=12)
    e = _eps(u, y)
    lin = O.Problem((n, n), (2 / n, 2 / n), 0.0, 1.0, 0.0)       # sum_d D_d as a linear operator
    second = 0.5 * e * beta * O.jac_apply(lin, None, y * y)
    err = O.jac_apply_fd(pb, u, y) - O.jac_apply(pb, u, y)
    k = _curvature_coefficient(err, second)
    assert abs(k - 1.0) < 0.1, k


def test_fd_jvp_scale_invariance():
    # eps ~ 1/||y||_inf: scaling the direction by a power of two scales eps by its inverse
    # exactly, so u + eps y is bitwise unchanged and J_FD(s y) = s J_FD(y) bitwise.
    n = 32
    pb = O.Problem((n, n), (2 / n, 2 / n), 1e-2, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(n)
    y = W.random_vector((n, n), seed=14)
    base = O.jac_apply_fd(pb, u, y)
    for s in (2.0 ** -20, 0.5, 8.0, 2.0 ** 30):
        assert np.array_equal(O.jac_apply_fd(pb, u, s * y), s * base)


def test_fd_jvp_zero_direction_and_linear_exactness():
    n = 32
    pl = O.Problem((n, n), (2 / n, 2 / n), 1.0, 10.0, 0.0)
    u = W.ic_problem1_2d(n)
    assert np.all(O.jac_apply_fd(pl, u, np.zeros((n, n))) == 0.0)
    # a linear f has no curvature: J_FD y = A y up to the roundoff floor eps_mach |A u| / eps
    y = W.random_vector((n, n), seed=13)
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pl, None, x), (n, n))
    ay = np.real(np.fft.ifft2(sym * np.fft.fft2(y)))
    got = O.jac_apply_fd(pl, u, y)
    assert np.linalg.norm(got - ay) <= 1e-6 * np.linalg.norm(ay)


def test_fd_remainder_matches_taylor_remainder():
    # F(x) - F(u) = g(x) - g(u) - g'(u)(x - u) for f = A + g; with FD Jacobians both
    # sides agree up to the FD error of J(u)x and J(u)u.
    n = 32
    pb = O.Problem((n, n), (2 / n, 2 / n), 1e-3, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(n)
    x = u + 0.01 * W.random_vector((n, n), seed=5)
    fu = O.rhs(pb, u)
    d_fd = O.nonlinear_remainder_fd(pb, u, x, fu) - O.nonlinear_remainder_fd(pb, u, u, fu)
    g = lambda z: z - z ** 3                                      # noqa: E731
    d_ex = g(x) - g(u) - (1 - 3 * u ** 2) * (x - u)
    # FD error of J(u)x ~ eps_x/2 |f''| |x|^2 with eps_x ~ 1.5e-8 (1+|u|)/|x|
    assert np.abs(d_fd - d_ex).max() <= 1e-7 + 1e-3 * np.abs(d_ex).max()


@pytest.mark.parametrize("l", [0, 1, 3])
@pytest.mark.parametrize("jac", ["fd", "linear_f"])
def test_blackbox_leja_vs_fft_exact(xi300, l, jac):
    n = 64
    pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 10.0, 0.0)
    dt = 10 * W.dt_cfl(n, 10.0)
    c, g = O.shift_scale(O.spectrum_bound(pb))
    u0 = W.ic_problem1_2d(n)
    r = O.real_leja_phi(pb, u0, dt, c, g, l, 1e-13, 1e-13, xi300, u_lin=u0, jac=jac)
    assert r.status == O.OK
    sym = refs.impulse_symbol(lambda v: O.jac_apply(pb, None, v), (n, n))
    ex = refs.fft_apply_phi(sym, u0, dt, l)
    rel = np.linalg.norm(r.outs[0] - ex) / np.linalg.norm(ex)
    # linear_f applies A exactly; fd adds ~eps_mach |A u| / eps relative noise per application
    assert rel <= (1e-11 if jac == "linear_f" else 1e-7), rel


@pytest.mark.parametrize("method", ["rosenbrock_euler", "exprb32", "exprb43", "epirk4s3a", "exprb42", "epirk5p1", "exprb53s3", "exprb54s4",
                                    "epirk4s3b", "epirk4s3"])
def test_fd_integrators_linear_exactness(xi300, method):
    n = 64
    pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 10.0, 0.0)
    c, g = O.shift_scale(O.spectrum_bound(pb))
    dt = 10 * W.dt_cfl(n, 10.0)
    u0 = W.ic_problem1_2d(n)
    r = O.step(pb, method, u0, dt, c, g, 1e-12, 1e-12, xi300, jac="fd")
    assert r.status == O.OK
    sym = refs.impulse_symbol(lambda x: O.jac_apply(pb, None, x), (n, n))
    ex = refs.fft_apply_phi(sym, u0, dt, 0)
    # F(x) - F(u) vanishes in exact arithmetic, but the literal FD remainder carries the quotient's
    # roundoff eps_mach |A x| / eps ~ 1e-8 |u| (times the tableau weights, up to 144; EPIRK4s3's phi_4
    # weights reach 34992 (R35): 243 x the noise): not 1e-11 as with the analytic remainder (R18)
    bound = 1e-5 if method == "epirk4s3" else 3e-8
    assert np.linalg.norm(r.u_high - ex) <= bound * np.linalg.norm(ex)


@pytest.mark.parametrize("method,order", [("rosenbrock_euler", 2), ("exprb32", 3), ("exprb43", 4)])
def test_fd_integrator_convergence_order(xi300, method, order):
    # black-box Allen-Cahn: same orders as with the exact Jacobian (FD error ~1e-8 << step error)
    n = 16
    pb = O.Problem((n, n), (2 / n, 2 / n), 2e-3, 0.0, 1.0)
    u0 = W.ic_allen_cahn_2d(n)
    T = 0.5
    uref = scipy.integrate.solve_ivp(lambda t, y: O.rhs(pb, y.reshape(n, n)).ravel(), (0, T), u0.ravel(),
                                     method="DOP853", rtol=1e-13, atol=1e-13).y[:, -1].reshape(n, n)
    errs = []
    for nsteps in (4, 8, 16):
        h = T / nsteps
        u = u0.copy()
        for _ in range(nsteps):
            c, g = O.shift_scale(O.spectrum_bound(pb, u))
            r = O.step(pb, method, u, h, c, g, 1e-13, 1e-13, xi300, jac="fd")
            assert r.status == O.OK
            u = r.u_high
        errs.append(np.linalg.norm(u - uref) / np.linalg.norm(uref))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - order) < 0.3, (errs, orders)
