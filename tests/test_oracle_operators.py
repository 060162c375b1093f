"""Pins for the oracle's operators, spectrum bound and power iteration.

The stencils are pinned by refinement order against analytic derivatives
(second-order centred / third-order upwind), by dissipativity (R10),
and by dense eigenvalues; the Allen-Cahn Jacobian by central differences of f.
"""
import numpy as np
import pytest
import scipy.linalg

import oracle as O
import workloads as W
from tests import refs


def _field_and_derivs(n):
    x, y = W.grid_2d(n)
    k = 2 * np.pi
    u = np.sin(k * x) * np.cos(k * y) + 0.5 * np.sin(2 * k * y)
    ux = k * np.cos(k * x) * np.cos(k * y)
    uy = -k * np.sin(k * x) * np.sin(k * y) + k * np.cos(2 * k * y)
    lap = -2 * k * k * np.sin(k * x) * np.cos(k * y) - 0.5 * 4 * k * k * np.sin(2 * k * y)
    return u, ux, uy, lap


def test_constant_field_maps_to_zero():
    pb = O.Problem((16, 24), (2 / 16, 2 / 24), 1.0, 10.0, 0.0)
    assert np.all(O.rhs(pb, np.full((16, 24), 3.25)) == 0.0)


def test_laplacian_second_order():
    errs = []
    for n in (32, 64, 128):
        u, ux, uy, lap = _field_and_derivs(n)
        pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 0.0, 0.0)
        errs.append(np.abs(O.rhs(pb, u).reshape(n, n) - lap).max())
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(orders - 2.0) < 0.1), orders


def test_upwind_third_order_and_sign():
    errs = []
    for n in (32, 64, 128):
        u, ux, uy, lap = _field_and_derivs(n)
        pb = O.Problem((n, n), (2 / n, 2 / n), 0.0, 1.0, 0.0)   # pure nu*(D_x + D_y)
        errs.append(np.abs(O.rhs(pb, u).reshape(n, n) - (ux + uy)).max())
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(orders - 3.0) < 0.15), orders


def test_advdiff_3d_orders():
    errs_d, errs_a = [], []
    for n in (16, 32, 64):
        c = W.coords(n)
        x, y, z = np.meshgrid(c, c, c, indexing="ij")
        k = 2 * np.pi
        u = np.sin(k * x) * np.sin(k * y) * np.sin(k * z)
        du = k * (np.cos(k * x) * np.sin(k * y) * np.sin(k * z) + np.sin(k * x) * np.cos(k * y) * np.sin(k * z)
                  + np.sin(k * x) * np.sin(k * y) * np.cos(k * z))
        pd = O.Problem((n, n, n), (2 / n,) * 3, 1.0, 0.0, 0.0)
        pa = O.Problem((n, n, n), (2 / n,) * 3, 0.0, 1.0, 0.0)
        errs_d.append(np.abs(O.rhs(pd, u).reshape(n, n, n) + 3 * k * k * u).max())
        errs_a.append(np.abs(O.rhs(pa, u).reshape(n, n, n) - du).max())
    od = np.log2(np.array(errs_d[:-1]) / np.array(errs_d[1:]))
    oa = np.log2(np.array(errs_a[:-1]) / np.array(errs_a[1:]))
    assert np.all(np.abs(od - 2.0) < 0.1), od
    assert np.all(np.abs(oa - 3.0) < 0.15), oa


def test_advdiff_dissipative_and_bound_dense():
    # R10: the +x-biased upwind stencil makes the spectrum lie in Re <= 0;
    # R9: |lambda_max| equals the closed form sum_d 4/dx^2 + 4nu/(3dx).
    for shape in [(16, 16), (8, 12)]:
        dx = tuple(2 / n for n in shape)
        pb = O.Problem(shape, dx, 1.0, 10.0, 0.0)
        N = int(np.prod(shape))
        M = refs.dense_matrix(lambda v: O.jac_apply(pb, None, v.reshape(shape)), N)
        ev = scipy.linalg.eigvals(M)
        assert ev.real.max() <= 1e-9 * np.abs(ev).max()
        if shape[0] == shape[1]:
            assert O.spectrum_bound(pb) == pytest.approx(np.abs(ev).max(), rel=1e-12)
        else:
            assert O.spectrum_bound(pb) >= np.abs(ev).max() * (1 - 1e-12)


def test_advdiff_bound_vs_fourier_grid():
    # closed form vs brute-force max over the full discrete Fourier grid
    for n in (64, 256):
        pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 10.0, 0.0)
        sym = refs.impulse_symbol(lambda v: O.jac_apply(pb, None, v), (n, n))
        assert O.spectrum_bound(pb) == pytest.approx(np.abs(sym).max(), rel=1e-12)


def test_allen_cahn_jacobian_central_difference():
    n = 24
    pb = O.Problem((n, n), (2 / n, 2 / n), 1e-2, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(n)
    v = W.random_vector((n, n), seed=3)
    eps = 1e-5
    fd = (O.rhs(pb, u + eps * v) - O.rhs(pb, u - eps * v)) / (2 * eps)
    jv = O.jac_apply(pb, u, v)
    assert np.linalg.norm(jv - fd) <= 1e-8 * np.linalg.norm(jv)


def test_nonlinear_remainder_definition():
    # F(x) = f(x) - J(u) x.  The oracle cancels the linear part exactly
    # (R18); check against the literal definition to roundoff.
    n = 32
    pb = O.Problem((n, n), (2 / n, 2 / n), 1e-3, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(n)
    x = u + 0.01 * W.random_vector((n, n), seed=5)
    lit = O.rhs(pb, x) - O.jac_apply(pb, u, x)
    got = O.nonlinear_remainder(pb, u, x)
    scale = np.abs(O.rhs(pb, x)).max()
    assert np.abs(got - lit).max() <= 1e-13 * scale
    # linear problem: F == 0 exactly
    pl = O.Problem((n, n), (2 / n, 2 / n), 1.0, 10.0, 0.0)
    assert np.all(O.nonlinear_remainder(pl, u, x) == 0.0)


def test_allen_cahn_gershgorin_bound_encloses():
    n = 12
    pb = O.Problem((n, n), (2 / n, 2 / n), 1e-2, 0.0, 1.0)
    u = 1.3 * W.ic_allen_cahn_2d(n)
    M = refs.dense_matrix(lambda v: O.jac_apply(pb, u, v.reshape(n, n)), n * n)
    ev = np.linalg.eigvalsh(0.5 * (M + M.T))
    b = O.spectrum_bound(pb, u)
    assert -ev.min() <= b * (1 + 1e-12)
    assert b == pytest.approx(8e-2 / (2 / n) ** 2 + max(0.0, 3 * np.max(u * u) - 1), rel=1e-14)


def test_power_iteration_vs_dense():
    # within 2% of the dominant magnitude after 50 iterations.
    for n in (16, 32):
        pb = O.Problem((n, n), (2 / n, 2 / n), 1.0, 10.0, 0.0)
        est = O.power_iteration(pb, None, 50)
        assert est <= O.spectrum_bound(pb) * (1 + 1e-12)
        assert est >= 0.98 * O.spectrum_bound(pb)
    # diagonal operator (diff = nu = 0): J = diag(1 - 3u^2)
    u = np.linspace(0.1, 2.0, 64).reshape(8, 8)
    pd = O.Problem((8, 8), (0.25, 0.25), 0.0, 0.0, 1.0)
    est = O.power_iteration(pd, u, 200)
    assert est == pytest.approx(np.max(np.abs(1 - 3 * u * u)), rel=1e-3)


def test_l2norm_scaled():
    assert O.l2norm_scaled(np.array([3.0, 4.0])) == pytest.approx(5 / np.sqrt(2), rel=1e-16)
    assert O.l2norm_scaled(np.zeros(7)) == 0.0
    assert O.l2norm_scaled(np.full(1001, -2.5)) == pytest.approx(2.5, rel=1e-15)


# ---------------------------------------------------------------- Problem III: viscous Burgers
def _burgers(n, beta=10.0):
    return O.Problem((n, n), (2 / n, 2 / n), 1.0, 0.0, 0.0, None, beta)


def test_burgers_flux_third_order():
    # (beta/2) sum_d D_d(u^2) -> beta u (u_x + u_y) at third order (P:549 upwind, R10)
    errs = []
    for n in (32, 64, 128):
        x, y = W.grid_2d(n)
        k = 2 * np.pi
        u = 2.0 + 0.3 * np.sin(k * x) * np.cos(k * y)
        ux = 0.3 * k * np.cos(k * x) * np.cos(k * y)
        uy = -0.3 * k * np.sin(k * x) * np.sin(k * y)
        pb = O.Problem((n, n), (2 / n, 2 / n), 0.0, 0.0, 0.0, None, 1.0)
        errs.append(np.abs(O.rhs(pb, u) - u * (ux + uy)).max())
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(orders - 3.0) < 0.2), orders


def test_burgers_jacobian_and_remainder():
    n = 32
    pb = _burgers(n)
    u = W.ic_burgers_2d(n)
    v = W.random_vector((n, n), seed=3)
    eps = 1e-6
    fd = (O.rhs(pb, u + eps * v) - O.rhs(pb, u - eps * v)) / (2 * eps)
    jv = O.jac_apply(pb, u, v)
    assert np.linalg.norm(jv - fd) <= 1e-8 * np.linalg.norm(jv)          # exact J (R13)
    x = u + 0.01 * v
    lit = O.rhs(pb, x) - O.jac_apply(pb, u, x)
    assert np.abs(O.nonlinear_remainder(pb, u, x) - lit).max() <= 1e-13 * np.abs(O.rhs(pb, x)).max()


def test_burgers_bound_encloses_power_iteration():
    for n in (16, 32):
        pb = _burgers(n)
        u = W.ic_burgers_2d(n)
        M = refs.dense_matrix(lambda v: O.jac_apply(pb, u, v.reshape(n, n)), n * n)
        lam = np.abs(np.linalg.eigvals(M)).max()
        assert lam <= O.spectrum_bound(pb, u) * (1 + 1e-12)
        assert O.power_iteration(pb, u, 200) <= O.spectrum_bound(pb, u)
