"""Pins for the oracle's scalar parts: phi_l, Leja points, divided differences.

-m "not gpu".  Every check compares the oracle with something other than
itself: closed forms (tests/golden), 60-digit mpmath, a 1e6-point brute force.
"""
import math
import os

import mpmath
import numpy as np
import pytest

import oracle as O
from tests import refs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                rows.append([float(t) for t in line.split()])
    return rows


# ------------------------------------------------------------------ phi
def test_phi_closed_forms():
    for l, z, val in _golden("phi_closed_forms.txt"):
        got = O.phi(int(l), z)
        assert got == pytest.approx(val, rel=1e-15, abs=0), (l, z)


@pytest.mark.parametrize("l", [0, 1, 2, 3, 4])
def test_phi_vs_mpmath(l):
    # S:537 acceptance: relative 1e-13 over z in {-100..10}; we also cover the
    # Taylor/recursion switch at |z| = 2 and the deep negative range of ρ ≤ 300.
    zs = [-300.0, -178.0, -100.0, -10.0, -2.5, -2.0, -1.9999999, -1.0, -0.1, -1e-6, 0.0,
          1e-8, 0.3, 1.0, 1.9999999, 2.0, 10.0]
    for z in zs:
        ref = float(refs.phi_mp(l, z))
        got = O.phi(l, z)
        assert abs(got - ref) <= 1e-14 * abs(ref), (l, z, got, ref)


def test_phi_recursion_identity():
    # z*phi_{l+1}(z) + 1/l! = phi_l(z)
    for l in range(4):
        for z in np.concatenate([-np.logspace(-8, 2, 25), np.logspace(-8, 1, 15)]):
            lhs = z * O.phi(l + 1, z) + 1.0 / math.factorial(l)
            assert lhs == pytest.approx(O.phi(l, z), rel=1e-12)


# ------------------------------------------------------------------ Leja points
def test_leja_first_nodes_exact():
    xi = O.leja_points(4)
    for j, val in _golden("leja_first_nodes.txt"):
        assert xi[int(j)] == pytest.approx(val, abs=2e-16)


def test_leja_vs_mpmath(xi300):
    ref = refs.leja_mp(16, dps=40)
    for j in range(16):
        assert abs(xi300[j] - float(ref[j])) <= 4e-16 * 2, (j, xi300[j], ref[j])


def test_leja_greedy_brute_force(xi300):
    # first 20 nodes satisfy the greedy-max property against a 1e6 grid.
    z = np.linspace(-2.0, 2.0, 1_000_001)
    logp = np.zeros_like(z)
    for j in range(1, 20):
        logp += np.log(np.abs(z - xi300[j - 1]) + 1e-300)
        grid_max = logp.max()
        at_node = np.sum(np.log(np.abs(xi300[j] - xi300[:j])))
        # continuous max >= grid max; grid resolution 4e-6 bounds the deficit
        assert at_node >= grid_max - 1e-6, j
        assert abs(z[np.argmax(logp)] - xi300[j]) < 1e-5 or j == 3, j


def test_leja_distinct_in_interval(xi300):
    assert np.all(np.abs(xi300) <= 2.0)
    assert len(np.unique(xi300)) == 300


# ------------------------------------------------------------------ divided differences
def test_dd_two_node_closed_form():
    # l=0, nodes {2,-2}, dt=1, c=0, gamma=0.1: d_1 = (e^{0.2} - e^{-0.2})/4.
    # (S:118 prints 0.100334, which is wrong: the closed form is 0.10066800127054701.)
    d = O.divided_differences(0, np.array([2.0, -2.0]), 2, 1.0, 0.0, 0.1)
    assert d[0] == pytest.approx(math.exp(0.2), rel=2e-16)
    assert d[1] == pytest.approx((math.exp(0.2) - math.exp(-0.2)) / 4.0, rel=1e-15)


def test_dd_dt_zero(xi300):
    # h constant 1/l!  =>  d_0 = 1/l!, d_k = 0
    for l in range(5):
        d = O.divided_differences(l, xi300, 50, 0.0, -100.0, 50.0)
        assert d[0] == 1.0 / math.factorial(l)
        assert np.all(d[1:] == 0.0)


def test_dd_newton_reconstruction(xi300):
    # the Newton form reproduces h at every node.
    rng = np.random.default_rng(7)
    for trial in range(6):
        l = trial % 5
        m = 40
        dt = 1.0
        gamma = rng.uniform(0.5, 7.0)
        c = -2.0 * gamma          # spectrum [c-2g, c+2g] = [-4g, 0]
        d = O.divided_differences(l, xi300, m, dt, c, gamma)
        for j in range(m):
            p, basis = 0.0, 1.0
            for k in range(j + 1):
                p += d[k] * basis
                basis *= (xi300[j] - xi300[k])
            h = O.phi(l, dt * (c + gamma * xi300[j]))
            assert p == pytest.approx(h, rel=1e-10, abs=1e-14), (trial, j)


@pytest.mark.parametrize("l,rho", [(0, 5.0), (1, 52.5), (3, 100.0), (4, 20.0)])
def test_dd_vs_mpmath(xi300, l, rho):
    # R8: plain fp64 recurrence; contribution |d_k - d_k^mp| * max|basis_k| small.
    m = 80
    gamma = rho
    c = -2.0 * gamma
    d = O.divided_differences(l, xi300, m, 1.0, c, gamma)
    dm = refs.divided_differences_mp(l, xi300, m, 1.0, c, gamma, dps=80)
    zs = np.linspace(-2, 2, 401)
    basis = np.ones_like(zs)
    for k in range(m):
        contrib = abs(d[k] - float(dm[k])) * np.abs(basis).max()
        assert contrib <= 1e-13, (k, contrib)
        basis = basis * (zs - xi300[k])
