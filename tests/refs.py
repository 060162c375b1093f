"""Independent reference computations used to PIN the oracle (test-only).

Nothing here calls the CUDA path.  Each helper computes a quantity by a route
other than the oracle's own code: arbitrary precision (mpmath), dense linear
algebra (scipy), or Fourier diagonalisation of the circulant stencil operator
(numpy FFT of the operator's impulse response).
"""
from __future__ import annotations

import math

import mpmath
import numpy as np
import scipy.linalg


# ---------------------------------------------------------------- phi functions
def phi_mp(l: int, z, dps: int = 60):
    """phi_l(z) in arbitrary precision from its Taylor series sum_k z^k/(k+l)!."""
    with mpmath.workdps(dps):
        z = mpmath.mpf(z) if not isinstance(z, mpmath.mpc) else z
        if abs(z) < 30:
            s = mpmath.mpf(0)
            term = mpmath.mpf(1) / mpmath.factorial(l)
            k = 0
            while True:
                s += term
                k += 1
                term = term * z / (k + l)
                if abs(term) < mpmath.mpf(10) ** (-dps) * max(abs(s), 1e-300) and k > 5:
                    break
            return s
        # large |z|: recursion in high precision is exact enough
        p = mpmath.exp(z)
        for j in range(l):
            p = (p - mpmath.mpf(1) / mpmath.factorial(j)) / z
        return p


def phi_complex(l: int, z: np.ndarray) -> np.ndarray:
    """phi_l on complex arrays: Taylor (40 terms) for |z| < 1, exp + recursion else."""
    z = np.asarray(z, dtype=np.complex128)
    out = np.empty_like(z)
    small = np.abs(z) < 1.0
    zs = z[small]
    term = np.full(zs.shape, 1.0 / math.factorial(l), dtype=np.complex128)
    s = term.copy()
    for k in range(1, 40):
        term = term * zs / (k + l)
        s = s + term
    out[small] = s
    zb = z[~small]
    p = np.exp(zb)
    for j in range(l):
        p = (p - 1.0 / math.factorial(j)) / zb
    out[~small] = p
    return out


# ---------------------------------------------------------------- Leja points
def leja_mp(count: int, dps: int = 50):
    """Greedy Leja points on [-2, 2] in arbitrary precision, via
    per-gap root finding of d/dz log prod |z - xi_k| with mpmath.findroot."""
    with mpmath.workdps(dps):
        xi = [mpmath.mpf(2), mpmath.mpf(-2)]
        while len(xi) < count:
            srt = sorted(xi)
            best = None
            for a, b in zip(srt[:-1], srt[1:]):
                g = lambda z: mpmath.fsum(1 / (z - x) for x in xi)
                # bisection to a bracket, then secant polish (robust)
                lo, hi = a, b
                for _ in range(dps * 4):
                    mid = (lo + hi) / 2
                    if g(mid) > 0:
                        lo = mid
                    else:
                        hi = mid
                z = (lo + hi) / 2
                L = mpmath.fsum(mpmath.log(abs(z - x)) for x in xi)
                if best is None or L > best[0] + mpmath.mpf(10) ** (-30) or \
                        (abs(L - best[0]) <= mpmath.mpf(10) ** (-30) and z > best[1]):
                    best = (L, z)
            xi.append(best[1])
        return xi


def divided_differences_mp(l, xi, m, dt, c, gamma, a=1.0, dps=80):
    with mpmath.workdps(dps):
        x = [mpmath.mpf(float(v)) for v in xi[:m]]
        d = [phi_mp(l, mpmath.mpf(a) * mpmath.mpf(dt) * (mpmath.mpf(c) + mpmath.mpf(gamma) * xv), dps)
             for xv in x]
        for i in range(1, m):
            for j in range(i, m):
                d[j] = (d[j] - d[i - 1]) / (x[j] - x[i - 1])
        return d


# ---------------------------------------------------------------- operators
def impulse_symbol(apply, shape) -> np.ndarray:
    """Eigenvalues of a circulant operator: FFT of its response to a delta.

    For a periodic constant-coefficient stencil A, A v = ifft(fft(A e_0) * fft(v)),
    so fft(A e_0) is the spectrum on the discrete Fourier grid."""
    e0 = np.zeros(shape)
    e0.flat[0] = 1.0
    return np.fft.fftn(apply(e0).reshape(shape))


def fft_apply_phi(symbol: np.ndarray, v: np.ndarray, dt: float, l: int) -> np.ndarray:
    """phi_l(dt A) v for circulant A with the given symbol (FFT-exact)."""
    vh = np.fft.fftn(v.reshape(symbol.shape))
    return np.real(np.fft.ifftn(phi_complex(l, dt * symbol) * vh))


def dense_matrix(apply, N: int) -> np.ndarray:
    M = np.zeros((N, N))
    for j in range(N):
        e = np.zeros(N)
        e[j] = 1.0
        M[:, j] = apply(e).ravel()
    return M


def dense_phi(M: np.ndarray, v: np.ndarray, dt: float, l: int) -> np.ndarray:
    """phi_l(dt M) v by the augmented-matrix exponential (scipy expm):
    B = [[dt M, v e_1^T], [0, J_l]] with J_l the l x l upper shift;
    phi_l(dt M) v = expm(B)[:N, N + l - 1]  (l >= 1), expm(dt M) v for l = 0."""
    N = M.shape[0]
    if l == 0:
        return scipy.linalg.expm(dt * M) @ v
    B = np.zeros((N + l, N + l))
    B[:N, :N] = dt * M
    B[:N, N] = v
    for i in range(l - 1):
        B[N + i, N + i + 1] = 1.0
    E = scipy.linalg.expm(B)
    return E[:N, N + l - 1]


# ---------------------------------------------------------------- spectral Leja
def spectral_leja_iters(symbol, v, dt, c, gamma, l, rtol, atol, xi, d=None, max_nodes=300):
    """Simulate the Leja recurrence (Eq. (2)) mode-by-mode in Fourier space.

    y_m(theta) = y_{m-1}(theta) * ((lambda(theta) - c)/gamma - xi_{m-1}); norms by
    Parseval.  Returns the iteration count of the stopping rule of P:155."""
    vh = np.fft.fftn(v.reshape(symbol.shape)).ravel()
    lam = symbol.ravel()
    N = vh.size
    if d is None:
        d = [float(x) for x in divided_differences_mp(l, xi, max_nodes, dt, c, gamma, dps=60)]
    yh = vh.copy()
    ph = d[0] * vh
    for m in range(1, max_nodes):
        yh = yh * ((lam - c) / gamma - xi[m - 1])
        ph = ph + d[m] * yh
        ny = np.sqrt(np.sum(np.abs(yh) ** 2) / N) / math.sqrt(N)
        npn = np.sqrt(np.sum(np.abs(ph) ** 2) / N) / math.sqrt(N)
        if abs(d[m]) * ny <= rtol * npn + atol:
            return m, np.real(np.fft.ifftn(ph.reshape(symbol.shape)))
    return None, None
