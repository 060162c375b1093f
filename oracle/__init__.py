"""CPU oracle for the LeXInt hot path (arxiv 2310.08344) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product package
``paper_2310_08344_b200`` never imports it and shares no code with it.

The arithmetic lives in ``lxoracle.c`` (plain fp64 C loops, each function
citing the paper passage it follows); this module only marshals numpy arrays
through ctypes.  ``ensure_built()`` compiles the C file with gcc if the shared
object is missing or stale (``__graft_entry__.build()`` calls it as well).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lxoracle.c")
_LIB = os.path.join(_HERE, "liblxoracle.so")
_LIB_OMP = os.path.join(_HERE, "liblxoracle_omp.so")   # same source with -fopenmp (bench cpu_baseline only)

OK, ERR_ARG, ERR_UNSUPPORTED, ERR_NOCONV, ERR_NONFINITE = 0, 1, 4, 5, 6
METHODS = {"rosenbrock_euler": 0, "exprb32": 1, "exprb43": 2, "epirk4s3a": 3, "exprb42": 4, "epirk5p1": 5, "exprb53s3": 6,
           "exprb54s4": 7, "epirk4s3b": 8, "epirk4s3": 9}
JAC = {"exact": 0, "fd": 1, "linear_f": 2}     # lxoracle.c OC_JAC_* (black-box RHS modes, reading R25)


def ensure_built(force: bool = False) -> str:
    """Compile lxoracle.c -> liblxoracle.so (plain -O2, no FMA contraction) and the OpenMP build
    liblxoracle_omp.so (same source and flags + -fopenmp; bit-identical results)."""
    for lib_path, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(lib_path) or os.path.getmtime(lib_path) < os.path.getmtime(_SRC):
            tmp = lib_path + ".tmp%d" % os.getpid()
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared"] + extra +
                                  ["-o", tmp, _SRC, "-lm"])
            os.replace(tmp, lib_path)
    return _LIB


_lib = None
_use_omp = False


def use_openmp(on: bool = True):
    """Switch this process to the OpenMP build (bench.py's all-core cpu_baseline / reference arm);
    results are bit-identical to the serial build."""
    global _lib, _use_omp
    if on != _use_omp:
        _use_omp = on
        _lib = None


def lib():
    global _lib
    if _lib is None:
        ensure_built()
        L = ctypes.CDLL(_LIB_OMP if _use_omp else _LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oc_l2norm_scaled.restype = ctypes.c_double
        L.oc_l2norm_scaled.argtypes = [dp, ctypes.c_long]
        L.oc_phi.restype = ctypes.c_double
        L.oc_phi.argtypes = [ctypes.c_int, ctypes.c_double]
        L.oc_leja_points.restype = ctypes.c_int
        L.oc_leja_points.argtypes = [ctypes.c_int, dp]
        L.oc_divided_differences.restype = ctypes.c_int
        L.oc_divided_differences.argtypes = [ctypes.c_int, dp, ctypes.c_int, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double, dp]
        pp = ctypes.POINTER(OcProblem)
        L.oc_rhs.argtypes = [pp, dp, dp]
        L.oc_jac_apply.argtypes = [pp, dp, dp, dp]
        L.oc_nonlinear_remainder.argtypes = [pp, dp, dp, dp]
        L.oc_jac_apply_slab.argtypes = [pp, ctypes.c_long, dp, dp, dp]
        L.oc_spectrum_bound.restype = ctypes.c_double
        L.oc_spectrum_bound.argtypes = [pp, dp]
        L.oc_power_iteration.restype = ctypes.c_double
        L.oc_power_iteration.argtypes = [pp, dp, ctypes.c_int]
        L.oc_real_leja_phi.restype = ctypes.c_int
        L.oc_real_leja_phi.argtypes = [pp, dp, dp, ctypes.POINTER(dp), dp, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_double, dp, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int), dp]
        L.oc_real_leja_phi_ex.restype = ctypes.c_int
        L.oc_real_leja_phi_ex.argtypes = [pp, ctypes.c_int, dp, dp, dp, ctypes.POINTER(dp), dp, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_double, dp, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_int), dp]
        L.oc_jac_apply_fd.argtypes = [pp, dp, dp, dp, dp]
        L.oc_nonlinear_remainder_fd.argtypes = [pp, dp, dp, dp, dp]
        L.oc_step_ex.restype = ctypes.c_int
        L.oc_step_ex.argtypes = [pp, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, dp,
                                 ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.oc_integrate_adaptive.restype = ctypes.c_int
        L.oc_integrate_adaptive.argtypes = [pp, ctypes.c_int, dp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_double, dp, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), dp, dp,
                                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.oc_step.restype = ctypes.c_int
        L.oc_step.argtypes = [pp, ctypes.c_int, dp, dp, dp, dp, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, ctypes.c_double, ctypes.c_double, dp, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_int)]
        _lib = L
    return _lib


class OcProblem(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int), ("n", ctypes.c_long * 3), ("dx", ctypes.c_double * 3),
                ("diff", ctypes.c_double), ("nu", ctypes.c_double), ("react", ctypes.c_double),
                ("flux", ctypes.c_double), ("source", ctypes.POINTER(ctypes.c_double))]


@dataclass(frozen=True, eq=False)
class Problem:
    """f(u) = diff*lap(u) + nu*sum_d D_d u + react*(u - u^3) [+ source] on a periodic grid."""
    shape: tuple
    dx: tuple
    diff: float = 1.0
    nu: float = 0.0
    react: float = 0.0
    source: np.ndarray | None = None
    flux: float = 0.0

    def c_struct(self) -> OcProblem:
        nd = len(self.shape)
        n = list(self.shape) + [1] * (3 - nd)
        dx = list(self.dx) + [1.0] * (3 - nd)
        src = None
        if self.source is not None:
            src = np.ascontiguousarray(self.source, dtype=np.float64)
            assert src.size == self.npoints
            object.__setattr__(self, "_src_keep", src)
        return OcProblem(nd, (ctypes.c_long * 3)(*n), (ctypes.c_double * 3)(*dx),
                         float(self.diff), float(self.nu), float(self.react), float(self.flux), _dp(src))

    @property
    def npoints(self) -> int:
        return int(np.prod(self.shape))


def _dp(a):
    if a is None:
        return ctypes.cast(None, ctypes.POINTER(ctypes.c_double))
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _vec(a, pb: Problem | None = None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if pb is not None:
        assert a.size == pb.npoints, (a.shape, pb.shape)
    return a


def l2norm_scaled(x) -> float:
    x = _vec(x)
    return lib().oc_l2norm_scaled(_dp(x), x.size)


def phi(l: int, z: float) -> float:
    return lib().oc_phi(int(l), float(z))


def leja_points(count: int) -> np.ndarray:
    xi = np.zeros(count)
    s = lib().oc_leja_points(int(count), _dp(xi))
    if s:
        raise ValueError("oc_leja_points status %d" % s)
    return xi


def divided_differences(l, xi, m, dt, c, gamma, a=1.0) -> np.ndarray:
    xi = _vec(xi)
    d = np.zeros(m)
    s = lib().oc_divided_differences(int(l), _dp(xi), int(m), float(dt), float(c), float(gamma),
                                     float(a), _dp(d))
    if s:
        raise ValueError("oc_divided_differences status %d" % s)
    return d


def rhs(pb: Problem, u) -> np.ndarray:
    u = _vec(u, pb)
    f = np.zeros_like(u)
    lib().oc_rhs(ctypes.byref(pb.c_struct()), _dp(u), _dp(f))
    return f


def jac_apply(pb: Problem, u, y) -> np.ndarray:
    y = _vec(y, pb)
    u = None if u is None else _vec(u, pb)
    w = np.zeros_like(y)
    lib().oc_jac_apply(ctypes.byref(pb.c_struct()), _dp(u), _dp(y), _dp(w))
    return w


def jac_apply_slab(pb: Problem, n_loc: int, u_loc, y_ghosted) -> np.ndarray:
    """J(u) y on a slab: y_ghosted has rows -1..n_loc+1 (1 ghost before, 2 after)."""
    row = int(np.prod(pb.shape[1:]))
    y = np.ascontiguousarray(y_ghosted, dtype=np.float64)
    assert y.size == (n_loc + 3) * row
    u = None if u_loc is None else np.ascontiguousarray(u_loc, dtype=np.float64)
    w = np.zeros(n_loc * row)
    lib().oc_jac_apply_slab(ctypes.byref(pb.c_struct()), int(n_loc), _dp(u), _dp(y), _dp(w))
    return w.reshape((n_loc,) + tuple(pb.shape[1:]))


def jac_apply_fd(pb: Problem, u, y, f_u=None) -> np.ndarray:
    """J(u) y by forward differences of f (reading R25)."""
    y = _vec(y, pb)
    u = _vec(u, pb)
    f_u = rhs(pb, u) if f_u is None else _vec(f_u, pb)
    w = np.zeros_like(y)
    lib().oc_jac_apply_fd(ctypes.byref(pb.c_struct()), _dp(u), _dp(f_u), _dp(y), _dp(w))
    return w


def nonlinear_remainder_fd(pb: Problem, u, x, f_u=None) -> np.ndarray:
    """F(x) = f(x) - J_FD(u) x, literally (alg:exprb32 Nonlinear_remainder)."""
    x = _vec(x, pb)
    u = _vec(u, pb)
    f_u = rhs(pb, u) if f_u is None else _vec(f_u, pb)
    out = np.zeros_like(x)
    lib().oc_nonlinear_remainder_fd(ctypes.byref(pb.c_struct()), _dp(u), _dp(f_u), _dp(x), _dp(out))
    return out


def nonlinear_remainder(pb: Problem, u, x) -> np.ndarray:
    x = _vec(x, pb)
    u = _vec(u, pb)
    out = np.zeros_like(x)
    lib().oc_nonlinear_remainder(ctypes.byref(pb.c_struct()), _dp(u), _dp(x), _dp(out))
    return out


def spectrum_bound(pb: Problem, u=None) -> float:
    u = None if u is None else _vec(u, pb)
    return lib().oc_spectrum_bound(ctypes.byref(pb.c_struct()), _dp(u))


def shift_scale(bound: float):
    """Listing alg:lexint: eig = -1.05*|lambda|; c = eig/2; Gamma = -eig/4."""
    eig = -1.05 * bound
    return eig / 2.0, -eig / 4.0


def power_iteration(pb: Problem, u=None, iters: int = 50) -> float:
    u = None if u is None else _vec(u, pb)
    return lib().oc_power_iteration(ctypes.byref(pb.c_struct()), _dp(u), int(iters))


@dataclass
class LejaResult:
    outs: list
    iters: int
    status: int
    margins: tuple


def real_leja_phi(pb: Problem, v, dt, c, gamma, l, rtol, atol, xi, *, u_lin=None,
                  coeffs: Sequence[float] = (1.0,), max_nodes: int | None = None,
                  jac: str = "exact") -> LejaResult:
    """jac: "exact" (J(u_lin) exact), "fd" (J(u_lin) by differences of f),
    "linear_f" (the operator is f itself: a linear black-box RHS)."""
    v = _vec(v, pb)
    u_lin = None if u_lin is None else _vec(u_lin, pb)
    xi = _vec(xi)
    max_nodes = len(xi) if max_nodes is None else max_nodes
    K = len(coeffs)
    outs = [np.zeros_like(v) for _ in range(K)]
    optr = (ctypes.POINTER(ctypes.c_double) * K)(*[_dp(o) for o in outs])
    cf = np.asarray(coeffs, dtype=np.float64)
    it = ctypes.c_int(0)
    mg = np.zeros(2)
    s = lib().oc_real_leja_phi_ex(ctypes.byref(pb.c_struct()), JAC[jac], _dp(u_lin), _dp(None), _dp(v), optr,
                                  _dp(cf), K, float(dt), float(c), float(gamma), int(l), float(rtol),
                                  float(atol), _dp(xi), int(max_nodes), ctypes.byref(it), _dp(mg))
    return LejaResult(outs, it.value, s, (float(mg[0]), float(mg[1])))


@dataclass
class StepResult:
    u_low: np.ndarray
    u_high: np.ndarray
    err: float
    iters: int
    status: int


def step(pb: Problem, method: str, u, dt, c, gamma, rtol, atol, xi, max_nodes=None,
         jac: str = "exact") -> StepResult:
    """jac: "exact" (exact J, analytic remainders R18) or "fd" (black-box f: J and the
    remainders F(x) = f(x) - J(u)x by finite differences)."""
    u = _vec(u, pb)
    xi = _vec(xi)
    max_nodes = len(xi) if max_nodes is None else max_nodes
    lo, hi = np.zeros_like(u), np.zeros_like(u)
    err = np.zeros(1)
    it = ctypes.c_int(0)
    s = lib().oc_step_ex(ctypes.byref(pb.c_struct()), JAC[jac], METHODS[method], _dp(u), _dp(lo), _dp(hi), _dp(err),
                      float(dt), float(c), float(gamma), float(rtol), float(atol), _dp(xi),
                      int(max_nodes), ctypes.byref(it))
    return StepResult(lo, hi, float(err[0]), it.value, s)


@dataclass
class AdaptiveResult:
    u: np.ndarray
    accepted: int
    rejected: int
    dts: np.ndarray        # every attempted step size, in order
    errs: np.ndarray       # its embedded error estimate
    acc: np.ndarray        # accepted?
    iters: int
    status: int


def integrate_adaptive(pb: Problem, method: str, u0, t_end, dt0, tol, rtol, atol, xi, max_nodes=None,
                       max_steps: int = 1000) -> AdaptiveResult:
    """Embedded-error step-size control (reading R32): see oc_integrate_adaptive."""
    u = _vec(u0, pb).copy()
    xi = _vec(xi)
    max_nodes = len(xi) if max_nodes is None else max_nodes
    dts, errs = np.zeros(max_steps), np.zeros(max_steps)
    acc = np.zeros(max_steps, dtype=np.int32)
    na, nr, it = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    s = lib().oc_integrate_adaptive(ctypes.byref(pb.c_struct()), METHODS[method], _dp(u), float(t_end), float(dt0),
                                    float(tol), float(rtol), float(atol), _dp(xi), int(max_nodes), int(max_steps),
                                    ctypes.byref(na), ctypes.byref(nr), _dp(dts), _dp(errs),
                                    acc.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), ctypes.byref(it))
    k = na.value + nr.value
    return AdaptiveResult(u, na.value, nr.value, dts[:k], errs[:k], acc[:k].astype(bool), it.value, s)
