"""Seeded synthetic inputs shaped like the paper's workloads (shared by the
oracle tests and the CUDA path; holds none of the method's arithmetic).

Everything here is *input*: grid coordinates, initial conditions, sources,
step sizes and the per-config parameter sets.  Neither the oracle nor the
product imports the other; both may import this module.

Grid convention: periodic [-1, 1)^d, x_i = -1 + i*dx,
dx = 2/n, row-major, dimension 0 slowest.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = 20231012


def coords(n: int) -> np.ndarray:
    dx = 2.0 / n
    return -1.0 + dx * np.arange(n, dtype=np.float64)


def grid_2d(n0: int, n1: int | None = None):
    n1 = n0 if n1 is None else n1
    return np.meshgrid(coords(n0), coords(n1), indexing="ij")


def ic_problem1_2d(n0: int, n1: int | None = None) -> np.ndarray:
    """Problem I/II initial condition: 1 + exp(-((x+.5)^2+(y+.5)^2)/0.01)."""
    x, y = grid_2d(n0, n1)
    return np.ascontiguousarray(1.0 + np.exp(-((x + 0.5) ** 2 + (y + 0.5) ** 2) / 0.01))


def source_problem2_2d(n0: int, n1: int | None = None) -> np.ndarray:
    """Problem II source S(x, y)."""
    x, y = grid_2d(n0, n1)
    return np.ascontiguousarray(np.exp(-((x + 0.4) ** 2 + (y - 0.6) ** 2) / 0.05)
                                + np.exp(-((x - 0.25) ** 2 + (y + 0.1) ** 2) / 0.04))


def ic_burgers_2d(n0: int, n1: int | None = None) -> np.ndarray:
    """Problem III initial condition."""
    x, y = grid_2d(n0, n1)
    return np.ascontiguousarray(2.0 + 1e-2 * (np.sin(2 * np.pi * x) + np.sin(2 * np.pi * y)
                                              + np.sin(8 * np.pi * x + 0.3) + np.sin(8 * np.pi * y + 0.3)))


def ic_allen_cahn_2d(n0: int, n1: int | None = None) -> np.ndarray:
    """Allen-Cahn initial condition (DESIGN reading R16; the P:593 shape, zero mean)."""
    x, y = grid_2d(n0, n1)
    return np.ascontiguousarray(0.5 * (np.sin(2 * np.pi * x) + np.sin(2 * np.pi * y)
                                       + np.sin(8 * np.pi * x + 0.3) + np.sin(8 * np.pi * y + 0.3)))


def ic_gaussian_3d(n: int) -> np.ndarray:
    """3D analogue of the Problem I initial condition (config 5)."""
    c = coords(n)
    x, y, z = np.meshgrid(c, c, c, indexing="ij")
    return np.ascontiguousarray(1.0 + np.exp(-((x + 0.5) ** 2 + (y + 0.5) ** 2 + (z + 0.5) ** 2) / 0.01))


def ic_random(shape, seed: int = SEED, amp: float = 0.1) -> np.ndarray:
    """Broadband robustness input: 1 + amp*U(-1, 1) i.i.d. per point (seeded PCG64)."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(1.0 + amp * rng.uniform(-1.0, 1.0, size=shape))


def random_vector(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(scale * rng.standard_normal(size=shape))


def dt_cfl(n: int, nu: float, ndim: int = 2) -> float:
    """Delta t_CFL (undefined in the paper, R11): min(dx/|nu|, dx^2/(2 ndim))."""
    dx = 2.0 / n
    diffusive = dx * dx / (2.0 * ndim)
    return min(dx / abs(nu), diffusive) if nu else diffusive


@dataclass(frozen=True)
class Workload:
    """Problem parameters of one BASELINE.json config (inputs, not arithmetic)."""
    name: str
    shape: tuple
    diff: float = 1.0
    nu: float = 10.0
    react: float = 0.0
    dt: float = 0.0
    rtol: float = 1e-10
    atol: float = 1e-10
    extra: dict = field(default_factory=dict)

    @property
    def dx(self) -> tuple:
        return tuple(2.0 / n for n in self.shape)

    @property
    def npoints(self) -> int:
        return int(np.prod(self.shape))


def config(idx: int, n: int | None = None, dt_mult: float = 10.0) -> Workload:
    """BASELINE.json configs (0-based index), optionally at a reduced size n."""
    if idx == 0:   # 64^2 advection-diffusion, one Rosenbrock-Euler step
        n = 64 if n is None else n
        return Workload("advdiff2d_rosenbrock_euler", (n, n), 1.0, 10.0, 0.0, dt_mult * dt_cfl(n, 10.0),
                        extra={"method": "rosenbrock_euler"})
    if idx == 1:   # 4096^2 advection-diffusion, phi_0..phi_3 via real Leja
        n = 4096 if n is None else n
        return Workload("advdiff2d_phi0-3", (n, n), 1.0, 10.0, 0.0, dt_mult * dt_cfl(n, 10.0),
                        extra={"ls": (0, 1, 2, 3)})
    if idx == 2:   # 2048^2 Allen-Cahn, EXPRB43, 100 steps (R16)
        n = 2048 if n is None else n
        return Workload("allen_cahn2d_exprb43", (n, n), 1e-4, 0.0, 1.0, 0.01,
                        extra={"method": "exprb43", "steps": 100})
    if idx == 3:   # 16384^2 advection-diffusion, slab-sharded
        n = 16384 if n is None else n
        return Workload("advdiff2d_phi0_slab", (n, n), 1.0, 10.0, 0.0, dt_mult * dt_cfl(n, 10.0),
                        extra={"ls": (0,)})
    if idx == 4:   # 512^3 advection-diffusion, EPIRK4s3A
        n = 512 if n is None else n
        return Workload("advdiff3d_epirk4s3a", (n, n, n), 1.0, 10.0, 0.0, dt_mult * dt_cfl(n, 10.0, 3),
                        extra={"method": "epirk4s3a"})
    raise ValueError(idx)
