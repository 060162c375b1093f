"""B200-native LeXInt hot path (arxiv 2310.08344): Python binding of the C ABI.

Argument marshalling only -- every step of the path runs in
``liblexint_b200.so`` (sm_100a CUDA kernels + C++ host runtime, declared in
``include/lexint.h``).  PyTorch is used for device memory, streams and
``torch.distributed`` plumbing.  There is no CPU fallback: if the shared
library is missing or cannot be loaded this package raises at import/use.

Names follow the C ABI: ``lx_leja_points``, ``lx_divided_differences``,
``lx_spectrum_estimate``, ``lx_spectrum_bound``, ``lx_real_leja_phi``,
``lx_real_leja_phi_vertical``, ``lx_step_<integrator>`` ...
Vectors may be CUDA tensors (device pointers, zero copy) or numpy arrays /
CPU tensors (host pointers: the library stages them through device buffers).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# LX_LIBRARY: load another build of the same library (A/B performance experiments only)
LIB_PATH = os.environ.get("LX_LIBRARY") or os.path.join(_PKG, "liblexint_b200.so")

LX_OK, LX_ERR_ARG, LX_ERR_DIM, LX_ERR_ALIAS, LX_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
LX_ERR_NOCONV, LX_ERR_NONFINITE, LX_ERR_UNKNOWN_INTEGRATOR, LX_ERR_CUDA, LX_ERR_NCCL = 5, 6, 7, 8, 9
LX_ERR_TIMEOUT = 10
LX_COMM_FORCE, LX_COMM_NO_PEER = 1, 2
STATUS_NAMES = {0: "LX_OK", 1: "LX_ERR_ARG", 2: "LX_ERR_DIM", 3: "LX_ERR_ALIAS", 4: "LX_ERR_UNSUPPORTED",
                5: "LX_ERR_NOCONV", 6: "LX_ERR_NONFINITE", 7: "LX_ERR_UNKNOWN_INTEGRATOR", 8: "LX_ERR_CUDA",
                9: "LX_ERR_NCCL", 10: "LX_ERR_TIMEOUT"}
(LX_ROSENBROCK_EULER, LX_EXPRB32, LX_EXPRB43, LX_EPIRK4S3A, LX_EXPRB42, LX_EPIRK5P1, LX_EXPRB53S3, LX_EXPRB54S4,
 LX_EPIRK4S3B, LX_EPIRK4S3) = range(10)
METHODS = {"rosenbrock_euler": 0, "exprb32": 1, "exprb43": 2, "epirk4s3a": 3, "exprb42": 4, "epirk5p1": 5,
           "exprb53s3": 6, "exprb54s4": 7, "epirk4s3b": 8, "epirk4s3": 9}

# Every symbol include/lexint.h declares (checked by tests/test_abi.py).
EXPORTS = ("lx_last_error", "lx_version", "lx_leja_points", "lx_phi_scalar", "lx_divided_differences",
           "lx_slab_range", "lx_ctx_create", "lx_ctx_destroy", "lx_nccl_unique_id", "lx_ctx_set_comm",
           "lx_ctx_local", "lx_ctx_synchronize", "lx_ctx_launch_count", "lx_ctx_iterations_per_pass", "lx_spectrum_estimate",
           "lx_spectrum_bound", "lx_shift_scale", "lx_real_leja_phi", "lx_real_leja_phi_vertical",
           "lx_step_rosenbrock_euler", "lx_step_exprb32", "lx_step_exprb43", "lx_step_epirk4s3a",
           "lx_step_exprb42", "lx_step_epirk5p1",
           "lx_step", "lx_rhs", "lx_integrate", "lx_local_group_create", "lx_local_group_destroy", "lx_ctx_set_comm_local",
           "lx_real_leja_phi_cb", "lx_step_cb", "lx_builtin_rhs", "lx_ctx_set_comm_ex", "lx_ctx_set_comm_local_ex",
           "lx_ctx_ipc_handle", "lx_ctx_set_comm_ipc", "lx_ctx_set_kernel", "lx_slab_halo_plan", "lx_integrate_adaptive",
           "lx_real_leja_phi_multi")

# void f(const double* in, double* out, void* user, void* cuda_stream)  (include/lexint.h lx_rhs_fn)
RHS_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class LxError(RuntimeError):
    def __init__(self, status: int, msg: str, iters: int | None = None):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status
        self.iters = iters


class LxProblem(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int), ("n", ctypes.c_int64 * 3), ("dx", ctypes.c_double * 3),
                ("diff", ctypes.c_double), ("nu", ctypes.c_double), ("react", ctypes.c_double),
                ("flux", ctypes.c_double), ("source", ctypes.c_void_p)]


@dataclass(frozen=True, eq=False)
class Problem:
    """du/dt = diff*lap(u) + nu*sum_d D_d u + (flux/2) sum_d D_d(u^2) + react*(u - u^3) [+ source]
    on a periodic GLOBAL grid (flux: viscous Burgers, Problem III).
    source: optional time-independent S (Problem II), the caller's local slab (tensor or ndarray)."""
    shape: tuple
    dx: tuple
    diff: float = 1.0
    nu: float = 0.0
    react: float = 0.0
    source: object = None
    flux: float = 0.0

    def c_struct(self) -> LxProblem:
        nd = len(self.shape)
        n = list(self.shape) + [1] * (3 - nd)
        dx = list(self.dx) + [1.0] * (3 - nd)
        return LxProblem(nd, (ctypes.c_int64 * 3)(*n), (ctypes.c_double * 3)(*dx), float(self.diff),
                         float(self.nu), float(self.react), float(self.flux), _ptr(self.source))

    @property
    def npoints(self) -> int:
        return int(np.prod(self.shape))


_lib = None


def lib() -> ctypes.CDLL:
    """Load liblexint_b200.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("liblexint_b200.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, dp, ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
        pbp = ctypes.POINTER(LxProblem)
        i64p = ctypes.POINTER(ctypes.c_int64)
        d = ctypes.c_double
        sig = {
            "lx_last_error": (ctypes.c_char_p, []),
            "lx_version": (ctypes.c_char_p, []),
            "lx_leja_points": (ctypes.c_int, [ctypes.c_int, dp]),
            "lx_phi_scalar": (ctypes.c_int, [ctypes.c_int, d, dp]),
            "lx_divided_differences": (ctypes.c_int, [ctypes.c_int, dp, ctypes.c_int, d, d, d, d, dp]),
            "lx_slab_range": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, i64p, i64p]),
            "lx_ctx_create": (ctypes.c_int, [pbp, ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(vp)]),
            "lx_ctx_destroy": (ctypes.c_int, [vp]),
            "lx_nccl_unique_id": (ctypes.c_int, [vp]),
            "lx_ctx_set_comm": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int]),
            "lx_ctx_local": (ctypes.c_int, [vp, i64p, i64p, i64p]),
            "lx_ctx_synchronize": (ctypes.c_int, [vp, ip, dp]),
            "lx_ctx_launch_count": (ctypes.c_int64, [vp]),
            "lx_ctx_iterations_per_pass": (ctypes.c_int, [vp]),
            "lx_spectrum_estimate": (ctypes.c_int, [vp, pbp, vp, ctypes.c_int, dp]),
            "lx_spectrum_bound": (ctypes.c_int, [vp, pbp, vp, dp]),
            "lx_shift_scale": (ctypes.c_int, [d, dp, dp]),
            "lx_real_leja_phi": (ctypes.c_int, [vp, pbp, vp, vp, vp, d, d, d, ctypes.c_int, d, d, ip]),
            "lx_real_leja_phi_vertical": (ctypes.c_int, [vp, pbp, vp, vp, ctypes.POINTER(vp), dp, ctypes.c_int,
                                                         d, d, d, ctypes.c_int, d, d, ip]),
            "lx_real_leja_phi_multi": (ctypes.c_int, [vp, pbp, vp, vp, ctypes.POINTER(vp), ip, dp, ctypes.c_int,
                                                      d, d, d, d, d, ip]),
            "lx_step": (ctypes.c_int, [vp, ctypes.c_int, pbp, vp, vp, vp, dp, d, d, d, d, d, ip]),
            "lx_step_rosenbrock_euler": (ctypes.c_int, [vp, pbp, vp, vp, d, d, d, d, d, ip]),
            "lx_step_exprb32": (ctypes.c_int, [vp, pbp, vp, vp, vp, dp, d, d, d, d, d, ip]),
            "lx_step_exprb43": (ctypes.c_int, [vp, pbp, vp, vp, vp, dp, d, d, d, d, d, ip]),
            "lx_step_epirk4s3a": (ctypes.c_int, [vp, pbp, vp, vp, vp, dp, d, d, d, d, d, ip]),
            "lx_step_exprb42": (ctypes.c_int, [vp, pbp, vp, vp, d, d, d, d, d, ip]),
            "lx_step_epirk5p1": (ctypes.c_int, [vp, pbp, vp, vp, d, d, d, d, d, ip]),
            "lx_rhs": (ctypes.c_int, [vp, pbp, vp, d, vp]),
            "lx_integrate": (ctypes.c_int, [vp, ctypes.c_int, pbp, vp, d, ctypes.c_int, d, d, ip, dp]),
            "lx_local_group_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(vp)]),
            "lx_local_group_destroy": (ctypes.c_int, [vp]),
            "lx_ctx_set_comm_local": (ctypes.c_int, [vp, vp, ctypes.c_int]),
            "lx_ctx_set_comm_ex": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
            "lx_ctx_set_comm_local_ex": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int]),
            "lx_ctx_ipc_handle": (ctypes.c_int, [vp, vp]),
            "lx_ctx_set_comm_ipc": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp]),
            "lx_ctx_set_kernel": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int]),
            "lx_integrate_adaptive": (ctypes.c_int, [vp, ctypes.c_int, pbp, vp, d, d, d, d, d, ctypes.c_int, ip, ip,
                                                     dp, dp, ip]),
            "lx_slab_halo_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                                 ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
            "lx_real_leja_phi_cb": (ctypes.c_int, [vp, vp, vp, vp, vp, ctypes.POINTER(vp), dp, ctypes.c_int,
                                                   d, d, d, ctypes.c_int, d, d, ip]),
            "lx_step_cb": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, vp, vp, vp, dp, d, d, d, d, d, ip]),
            "lx_builtin_rhs": (None, [vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, iters: int | None = None):
    if status != LX_OK:
        raise LxError(status, lib().lx_last_error().decode(), iters)


def _ptr(x):
    """Raw pointer of a torch tensor (device or host) or numpy array (host)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.dtype == np.float64 and x.flags.c_contiguous, "float64 C-contiguous arrays only"
        return x.ctypes.data
    # torch.Tensor
    assert x.dtype.is_floating_point and x.element_size() == 8 and x.is_contiguous(), "fp64 contiguous tensors only"
    return x.data_ptr()


# ------------------------------------------------------------------ host math
def lx_leja_points(count: int) -> np.ndarray:
    xi = np.zeros(count)
    _check(lib().lx_leja_points(count, xi.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return xi


def lx_phi_scalar(l: int, z: float) -> float:
    out = ctypes.c_double()
    _check(lib().lx_phi_scalar(int(l), float(z), ctypes.byref(out)))
    return out.value


def lx_divided_differences(l, xi, m, dt, c, gamma, a=1.0) -> np.ndarray:
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    d = np.zeros(m)
    dp = ctypes.POINTER(ctypes.c_double)
    _check(lib().lx_divided_differences(int(l), xi.ctypes.data_as(dp), int(m), float(dt), float(c), float(gamma),
                                        float(a), d.ctypes.data_as(dp)))
    return d


def lx_slab_halo_plan(rank: int, nranks: int, n_loc: int, mode: int) -> list:
    """The library's halo exchange plan (lexint.h): [(kind, peer, first_row, nrows, ghost_slot)]."""
    ops = (ctypes.c_int * 40)()
    n = lib().lx_slab_halo_plan(int(rank), int(nranks), int(n_loc), int(mode), ops, 8)
    if n < 0:
        raise LxError(LX_ERR_ARG, "lx_slab_halo_plan: bad arguments")
    return [("send" if ops[5 * i] == 0 else "recv",) + tuple(ops[5 * i + 1:5 * i + 5]) for i in range(n)]


def lx_slab_range(n0: int, rank: int, nranks: int):
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().lx_slab_range(int(n0), int(rank), int(nranks), ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def lx_shift_scale(lambda_abs: float):
    c, g = ctypes.c_double(), ctypes.c_double()
    _check(lib().lx_shift_scale(float(lambda_abs), ctypes.byref(c), ctypes.byref(g)))
    return c.value, g.value


def lx_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().lx_nccl_unique_id(buf))
    return buf.raw


# ------------------------------------------------------------------ context
class LocalGroup:
    """Virtual ranks of one process on one GPU (lx_local_group): same slab protocol as NCCL."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        _check(lib().lx_local_group_create(int(nranks), ctypes.byref(h)))
        self.handle = h
        self.nranks = nranks

    def close(self):
        if self.handle:
            lib().lx_local_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """Owns an lx_ctx (scratch allocated once)."""

    def __init__(self, problem: Problem, max_nodes: int = 300, device: int = -1, stream=None):
        """stream: torch.cuda.Stream / raw cudaStream_t handle; default = torch's current
        stream (so library work is ordered with the caller's torch ops)."""
        self.problem = problem
        self._pb = problem.c_struct()
        h = ctypes.c_void_p()
        sp = None
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    # the current stream OF THE CONTEXT'S DEVICE (not of whatever device is current)
                    stream = torch.cuda.current_stream(device if device >= 0 else None)
            except ImportError:
                pass
        if stream is not None:
            dev = getattr(stream, "device", None)
            if device >= 0 and dev is not None and getattr(dev, "index", device) not in (None, device):
                raise LxError(LX_ERR_ARG, "stream belongs to device %s, context to device %d" % (dev, device))
            sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
            if sp == 0:
                sp = 1   # the legacy default stream (cudaStreamLegacy); NULL would mean "own stream"
        _check(lib().lx_ctx_create(ctypes.byref(self._pb), int(max_nodes), int(device), sp, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib().lx_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_comm(self, uid: bytes, rank: int, nranks: int, flags: int = 0):
        """flags: LX_COMM_FORCE (communicator even for one rank), LX_COMM_NO_PEER (no peer-memory kernel)."""
        buf = ctypes.create_string_buffer(uid, 128)
        _check(lib().lx_ctx_set_comm_ex(self.handle, buf, int(rank), int(nranks), int(flags)))

    def set_comm_local(self, group: "LocalGroup", rank: int, flags: int = 0):
        self._group = group   # keep the group alive while the context uses it
        _check(lib().lx_ctx_set_comm_local_ex(self.handle, group.handle, int(rank), int(flags)))

    def ipc_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this context's peer-memory exchange block (lx_ctx_ipc_handle)."""
        buf = ctypes.create_string_buffer(64)
        _check(lib().lx_ctx_ipc_handle(self.handle, buf))
        return buf.raw

    def set_comm_ipc(self, rank: int, handles: list):
        """Peer-memory communicator from every rank's ipc_handle() (rank order)."""
        buf = ctypes.create_string_buffer(b"".join(handles), 64 * len(handles))
        _check(lib().lx_ctx_set_comm_ipc(self.handle, int(rank), len(handles), buf))

    def set_kernel(self, iterations_per_pass: int = 0, kernel3d: int = 0):
        """lx_ctx_set_kernel: 2D Leja iterations per HBM pass (0 auto, 1, 2); 3D kernel (0 auto, 1 warp tiles)."""
        _check(lib().lx_ctx_set_kernel(self.handle, int(iterations_per_pass), int(kernel3d)))

    def local(self):
        b, e, n = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().lx_ctx_local(self.handle, ctypes.byref(b), ctypes.byref(e), ctypes.byref(n)))
        return b.value, e.value, n.value

    def synchronize(self):
        it, err = ctypes.c_int(), ctypes.c_double()
        st = lib().lx_ctx_synchronize(self.handle, ctypes.byref(it), ctypes.byref(err))
        _check(st, it.value)
        return it.value, err.value

    @property
    def iterations_per_pass(self) -> int:
        """2 when this context's Leja calls use the temporally blocked kernel, else 1."""
        return int(lib().lx_ctx_iterations_per_pass(self.handle))

    @property
    def launch_count(self) -> int:
        return int(lib().lx_ctx_launch_count(self.handle))


def _pb(ctx: Context, problem: Problem | None):
    return ctypes.byref(problem.c_struct() if problem is not None else ctx._pb)


def lx_spectrum_bound(ctx: Context, u=None, problem: Problem | None = None) -> float:
    out = ctypes.c_double()
    _check(lib().lx_spectrum_bound(ctx.handle, _pb(ctx, problem), _ptr(u), ctypes.byref(out)))
    return out.value


def lx_spectrum_estimate(ctx: Context, u=None, iters: int = 50, problem: Problem | None = None) -> float:
    out = ctypes.c_double()
    _check(lib().lx_spectrum_estimate(ctx.handle, _pb(ctx, problem), _ptr(u), int(iters), ctypes.byref(out)))
    return out.value


def lx_real_leja_phi(ctx: Context, v, out, dt, c, gamma, l, rtol, atol, u_lin=None,
                     problem: Problem | None = None, sync: bool = True):
    """out <- phi_l(dt J(u_lin)) v.  Returns the Leja iteration count (None if sync=False)."""
    it = ctypes.c_int(0)
    st = lib().lx_real_leja_phi(ctx.handle, _pb(ctx, problem), _ptr(u_lin), _ptr(v), _ptr(out), float(dt), float(c),
                                float(gamma), int(l), float(rtol), float(atol), ctypes.byref(it) if sync else None)
    _check(st, it.value)
    return it.value if sync else None


def lx_real_leja_phi_vertical(ctx: Context, v, outs: Sequence, coeffs: Sequence[float], dt, c, gamma, l, rtol,
                              atol, u_lin=None, problem: Problem | None = None, sync: bool = True):
    K = len(outs)
    arr = (ctypes.c_void_p * K)(*[_ptr(o) for o in outs])
    cf = (ctypes.c_double * K)(*[float(a) for a in coeffs])
    it = ctypes.c_int(0)
    st = lib().lx_real_leja_phi_vertical(ctx.handle, _pb(ctx, problem), _ptr(u_lin), _ptr(v), arr, cf, K,
                                         float(dt), float(c), float(gamma), int(l), float(rtol), float(atol),
                                         ctypes.byref(it) if sync else None)
    _check(st, it.value)
    return it.value if sync else None


def lx_real_leja_phi_multi(ctx: Context, v, outs: Sequence, ls: Sequence[int], coeffs: Sequence[float], dt, c, gamma,
                           rtol, atol, u_lin=None, problem: Problem | None = None, sync: bool = True):
    """outs[k] = phi_{ls[k]}(coeffs[k] dt J) v, one shared Newton basis (lexint.h)."""
    K = len(outs)
    arr = (ctypes.c_void_p * K)(*[_ptr(o) for o in outs])
    li = (ctypes.c_int * K)(*[int(x) for x in ls])
    cf = (ctypes.c_double * K)(*[float(a) for a in coeffs])
    it = ctypes.c_int(0)
    st = lib().lx_real_leja_phi_multi(ctx.handle, _pb(ctx, problem), _ptr(u_lin), _ptr(v), arr, li, cf, K,
                                      float(dt), float(c), float(gamma), float(rtol), float(atol),
                                      ctypes.byref(it) if sync else None)
    _check(st, it.value)
    return it.value if sync else None


def lx_step(ctx: Context, method, u, u_low, u_high, dt, c, gamma, rtol, atol, problem: Problem | None = None,
            sync: bool = True):
    """One exponential-integrator step.  Returns (iters, err) (None, None if sync=False)."""
    m = METHODS[method] if isinstance(method, str) else int(method)
    it, err = ctypes.c_int(0), ctypes.c_double(0.0)
    st = lib().lx_step(ctx.handle, m, _pb(ctx, problem), _ptr(u), _ptr(u_low), _ptr(u_high),
                       ctypes.byref(err) if sync else None, float(dt), float(c), float(gamma), float(rtol),
                       float(atol), ctypes.byref(it) if sync else None)
    _check(st, it.value)
    return (it.value, err.value) if sync else (None, None)


def lx_step_rosenbrock_euler(ctx, u, u_out, dt, c, gamma, rtol, atol, problem=None):
    return lx_step(ctx, LX_ROSENBROCK_EULER, u, None, u_out, dt, c, gamma, rtol, atol, problem)[0]


def lx_step_exprb42(ctx, u, u_out, dt, c, gamma, rtol, atol, problem=None):
    return lx_step(ctx, LX_EXPRB42, u, None, u_out, dt, c, gamma, rtol, atol, problem)[0]


def lx_step_epirk5p1(ctx, u, u_out, dt, c, gamma, rtol, atol, problem=None):
    return lx_step(ctx, LX_EPIRK5P1, u, None, u_out, dt, c, gamma, rtol, atol, problem)[0]


def lx_step_exprb32(ctx, u, u_low, u_high, dt, c, gamma, rtol, atol, problem=None):
    return lx_step(ctx, LX_EXPRB32, u, u_low, u_high, dt, c, gamma, rtol, atol, problem)


def lx_step_exprb43(ctx, u, u_low, u_high, dt, c, gamma, rtol, atol, problem=None):
    return lx_step(ctx, LX_EXPRB43, u, u_low, u_high, dt, c, gamma, rtol, atol, problem)


def lx_step_epirk4s3a(ctx, u, u_low, u_high, dt, c, gamma, rtol, atol, problem=None):
    return lx_step(ctx, LX_EPIRK4S3A, u, u_low, u_high, dt, c, gamma, rtol, atol, problem)


def lx_integrate(ctx: Context, method, u, dt, nsteps, rtol, atol, problem: Problem | None = None,
                 sync: bool = True):
    """nsteps exponential-integrator steps in place on u with the spectrum (c, gamma) recomputed on the
    device every step (the paper's time loop).  Returns (total Leja iterations, last err)."""
    m = METHODS[method] if isinstance(method, str) else int(method)
    it, err = ctypes.c_int(0), ctypes.c_double(0.0)
    st = lib().lx_integrate(ctx.handle, m, _pb(ctx, problem), _ptr(u), float(dt), int(nsteps), float(rtol),
                            float(atol), ctypes.byref(it) if sync else None, ctypes.byref(err) if sync else None)
    _check(st, it.value)
    return (it.value, err.value) if sync else (None, None)


def lx_integrate_adaptive(ctx: Context, method, u, t_end, dt0, tol, rtol, atol, max_steps: int = 1000,
                          problem: Problem | None = None):
    """Embedded-error step-size control (lexint.h; reading R32) in place on device u.
    Returns (accepted, rejected, step sizes tried, their errors, Leja iterations)."""
    m = METHODS[method] if isinstance(method, str) else int(method)
    na, nr, it = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    dts = np.zeros(max_steps)
    errs = np.zeros(max_steps)
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib().lx_integrate_adaptive(ctx.handle, m, _pb(ctx, problem), _ptr(u), float(t_end), float(dt0), float(tol),
                                     float(rtol), float(atol), int(max_steps), ctypes.byref(na), ctypes.byref(nr),
                                     dts.ctypes.data_as(dp), errs.ctypes.data_as(dp), ctypes.byref(it))
    _check(st, it.value)
    k = na.value + nr.value
    return na.value, nr.value, dts[:k], errs[:k], it.value


def lx_rhs(ctx: Context, u, f_out, scale: float = 1.0, problem: Problem | None = None):
    _check(lib().lx_rhs(ctx.handle, _pb(ctx, problem), _ptr(u), float(scale), _ptr(f_out)))


# ------------------------------------------------------------------ black-box RHS
class LxBuiltinRhsUser(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("pb", ctypes.POINTER(LxProblem))]


class Rhs:
    """A black-box right-hand side f for lx_real_leja_phi_cb / lx_step_cb.

    Rhs.builtin(ctx): the library's own stencil f of ctx's problem, called natively (no Python
    in the loop).  Rhs.from_python(fn): fn(in_ptr, out_ptr, stream_handle) is called from the
    library through a ctypes trampoline; it must enqueue its device work on that stream."""

    def __init__(self, fn_ptr, user_ptr, keep=()):
        self.fn = fn_ptr
        self.user = user_ptr
        self._keep = keep
        self.error = None     # first exception raised inside a Python callback (re-raised after the call)

    def _raise(self):
        if self.error is not None:
            e, self.error = self.error, None
            raise RuntimeError("black-box RHS callback failed") from e

    @classmethod
    def builtin(cls, ctx: "Context", problem: Problem | None = None) -> "Rhs":
        pb = problem.c_struct() if problem is not None else ctx._pb
        u = LxBuiltinRhsUser(ctx.handle.value, ctypes.pointer(pb))
        fn = ctypes.cast(lib().lx_builtin_rhs, ctypes.c_void_p).value
        return cls(fn, ctypes.addressof(u), keep=(u, pb))

    @classmethod
    def from_torch(cls, fn, shape) -> "Rhs":
        """fn(x, out): a torch implementation of f on CUDA tensors of `shape` (fp64); it runs on the
        library's stream (torch.cuda.ExternalStream).  User code -- the library only calls it."""
        import torch

        class _View:
            def __init__(self, ptr):
                self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
                                                 "version": 3, "strides": None, "stream": None}

        def call(inp, out, stream):
            # the legacy default stream (handle 0 or cudaStreamLegacy = 1) is torch's default stream
            st = torch.cuda.default_stream() if not stream or stream == 1 else torch.cuda.ExternalStream(stream)
            with torch.cuda.stream(st):
                fn(torch.as_tensor(_View(inp), device="cuda"), torch.as_tensor(_View(out), device="cuda"))
        return cls.from_python(call)

    @classmethod
    def from_python(cls, fn) -> "Rhs":
        holder = []

        def tramp(inp, out, user, stream):
            try:
                fn(inp, out, stream)
            except BaseException as e:   # never unwind through the C frames
                if holder and holder[0].error is None:
                    holder[0].error = e
        cb = RHS_FN(tramp)
        r = cls(ctypes.cast(cb, ctypes.c_void_p).value, None, keep=(cb,))
        holder.append(r)
        return r


def lx_real_leja_phi_cb(ctx: Context, rhs: Rhs, v, outs: Sequence, coeffs: Sequence[float], dt, c, gamma, l,
                        rtol, atol, u=None) -> int:
    """phi_l(a_k dt J) v with J known only through rhs: J(u) by finite differences when u is
    given, else J y = f(y) (linear f).  Returns the Leja iteration count."""
    K = len(outs)
    arr = (ctypes.c_void_p * K)(*[_ptr(o) for o in outs])
    cf = (ctypes.c_double * K)(*[float(a) for a in coeffs])
    it = ctypes.c_int(0)
    st = lib().lx_real_leja_phi_cb(ctx.handle, rhs.fn, rhs.user, _ptr(u), _ptr(v), arr, cf, K, float(dt), float(c),
                                   float(gamma), int(l), float(rtol), float(atol), ctypes.byref(it))
    rhs._raise()
    _check(st, it.value)
    return it.value


def lx_step_cb(ctx: Context, method, rhs: Rhs, u, u_low, u_high, dt, c, gamma, rtol, atol):
    """One integrator step on a black-box f (FD Jacobians and remainders).  Returns (iters, err)."""
    m = METHODS[method] if isinstance(method, str) else int(method)
    it, err = ctypes.c_int(0), ctypes.c_double(0.0)
    st = lib().lx_step_cb(ctx.handle, m, rhs.fn, rhs.user, _ptr(u), _ptr(u_low), _ptr(u_high), ctypes.byref(err),
                          float(dt), float(c), float(gamma), float(rtol), float(atol), ctypes.byref(it))
    rhs._raise()
    _check(st, it.value)
    return it.value, err.value
