#!/usr/bin/env python
"""Measure every BASELINE.json config on one GPU (device-timed, CUDA events).

Prints one JSON object per config: Leja iterations, time, achieved algorithmic
GB/s of the Leja kernels and the fraction of the measured HBM copy peak.
Not the driver's bench line (bench.py is); used to fill profiles/.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_08344_b200 as lx  # noqa: E402
import workloads as W  # noqa: E402
from bench import leja_bytes_per_point, leja_bytes_per_point_vertical_tb2  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def timed(stream, fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    out = [fn() for _ in range(reps)]
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def cfg0(stream):
    wl = W.config(0)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_problem1_2d(64)).cuda()
    out = torch.empty_like(u)
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
    for _ in range(5):
        it = lx.lx_step_rosenbrock_euler(ctx, u, out, wl.dt, c, g, wl.rtol, wl.atol)
    ms, _ = timed(stream, lambda: lx.lx_step(ctx, "rosenbrock_euler", u, None, out, wl.dt, c, g, wl.rtol,
                                             wl.atol, sync=False), 50)
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        lx.lx_step_rosenbrock_euler(ctx, u, out, wl.dt, c, g, wl.rtol, wl.atol)
    host_us = (time.perf_counter() - t0) / 50 * 1e6
    return {"config": 0, "workload": wl.name, "grid": [64, 64], "leja_iters": it, "device_us_per_step": ms * 1e3,
            "sync_us_per_step": host_us, "note": "L1/L2 resident, launch/latency bound: no roofline claim"}


def cfg_leja(stream, n, ls, name, reps=3, mult=10.0):
    """phi_l Leja calls on the n^2 Problem-I Gaussian at mult x dt_CFL (config 1: mult = 10; the dt sweep
    1 / 10 / 100 x CFL of SURVEY 8(d))."""
    wl = W.config(1, n=n)
    dt = wl.dt * mult / 10.0
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_problem1_2d(n)).cuda()
    out = torch.empty_like(u)
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
    res = []
    for l in ls:
        it = lx.lx_real_leja_phi(ctx, u, out, dt, c, g, l, wl.rtol, wl.atol)
        ms, _ = timed(stream, lambda: lx.lx_real_leja_phi(ctx, u, out, dt, c, g, l, wl.rtol, wl.atol,
                                                           sync=False), reps)
        ctx.synchronize()
        tb2 = ctx.iterations_per_pass == 2
        byt = u.numel() * leja_bytes_per_point(it, tb2)        # the kernel's own algorithmic bytes
        byt1 = u.numel() * leja_bytes_per_point(it, False)     # one-pass accounting (32 B/pt per iteration)
        res.append({"l": l, "iters": it, "ms": ms, "GBps": byt / ms / 1e6, "frac": byt / ms / 1e6 / PEAK,
                    "one_pass_equiv_frac": byt1 / ms / 1e6 / PEAK})
    ctx.close()
    return {"config": name, "grid": [n, n], "dt_cfl_mult": mult, "calls": res,
            "leja_it_per_s": sum(r["iters"] for r in res) / sum(r["ms"] for r in res) * 1e3}


def cfg2(stream, n=2048, steps=20):
    wl = W.config(2, n=n)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
    lo, hi = torch.empty_like(u), torch.empty_like(u)
    its, errs = [], []
    for _ in range(2):   # warm-up (lazy module loading, first-use allocations) on a copy of the state
        uw = u.clone()
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, uw))
        lx.lx_step(ctx, "exprb43", uw, lo, hi, wl.dt, c, g, wl.rtol, wl.atol)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for s in range(steps):
        c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, u))
        it, err = lx.lx_step(ctx, "exprb43", u, lo, hi, wl.dt, c, g, wl.rtol, wl.atol)
        its.append(it)
        errs.append(err)
        u, hi = hi, u
    b.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = a.elapsed_time(b)
    # the same run through lx_integrate (device-side spectrum, no host round trips); twice, the
    # second timed
    for _ in range(2):
        u2 = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
        torch.cuda.synchronize()
        a.record(stream)
        lx.lx_integrate(ctx, "exprb43", u2, wl.dt, steps, wl.rtol, wl.atol, sync=False)
        b.record(stream)
        torch.cuda.synchronize()
        it2, err2 = ctx.synchronize()
        ms2 = a.elapsed_time(b)
    ctx.close()
    return {"config": 2, "workload": wl.name, "grid": [n, n], "steps": steps, "leja_iters_per_step": its,
            "err": errs[-1], "steps_per_s_device": steps / (ms * 1e-3), "steps_per_s_wall": steps / wall,
            "ms_per_step": ms / steps, "integrate_steps_per_s": steps / (ms2 * 1e-3),
            "integrate_iters": it2, "integrate_err": err2, "integrate_vs_loop_max_abs": float((u2 - u).abs().max())}


def cfg4(stream, n=512):
    wl = W.config(4, n=n)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=stream)
    c1 = W.coords(n)
    u = torch.empty(wl.shape, dtype=torch.float64, device="cuda")
    for i in range(n):   # 3D Gaussian built slab by slab (host memory)
        x = c1[i]
        y, z = np.meshgrid(c1, c1, indexing="ij")
        u[i] = torch.from_numpy(1.0 + np.exp(-((x + .5) ** 2 + (y + .5) ** 2 + (z + .5) ** 2) / 0.01))
    lo, hi = torch.empty_like(u), torch.empty_like(u)
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
    it, err = lx.lx_step(ctx, "epirk4s3a", u, lo, hi, wl.dt, c, g, wl.rtol, wl.atol)
    ms, _ = timed(stream, lambda: lx.lx_step(ctx, "epirk4s3a", u, lo, hi, wl.dt, c, g, wl.rtol, wl.atol,
                                             sync=False), 2)
    ctx.synchronize()
    out = torch.empty_like(u)
    it0 = lx.lx_real_leja_phi(ctx, u, out, wl.dt, c, g, 0, wl.rtol, wl.atol)
    ms0, _ = timed(stream, lambda: lx.lx_real_leja_phi(ctx, u, out, wl.dt, c, g, 0, wl.rtol, wl.atol, sync=False), 2)
    ctx.synchronize()
    tb = ctx.iterations_per_pass == 2
    # the kernel's own algorithmic bytes (repeated call: predicted final iteration), and the
    # one-pass accounting (32 B/pt per iteration) for comparison
    byt = u.numel() * (leja_bytes_per_point_vertical_tb2([it0], predicted=True) if tb else 24 + 32 * (it0 - 1))
    byt1 = u.numel() * (24 + 32 * (it0 - 1))
    ctx.close()
    return {"config": 4, "workload": wl.name, "grid": list(wl.shape), "epirk4s3a_iters": it, "epirk4s3a_ms": ms,
            "phi0_iters": it0, "phi0_ms": ms0, "iterations_per_pass": 2 if tb else 1,
            "phi0_GBps": byt / ms0 / 1e6, "phi0_frac": byt / ms0 / 1e6 / PEAK,
            "phi0_one_pass_equiv_frac": byt1 / ms0 / 1e6 / PEAK}


def cfg_burgers(stream, n=4096, mult=10.0, steps=3):
    """Problem III: viscous Burgers, EXPRB32 (the paper's Table 2 integrators)."""
    dx = (2.0 / n, 2.0 / n)
    pb = lx.Problem((n, n), dx, 1.0, 0.0, 0.0, None, 10.0)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_burgers_2d(n)).cuda()
    dt = mult * W.dt_cfl(n, 20.0)
    it, _ = lx.lx_integrate(ctx, "exprb32", u, dt, 1, 1e-10, 1e-10)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    lx.lx_integrate(ctx, "exprb32", u, dt, steps, 1e-10, 1e-10, sync=False)
    b.record(stream)
    torch.cuda.synchronize()
    its, err = ctx.synchronize()
    ms = a.elapsed_time(b)
    # one Burgers Leja call (J(u) flux form), phi_1 of f*dt
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, u))
    f = torch.empty_like(u)
    lx.lx_rhs(ctx, u, f, dt)
    out = torch.empty_like(u)
    m = lx.lx_real_leja_phi(ctx, f, out, dt, c, g, 1, 1e-10, 1e-10, u_lin=u)
    ms1, _ = timed(stream, lambda: lx.lx_real_leja_phi(ctx, f, out, dt, c, g, 1, 1e-10, 1e-10, u_lin=u,
                                                        sync=False), 3)
    ctx.synchronize()
    byt = u.numel() * (32 + 40 * (m - 1))   # iteration 1: v, u read, y, p written; then y, p, u read, y, p written
    ctx.close()
    return {"config": "Problem III (Burgers) exprb32", "grid": [n, n], "dt_cfl_mult": mult, "steps": steps,
            "leja_iters": its, "ms_per_step": ms / steps, "steps_per_s": steps / (ms * 1e-3), "err": err,
            "phi1_iters": m, "phi1_ms": ms1, "phi1_GBps": byt / ms1 / 1e6, "phi1_frac": byt / ms1 / 1e6 / PEAK,
            "algorithmic_bytes_note": "40 B/pt per iteration (y, p, u reads; y, p writes)"}


def cfg_blackbox(stream, n=4096, n_fd=2048):
    """the black-box RHS path (user f through lx_rhs_fn, FD Jacobian)."""
    wl = W.config(1, n=n)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_problem1_2d(n)).cuda()
    out = torch.empty_like(u)
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
    rhs = lx.Rhs.builtin(ctx)
    it = lx.lx_real_leja_phi_cb(ctx, rhs, u, [out], [1.0], wl.dt, c, g, 0, wl.rtol, wl.atol)
    ms, _ = timed(stream, lambda: lx.lx_real_leja_phi_cb(ctx, rhs, u, [out], [1.0], wl.dt, c, g, 0, wl.rtol,
                                                          wl.atol), 3)
    # per iteration: builtin f(y) 16 B/pt + update (read f(y), y, p; write y, p) 40 B/pt
    lin = {"mode": "linear operator (J y = f(y)), builtin stencil f", "grid": [n, n], "l": 0, "iters": it,
           "ms": ms, "leja_it_per_s": it / ms * 1e3, "algorithmic_B_per_pt_iter": 56,
           "frac": u.numel() * 56 * it / ms / 1e6 / PEAK}
    ctx.close()
    wl = W.config(2, n=n_fd)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_allen_cahn_2d(n_fd)).cuda()
    v = torch.empty_like(u)
    lx.lx_rhs(ctx, u, v, wl.dt)
    out = torch.empty_like(u)
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx, u))
    rhs = lx.Rhs.builtin(ctx)
    it = lx.lx_real_leja_phi_cb(ctx, rhs, v, [out], [1.0], wl.dt, c, g, 1, wl.rtol, wl.atol, u=u)
    ms, _ = timed(stream, lambda: lx.lx_real_leja_phi_cb(ctx, rhs, v, [out], [1.0], wl.dt, c, g, 1, wl.rtol,
                                                          wl.atol, u=u), 3)
    it_s, err = lx.lx_step_cb(ctx, "exprb43", rhs, u, torch.empty_like(u), torch.empty_like(u), wl.dt, c, g,
                              wl.rtol, wl.atol)
    ms_s, _ = timed(stream, lambda: lx.lx_step_cb(ctx, "exprb43", rhs, u, out, v, wl.dt, c, g, wl.rtol, wl.atol), 2)
    # per iteration: perturb (u, y -> w) 24 + f(w) 16 + update (f(w), f(u), y, p -> y, p) 48 B/pt
    fd = {"mode": "FD Jacobian of the builtin Allen-Cahn f (R25)", "grid": [n_fd, n_fd], "l": 1, "iters": it,
          "ms": ms, "leja_it_per_s": it / ms * 1e3, "algorithmic_B_per_pt_iter": 88,
          "frac": u.numel() * 88 * it / ms / 1e6 / PEAK, "exprb43_step_iters": it_s, "exprb43_step_ms": ms_s,
          "note": "host waits on each iteration's device decision (one iteration in flight)"}
    ctx.close()
    return {"config": "f-1 black-box RHS", "linear": lin, "fd": fd}


def cfg_catalogue(stream, n=2048, steps=20):
    """Problem II (source) and the 5th-order methods through lx_integrate."""
    out = {"config": "f-2 / f-4"}
    wl = W.config(1, n=n)
    S = torch.from_numpy(W.source_problem2_2d(n)).cuda()
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react, S)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_problem1_2d(n)).cuda()
    it, _ = lx.lx_integrate(ctx, "rosenbrock_euler", u, wl.dt, 1, wl.rtol, wl.atol)
    ms, _ = timed(stream, lambda: lx.lx_integrate(ctx, "rosenbrock_euler", u, wl.dt, steps, wl.rtol, wl.atol,
                                                   sync=False), 1)
    its, _ = ctx.synchronize()
    out["problem2_rosenbrock_euler"] = {"grid": [n, n], "steps": steps, "ms_per_step": ms / steps,
                                        "steps_per_s": steps / ms * 1e3, "leja_iters_per_step": its / steps}
    ctx.close()
    wl = W.config(2, n=n)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    for m in ("epirk5p1", "exprb53s3", "exprb43"):
        ctx = lx.Context(pb, stream=stream)
        u = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
        lx.lx_integrate(ctx, m, u, wl.dt, 2, wl.rtol, wl.atol)
        ms, _ = timed(stream, lambda: lx.lx_integrate(ctx, m, u, wl.dt, steps, wl.rtol, wl.atol, sync=False), 1)
        its, err = ctx.synchronize()
        out["allen_cahn_" + m] = {"grid": [n, n], "steps": steps, "ms_per_step": ms / steps,
                                  "steps_per_s": steps / ms * 1e3, "leja_iters_per_step": its / steps,
                                  "last_err": err}
        ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="0,1,2,3,4,5,6,7,8")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    want = set(int(x) for x in a.only.split(","))
    if 0 in want:
        print(json.dumps(cfg0(s)), flush=True)
    if 1 in want:
        print(json.dumps(cfg_leja(s, 4096, (0, 1, 2, 3), 1)), flush=True)
    if 2 in want:
        print(json.dumps(cfg2(s)), flush=True)
    if 3 in want:
        print(json.dumps(cfg_leja(s, 16384, (0,), "3 (N=1)", reps=2)), flush=True)
    if 4 in want:
        print(json.dumps(cfg4(s)), flush=True)
    if 5 in want:
        print(json.dumps(cfg_burgers(s)), flush=True)
    if 6 in want:
        print(json.dumps(cfg_blackbox(s)), flush=True)
    if 7 in want:
        print(json.dumps(cfg_catalogue(s)), flush=True)
    if 8 in want:   # config-1 dt sweep (1 and 100 x CFL; 10 x CFL is row 1)
        for mult in (1.0, 100.0):
            print(json.dumps(cfg_leja(s, 4096, (0, 1, 2, 3), "1 (dt sweep)", mult=mult)), flush=True)


if __name__ == "__main__":
    main()
