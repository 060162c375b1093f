#!/usr/bin/env python
"""Benchmark of the B200-native LeXInt hot path (BASELINE.json metric).

Workload at N=1 (BASELINE.json configs[1]): 2D linear advection-diffusion on a
4096^2 periodic grid (nu = 10, Problem-I Gaussian IC), fp64;
phi_0..phi_3(dt A) u_0 by real Leja interpolation at dt = 10 dt_CFL with
rtol = atol = 1e-10.  One bench STEP = the whole hot path over that input:
spectrum bound -> (c, gamma) -> for l in 0..3: divided differences (host) +
one persistent fused Leja kernel (device-side stopping decision).

value   = Leja iterations / s (device-timed, inputs resident in HBM)
e2e     = same metric through the C-ABI with HOST (pinned) buffers, copies inside
roofline: dominant kernel k_leja2d_tb2<1,false> (two Leja iterations per HBM pass),
          algorithmic bytes N*(24 + 32*(ceil(m/2)-1) [+24 if m odd]) per launch
          (leja_bytes_per_point; one-step schedule: N*(24 + 32*(m-1)))
          / CUDA-event duration.
cpu_baseline / --impl reference: the oracle (oracle/) on the host cores.

N>1 (torchrun): weak scaling -- each rank owns a 4096-row slab of a
(4096*N) x 4096 grid (slab decomposition, NCCL halos + norm allgather); value
counts 4096^2-equivalent Leja iterations of all ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "Leja iterations/s and EXPRB steps/s (fp64) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Leja it/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                                 f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline(n: int, iters: int = 2, reps: int = 1):
    """Oracle (as it stands, single-threaded C) on a bounded sample of the workload."""
    import oracle as O
    wl = W.config(1, n=n)
    ob = O.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    u0 = W.ic_problem1_2d(n)
    xi = O.leja_points(300)
    c, g = O.shift_scale(O.spectrum_bound(ob))
    tot_it, t = 0, 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        r = O.real_leja_phi(ob, u0, wl.dt, c, g, 0, wl.rtol, wl.atol, xi, max_nodes=iters + 1)
        t += time.perf_counter() - t0
        tot_it += r.iters
    return {"value": tot_it / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": "oracle real_leja_phi phi_0 on the full %dx%d grid, first %d Leja iterations "
                      "(node cap %d) x %d, single-threaded plain C" % (n, n, iters, iters + 1, reps)}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    n = args.n or 4096
    per_step = args.ref_iters
    cfg = {"workload": W.config(1, n=n).name, "grid": [n, n], "ls": [0, 1, 2, 3], "dt_cfl_mult": 10.0,
           "tol": 1e-10, "inputs": "synthetic Problem-I Gaussian IC (P:562)"}
    for _ in range(args.warmup):
        cpu_baseline(n, per_step)
    t0 = time.perf_counter()
    tot = 0
    for _ in range(args.steps):
        r = cpu_baseline(n, per_step)
        tot += per_step
    dt = time.perf_counter() - t0
    val = tot / dt
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": r["sample"]},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def leja_bytes_per_point(m, tb2):
    """Algorithmic HBM bytes per grid point of one Leja call with m iterations (roofline).

    one-step kernel: iteration 1 reads v, writes y, p (24 B); every later one reads y, p and writes
    y, p (32 B).  two-step kernel (temporal blocking): pass 1 = iterations 1, 2 reads v, writes y, p
    (24 B); each later pass (two iterations) reads y, p and writes y, p (32 B); a call that stops on
    the first iteration of its last pass adds the rollback pass (read y, p; write p: 24 B)."""
    if not tb2:
        return 24 + 32 * (m - 1)
    passes = (m + 1) // 2
    return 24 + 32 * (passes - 1) + (24 if m % 2 == 1 else 0)


def _traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "leja_traffic.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d
        except Exception:
            return None
    return None


def exprb43_steps(lx, torch, stream, n=2048, warm=2, steps=20):
    """EXPRB steps/s: Allen-Cahn 2048^2 (config 2 shape), EXPRB43, spectrum (Gershgorin) and
    (c, gamma) recomputed on the device every step -- lx_integrate, the paper's time loop."""
    wl = W.config(2, n=n)
    pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    ctx = lx.Context(pb, stream=stream)
    u = torch.from_numpy(W.ic_allen_cahn_2d(n)).cuda()
    it_w, _ = lx.lx_integrate(ctx, "exprb43", u, wl.dt, warm, wl.rtol, wl.atol)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    l0 = ctx.launch_count
    a.record(stream)
    lx.lx_integrate(ctx, "exprb43", u, wl.dt, steps, wl.rtol, wl.atol, sync=False)
    b.record(stream)
    torch.cuda.synchronize()
    its, err = ctx.synchronize()
    ms = a.elapsed_time(b)
    launches = ctx.launch_count - l0
    ctx.close()
    return {"metric": "EXPRB43 steps/s", "value": steps / (ms * 1e-3), "unit": "steps/s",
            "workload": wl.name, "grid": [n, n], "steps_timed": steps, "after_steps": warm,
            "ms_per_step": ms / steps, "leja_iters_timed": its, "leja_iters_per_step": its / steps,
            "last_err": err, "gpu_launches": launches,
            "note": "lx_integrate (one async call): Gershgorin bound + (c, gamma) on the device every step, "
                    "no host round trips; device-timed"}


def run_ours(args):
    import torch

    import paper_2310_08344_b200 as lx

    ws, rank, local = _dist()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    n = args.n or 4096
    wl = W.config(1, n=n)
    if ws > 1:
        import torch.distributed as dist
        from paper_2310_08344_b200 import dist as lxd
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # weak scaling: a (n*ws) x n grid at the SAME spacing, Problem-I IC replicated per
        # slab (x-periodic images) -> every rank does exactly the N=1 work + halos/gathers
        pb = lx.Problem((n * ws, n), wl.dx, wl.diff, wl.nu, wl.react)
    else:
        pb = lx.Problem(wl.shape, wl.dx, wl.diff, wl.nu, wl.react)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = lx.Context(pb, stream=stream)
    if ws > 1:
        b, e = lxd.attach(ctx)
        assert e - b == n, (b, e)
    u0_h = W.ic_problem1_2d(n)
    u0 = torch.from_numpy(u0_h).cuda()
    outs = [torch.empty_like(u0) for _ in range(4)]
    N = u0.numel()

    def step(ev=None):
        bound = lx.lx_spectrum_bound(ctx)
        c, g = lx.lx_shift_scale(bound)
        for l in range(4):
            if ev is not None:
                ev[l][0].record(stream)
            lx.lx_real_leja_phi(ctx, u0, outs[l], wl.dt, c, g, l, wl.rtol, wl.atol, sync=False)
            if ev is not None:
                ev[l][1].record(stream)

    # iteration counts per call (untimed, sync)
    c, g = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
    iters = [lx.lx_real_leja_phi(ctx, u0, outs[l], wl.dt, c, g, l, wl.rtol, wl.atol) for l in range(4)]
    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
        torch.cuda.synchronize()

    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in range(4)]
           for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()
        start.record(stream)
        for s in range(args.steps):
            step(evs[s])
        stop.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
    launches = ctx.launch_count - launches0
    total_iters, _ = ctx.synchronize()
    ms = start.elapsed_time(stop)
    if ws > 1:
        ms = lxd.max_over_ranks(ms, device=u0.device)
    assert total_iters == args.steps * sum(iters), (total_iters, iters)
    value = ws * total_iters / (ms * 1e-3)   # 4096^2-equivalent Leja iterations of all ranks

    # roofline of the dominant kernel (persistent Leja kernel, one launch per call)
    durs = np.array([[evs[s][l][0].elapsed_time(evs[s][l][1]) for l in range(4)] for s in range(args.steps)])
    tb2 = ctx.iterations_per_pass == 2   # the library's kernel choice for this context (lexint.h)
    bytes_per_call = np.array([N * leja_bytes_per_point(m, tb2) for m in iters], dtype=np.float64)
    per_call_ms = durs.mean(axis=0)
    achieved = float(bytes_per_call.sum() / (per_call_ms.sum() * 1e-3) / 1e9)
    peak, peak_kind = _peaks()
    tr = _traffic_from_profiles()
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": (tr or {}).get("traffic_bytes_per_launch"),
            "kernel": ("k_leja2d_tb2<1,false> (persistent, 2 Leja iterations per HBM pass, 1 launch per call)"
                       if tb2 else "k_leja2d<1,false> (persistent, 1 launch per Leja call)"),
            "one_step_equivalent_frac": float(N * sum(leja_bytes_per_point(m, False) for m in iters)
                                              / (per_call_ms.sum() * 1e-3) / 1e9 / peak),
            "algorithmic_bytes_per_launch": [float(b) for b in bytes_per_call],
            "launch_ms": [float(x) for x in per_call_ms],
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (%s)" % peak_kind,
            "frac_of_8TBs_spec": achieved / 8000.0,
            "kernel_share_of_step": float(per_call_ms.sum() / (ms / args.steps))}

    # e2e through the public API with the step's input in pinned HOST memory and its results read back to
    # pinned host memory inside the timed region: per step one H2D of u0 (copy stream), the 4
    # lx_real_leja_phi calls on the context stream, and a D2H of each phi_l output on a second copy stream
    # as soon as its call ends (overlapping the next calls; H2D and D2H run full duplex)
    uh = torch.from_numpy(u0_h).pin_memory()
    oh = [torch.empty(wl.shape, dtype=torch.float64).pin_memory() for _ in range(4)]
    ud = torch.empty_like(u0)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = torch.cuda.Event()
    ev_call = [torch.cuda.Event() for _ in range(4)]
    ev_read = [torch.cuda.Event() for _ in range(4)]
    for e in ev_read:
        e.record(s_out)
    e2e_steps = max(2, min(args.steps, 6))

    def step_e2e():
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_call[3])               # the previous step's last call has read ud
            ud.copy_(uh, non_blocking=True)
            ev_in.record(s_in)
        stream.wait_event(ev_in)
        c2, g2 = lx.lx_shift_scale(lx.lx_spectrum_bound(ctx))
        for l in range(4):
            stream.wait_event(ev_read[l])             # outs[l] of the previous step has been read back
            lx.lx_real_leja_phi(ctx, ud, outs[l], wl.dt, c2, g2, l, wl.rtol, wl.atol, sync=False)
            ev_call[l].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_call[l])
                oh[l].copy_(outs[l], non_blocking=True)
                ev_read[l].record(s_out)

    step_e2e()
    torch.cuda.synchronize()
    ctx.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e()
    torch.cuda.synchronize()
    e_t = time.perf_counter() - t0
    e_it, _ = ctx.synchronize()
    assert e_it == e2e_steps * sum(iters), (e_it, iters)
    for l in range(4):   # the read-back results are the step's outputs
        assert torch.equal(oh[l], outs[l].cpu())
    if ws > 1:
        e_t = lxd.max_over_ranks(e_t, device=u0.device)
    e2e = {"value": ws * e_it / e_t, "unit": UNIT, "h2d_bytes_per_step": N * 8, "d2h_bytes_per_step": 4 * N * 8,
           "steps": e2e_steps, "note": "per step: H2D of u0 from pinned host memory, 4 lx_real_leja_phi calls, "
           "D2H of each phi_l output to pinned host memory overlapped with the next call (wall clock)"}

    # secondary metric of BASELINE.json: EXPRB steps/s (config 2 shape: Allen-Cahn 2048^2, EXPRB43,
    # Gershgorin (c, gamma) recomputed every step).  Single-GPU only.
    exprb = None
    if ws == 1 and not args.no_exprb:
        exprb = exprb43_steps(lx, torch, stream)

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(n, args.ref_iters)
    cfg = {"workload": wl.name, "grid": list(pb.shape), "per_rank_grid": [n, n], "ls": [0, 1, 2, 3], "dt_cfl_mult": 10.0, "dt": wl.dt,
           "tol": 1e-10, "leja_iters_per_call": iters, "leja_iters_per_step": sum(iters),
           "l2_policy": "inputs larger than L2 (each fp64 vector %.0f MB > 126 MB L2)" % (N * 8 / 1e6),
           "inputs": "synthetic Problem-I Gaussian IC (P:562), nu=10" + (" replicated per slab" if ws > 1 else ""),
           "parallelism": ("slab%d (NCCL halos + partial allgather per Leja iteration)" % ws) if ws > 1 else "single GPU"}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg, "roofline": roof,
           "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
           "exprb43": exprb}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="grid side override (default 4096)")
    ap.add_argument("--ref-iters", type=int, default=2, help="oracle Leja iterations per cpu sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-exprb", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
