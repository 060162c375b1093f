"""Multi-rank slab decomposition on ONE GPU.

Virtual ranks (host threads) with the in-process transport run exactly the protocols of the
multi-GPU path: 2D Leja calls with >= 16 rows per rank take the persistent peer-memory slab kernel
(k_leja2d_tb2<K, DIAG, true>: halo rows stored into the neighbours' ghost blocks from inside the
pass, per-rank partials exchanged at the pass barrier); everything else the per-iteration step
protocol (step kernels, 1+2-row halo exchange, rank-order sum of the gathered partials).  Results
must match the oracle (same iterations, rel L2 <= 1e-10) and -- since the per-point arithmetic is
identical and only the norm summation order differs -- equal the single-domain CUDA result of the
same kernel family bitwise.  A two-process test maps the exchange blocks through CUDA IPC."""
import threading

import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2310_08344_b200 as lx  # noqa: E402

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _run_ranks(P, fn):
    """Run fn(rank, group) on P threads; collect results / exceptions."""
    group = lx.LocalGroup(P)
    res, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                res[r] = fn(r, group, s)
            s.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return res


@pytest.mark.parametrize("P,shape", [(2, (64, 64)), (3, (50, 70)), (4, (130, 66)), (8, (64, 128))])
def test_slab_leja_matches_oracle_and_single_domain(xi300, P, shape):
    # peer-memory slab kernel when every rank has >= 16 rows (two iterations per pass: compared with the
    # single-domain two-step kernel), else the step protocol (compared with the one-step kernel)
    peer = shape[0] // P >= 16 and shape[1] >= 64
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    v = W.ic_problem1_2d(*shape)
    dt = 10 * min(W.dt_cfl(n, 10.0) for n in shape)
    c, g = O.shift_scale(O.spectrum_bound(ob))

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r)
        assert ctx.iterations_per_pass == (2 if peer else 1)
        b, e, _ = ctx.local()
        vloc = torch.from_numpy(v[b:e]).cuda()
        outs = []
        for l in (0, 1, 3):
            o = torch.empty_like(vloc)
            it = lx.lx_real_leja_phi(ctx, vloc, o, dt, c, g, l, TOL, TOL)
            outs.append((it, o.cpu().numpy()))
        ctx.close()
        return b, e, outs

    res = _run_ranks(P, rank_fn)
    with lx.Context(pb) as ctx1:
        ctx1.set_kernel(2 if peer else 1)
        for idx, l in enumerate((0, 1, 3)):
            full = np.concatenate([res[r][2][idx][1] for r in range(P)], axis=0)
            its = {res[r][2][idx][0] for r in range(P)}
            ref = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300)
            assert its == {ref.iters}, (l, its, ref.iters)
            assert np.linalg.norm(full - ref.outs[0]) <= TOL * np.linalg.norm(ref.outs[0])
            one = torch.empty(shape, dtype=torch.float64, device="cuda")
            lx.lx_real_leja_phi(ctx1, torch.from_numpy(v).cuda(), one, dt, c, g, l, TOL, TOL)
            np.testing.assert_array_equal(full, one.cpu().numpy())


@pytest.mark.parametrize("method", ["exprb32", "exprb43", "epirk4s3a", "epirk5p1", "exprb53s3", "exprb54s4",
                                    "epirk4s3b", "epirk4s3"])
def test_slab_steps_allen_cahn(xi300, method):
    P, shape = 2, (96, 64)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1e-4, 0.0, 1.0)
    ob = O.Problem(shape, dx, 1e-4, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(*shape)

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r)
        b, e, _ = ctx.local()
        ul = torch.from_numpy(u[b:e]).cuda()
        bound = lx.lx_spectrum_bound(ctx, ul)
        cc, gg = lx.lx_shift_scale(bound)
        lo, hi = torch.empty_like(ul), torch.empty_like(ul)
        it, err = lx.lx_step(ctx, method, ul, lo, hi, 0.01, cc, gg, TOL, TOL)
        est = lx.lx_spectrum_estimate(ctx, ul, 30)
        ctx.close()
        return bound, it, err, lo.cpu().numpy(), hi.cpu().numpy(), est

    res = _run_ranks(P, rank_fn)
    bound = O.spectrum_bound(ob, u)
    assert {r[0] for r in res} == {bound}
    c, g = O.shift_scale(bound)
    ref = O.step(ob, method, u, 0.01, c, g, TOL, TOL, xi300)
    assert {r[1] for r in res} == {ref.iters}
    hi = np.concatenate([r[4] for r in res])
    lo = np.concatenate([r[3] for r in res])
    assert np.linalg.norm(hi - ref.u_high) <= TOL * np.linalg.norm(ref.u_high)
    assert np.linalg.norm(lo - ref.u_low) <= TOL * np.linalg.norm(ref.u_low)
    assert len({r[2] for r in res}) == 1 and res[0][2] == pytest.approx(ref.err, rel=1e-8)
    assert len({r[5] for r in res}) == 1
    assert res[0][5] == pytest.approx(O.power_iteration(ob, u, 30), rel=1e-10)


@pytest.mark.parametrize("P", [2, 4])
def test_slab_3d_epirk(xi300, P):
    shape = (24, 16, 32)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    u = W.ic_random(shape, seed=11, amp=0.3)
    dt = 5 * W.dt_cfl(32, 10.0, 3)
    c, g = O.shift_scale(O.spectrum_bound(ob))

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r)
        b, e, _ = ctx.local()
        ul = torch.from_numpy(u[b:e]).cuda()
        lo, hi = torch.empty_like(ul), torch.empty_like(ul)
        it, err = lx.lx_step(ctx, "epirk4s3a", ul, lo, hi, dt, c, g, TOL, TOL)
        ctx.close()
        return it, hi.cpu().numpy()

    res = _run_ranks(P, rank_fn)
    ref = O.step(ob, "epirk4s3a", u, dt, c, g, TOL, TOL, xi300)
    assert {r[0] for r in res} == {ref.iters}
    hi = np.concatenate([r[1] for r in res])
    assert np.linalg.norm(hi - ref.u_high) <= TOL * np.linalg.norm(ref.u_high)


def test_nccl_transport_world_size_one():
    # the real NCCL transport (not the in-process one) on one GPU: a communicator of size 1 exchanges halos
    # with itself; results must match the single-domain path (tools/nccl_selfcheck.py, own process)
    import json
    import subprocess
    import sys
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    r = subprocess.run([sys.executable, root + "/tools/nccl_selfcheck.py"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["ok"], res


def _slab_vs_single(xi300, P, shape, K, react, l, flags=0, mult=10.0):
    """P virtual ranks through the peer-memory slab kernel vs the single-domain two-step kernel
    (bitwise) and the oracle (same iterations, 1e-10)."""
    diff, nu = (1e-4, 0.0) if react else (1.0, 10.0)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, diff, nu, react)
    ob = O.Problem(shape, dx, diff, nu, react)
    u = W.ic_allen_cahn_2d(*shape) if react else None
    v = W.ic_random(shape, seed=41, amp=0.2)
    dt = 0.01 if react else mult * min(W.dt_cfl(n, 10.0) for n in shape)
    c, g = O.shift_scale(O.spectrum_bound(ob, u))
    coeffs = (0.25, 0.5, 0.75, 1.0)[-K:]

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r, flags)
        assert ctx.iterations_per_pass == 2
        b, e, _ = ctx.local()
        ul = torch.from_numpy(u[b:e]).cuda() if react else None
        vl = torch.from_numpy(v[b:e]).cuda()
        outs = [torch.full_like(vl, float("nan")) for _ in range(K)]
        it = lx.lx_real_leja_phi_vertical(ctx, vl, outs, coeffs, dt, c, g, l, TOL, TOL, u_lin=ul)
        it2 = lx.lx_real_leja_phi_vertical(ctx, vl, outs, coeffs, dt, c, g, l, TOL, TOL, u_lin=ul)   # reuse
        ctx.close()
        return it, it2, [o.cpu().numpy() for o in outs]

    res = _run_ranks(P, rank_fn)
    with lx.Context(pb) as ctx1:
        ctx1.set_kernel(2)
        ones = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(K)]
        it1 = lx.lx_real_leja_phi_vertical(ctx1, torch.from_numpy(v).cuda(), ones, coeffs, dt, c, g, l, TOL, TOL,
                                           u_lin=torch.from_numpy(u).cuda() if react else None)
    ref = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300, coeffs=coeffs, u_lin=u)
    assert {(r[0], r[1]) for r in res} == {(ref.iters, ref.iters)} and it1 == ref.iters
    for k in range(K):
        full = np.concatenate([res[r][2][k] for r in range(P)], axis=0)
        np.testing.assert_array_equal(full, ones[k].cpu().numpy())
        assert np.linalg.norm(full - ref.outs[k]) <= TOL * np.linalg.norm(ref.outs[k])


@pytest.mark.parametrize("P,shape,K,react,l", [(2, (96, 130), 1, 0.0, 0), (4, (131, 64), 2, 0.0, 1),
                                               (3, (200, 122), 3, 1.0, 1), (8, (256, 182), 4, 0.0, 3),
                                               (2, (1024, 256), 1, 1.0, 0)])
def test_peer_slab_kernel_bitwise(xi300, P, shape, K, react, l):
    # ragged slabs (131 rows over 4 ranks), ragged 60-column bands, K = 1..4 (rollbacks), Allen-Cahn J
    _slab_vs_single(xi300, P, shape, K, react, l)


def test_peer_slab_kernel_one_rank_is_single_domain(xi300):
    # LX_COMM_FORCE with one virtual rank: the slab kernel with itself as both neighbours (its ghost rows
    # are its own periodic images) -- bitwise the single-domain two-step kernel
    _slab_vs_single(xi300, 1, (128, 128), 2, 0.0, 1, flags=lx.LX_COMM_FORCE)


def test_no_peer_flag_uses_step_protocol(xi300):
    shape = (64, 64)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r, lx.LX_COMM_NO_PEER)
        ipp = ctx.iterations_per_pass
        ctx.close()
        return ipp

    assert _run_ranks(2, rank_fn) == [1, 1]
    with lx.Context(pb) as ctx:   # one rank without FORCE: the single-domain context
        ctx.set_comm_local(lx.LocalGroup(1), 0)
        assert ctx.local() == (0, 64, 64 * 64)


def test_peer_slab_kernel_two_processes_ipc(xi300):
    # two processes on one GPU, exchange blocks mapped with CUDA IPC (tools/ipc_slab_check.py)
    import json
    import os
    import subprocess
    import sys
    shape = (96, 128)
    dx = tuple(2.0 / n for n in shape)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    c, g = O.shift_scale(O.spectrum_bound(ob))
    dt = 10 * min(W.dt_cfl(n, 10.0) for n in shape)
    ls = [0, 1, 3]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    arg = json.dumps({"dt": dt, "c": c, "g": g, "ls": ls, "tol": TOL})
    r = subprocess.run([sys.executable, root + "/tools/ipc_slab_check.py", arg], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    ranks = sorted(json.loads(r.stdout.strip().splitlines()[-1])["ranks"], key=lambda x: x["rank"])
    assert [x["ipp"] for x in ranks] == [2, 2]
    v = W.ic_random(shape, seed=51, amp=0.2)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    with lx.Context(pb) as ctx1:
        ctx1.set_kernel(2)
        for idx, l in enumerate(ls):
            full = np.concatenate([np.array(x["res"][idx][1]) for x in ranks], axis=0)
            ref = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300)
            assert {x["res"][idx][0] for x in ranks} == {ref.iters}
            assert np.linalg.norm(full - ref.outs[0]) <= TOL * np.linalg.norm(ref.outs[0])
            one = torch.empty(shape, dtype=torch.float64, device="cuda")
            lx.lx_real_leja_phi(ctx1, torch.from_numpy(v).cuda(), one, dt, c, g, l, TOL, TOL)
            np.testing.assert_array_equal(full, one.cpu().numpy())


def _slab3d_vs_single(xi300, P, shape, K, l, flags=0, mult=5.0):
    """3D: P virtual ranks through the peer-memory two-step plane-sweep kernel (k_leja3d_tb2<K, true>:
    ghost planes stored into the neighbours' exchange blocks by stage B, norm partials exchanged at every
    pass barrier) vs the single-domain k_leja3d_tb2 (bitwise) and the oracle (same iterations, 1e-10)."""
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    v = W.ic_random(shape, seed=43, amp=0.2)
    dt = mult * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    c, g = O.shift_scale(O.spectrum_bound(ob))
    coeffs = (0.25, 0.5, 0.75, 1.0)[-K:]

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r, flags)
        assert ctx.iterations_per_pass == 2
        b, e, _ = ctx.local()
        vl = torch.from_numpy(v[b:e]).cuda()
        outs = [torch.full_like(vl, float("nan")) for _ in range(K)]
        it = lx.lx_real_leja_phi_vertical(ctx, vl, outs, coeffs, dt, c, g, l, TOL, TOL)
        it2 = lx.lx_real_leja_phi_vertical(ctx, vl, outs, coeffs, dt, c, g, l, TOL, TOL)   # reuse
        ctx.close()
        return it, it2, [o.cpu().numpy() for o in outs]

    res = _run_ranks(P, rank_fn)
    with lx.Context(pb) as ctx1:
        ctx1.set_kernel(2)
        assert ctx1.iterations_per_pass == 2
        ones = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(K)]
        it1 = lx.lx_real_leja_phi_vertical(ctx1, torch.from_numpy(v).cuda(), ones, coeffs, dt, c, g, l, TOL, TOL)
    ref = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300, coeffs=coeffs)
    assert {(r[0], r[1]) for r in res} == {(ref.iters, ref.iters)} and it1 == ref.iters
    for k in range(K):
        full = np.concatenate([res[r][2][k] for r in range(P)], axis=0)
        np.testing.assert_array_equal(full, ones[k].cpu().numpy())
        assert np.linalg.norm(full - ref.outs[k]) <= TOL * np.linalg.norm(ref.outs[k])


@pytest.mark.parametrize("P,shape,K,l", [(2, (24, 16, 64), 1, 0), (4, (37, 32, 64), 2, 1), (4, (16, 16, 128), 3, 0),
                                         (8, (64, 16, 64), 4, 3), (3, (40, 16, 64), 1, 2)])
def test_peer_slab_3d_kernel_bitwise(xi300, P, shape, K, l):
    # ragged slabs (37 planes over 4 ranks), the minimum of 4 planes per rank (16 / 4: every plane is a
    # boundary plane of one or both neighbours), K = 1..4 (rollbacks), phi_0..phi_3
    _slab3d_vs_single(xi300, P, shape, K, l)


def test_peer_slab_3d_one_rank_is_single_domain(xi300):
    # one virtual rank with LX_COMM_FORCE: its ghost planes are its own periodic images
    _slab3d_vs_single(xi300, 1, (20, 16, 64), 2, 1, flags=lx.LX_COMM_FORCE)


def test_peer_slab_3d_epirk_step(xi300):
    # a whole EPIRK4s3A step (config 5's integrator) with the 3D Leja calls on the peer-memory kernel and
    # the stage kernels on the step protocol
    P, shape = 2, (32, 16, 64)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    u = W.ic_random(shape, seed=17, amp=0.3)
    dt = 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    c, g = O.shift_scale(O.spectrum_bound(ob))

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r)
        assert ctx.iterations_per_pass == 2
        b, e, _ = ctx.local()
        ul = torch.from_numpy(u[b:e]).cuda()
        lo, hi = torch.empty_like(ul), torch.empty_like(ul)
        it, err = lx.lx_step(ctx, "epirk4s3a", ul, lo, hi, dt, c, g, TOL, TOL)
        ctx.close()
        return it, err, lo.cpu().numpy(), hi.cpu().numpy()

    res = _run_ranks(P, rank_fn)
    ref = O.step(ob, "epirk4s3a", u, dt, c, g, TOL, TOL, xi300)
    assert {r[0] for r in res} == {ref.iters}
    hi = np.concatenate([r[3] for r in res])
    lo = np.concatenate([r[2] for r in res])
    assert np.linalg.norm(hi - ref.u_high) <= TOL * np.linalg.norm(ref.u_high)
    assert np.linalg.norm(lo - ref.u_low) <= TOL * np.linalg.norm(ref.u_low)


def test_peer_slab_3d_kernel_two_processes_ipc(xi300):
    # two processes on one GPU, 3D ghost planes through CUDA IPC mappings of the exchange blocks
    import json
    import os
    import subprocess
    import sys
    shape = (16, 16, 64)
    dx = tuple(2.0 / n for n in shape)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    c, g = O.shift_scale(O.spectrum_bound(ob))
    dt = 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    ls = [0, 2]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    arg = json.dumps({"dt": dt, "c": c, "g": g, "ls": ls, "tol": TOL, "shape": list(shape)})
    r = subprocess.run([sys.executable, root + "/tools/ipc_slab_check.py", arg], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    ranks = sorted(json.loads(r.stdout.strip().splitlines()[-1])["ranks"], key=lambda x: x["rank"])
    assert [x["ipp"] for x in ranks] == [2, 2]
    v = W.ic_random(shape, seed=51, amp=0.2)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    with lx.Context(pb) as ctx1:
        ctx1.set_kernel(2)
        for idx, l in enumerate(ls):
            full = np.concatenate([np.array(x["res"][idx][1]) for x in ranks], axis=0)
            ref = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300)
            assert {x["res"][idx][0] for x in ranks} == {ref.iters}
            assert np.linalg.norm(full - ref.outs[0]) <= TOL * np.linalg.norm(ref.outs[0])
            one = torch.empty(shape, dtype=torch.float64, device="cuda")
            lx.lx_real_leja_phi(ctx1, torch.from_numpy(v).cuda(), one, dt, c, g, l, TOL, TOL)
            np.testing.assert_array_equal(full, one.cpu().numpy())


@pytest.mark.parametrize("shape", [(96, 130), (32, 16, 64)])
def test_slab_multi_phi(xi300, shape):
    # lx_real_leja_phi_multi on 2 virtual ranks (2D / 3D peer-memory slab kernels, per-accumulator phi index
    # in the in-kernel coefficients and in the prebuilt tables) against the oracle's separate calls
    P, ls, coeffs = 2, (0, 1, 3), (1.0, 1.0, 1.0)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    v = W.ic_random(shape, seed=12, amp=0.2)
    dt = (10 if len(shape) == 2 else 5) * min(W.dt_cfl(n, 10.0, len(shape)) for n in shape)
    c, g = O.shift_scale(O.spectrum_bound(ob))

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r)
        b, e, _ = ctx.local()
        vl = torch.from_numpy(v[b:e]).cuda()
        outs = [torch.empty_like(vl) for _ in ls]
        it = lx.lx_real_leja_phi_multi(ctx, vl, outs, ls, coeffs, dt, c, g, TOL, TOL)
        ctx.close()
        return it, [o.cpu().numpy() for o in outs]

    res = _run_ranks(P, rank_fn)
    refs_ = [O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300) for l in ls]
    assert {r[0] for r in res} == {max(x.iters for x in refs_)}
    for k, ref in enumerate(refs_):
        full = np.concatenate([res[r][1][k] for r in range(P)], axis=0)
        assert np.linalg.norm(full - ref.outs[0]) <= TOL * np.linalg.norm(ref.outs[0])


@pytest.mark.parametrize("method", ["exprb43", "epirk4s3a"])
def test_slab_integrate_and_adaptive(xi300, method):
    # the paper's time loop on 2 virtual ranks: lx_integrate (device spectrum bound with the cross-rank max,
    # (c, gamma) on the device every step) and lx_integrate_adaptive (R32: the cross-rank embedded error
    # drives identical accept / reject decisions on every rank) against the oracle's single-domain loops
    P, shape = 2, (96, 64)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1e-3, 0.0, 1.0)
    ob = O.Problem(shape, dx, 1e-3, 0.0, 1.0)
    u = W.ic_allen_cahn_2d(*shape)
    dt, nsteps = 0.01, 3
    t_end, dt0, tol = 0.2, 0.2, 1e-7

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r)
        b, e, _ = ctx.local()
        ul = torch.from_numpy(u[b:e]).cuda()
        it, err = lx.lx_integrate(ctx, method, ul, dt, nsteps, TOL, TOL)
        ua = torch.from_numpy(u[b:e]).cuda()
        acc, rej, dts, errs, its = lx.lx_integrate_adaptive(ctx, method, ua, t_end, dt0, tol, 1e-12, 1e-12)
        ctx.close()
        return it, err, ul.cpu().numpy(), (acc, rej, list(dts), its), ua.cpu().numpy()

    res = _run_ranks(P, rank_fn)
    uo, tot = u.copy(), 0
    for _ in range(nsteps):
        c, g = O.shift_scale(O.spectrum_bound(ob, uo))
        r = O.step(ob, method, uo, dt, c, g, TOL, TOL, xi300)
        tot += r.iters
        uo = r.u_high
    assert {x[0] for x in res} == {tot}
    full = np.concatenate([x[2] for x in res])
    assert np.linalg.norm(full - uo) <= TOL * np.linalg.norm(uo)
    ref = O.integrate_adaptive(ob, method, u, t_end, dt0, tol, 1e-12, 1e-12, xi300)
    assert ref.status == O.OK
    for x in res:
        acc, rej, dts, its = x[3]
        assert (acc, rej, its) == (ref.accepted, ref.rejected, ref.iters)
        np.testing.assert_allclose(dts, ref.dts, rtol=1e-8)
    fa = np.concatenate([x[4] for x in res])
    assert np.linalg.norm(fa - ref.u) <= 1e-9 * np.linalg.norm(ref.u)
