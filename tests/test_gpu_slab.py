"""Multi-rank slab decomposition on ONE GPU: virtual ranks (host threads) with the
in-process transport run exactly the protocol of the NCCL path (step kernels,
1+2-row halo exchange, rank-order sum of the gathered partials).  Results must
match the oracle (same iterations, rel L2 <= 1e-10) and -- since the per-point
arithmetic is identical and only the norm summation order differs -- equal the
single-domain CUDA result bitwise."""
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
def test_slab_leja_matches_oracle_and_single_domain(xi300, monkeypatch, P, shape):
    monkeypatch.setenv("LX_TBLOCK", "1")   # single-domain reference: the one-step kernel (same arithmetic)
    dx = tuple(2.0 / n for n in shape)
    pb = lx.Problem(shape, dx, 1.0, 10.0, 0.0)
    ob = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    v = W.ic_problem1_2d(*shape)
    dt = 10 * min(W.dt_cfl(n, 10.0) for n in shape)
    c, g = O.shift_scale(O.spectrum_bound(ob))

    def rank_fn(r, group, s):
        ctx = lx.Context(pb, stream=s)
        ctx.set_comm_local(group, r)
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
        for idx, l in enumerate((0, 1, 3)):
            full = np.concatenate([res[r][2][idx][1] for r in range(P)], axis=0)
            its = {res[r][2][idx][0] for r in range(P)}
            ref = O.real_leja_phi(ob, v, dt, c, g, l, TOL, TOL, xi300)
            assert its == {ref.iters}, (l, its, ref.iters)
            assert np.linalg.norm(full - ref.outs[0]) <= TOL * np.linalg.norm(ref.outs[0])
            one = torch.empty(shape, dtype=torch.float64, device="cuda")
            lx.lx_real_leja_phi(ctx1, torch.from_numpy(v).cuda(), one, dt, c, g, l, TOL, TOL)
            np.testing.assert_array_equal(full, one.cpu().numpy())


@pytest.mark.parametrize("method", ["exprb32", "exprb43", "epirk4s3a", "epirk5p1", "exprb53s3"])
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
