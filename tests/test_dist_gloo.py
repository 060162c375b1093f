"""World-size-2 (and 3) CPU tests of the multi-process slab path with the gloo backend.

* the NCCL unique id bootstrap through torch.distributed (same 128 bytes on all ranks);
* slab ranges, max-over-ranks timing reduction;
* oracle-based emulations of the two slab protocols that follow the LIBRARY's exchange plan
  (lx_slab_halo_plan from liblexint_b200.so, host-only, executed with gloo send/recv) and the
  rank-order sum of the per-rank partials: mode 0, the step protocol (one Leja iteration per
  exchange, 3 ghost rows); mode 1, the two-step slab kernel (two iterations per exchange, 6 ghost
  rows, the first iteration recomputed on the halo-extended slab).  The fields must equal the
  single-domain oracle BITWISE and stop at the same iteration.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(gh, n_loc, rank, world, mode):
    """Fill the ghost rows of gh (local rows stored from index G, G = 1 (mode 0) or 2 (mode 1); ghost slot
    0.. = rows -G..-1, then rows n_loc.. ) per the library's plan."""
    from paper_2310_08344_b200 import lx_slab_halo_plan
    G = 1 if mode == 0 else 2
    reqs = []
    for kind, peer, first, nrows, slot in lx_slab_halo_plan(rank, world, n_loc, mode):
        if kind == "send":
            buf = torch.from_numpy(np.ascontiguousarray(gh[G + first:G + first + nrows]))
            reqs.append(dist.isend(buf, peer))
        else:
            buf = torch.empty((nrows,) + gh.shape[1:], dtype=torch.float64)
            dist.recv(buf, peer)
            rows = [slot + i if slot + i < G else n_loc + slot + i for i in range(nrows)]   # slot -> gh index
            gh[rows] = buf.numpy()
    for r in reqs:
        r.wait()


def _case(shape):
    """Input, dt and (c, gamma) of the emulated slab run: the Problem-I Gaussian (2D, 10 x CFL) or a
    seeded random field (3D, 5 x CFL; the 3D slab kernel follows the mode-1 plan with planes)."""
    import oracle as O
    import workloads as W
    dx = tuple(2.0 / n for n in shape)
    pb = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    if len(shape) == 2:
        v = W.ic_problem1_2d(*shape)
        dt = 10 * W.dt_cfl(shape[0], 10.0)
    else:
        v = W.ic_random(shape, seed=29, amp=0.2)
        dt = 5 * min(W.dt_cfl(n, 10.0, 3) for n in shape)
    c, g = O.shift_scale(O.spectrum_bound(pb))
    return pb, v, dt, c, g


def _worker(rank, world, port, result_dir, mode, shape=(40, 24)):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    import workloads as W
    from paper_2310_08344_b200 import dist as lxd

    # 1. bootstrap of the library communicator id
    uid = lxd.share_unique_id()
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    assert len(uid) == 128 and all(i == uid for i in ids)
    # 2. slabs and timing reduction
    n0 = shape[0]
    sl = lxd.slabs(n0, world)
    b, e = sl[rank]
    assert lxd.max_over_ranks(float(rank) + 0.5) == world - 0.5
    # 3. emulated slab Leja iterations (oracle arithmetic, the library's exchange plan)
    pb, v, dt, c, g = _case(shape)
    xi = O.leja_points(300)
    d = O.divided_differences(1, xi, 300, dt, c, g)
    n_loc = e - b
    N = v.size
    G = 1 if mode == 0 else 2
    y = np.zeros((n_loc + G + (2 if mode == 0 else 4),) + tuple(shape[1:]))   # ghost rows -G..-1, local, n..
    y[G:G + n_loc] = v[b:e]
    p = d[0] * v[b:e]

    def step(ygh_ext, n_ext, m):
        # one Leja iteration (Eq. (2)) on n_ext rows whose ghosted input ygh_ext has 1 row before, 2 after
        w = O.jac_apply_slab(pb, n_ext, None, ygh_ext)
        yin = ygh_ext[1:n_ext + 1]
        return (w - c * yin) / g - xi[m - 1] * yin

    def converged(m, ynew, pnew):
        part = torch.tensor([np.sum(ynew * ynew), np.sum(pnew * pnew)], dtype=torch.float64)
        allp = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, part)
        sy = sp = 0.0
        for t in allp:            # rank order
            sy += float(t[0])
            sp += float(t[1])
        return abs(d[m]) * np.sqrt(sy / N) <= 1e-10 * np.sqrt(sp / N) + 1e-10

    iters = None
    m = 1
    while m < 300 and iters is None:
        _exchange(y, n_loc, rank, world, mode)
        if mode == 0:
            ynew = step(y, n_loc, m)
            p = p + d[m] * ynew
            y[1:n_loc + 1] = ynew
            if converged(m, ynew, p):
                iters = m
            m += 1
        else:
            # two iterations per exchange: y_m on rows -1 .. n+1 from y_{m-1} rows -2 .. n+3, then y_{m+1}
            ym_ext = step(y, n_loc + 3, m)                 # rows -1 .. n+1
            ym = ym_ext[1:n_loc + 1]
            p = p + d[m] * ym
            if converged(m, ym, p):
                iters = m
                break
            ym1 = step(ym_ext, n_loc, m + 1)
            p = p + d[m + 1] * ym1
            y[2:n_loc + 2] = ym1
            if converged(m + 1, ym1, p):
                iters = m + 1
            m += 2
    np.save(os.path.join(result_dir, "p%d.npy" % rank), p)
    np.save(os.path.join(result_dir, "it%d.npy" % rank), np.array([iters, b, e]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode,shape", [(2, 0, (40, 24)), (3, 0, (40, 24)), (2, 1, (40, 24)), (3, 1, (40, 24)),
                                              (2, 1, (24, 8, 8)), (3, 1, (20, 8, 6))])
def test_gloo_slab_protocol(tmp_path, world, mode, shape):
    # 3D rows: the 3D peer-memory slab kernel's ghost PLANES follow the same mode-1 plan (rows = planes;
    # 20 planes over 3 ranks: ragged slabs of 7 / 7 / 6)
    import oracle as O
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), mode, shape), nprocs=world, join=True,
                       start_method="spawn")
    pb, v, dt, c, g = _case(shape)
    xi = O.leja_points(300)
    ref = O.real_leja_phi(pb, v, dt, c, g, 1, 1e-10, 1e-10, xi)
    parts, its = [], set()
    for r in range(world):
        parts.append(np.load(tmp_path / ("p%d.npy" % r)))
        its.add(int(np.load(tmp_path / ("it%d.npy" % r))[0]))
    assert its == {ref.iters}
    # the recurrence's field values are bitwise those of the single-domain oracle
    # (only the norm summation order differs); literal (w - c y)/gamma form as the oracle
    np.testing.assert_array_equal(np.concatenate(parts), ref.outs[0])


def test_halo_plan_shapes():
    # the plan's rows reach what the +x-biased stencil needs (i-1, i+1, i+2 per iteration; twice that for
    # the two-step kernel), sends and receives pair up across ranks, and two ranks still match in order
    from paper_2310_08344_b200 import lx_slab_halo_plan
    for world in (1, 2, 3, 8):
        for mode, (nu, nd) in ((0, (2, 1)), (1, (4, 2))):
            plans = [lx_slab_halo_plan(r, world, 16, mode) for r in range(world)]
            for r, plan in enumerate(plans):
                assert [op[0] for op in plan] == ["send", "recv", "send", "recv"]
                assert plan[0][1] == (r - 1) % world and plan[0][2:4] == (0, nu)
                assert plan[2][1] == (r + 1) % world and plan[2][2:4] == (16 - nd, nd)
                # my i-th send is received by its peer as that peer's op with the same direction
                for i in (0, 2):
                    peer = plan[i][1]
                    recv = plans[peer][i + 1]
                    assert recv[0] == "recv" and recv[1] == r and recv[3] == plan[i][3]
                    assert recv[4] == plan[i][4]
