"""World-size-2 (and 3) CPU tests of the multi-process slab path with the gloo backend.

* the NCCL unique id bootstrap through torch.distributed (same 128 bytes on all ranks);
* slab ranges, max-over-ranks timing reduction;
* an oracle-based emulation of the slab Leja iteration that follows the product's
  exchange protocol (dist.halo_plan, executed with gloo send/recv) and the
  rank-order sum of gathered partials: the fields must equal the single-domain
  oracle BITWISE and stop at the same iteration.
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


def _exchange(slab_gh, n_loc, rank, world):
    """Fill ghost rows of slab_gh (rows -1..n_loc+1 stored at 0..n_loc+2) per halo_plan."""
    from paper_2310_08344_b200.dist import halo_plan
    reqs = []
    for op in halo_plan(rank, world, n_loc):
        if op.kind == "send":
            buf = torch.from_numpy(np.ascontiguousarray(slab_gh[[r + 1 for r in op.rows]]))
            reqs.append(dist.isend(buf, op.peer))
        else:
            buf = torch.empty((len(op.rows),) + slab_gh.shape[1:], dtype=torch.float64)
            dist.recv(buf, op.peer)
            slots = [0] if op.rows == (0,) else [n_loc + 1, n_loc + 2]
            slab_gh[slots] = buf.numpy()
    for r in reqs:
        r.wait()


def _worker(rank, world, port, result_dir):
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
    n0, n1 = 40, 24
    sl = lxd.slabs(n0, world)
    b, e = sl[rank]
    assert lxd.max_over_ranks(float(rank) + 0.5) == world - 0.5
    # 3. emulated slab Leja iteration (oracle arithmetic, product protocol)
    shape = (n0, n1)
    dx = (2.0 / n0, 2.0 / n1)
    pb = O.Problem(shape, dx, 1.0, 10.0, 0.0)
    v = W.ic_problem1_2d(n0, n1)
    xi = O.leja_points(300)
    dt = 10 * W.dt_cfl(n0, 10.0)
    c, g = O.shift_scale(O.spectrum_bound(pb))
    d = O.divided_differences(1, xi, 300, dt, c, g)
    n_loc = e - b
    y = np.zeros((n_loc + 3, n1))
    y[1:n_loc + 1] = v[b:e]
    p = d[0] * v[b:e]
    N = n0 * n1
    iters = None
    for m in range(1, 300):
        _exchange(y, n_loc, rank, world)
        w = O.jac_apply_slab(pb, n_loc, None, y)
        yin = y[1:n_loc + 1]
        ynew = (w - c * yin) / g - xi[m - 1] * yin
        p = p + d[m] * ynew
        y[1:n_loc + 1] = ynew
        part = torch.tensor([np.sum(ynew * ynew), np.sum(p * p)], dtype=torch.float64)
        allp = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, part)
        sy = 0.0
        sp = 0.0
        for t in allp:            # rank order
            sy += float(t[0])
            sp += float(t[1])
        if abs(d[m]) * np.sqrt(sy / N) <= 1e-10 * np.sqrt(sp / N) + 1e-10:
            iters = m
            break
    np.save(os.path.join(result_dir, "p%d.npy" % rank), p)
    np.save(os.path.join(result_dir, "it%d.npy" % rank), np.array([iters, b, e]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_protocol(tmp_path, world):
    import oracle as O
    import workloads as W
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    n0, n1 = 40, 24
    pb = O.Problem((n0, n1), (2.0 / n0, 2.0 / n1), 1.0, 10.0, 0.0)
    v = W.ic_problem1_2d(n0, n1)
    xi = O.leja_points(300)
    dt = 10 * W.dt_cfl(n0, 10.0)
    c, g = O.shift_scale(O.spectrum_bound(pb))
    ref = O.real_leja_phi(pb, v, dt, c, g, 1, 1e-10, 1e-10, xi)
    parts, its = [], set()
    for r in range(world):
        parts.append(np.load(tmp_path / ("p%d.npy" % r)))
        its.add(int(np.load(tmp_path / ("it%d.npy" % r))[0]))
    assert its == {ref.iters}
    # the recurrence's field values are bitwise those of the single-domain oracle
    # (only the norm summation order differs); literal (w - c y)/gamma form as the oracle
    np.testing.assert_array_equal(np.concatenate(parts), ref.outs[0])
