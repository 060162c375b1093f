"""Host-side accounting used by bench.py's roofline (CPU, no GPU).

The algorithmic bytes of a Leja call are checked against an explicit pass-by-pass model of
what each kernel reads and writes (one N-vector = 8 B/pt): the one-pass kernel does one pass per
iteration; the two-step kernel does one pass per pair of iterations plus a rollback pass when the call
stops on the first iteration of a pair.
"""
import pytest

import bench


def _passes_one_step(m):
    traffic = 0
    for it in range(1, m + 1):
        if it == 1:
            traffic += 8 * (1 + 2)          # read v; write y_1, p_1
        else:
            traffic += 8 * (2 + 2)          # read y, p; write y, p
    return traffic


def _passes_two_step(m):
    traffic = 0
    npass = (m + 1) // 2
    for q in range(npass):
        traffic += 8 * (1 + 2) if q == 0 else 8 * (2 + 2)
    if m % 2 == 1:                           # stopped on the first iteration of the last pass: rollback
        traffic += 8 * (2 + 1)               # read y, p; write p
    return traffic


@pytest.mark.parametrize("m", list(range(1, 41)))
def test_leja_bytes_per_point_matches_pass_model(m):
    assert bench.leja_bytes_per_point(m, False) == _passes_one_step(m)
    assert bench.leja_bytes_per_point(m, True) == _passes_two_step(m)


def test_config1_bytes_per_step():
    # config 1 (4096^2, phi_0..phi_3 at 10 dt_CFL): 16/16/14/10 iterations (SURVEY 8(c) spectral simulation)
    iters = (16, 16, 14, 10)
    one = sum(bench.leja_bytes_per_point(m, False) for m in iters)
    two = sum(bench.leja_bytes_per_point(m, True) for m in iters)
    assert one == 8 * (3 + 4 * 15) + 8 * (3 + 4 * 15) + 8 * (3 + 4 * 13) + 8 * (3 + 4 * 9)
    assert two == 8 * (3 + 4 * 7) * 2 + 8 * (3 + 4 * 6) + 8 * (3 + 4 * 4)
    assert 2.0 < one / two < 2.1        # two iterations per pass (and the first pass reads v only)


def _passes_vertical(m_k):
    # one pass per iteration; iteration 1 reads v and writes y and every accumulator; iteration m >= 2
    # reads/writes y and every accumulator still active at m (converged at m_k >= m)
    traffic = 0
    for m in range(1, max(m_k) + 1):
        if m == 1:
            traffic += 8 * (1 + 1 + len(m_k))
        else:
            traffic += 8 * 2 + 16 * sum(1 for mk in m_k if mk >= m)
    return traffic


@pytest.mark.parametrize("m_k", [(1,), (5, 7, 9), (13, 14, 16), (3, 3)])
def test_vertical_bytes_match_pass_model(m_k):
    assert bench.leja_bytes_per_point_vertical(list(m_k)) == _passes_vertical(m_k)


def _passes_vertical_tb2(m_k):
    # 3D two-step kernel: pass q performs iterations 2q+1, 2q+2 and touches y plus the accumulators it
    # updates or rolls back; simulated iteration by iteration
    M = max(m_k)
    traffic = 0
    pending = set()                          # accumulators whose p holds one term too many
    for q in range((M + 1) // 2):
        m = 2 * q + 1
        if q == 0:
            traffic += 8 * (1 + 1 + len(m_k))    # read v; write y_2 and every p
        else:
            touched = {k for k, mk in enumerate(m_k) if mk >= m} | pending
            traffic += 8 * 2 + 16 * len(touched)
        pending = {k for k, mk in enumerate(m_k) if mk == m}   # stopped on the first iteration of pass q
    if pending:                              # end-of-call fix-up
        traffic += 8 + 16 * len(pending)
    return traffic


@pytest.mark.parametrize("m_k", [(1,), (2,), (5, 7, 9), (13, 14, 16), (3, 3), (4, 5, 6), (9, 11, 12), (7, 8, 8, 9)])
def test_vertical_tb2_bytes_match_pass_model(m_k):
    assert bench.leja_bytes_per_point_vertical_tb2(list(m_k)) == _passes_vertical_tb2(m_k)


@pytest.mark.parametrize("m", list(range(1, 30)))
def test_vertical_tb2_single_accumulator_is_two_step(m):
    assert bench.leja_bytes_per_point_vertical_tb2([m]) == bench.leja_bytes_per_point(m, True)


@pytest.mark.parametrize("m_k", [(1,), (5,), (3, 5, 7), (13, 14, 16), (9, 11, 11)])
def test_vertical_tb2_predicted_final_iteration(m_k):
    # a predicted odd final iteration M: the last pass performs only iteration M, no end-of-call rollback
    full = bench.leja_bytes_per_point_vertical_tb2(list(m_k))
    pred = bench.leja_bytes_per_point_vertical_tb2(list(m_k), predicted=True)
    M = max(m_k)
    if M % 2:
        assert full - pred == 8 + 16 * sum(1 for mk in m_k if mk == M)
    else:
        assert pred == full
