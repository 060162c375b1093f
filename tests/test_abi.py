"""CPU checks of the C-ABI library: it loads, exports every symbol declared in
include/lexint.h, and its host-side math (no device work) agrees with the
independent oracle.  -m "not gpu": no device compute calls here."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2310_08344_b200 as lx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "lexint.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lx_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_all_declared_symbols():
    L = lx.lib()
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(lx.EXPORTS)
    assert b"sm_100a" in L.lx_version()


def test_library_is_sm100a_fatbin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lx.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_leja_points_match_oracle(xi300):
    xi = lx.lx_leja_points(300)
    assert np.max(np.abs(xi - xi300)) <= 2e-15   # root of g located to a few ulps by two methods


@pytest.mark.parametrize("l", range(5))
def test_host_phi_matches_oracle(l):
    for z in [-300.0, -50.0, -2.0, -1.999, -0.5, -1e-9, 0.0, 0.7, 1.99, 2.0, 8.0]:
        a, b = lx.lx_phi_scalar(l, z), O.phi(l, z)
        assert a == pytest.approx(b, rel=3e-15, abs=1e-300), (l, z)


def test_host_divided_differences_match_oracle(xi300):
    for l, rho in [(0, 5.0), (1, 30.0), (3, 60.0), (4, 2.0)]:
        g = rho
        c = -2 * g
        a = lx.lx_divided_differences(l, xi300, 300, 1.0, c, g)
        b = O.divided_differences(l, xi300, 300, 1.0, c, g)
        # same recurrence, independent code: bitwise or ulp-level agreement of the
        # contributions |d_k| * max|basis_k| (basis <= 4^k on [-2, 2])
        zs = np.linspace(-2, 2, 201)
        basis = np.ones_like(zs)
        for k in range(120):
            assert abs(a[k] - b[k]) * np.abs(basis).max() <= 1e-14, (l, k)
            basis = basis * (zs - xi300[k])


def test_host_error_paths():
    with pytest.raises(lx.LxError) as e:
        lx.lx_phi_scalar(5, 0.0)
    assert e.value.status == lx.LX_ERR_UNSUPPORTED
    with pytest.raises(lx.LxError):
        lx.lx_leja_points(0)
    assert lx.lx_shift_scale(100.0) == (-52.5, 26.25)
    c, g = lx.lx_shift_scale(4 / (2 / 256) ** 2)
    assert c == pytest.approx(-34406.4, rel=1e-15) and g == pytest.approx(17203.2, rel=1e-15)


def test_slab_range_partitions():
    for n0 in (7, 64, 4096, 16384):
        for P in (1, 2, 3, 4, 8):
            rows = [lx.lx_slab_range(n0, r, P) for r in range(P)]
            assert rows[0][0] == 0 and rows[-1][1] == n0
            assert all(rows[i][1] == rows[i + 1][0] for i in range(P - 1))
            assert max(e - b for b, e in rows) - min(e - b for b, e in rows) <= 1
