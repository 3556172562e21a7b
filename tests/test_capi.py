"""CPU: the C-ABI library loads without a GPU, exports every symbol the public
header declares, and its pure host logic (z-slab partition) follows
partition_rows (parallel.cpp:50-71; test_parallel.cpp:20-63)."""
import ctypes as C
import os
import re

import pytest

from paper_1906_04051_b200 import _capi
from paper_1906_04051_b200.build import ROOT, build_library


@pytest.fixture(scope="module")
def lib():
    build_library()
    return _capi.lib()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "pgmres.h")).read()
    declared = set(re.findall(r"\b(pgm_[a-z_]+)\s*\(", hdr))
    assert declared == set(_capi.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def _part(lib, n_axis, p, w):
    out = _capi.Partition()
    rc = lib.pgm_partition_rows(n_axis, p, w, C.byref(out))
    return rc, (out.row_begin, out.row_end, out.halo_lo, out.halo_hi)


def test_partition_rows_matches_reference(lib):
    # n_e = 2: 5 planes of 25 nodes over 2 workers -> 3 + 2 planes, 2-plane halos
    assert _part(lib, 5, 2, 0) == (0, (0, 75, 0, 50))
    assert _part(lib, 5, 2, 1) == (0, (75, 125, 50, 0))
    for na in (3, 5, 7):
        plane = na * na
        for p in range(1, na + 1):
            cursor = 0
            for w in range(p):
                rc, (b, e, lo, hi) = _part(lib, na, p, w)
                assert rc == 0 and b == cursor and b % plane == 0
                sizes = [(_part(lib, na, p, q)[1][1] - _part(lib, na, p, q)[1][0]) // plane
                         for q in range(p)]
                assert max(sizes) - min(sizes) <= 1
                assert lo == min(2, b // plane) * plane
                assert hi == min(2, na - e // plane) * plane
                cursor = e
            assert cursor == na ** 3


def test_partition_rejects_bad_worker_counts(lib):
    assert _part(lib, 5, 0, 0)[0] == _capi.PGM_EINVAL
    assert _part(lib, 5, 6, 0)[0] == _capi.PGM_EINVAL
    assert _part(lib, 5, 5, 4)[0] == 0


def test_newton_config_and_report_mirror_reference():
    """NewtonConfig defaults (newton.hpp:15-23), ctypes layout of the C struct,
    and NewtonReport::write_csv (newton.cpp:12-19: header, precision 17)."""
    import paper_1906_04051_b200 as pg

    c = pg.NewtonConfig()
    assert (c.max_iters, c.update_tol, c.use_deflation, c.continuation,
            c.continuation_steps) == (30, 1e-8, True, False, 4)
    assert (c.gmres.m, c.gmres.max_restarts, c.gmres.rel_tol) == (50, 100, 1e-10)
    cc = c._c()
    assert cc.max_iters == 30 and cc.gmres.m == 50 and cc.deflation.r_max == 20
    assert C.sizeof(_capi.NewtonRecordC) == 48
    rep = pg.NewtonReport([pg.NewtonIterRecord(1, 6.8, 0.7895591656135857, 0.12056974500368113,
                                               2, 66)], True)
    assert rep.write_csv() == ("iter,update_inf_norm,residual_2norm,gmres_restarts\n"
                               "1,0.78955916561358575,0.12056974500368113,2\n")
    with pytest.raises(ValueError):
        pg.NewtonConfig(max_iters=-1)._c()
