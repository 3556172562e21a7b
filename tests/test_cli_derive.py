"""CPU: the speedup subcommand's derived columns (bratu_bench.cpp:282-307;
test_cli.cpp:225-248) and the profile -> TimingBreakdown mapping."""
import numpy as np
import pytest

from paper_1906_04051_b200 import cli


def test_speedup_rows_derivations():
    rows = cli.speedup_rows(1000, [(1, 2.0, (1.5, 0.0, 0.5)), (4, 0.8, (2.0, 0.4, 0.8)),
                                   (8, 0.5, (2.4, 0.8, 0.8))])
    assert [r["p"] for r in rows] == [1, 4, 8]
    for r in rows:
        assert r["speedup"] == pytest.approx(2.0 / r["median_s"], rel=1e-12)
        assert r["relative_speed"] == pytest.approx(2.0 / r["median_s"], rel=1e-12)
        assert r["compute_pct"] + r["local_comm_pct"] + r["global_comm_pct"] == pytest.approx(100)
    assert rows[0]["compute_pct"] == pytest.approx(75.0) and rows[0]["local_comm_pct"] == 0.0
    assert rows[1]["local_comm_pct"] == pytest.approx(100 * 0.4 / 3.2)


class _FakeEx:
    def __init__(self, cls, ms):
        self._p = (np.array(cls, np.uint32), None, None, np.array(ms, np.float64))

    def profile(self):
        return self._p


def test_breakdown_from_profile_classes():
    # class 10 = halo planes (local), 11 = allreduce + finisher (global)
    ex = _FakeEx([0, 2, 10, 11, 10, 3], [5.0, 1.0, 0.5, 0.25, 0.5, 0.1])
    compute, local, glob = cli.breakdown(ex, 0.010)
    assert local == pytest.approx(1e-3) and glob == pytest.approx(0.25e-3)
    assert compute == pytest.approx(0.010 - 1.25e-3)
