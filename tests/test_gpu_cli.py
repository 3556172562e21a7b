"""GPU: the bratu_bench equivalents (paper_1906_04051_b200.cli) keep the
reference CLI's CSV schemas and config echo (tools/bratu_bench.cpp:83-99,
180-380) and their numbers match the reference solver."""
import io
import os
import struct
import sys
from contextlib import redirect_stdout

import numpy as np
import pytest

from paper_1906_04051_b200 import cli

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_cli_convergence_matches_reference(cuda, ref, tmp_path):
    out = tmp_path / "conv.csv"
    rc = cli.main(["convergence", "--ne", "10", "--m", "30", "--restarts", "4",
                   "--out", str(out), "--json", str(tmp_path / "conv.json")])
    assert rc == 0
    lines = out.read_text().splitlines()
    echo = [ln for ln in lines if ln.startswith("# ")]
    assert echo[0] == "# subcommand=convergence" and "# m=30" in echo
    body = [ln for ln in lines if not ln.startswith("#")]
    assert body[0] == "restart,explicit_residual,variant"
    rows = [ln.split(",") for ln in body[1:]]
    assert [r[2] for r in rows] == ["deflated"] * 5 + ["undeflated"] * 5
    A, b = ref.first_newton_system(10)
    for variant, defl in (("deflated", True), ("undeflated", False)):
        r = ref.solve(A, b, m=30, max_restarts=4, fixed_iterations=True, deflation=defl)
        got = np.array([float(x[1]) for x in rows if x[2] == variant])
        want = np.concatenate([[r.beta0], r.explicit_residual])
        assert np.max(np.abs(got - want)) <= 1e-10 * r.beta0
    assert (tmp_path / "conv.json").exists()


def _speedup_rows(argv):
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv)
    assert rc == 0
    body = [ln for ln in buf.getvalue().splitlines() if not ln.startswith("#")]
    assert body[0] == ("dof,p,median_s,speedup,relative_speed,compute_pct,local_comm_pct,"
                       "global_comm_pct")
    return [ln.split(",") for ln in body[1:]]


def test_cli_speedup_schema(cuda):
    rows = _speedup_rows(["speedup", "--ne", "6", "--m", "10", "--restarts", "2", "--reps", "2"])
    assert len(rows) == 1
    dof, p, med = rows[0][:3]
    assert int(dof) == 13 ** 3 and int(p) == 1 and float(med) > 0
    assert float(rows[0][3]) == 1.0 and float(rows[0][5]) == pytest.approx(100.0)


def test_cli_speedup_derived_columns(cuda):
    """test_cli.cpp:225-248 on the GPU: the p = 1 baseline row is inserted,
    speedup = T1 / Tp, relative_speed = slowest / Tp, and the compute /
    local / global percentages sum to 100 (p = 2: two in-process ranks on one
    GPU with host-staged collectives, so the halo and allreduce shares are
    measured)."""
    rows = _speedup_rows(["speedup", "--ne", "6", "--m", "10", "--restarts", "2", "--reps", "1",
                          "--loopback", "2"])
    assert [r[1] for r in rows] == ["1", "2"]
    t1, t2 = float(rows[0][2]), float(rows[1][2])
    slowest = max(t1, t2)
    for r in rows:
        med = float(r[2])
        assert float(r[3]) == pytest.approx(t1 / med, rel=1e-9)
        assert float(r[4]) == pytest.approx(slowest / med, rel=1e-9)
        assert float(r[5]) + float(r[6]) + float(r[7]) == pytest.approx(100.0, abs=1e-6)
    assert float(rows[0][6]) == 0.0 and float(rows[0][7]) == 0.0
    assert float(rows[1][6]) > 0.0 and float(rows[1][7]) > 0.0


def test_cli_solve_writes_solution_and_trace(cuda, tmp_path, golden):
    path = tmp_path / "u.bin"
    rc = cli.main(["solve", "--ne", "8", "--out", str(path)])
    assert rc == 0
    raw = path.read_bytes()
    (n,) = struct.unpack("<Q", raw[:8])
    u = np.frombuffer(raw[8:], "<f8")
    assert n == 17 ** 3 == u.size
    g = golden("newton_ne8")
    assert np.linalg.norm(u - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])
    trace = (tmp_path / "u.bin.trace.csv").read_text().splitlines()
    assert trace[0] == "# subcommand=solve"
    assert "iter,update_inf_norm,residual_2norm,gmres_restarts" in trace
