"""bratu_bench equivalents on the GPU (tools/bratu_bench.cpp).

    python -m paper_1906_04051_b200.cli convergence --ne 10 --m 30 --restarts 6
    python -m paper_1906_04051_b200.cli speedup --ne 50,125 --reps 3
    python -m paper_1906_04051_b200.cli solve --ne 8 --out solution.bin

Same options, CSV schemas, "# key=value" config echo (precision 17) and JSON
mirror as the reference CLI (bratu_bench.cpp:36-110), with `p` counting GPUs
instead of worker threads: run under torchrun (one process per GPU) for
p > 1; rank 0 writes the output.  Everything runs through the library
(device assembly, pgm_solve, pgm_newton_solve); nothing falls back to the CPU.
"""
from __future__ import annotations

import argparse
import io
import json
import os
import struct
import sys
import time

import numpy as np

from . import dgmres as pg

EXIT_OK, EXIT_SOLVER_FAILURE = 0, 3


def _g17(v) -> str:
    return format(float(v), ".17g")


def _parse(argv):
    ap = argparse.ArgumentParser(prog="bratu_bench (GPU)", description=__doc__.splitlines()[0])
    ap.add_argument("subcommand", choices=["convergence", "speedup", "solve"])
    ap.add_argument("--ne", default="10", help="elements per axis (list)")
    ap.add_argument("--lambda", dest="lam", type=float, default=6.8, help="reaction coefficient")
    ap.add_argument("--m", type=int, default=50, help="restart length")
    ap.add_argument("--restarts", type=int, default=100, help="restart count / outer cap")
    ap.add_argument("--rmax", type=int, default=20, help="deflation basis cap")
    ap.add_argument("--out", default="", help="output file (CSV, or solution file for solve)")
    ap.add_argument("--json", dest="json_path", default="", help="JSON mirror path")
    ap.add_argument("--reps", type=int, default=3, help="timed repetitions after one warm-up")
    ap.add_argument("--fixed-iterations", action="store_true")
    ap.add_argument("--continuation", action="store_true")
    ap.add_argument("--loopback", type=int, default=0,
                    help="speedup only: p = N in-process ranks sharing GPU 0 (host-staged "
                         "collectives; a one-GPU check of the p > 1 rows)")
    a = ap.parse_args(argv)
    a.ne = [int(v) for v in str(a.ne).split(",") if v]
    for name in ("m", "restarts", "rmax", "reps"):
        if getattr(a, name) <= 0:
            ap.error(f"--{name} must be positive")
    return a


def _world():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def config_echo(a, cmd):
    """bratu_bench.cpp:51-73 (threads -> gpus)."""
    world = _world()[0]
    return [("subcommand", cmd), ("ne", ",".join(str(v) for v in a.ne)),
            ("lambda", _g17(a.lam)), ("m", str(a.m)), ("restarts", str(a.restarts)),
            ("rmax", str(a.rmax)), ("gpus", str(world)), ("deterministic", "1"),
            ("reps", str(a.reps)), ("fixed_iterations", "1" if a.fixed_iterations else "0"),
            ("continuation", "1" if a.continuation else "0")]


class _Sink:
    """CsvSink (bratu_bench.cpp:83-99): config echo, then the table."""

    def __init__(self, a, cmd, enabled=True):
        self.enabled = enabled
        self.buf = io.StringIO()
        for k, v in config_echo(a, cmd):
            self.buf.write(f"# {k}={v}\n")
        self.path = a.out

    def write(self, s):
        self.buf.write(s)

    def close(self):
        if not self.enabled:
            return
        if self.path:
            with open(self.path, "w") as f:
                f.write(self.buf.getvalue())
        else:
            sys.stdout.write(self.buf.getvalue())
            sys.stdout.flush()


def _json_mirror(a, cmd, rows, enabled=True):
    if not a.json_path or not enabled:
        return
    with open(a.json_path, "w") as f:
        json.dump({"config": dict(config_echo(a, cmd)), "rows": rows}, f, indent=2)
        f.write("\n")


def _dist_init(local):
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def _executor(ne):
    world, rank, local = _world()
    na = 2 * ne + 1
    if world == 1:
        return pg.DeviceExecutor(0), None
    import torch

    dist = _dist_init(local)
    idt = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(pg.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    ex = pg.DeviceExecutor(local, n_global=na ** 3, n_axis=na, rank=rank, world=world,
                           nccl_id=bytes(idt.cpu().numpy()))
    return ex, dist


def cmd_convergence(a) -> int:
    """cmd_convergence (bratu_bench.cpp:180-233): fixed-iteration deflated and
    undeflated runs, restart-by-restart explicit residuals."""
    ne = a.ne[0]
    ex, dist = _executor(ne)
    A, b = ex.assemble_bratu(ne, a.lam, device=True)
    dA = ex.upload(A)
    import torch

    cfg = pg.GmresConfig(m=a.m, max_restarts=a.restarts, fixed_iterations=True)
    d = pg.Deflator(pg.DeflationConfig(r_max=a.rmax), ex)
    x = torch.zeros(ex.n_own, dtype=torch.float64, device=f"cuda:{ex.device}")
    defl = pg.deflated_gmres(dA, b, x, cfg, d, ex)
    x.zero_()
    plain = pg.gmres_restarted(dA, None, b, x, cfg, ex)
    lead = _world()[1] == 0
    sink = _Sink(a, "convergence", lead)
    sink.write("restart,explicit_residual,variant\n")
    rows = []
    for rep, variant in ((defl, "deflated"), (plain, "undeflated")):
        sink.write(f"0,{_g17(rep.beta0)},{variant}\n")
        rows.append({"restart": 0, "explicit_residual": rep.beta0, "variant": variant})
        for j, e in enumerate(rep.explicit_residual):
            sink.write(f"{j + 1},{_g17(e)},{variant}\n")
            rows.append({"restart": j + 1, "explicit_residual": float(e), "variant": variant})
    sink.close()
    _json_mirror(a, "convergence", rows, lead)
    return EXIT_OK


PC_HALO, PC_ALLREDUCE = 10, 11  # pgm_context_profile classes (include/pgmres.h)


def breakdown(ex, total_s):
    """TimingBreakdown (parallel.hpp:47-62) of the last solve from the
    per-launch CUDA-event profile: local = halo planes (class 10, the
    reference's halo gathers, parallel.cpp:249-253), global = the collective
    reduction + replicated finisher (class 11, its reductions and barrier
    waits, parallel.cpp:297-300), compute = the rest of the device time.
    Returns (compute_s, local_s, global_s)."""
    cls, _cyc, _k, ms = ex.profile()
    local = float(ms[cls == PC_HALO].sum()) * 1e-3
    glob = float(ms[cls == PC_ALLREDUCE].sum()) * 1e-3
    return max(total_s - local - glob, 0.0), local, glob


def _pct(v, parts):
    t = sum(parts)
    return 100.0 * v / t if t > 0 else 0.0


def speedup_rows(dof, results):
    """Rows of one mesh from [(p, median_s, (compute_s, local_s, global_s))]
    with p = 1 first (bratu_bench.cpp:282-307): speedup = T1 / Tp,
    relative_speed = slowest / Tp, percentages of the summed clocks
    (TimingBreakdown, parallel.hpp:47-62)."""
    t1 = next((m for p, m, _ in results if p == 1), 0.0)
    rows = [{"dof": dof, "p": p, "median_s": med,
             "speedup": t1 / med if t1 > 0 else 1.0, "relative_speed": 1.0,
             "compute_pct": _pct(parts[0], parts), "local_comm_pct": _pct(parts[1], parts),
             "global_comm_pct": _pct(parts[2], parts)} for p, med, parts in results]
    if rows:
        slowest = max(r["median_s"] for r in rows)
        for r in rows:
            r["relative_speed"] = slowest / r["median_s"]
    return rows


def _timed_solves(ex, dist, dA, b, cfg, rmax, reps):
    """One warm-up + `reps` fixed-iteration deflated solves with a fresh
    Deflator each (bratu_bench.cpp:282-300); the median by device time (max
    over ranks) and its breakdown."""
    import torch

    x = torch.zeros(ex.n_own, dtype=torch.float64, device=f"cuda:{ex.device}")
    samples = []
    ex.set_profiling(True)
    try:
        for rep in range(reps + 1):
            d = pg.Deflator(pg.DeflationConfig(r_max=rmax), ex)
            x.zero_()
            r = pg.deflated_gmres(dA, b, x, cfg, d, ex)
            parts = breakdown(ex, r.solve_seconds)
            t = r.solve_seconds
            if dist is not None:
                tt = torch.tensor([t, *parts], dtype=torch.float64, device=x.device)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt[0].item())
                # the reference sums its per-worker clocks (parallel.cpp:219-228)
                ps = torch.tensor(parts, dtype=torch.float64, device=x.device)
                dist.all_reduce(ps)
                parts = tuple(float(v) for v in ps.cpu())
            if rep > 0:  # drop the warm-up
                samples.append((t, parts))
            del d
    finally:
        ex.set_profiling(False)
    samples.sort(key=lambda s: s[0])
    return samples[len(samples) // 2]


def _loopback_solves(ne, world, a, cfg):
    """The p = world row with `world` in-process ranks on GPU 0 (LoopbackGroup,
    one host thread per rank, host-staged collectives so the allreduce is
    timed separately): max over ranks of the device time, summed clocks."""
    import threading

    os.environ["PGMRES_PEER"] = "0"
    na = 2 * ne + 1
    grp = pg.LoopbackGroup(world)
    out, err = {}, []

    def body(r):
        try:
            ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world,
                                   loopback=grp)
            A, b = ex.assemble_bratu(ne, a.lam, device=True)
            dA = ex.upload(A)
            out[r] = _timed_solves(ex, None, dA, b, cfg, a.rmax, a.reps)
            del dA
            ex.close()
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    med = max(out[r][0] for r in range(world))
    parts = tuple(sum(out[r][1][i] for r in range(world)) for i in range(3))
    return med, parts


def cmd_speedup(a) -> int:
    """cmd_speedup (bratu_bench.cpp:235-329) with p = GPUs.  The p = 1
    baseline row is always inserted (bratu_bench.cpp:235-239): under torchrun
    rank 0 first solves alone on its GPU, then all ranks solve the z-slab
    partitioned system.  Per row: median device time of `reps`
    fixed-iteration deflated solves after one warm-up, speedup = T1 / Tp,
    relative_speed = slowest / Tp over the mesh's rows, and the
    compute / local / global split from the per-kernel profile (breakdown)."""
    world, rank, local = _world()
    if a.loopback > 1 and world > 1:
        raise SystemExit("--loopback runs in one process; do not combine it with torchrun")
    ps = sorted({1, a.loopback if a.loopback > 1 else world})
    rows = []
    for ne in a.ne:
        cfg = pg.GmresConfig(m=a.m, max_restarts=a.restarts, fixed_iterations=True)
        results = []
        for p in ps:
            if p > 1 and a.loopback > 1:
                res = _loopback_solves(ne, p, a, cfg)
            elif p == 1 and world > 1:
                dist = _dist_init(local)
                res = None
                if rank == 0:
                    ex = pg.DeviceExecutor(local)
                    A, b = ex.assemble_bratu(ne, a.lam, device=True)
                    dA = ex.upload(A)
                    res = _timed_solves(ex, None, dA, b, cfg, a.rmax, a.reps)
                    del dA
                    ex.close()
                dist.barrier()
            else:
                ex, dist = _executor(ne)
                A, b = ex.assemble_bratu(ne, a.lam, device=True)
                dA = ex.upload(A)
                res = _timed_solves(ex, dist, dA, b, cfg, a.rmax, a.reps)
                del dA
                ex.close()
            if rank != 0:
                continue
            results.append((p, res[0], res[1]))
        rows.extend(speedup_rows((2 * ne + 1) ** 3, results))
    lead = rank == 0
    sink = _Sink(a, "speedup", lead)
    sink.write("dof,p,median_s,speedup,relative_speed,compute_pct,local_comm_pct,"
               "global_comm_pct\n")
    for r in rows:
        sink.write(f"{r['dof']},{r['p']},{_g17(r['median_s'])},{_g17(r['speedup'])},"
                   f"{_g17(r['relative_speed'])},{_g17(r['compute_pct'])},"
                   f"{_g17(r['local_comm_pct'])},{_g17(r['global_comm_pct'])}\n")
    sink.close()
    _json_mirror(a, "speedup", rows, lead)
    return EXIT_OK if (rows or not lead) else EXIT_SOLVER_FAILURE


def cmd_solve(a) -> int:
    """cmd_solve (bratu_bench.cpp:331-380): Newton solve, solution binary
    (u64 dof + f64 values) and <out>.trace.csv with the config echo."""
    ne = a.ne[0]
    ex, dist = _executor(ne)
    n = (2 * ne + 1) ** 3
    u = np.zeros(n)
    cfg = pg.NewtonConfig(gmres=pg.GmresConfig(m=a.m, max_restarts=a.restarts, rel_tol=1e-10,
                                               fixed_iterations=a.fixed_iterations),
                          deflation=pg.DeflationConfig(r_max=a.rmax),
                          continuation=a.continuation)
    t0 = time.perf_counter()
    rep = pg.newton_solve(ne, a.lam, u, cfg, ex)
    wall = time.perf_counter() - t0
    if dist is not None:  # every rank wrote its owned rows into its copy of u
        import torch

        ut = torch.from_numpy(u).to(f"cuda:{ex.device}")
        dist.all_reduce(ut)
        u = ut.cpu().numpy()
    if _world()[1] != 0:
        return EXIT_OK if rep.converged else EXIT_SOLVER_FAILURE
    path = a.out or "solution.bin"
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", n))
        f.write(np.ascontiguousarray(u, "<f8").tobytes())
    with open(path + ".trace.csv", "w") as f:
        for k, v in config_echo(a, "solve"):
            f.write(f"# {k}={v}\n")
        rep.write_csv(f)
    _json_mirror(a, "solve", [{"iter": r.iter, "lambda": r.lam, "update_inf_norm": r.update_inf,
                               "residual_2norm": r.residual_norm,
                               "gmres_restarts": r.gmres_restarts,
                               "gmres_inner": r.gmres_inner} for r in rep.iters])
    if not rep.converged:
        print(f"solve: no convergence within {cfg.max_iters} iterations (final update "
              f"{rep.final_update})", file=sys.stderr)
        return EXIT_SOLVER_FAILURE
    print(f"solve: converged in {len(rep.iters)} iterations ({wall:.3f} s), solution written "
          f"to {path}", file=sys.stderr)
    return EXIT_OK


def main(argv=None) -> int:
    a = _parse(sys.argv[1:] if argv is None else argv)
    return {"convergence": cmd_convergence, "speedup": cmd_speedup, "solve": cmd_solve}[
        a.subcommand](a)


if __name__ == "__main__":
    sys.exit(main())
