#!/usr/bin/env python
"""Benchmark of the deflated PGMRES hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pgmres|reference]

One step = one complete deflated_gmres solve of the first Newton system
J(0) x = -R(0) of the 3-D Bratu FEM problem (lambda = 6.8, x0 = 0),
GMRES(50) + deflation (r_max = 20), rel_tol = 1e-10.  Default workload is
BASELINE config 3, the largest benchmark mesh, quoted "at 1/2/4/8 B200":
n_e = 125, 15,813,251 DOF, 991,266,025 nnz (the matrix, 11.9 GB, dwarfs the
126 MB L2, so no L2 flush is needed); --gpus N row-block partitions it
(strong scaling).  --ne 50 is BASELINE config 2 (1,030,301 DOF).

`value`  : GMRES iterations/s with inputs resident in HBM (CUDA events on the
           library stream, max over ranks).
`e2e`    : same metric through the public API with HOST buffers: full CSR
           upload + b + x0 host->device, solve, x device->host, every step.
`roofline`: the step SpMV kernel (SpMV fused with the deflation correction and
           the Arnoldi step's dot products), algorithmic bytes / its CUDA-event
           duration; `traffic` / `frac_dram` from the committed ncu launch list.
`cpu_baseline`: the reference CPU solver (oracle/_ref, the reference's own
           sources) on a bounded sample of the same system, all host cores.
--impl reference: the reference CPU solver itself, rank 0 only (a bounded
           sample per step: one fixed restart cycle on n_e > 50).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if os.environ.get("PGMRES_PEER") == "1":  # before CUDA starts (pgm_peer_import requires it)
    os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, ROOT)

LAMBDA = 6.8
_OUT = sys.stdout
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pgmres", choices=["pgmres", "reference"])
    ap.add_argument("--ne", type=int, default=125,
                    help="mesh: n_e = 125 is BASELINE config 3 (the largest benchmark mesh, "
                         "15.8 M DOF, quoted at 1/2/4/8 B200); n_e = 50 is config 2")
    ap.add_argument("--m", type=int, default=50)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--nccl-selftest", action="store_true",
                    help="N=1 in collective mode (1-rank NCCL communicator): every reduction "
                         "pays an ncclAllReduce + k_finish, as on each rank of an N-GPU run")
    return ap.parse_args()


def metric_name(a):
    return (f"PGMRES fp64 GMRES iterations/s (deflated GMRES({a.m}), rel_tol {a.tol:g}, "
            f"time-to-solution per step)")


def workload(a, n, nnz):
    tag = {125: "BASELINE config 3 (4000x4000-equivalent, largest benchmark mesh)",
           50: "BASELINE config 2 (1000x1000-equivalent)"}.get(a.ne, "custom mesh")
    nnz_s = f"{nnz:,}" if nnz is not None else "-"
    return {"workload": f"{tag}: 3-D Bratu first Newton system, n_e={a.ne} "
                        f"({n:,} DOF, {nnz_s} nnz), GMRES({a.m}) + deflation r_max=20, "
                        f"rel_tol={a.tol:g}, x0=0",
            "n_e": a.ne, "dof": n, "nnz": nnz, "m": a.m, "rel_tol": a.tol, "r_max": 20,
            "lambda": LAMBDA,
            "l2": "inputs larger than L2 (matrix 12*nnz bytes >> 126 MB); no flush",
            "parallelism": f"z-slab row blocks x{a.gpus}" if a.gpus > 1 else "1 GPU"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return PEAKS_FALLBACK["hbm_gbs"], "fallback"


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def step_spmv_bytes(n, nnz, k, r):
    """Algorithmic HBM bytes of one fused step-SpMV launch:
    SpMV 12 nnz + 4(n+1) + 8n (x) + 8n (w), + 8n(k+1) basis reads for the
    CGS2 pass-1 dots, + 8n r AU reads for the deflation correction."""
    return 12 * nnz + 4 * (n + 1) + 16 * n + 8 * n * (k + 1) + 8 * n * r


def class_bytes(cls, n, nnz, k, r, steps, dcgs2=True):
    spmv = 12 * nnz + 4 * (n + 1) + 16 * n
    if cls == 0:
        if dcgs2:  # DCGS2 step SpMV: epilogue reads W_0..W_{k-1} (both dot families), u, U, AU
            return spmv + 8 * n * (max(k, 1) + 1 + 2 * r)
        return step_spmv_bytes(n, nnz, k, r)
    if cls == 1:  # CGS2 pass B: w1 = w - V h1 (read V_0..k, w, U_0..r-1; write w); V^T w1, ||w1||, U^T w1
        return 8 * n * (k + 3 + r)
    if cls == 2:
        if dcgs2:  # DCGS2 update: read W_0..W_{k-1}, u_k, y; write q_k, u_{k+1}
            return 8 * n * (k + 4)
        return 8 * n * (k + 3)  # CGS2 pass C: w2 = w1 - V h2
    if cls == 3:  # x += V y + U c
        return 8 * n * (steps + r + 2)
    if cls == 8:  # r = b - A x, ||r||, U^T r
        return spmv + 8 * n + 8 * n * r
    return 0


def run_gpu(a):
    import torch

    import paper_1906_04051_b200 as pg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    na = 2 * a.ne + 1
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines on stderr
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_1906_04051_b200.dgmres import nccl_unique_id

        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy())
    elif a.nccl_selftest:
        from paper_1906_04051_b200.dgmres import nccl_unique_id

        nccl_id = nccl_unique_id()
    ex = pg.DeviceExecutor(local, n_global=na ** 3, n_axis=na if world > 1 else 0, rank=rank,
                           world=world, nccl_id=nccl_id)
    if dist and os.environ.get("PGMRES_PEER") == "1":
        # fused peer-memory allreduce inside the reduction kernels (CUDA IPC
        # windows over NVLink) instead of NCCL allreduce + k_finish
        mine = torch.frombuffer(bytearray(ex.peer_export()), dtype=torch.uint8).cuda()
        allh = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allh, mine)
        ex.peer_import([bytes(h.cpu().numpy()) for h in allh])
    A_d, b_d = ex.assemble_bratu(a.ne, LAMBDA, device=True)
    n = ex.n_own
    nnz_local = A_d.nnz
    dA = ex.upload(A_d)
    ext = torch.cuda.ExternalStream(ex.stream())
    x_d = torch.zeros(n, dtype=torch.float64, device="cuda")
    d = pg.Deflator(pg.DeflationConfig(r_max=20), ex)
    cfg = pg.GmresConfig(m=a.m, max_restarts=100, rel_tol=a.tol)

    def step():
        d.reset()
        with torch.cuda.stream(ext):
            x_d.zero_()
        return pg.deflated_gmres(dA, b_d, x_d, cfg, d, ex)

    for _ in range(a.warmup):
        rep = step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    iters = 0
    launches = 0
    reps = []
    torch.cuda.synchronize()
    ev0.record(ext)
    for _ in range(a.steps):
        rep = step()
        iters += rep.total_inner
        launches += ex.launch_count()
        reps.append(rep)
    ev1.record(ext)
    torch.cuda.synchronize()
    clk = clocks.stop()
    t = ev0.elapsed_time(ev1) / 1e3
    if dist:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    value = iters / t
    ms_per_step = 1e3 * t / a.steps
    last = reps[-1]

    # ---- roofline: per-launch CUDA-event profile of one more solve -------------
    ex.set_profiling(True)
    prep = step()
    ex.set_profiling(False)
    cls, cyc, kk, ms = ex.profile()
    hist = d.history()
    rank_of = {0: 0}
    for h in hist:
        rank_of[h.restart + 1] = h.r
    steps_of = {}
    for r_, k_ in zip(prep.inner_restart, prep.inner_step):
        steps_of[int(r_)] = max(steps_of.get(int(r_), 0), int(k_) + 1)
    n_g = na ** 3 if world > 1 else n
    per = {}
    for c, y, k, t_ms in zip(cls, cyc, kk, ms):
        c, y, k = int(c), int(y), int(k)
        if c in (0, 1, 2) and (y not in steps_of or k >= steps_of[y]):
            continue  # early-exit launch after the cycle stopped
        rr = rank_of.get(y, 0)
        b = class_bytes(c, n, nnz_local, k, rr, steps_of.get(y, a.m),
                        os.environ.get("PGMRES_DCGS2", "1") != "0")
        e = per.setdefault(c, [0.0, 0.0, 0])
        e[0] += b
        e[1] += t_ms / 1e3
        e[2] += 1
    dc = os.environ.get("PGMRES_DCGS2", "1") != "0"
    names = {0: "step_spmv", 1: "cgs2_passB_update_dots",
             2: "dcgs2_update" if dc else "cgs2_passC_update", 3: "x_update",
             4: "ritz", 5: "push_sweeps", 6: "push_spmv", 7: "rotate", 8: "residual_spmv",
             9: "other"}
    prof_total = float(ms.sum()) / 1e3
    kernels = {names[c]: {"launches": v[2], "ms_total": round(1e3 * v[1], 3),
                          "share": round(v[1] / prof_total, 4) if prof_total else None,
                          "GBps": round(v[0] / v[1] / 1e9, 1) if v[0] and v[1] else None}
               for c, v in sorted(per.items())}
    peak, peak_kind = peaks()
    sp = per.get(0, [0, 1, 1])
    achieved = sp[0] / sp[1] / 1e9
    traffic = None  # measured DRAM bytes per launch of this kernel (ncu, profiles/)
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and a.m == 50 and world == 1:
        with open(tp) as f:
            traffic = json.load(f).get(f"n_e={a.ne}", {}).get(
                "k_spmv<DStepEpi>" if os.environ.get("PGMRES_DCGS2", "1") != "0"
                else "k_spmv<StepEpi>", {}).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "frac_dram": (round(traffic / (sp[1] / max(1, sp[2])) / 1e9 / peak, 4)
                              if traffic else None),
                "note": "achieved/frac use SURVEY 8(d) algorithmic bytes (12 B per nonzero); "
                        "the kernel stores 16-bit column deltas (10 B), so frac_dram "
                        "(ncu-measured DRAM bytes / launch time) is the physical fraction",
                "kernel": ("k_spmv<DStepEpi> (SpMV + AU c deflation + the DCGS2 step's dots)"
                           if dc else
                           "k_spmv<StepEpi> (SpMV + AU c deflation + CGS2 pass-1 dots)"),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "bytes_per_launch_avg": int(sp[0] / max(1, sp[2])),
                "launch_ms_avg": round(1e3 * sp[1] / max(1, sp[2]), 4)}
    tot_bytes = sum(v[0] for v in per.values())
    tot_time = sum(v[1] for v in per.values())
    solve_frac = (tot_bytes / prof_total / 1e9) / peak if prof_total else None

    # ---- standalone SpMV microbenchmark: y = A x with x ~ U(-1, 1)
    # from std::mt19937(11) as acceptance.cpp:437-443 (bit-identical stream)
    from paper_1906_04051_b200.rng import acceptance_vectors

    part = ex.partition() if world > 1 else {"row_begin": 0, "row_end": n}
    xv = acceptance_vectors(n_g if world > 1 else n)[0][part["row_begin"]:part["row_end"]]
    xs = torch.from_numpy(np.ascontiguousarray(xv)).cuda()
    ys = torch.empty_like(xs)
    for _ in range(3):
        ex.spmv(dA, xs, ys)
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    reps = 20
    s0.record(ext)
    for _ in range(reps):
        ex.spmv(dA, xs, ys)
    s1.record(ext)
    torch.cuda.synchronize()
    t_sp = s0.elapsed_time(s1) / 1e3 / reps
    if dist:
        tt = torch.tensor([t_sp], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_sp = float(tt.item())
    b_sp = 12 * nnz_local + 4 * (n + 1) + 16 * n
    spmv_micro = {"kernel": "k_spmv<PlainEpi> via pgm_spmv", "x": "U(-1,1), std::mt19937(11) "
                  "stream of acceptance.cpp:437-443", "launches": reps,
                  "us_per_launch": round(1e6 * t_sp, 2),
                  "GBps": round(b_sp / t_sp / 1e9, 1), "frac": round(b_sp / t_sp / 1e9 / peak, 4),
                  "bytes_per_launch": int(b_sp),
                  "note": "SURVEY 8(d) B_spmv = 12 nnz + 4(n+1) + 16n; the kernel stores "
                          "16-bit column deltas when gaps fit (10 B / nnz)"}
    del xs, ys

    # ---- e2e through the public API with host buffers --------------------------
    e2e = None
    if not a.no_e2e:
        rp_h = torch.empty(n + 1, dtype=torch.int32, pin_memory=True)
        ci_h = torch.empty(nnz_local, dtype=torch.int32, pin_memory=True)
        va_h = torch.empty(nnz_local, dtype=torch.float64, pin_memory=True)
        b_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
        x_h = torch.zeros(n, dtype=torch.float64, pin_memory=True)
        rp_h.copy_(A_d.row_ptr)
        ci_h.copy_(A_d.col_idx)
        va_h.copy_(A_d.values)
        b_h.copy_(b_d)
        A_h = pg.CsrMatrix(n, rp_h.numpy().view(np.uint32), ci_h.numpy().view(np.uint32),
                           va_h.numpy())
        bn, xn = b_h.numpy(), x_h.numpy()

        def e2e_step():
            d.reset()
            xn[:] = 0.0
            return pg.deflated_gmres(A_h, bn, xn, cfg, d, ex)

        e2e_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e_iters = 0
        e0.record(ext)
        for _ in range(a.steps):
            e_iters += e2e_step().total_inner
        e1.record(ext)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / 1e3
        if dist:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": round(e_iters / te, 2), "unit": "iter/s",
               "h2d_bytes_per_step": int(4 * (n + 1) + 12 * nnz_local + 16 * n),
               "d2h_bytes_per_step": int(8 * n),
               "ms_per_step": round(1e3 * te / a.steps, 3),
               "path": "deflated_gmres(CsrMatrix host arrays, numpy b, x) -> pgm_matrix_upload"
                       " + pgm_solve(host pointers); host arrays pinned"}
        # the drop-in's real input: pageable host memory (a std::vector in the
        # reference's CsrMatrix, numpy arrays here)
        del A_h
        A_p = pg.CsrMatrix(n, np.array(rp_h.numpy().view(np.uint32)),
                           np.array(ci_h.numpy().view(np.uint32)), np.array(va_h.numpy()))
        bp_, xp_ = np.array(bn), np.zeros(n)
        del rp_h, ci_h, va_h

        def pageable_step():
            d.reset()
            xp_[:] = 0.0
            return pg.deflated_gmres(A_p, bp_, xp_, cfg, d, ex)

        pageable_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ksteps = max(1, min(a.steps, 3))
        e0.record(ext)
        p_iters = 0
        for _ in range(ksteps):
            p_iters += pageable_step().total_inner
        e1.record(ext)
        torch.cuda.synchronize()
        tp_ = e0.elapsed_time(e1) / 1e3
        if dist:
            tt = torch.tensor([tp_], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tp_ = float(tt.item())
        e2e["pageable"] = {"value": round(p_iters / tp_, 2), "unit": "iter/s",
                           "steps": ksteps, "ms_per_step": round(1e3 * tp_ / ksteps, 3),
                           "path": "same call with pageable numpy arrays"}
        del A_p

    out = {
        "metric": metric_name(a), "value": round(value, 2), "unit": "iter/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: Bratu FEM Jacobian/residual assembled on the GPU by "
                "pgm_bratu_assemble (bit-identical to the reference assembly at u=0)",
        "config": workload(a, n_g, A_d.nnz if world == 1 else None),
        "gpu_launches": int(launches),
        "iterations_per_step": int(last.total_inner), "restarts_per_step": int(last.restarts),
        "final_relative": last.final_relative,
        "time_to_solution_s": round(ms_per_step / 1e3, 5),
        "roofline": roofline,
        "solve_roofline": {"frac": round(solve_frac, 4) if solve_frac else None,
                           "achieved_GBps": round(tot_bytes / prof_total / 1e9, 1)
                           if prof_total else None,
                           "note": "all hot-path kernels of one profiled solve, algorithmic "
                                   "bytes / summed kernel time"},
        "spmv_GBps": round(achieved, 1),
        "spmv_micro": spmv_micro,
        "kernels": kernels,
        "clocks": clk,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(a)
    if rank == 0:
        print(json.dumps(out), file=_OUT, flush=True)
    if dist:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def _ref_threads(na):
    return max(1, min(os.cpu_count() or 1, na))


def cpu_baseline(a):
    """The reference CPU solver (oracle/_ref: its own sources) on a bounded
    sample of the same system: 2 fixed restart cycles (2m inner iterations)."""
    from oracle import refbind as R

    na = 2 * a.ne + 1
    th = _ref_threads(na)
    A, b = R.first_newton_system(a.ne, LAMBDA, threads=th)
    cycles = 2 if a.ne <= 50 else 1  # ~2-40 s of CPU work
    r = R.solve(A, b, m=a.m, max_restarts=cycles, fixed_iterations=True, ne=a.ne, threads=th)
    return {"value": round(r.total_inner / r.wall_s, 3), "unit": "iter/s", "cores": th,
            "kind": "reference",
            "sample": f"{cycles} fixed restart cycle(s) ({r.total_inner} inner iterations) of deflated "
                      f"GMRES({a.m}) on the same n_e={a.ne} system, deterministic executor, "
                      f"{th} threads, {r.wall_s:.2f} s",
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(a):
    """The reference's own CPU solver (oracle/_ref: its sources compiled
    verbatim) on this host, all host threads, rank 0 only.  One step = the
    next restart cycle of ONE deflated GMRES(m) solve of the same system
    (x and the Deflator carried between steps, refbind.RefSession): the K
    timed steps are cycles 0..K-1 of the real solve from x0 = 0, so the
    deflation rank grows 0, 1, 2, ... as in the GPU arm's solve (r <= 20).
    The W warm-up cycles run first and are then discarded (x, Deflator reset).
    On n_e <= 50 one step is the complete tolerance solve instead.  A p = 1
    sample (one fixed cycle from x0 = 0, one thread) is reported beside it
    (bratu_bench speedup's baseline, bratu_bench.cpp:235-239)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import refbind as R

    na = 2 * a.ne + 1
    th = _ref_threads(na)
    t0 = time.perf_counter()
    S = R.RefSession(a.ne, LAMBDA, threads=th)
    setup_s = time.perf_counter() - t0
    nnz = int(S.nnz)
    full = a.ne <= 50
    if full:
        run = lambda: S.run(m=a.m, max_restarts=100, rel_tol=a.tol, fixed_iterations=False)  # noqa: E731
        desc = "the complete tolerance solve"
    else:
        run = lambda: S.run(m=a.m, max_restarts=1, fixed_iterations=True)  # noqa: E731
        desc = (f"the next restart cycle ({a.m} inner iterations) of one deflated solve "
                f"from x0 = 0 (timed steps = cycles 0..{a.steps - 1}, deflation rank "
                f"0..{min(a.steps - 1, 20)})")
    for _ in range(a.warmup):
        if full:
            S.reset()
        run()
    S.reset()
    iters, secs, ranks, rk = 0, 0.0, [], 0
    for _ in range(a.steps):
        if full:
            S.reset()
            rk = 0
        ranks.append(rk)  # deflation rank during this step's (first) cycle
        r = run()
        iters += r.total_inner
        secs += r.wall_s
        rk = int(r.rank)
    v = iters / secs
    del S
    p1 = None
    # p = 1 costs ~a cycle x the thread count: default on up to n_e = 80
    # (PGMRES_REF_P1=1 forces it, =0 skips it)
    p1_mode = os.environ.get("PGMRES_REF_P1", "auto")
    want_p1 = p1_mode == "1" or (p1_mode == "auto" and a.ne <= 80)
    if not want_p1:
        p1 = {"skipped": "p = 1 sample skipped above n_e = 80 to bound the run "
                         "(PGMRES_REF_P1=1 forces it; profiles/ holds a measured one)"}
    if want_p1 and th > 1:
        S1 = R.RefSession(a.ne, LAMBDA, threads=1, assembly_threads=th)
        r1 = S1.run(m=a.m, max_restarts=1, fixed_iterations=True)
        p1 = {"value": round(r1.total_inner / r1.wall_s, 4), "unit": "iter/s", "cores": 1,
              "sample": f"1 fixed restart cycle ({r1.total_inner} inner iterations) from "
                        f"x0 = 0 (deflation rank 0), {r1.wall_s:.2f} s",
              "all_cores_speedup": round(v / (r1.total_inner / r1.wall_s), 2)}
        del S1
    out = {"metric": metric_name(a), "value": round(v, 3), "unit": "iter/s", "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 * secs / a.steps, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic: Bratu FEM first Newton system (reference assembly)",
           "config": workload(a, na ** 3, nnz), "impl": "reference",
           "cpu_baseline": {"value": round(v, 3), "unit": "iter/s", "cores": th,
                            "kind": "reference",
                            "sample": f"{desc} per step; reference deflated_gmres (oracle/_ref), "
                                      f"deterministic executor, {th} threads; ranks per step "
                                      f"{ranks}",
                            "cpu_model": _cpu_model(), "p1": p1,
                            "setup_s": round(setup_s, 2)},
           "e2e": {"value": round(v, 3), "unit": "iter/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), file=_OUT, flush=True)


def self_launch(a) -> int:
    """`python bench.py --gpus N` outside torchrun: launch N ranks (one process
    per GPU, torch.distributed.run on 127.0.0.1) and forward rank 0's line."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < a.gpus:
        print(f"bench.py: --gpus {a.gpus} needs {a.gpus} GPUs, this node has {have}",
              file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    res = subprocess.run(cmd, stdout=subprocess.PIPE, text=True, env=env)
    for ln in res.stdout.splitlines():
        if ln.startswith("{"):
            print(ln, file=_OUT, flush=True)
    return res.returncode


def main():
    # exactly one JSON line on stdout: libraries (NCCL's version banner, ...)
    # print to fd 1, so fd 1 points at stderr until the result is printed
    saved = os.dup(1)
    os.dup2(2, 1)
    global _OUT
    _OUT = os.fdopen(saved, "w")
    a = parse()
    if a.impl == "pgmres" and a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    if a.impl == "reference":
        run_reference(a)
    else:
        run_gpu(a)


if __name__ == "__main__":
    main()
