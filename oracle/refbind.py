"""ctypes binding to oracle/_ref/libdgmres_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the reference's own C++ sources (compiled verbatim from
/root/reference/proj/src by oracle/Makefile) plus oracle/ref_driver.cpp.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module; the
product path (paper_1906_04051_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libdgmres_ref.so")
REF_SRC = "/root/reference/proj"

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class RefdConfig(C.Structure):
    _fields_ = [
        ("m", C.c_uint32), ("max_restarts", C.c_uint32), ("rel_tol", C.c_double),
        ("fixed_iterations", C.c_int32), ("breakdown_scale", C.c_double),
        ("use_deflation", C.c_int32), ("r_max", C.c_uint32), ("drop", C.c_uint32),
        ("accept_tol", C.c_double), ("inv_power_maxit", C.c_uint32),
        ("inv_power_tol", C.c_double), ("power_maxit", C.c_uint32),
        ("ne", C.c_uint32), ("threads", C.c_uint32), ("deterministic", C.c_int32),
        ("audit", C.c_int32),
    ]


class RefdReport(C.Structure):
    _fields_ = [
        ("beta0", C.c_double), ("restarts", C.c_uint32), ("total_inner", C.c_uint64),
        ("converged", C.c_int32), ("breakdown", C.c_int32), ("final_relative", C.c_double),
        ("n_inner", C.c_uint32), ("rank", C.c_uint32), ("skipped", C.c_uint32),
        ("n_hist", C.c_uint32), ("mu", C.c_double), ("ortho_max", C.c_double),
        ("tmatch_max", C.c_double), ("rank_max", C.c_uint32), ("wall_s", C.c_double),
    ]


class RefdNewtonRec(C.Structure):
    _fields_ = [
        ("iter", C.c_uint32), ("lam", C.c_double), ("update_inf", C.c_double),
        ("residual_norm", C.c_double), ("gmres_restarts", C.c_uint32),
        ("gmres_inner", C.c_uint64),
    ]


def build(quiet: bool = True) -> str:
    """Compile oracle/_ref from the reference sources (only where they exist)."""
    if not os.path.isdir(REF_SRC):
        if os.path.exists(LIB_PATH):
            return LIB_PATH
        raise RuntimeError("reference sources absent and oracle/_ref not prebuilt")
    subprocess.run(["make", "-s", "-j8", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.refd_last_error.restype = C.c_char_p
        L.refd_system_create.restype = C.c_void_p
        L.refd_system_create.argtypes = [C.c_uint32, C.c_double, C.c_void_p, C.c_uint32]
        L.refd_system_n.restype = C.c_uint32
        L.refd_system_n.argtypes = [C.c_void_p]
        L.refd_system_nnz.restype = C.c_uint64
        L.refd_system_nnz.argtypes = [C.c_void_p]
        L.refd_system_export.argtypes = [C.c_void_p, u32p, u32p, f64p, f64p]
        L.refd_system_free.argtypes = [C.c_void_p]
        L.refd_pattern_nnz.restype = C.c_uint64
        L.refd_pattern_nnz.argtypes = [C.c_uint32]
        L.refd_residual.argtypes = [C.c_uint32, C.c_double, f64p, f64p]
        L.refd_spmv.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, f64p, f64p, f64p]
        L.refd_executor_kernels.argtypes = [C.c_uint32, C.c_uint32, C.c_int32, C.c_uint32,
                                            C.c_uint64, u32p, u32p, f64p, f64p, f64p, f64p,
                                            f64p]
        L.refd_solve.argtypes = [C.POINTER(RefdConfig), C.c_uint32, C.c_uint64, u32p, u32p,
                                 f64p, f64p, f64p, C.POINTER(RefdReport),
                                 u32p, u32p, f64p, f64p, u32p, u32p, f64p, f64p,
                                 C.c_void_p, C.c_void_p]
        L.refd_deflator_create.restype = C.c_void_p
        L.refd_deflator_create.argtypes = [C.c_uint32, C.c_uint32]
        L.refd_deflator_free.argtypes = [C.c_void_p]
        L.refd_deflator_push.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u32p, u32p, f64p,
                                         f64p]
        L.refd_deflator_truncate.argtypes = [C.c_void_p]
        L.refd_deflator_observe.argtypes = [C.c_void_p, C.c_double]
        L.refd_deflator_reset.argtypes = [C.c_void_p]
        L.refd_deflator_apply.argtypes = [C.c_void_p, C.c_uint32, f64p, f64p]
        L.refd_deflator_state.argtypes = [C.c_void_p, C.POINTER(C.c_uint32),
                                          C.POINTER(C.c_double), C.POINTER(C.c_uint32),
                                          C.c_void_p, C.c_void_p, C.c_uint32]
        L.refd_newton.argtypes = [C.c_uint32, C.c_double, C.c_uint32, C.c_double, C.c_uint32,
                                  C.c_uint32, C.c_double, C.c_int32, C.c_int32, C.c_uint32,
                                  C.c_uint32, f64p, C.POINTER(RefdNewtonRec), C.c_uint32,
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.refd_session_create.restype = C.c_void_p
        L.refd_session_create.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32]
        L.refd_session_run.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double,
                                       C.c_int32, C.POINTER(RefdReport)]
        L.refd_session_reset.argtypes = [C.c_void_p]
        L.refd_session_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _err():
    return lib().refd_last_error().decode()


@dataclass
class Csr:
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)


def first_newton_system(ne: int, lam: float = 6.8, u=None, threads: int = 0):
    """J(u), -R(u) via the reference assembly (u = 0: the first Newton system)."""
    L = lib()
    up = None
    if u is not None:
        u = np.ascontiguousarray(u, dtype=np.float64)
        up = u.ctypes.data
    h = L.refd_system_create(ne, lam, up, threads)
    if not h:
        raise RuntimeError(_err())
    try:
        n, nnz = L.refd_system_n(h), L.refd_system_nnz(h)
        rp = np.empty(n + 1, np.uint32)
        ci = np.empty(nnz, np.uint32)
        v = np.empty(nnz, np.float64)
        rhs = np.empty(n, np.float64)
        L.refd_system_export(h, rp, ci, v, rhs)
    finally:
        L.refd_system_free(h)
    return Csr(n, rp, ci, v), rhs


def residual(ne: int, lam: float, u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    r = np.empty_like(u)
    if lib().refd_residual(ne, lam, u, r) != 0:
        raise RuntimeError(_err())
    return r


def spmv(A: Csr, x: np.ndarray) -> np.ndarray:
    y = np.empty(A.n, np.float64)
    lib().refd_spmv(A.n, A.nnz, A.row_ptr, A.col_idx, A.values,
                    np.ascontiguousarray(x, np.float64), y)
    return y


def executor_kernels(ne, threads, deterministic, A: Csr, x, w):
    y = np.empty(A.n)
    d = np.empty(2)
    rc = lib().refd_executor_kernels(ne, threads, int(deterministic), A.n, A.nnz, A.row_ptr,
                                     A.col_idx, A.values, np.ascontiguousarray(x, np.float64),
                                     np.ascontiguousarray(w, np.float64), y, d)
    if rc:
        raise RuntimeError(_err())
    return y, d[0], d[1]


@dataclass
class RefResult:
    x: np.ndarray
    beta0: float
    restarts: int
    total_inner: int
    converged: bool
    breakdown: bool
    final_relative: float
    inner_restart: np.ndarray
    inner_step: np.ndarray
    monitored: np.ndarray
    explicit_residual: np.ndarray
    rank: int
    mu: float
    skipped: int
    hist_restart: np.ndarray
    hist_r: np.ndarray
    hist_mu: np.ndarray
    hist_theta: np.ndarray
    T: np.ndarray | None
    U: np.ndarray | None
    ortho_max: float
    tmatch_max: float
    rank_max: int
    wall_s: float
    extra: dict = field(default_factory=dict)


def solve(A: Csr, b, x0=None, *, m=50, max_restarts=100, rel_tol=1e-8, fixed_iterations=False,
          breakdown_scale=1e-14, deflation=True, r_max=20, drop=1, accept_tol=1e-8,
          inv_power_maxit=500, inv_power_tol=1e-10, power_maxit=200, ne=0, threads=0,
          deterministic=True, audit=False, want_basis=False) -> RefResult:
    """deflated_gmres (deflation=True) or gmres_restarted(opA, nullptr) on CSR A."""
    L = lib()
    n = A.n
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64, copy=True)
    cfg = RefdConfig(m, max_restarts, rel_tol, int(fixed_iterations), breakdown_scale,
                     int(deflation), r_max, drop, accept_tol, inv_power_maxit, inv_power_tol,
                     power_maxit, ne, threads, int(deterministic), int(audit))
    cap = max(1, m * max_restarts)
    ir = np.zeros(cap, np.uint32)
    ik = np.zeros(cap, np.uint32)
    im = np.zeros(cap)
    ex = np.zeros(max(1, max_restarts))
    hr = np.zeros(max(1, max_restarts), np.uint32)
    hrr = np.zeros(max(1, max_restarts), np.uint32)
    hmu = np.zeros(max(1, max_restarts))
    hth = np.zeros(max(1, max_restarts))
    T = np.zeros((r_max + 1) ** 2)
    U = np.zeros(n * (r_max + 1)) if want_basis else None
    rep = RefdReport()
    rc = L.refd_solve(C.byref(cfg), n, A.nnz, A.row_ptr, A.col_idx, A.values, b, x,
                      C.byref(rep), ir, ik, im, ex, hr, hrr, hmu, hth, T.ctypes.data,
                      U.ctypes.data if U is not None else None)
    if rc:
        raise RuntimeError(_err())
    ni, nh, r = rep.n_inner, rep.n_hist, rep.rank
    return RefResult(
        x=x, beta0=rep.beta0, restarts=rep.restarts, total_inner=rep.total_inner,
        converged=bool(rep.converged), breakdown=bool(rep.breakdown),
        final_relative=rep.final_relative, inner_restart=ir[:ni].copy(),
        inner_step=ik[:ni].copy(), monitored=im[:ni].copy(),
        explicit_residual=ex[:rep.restarts].copy(), rank=r, mu=rep.mu, skipped=rep.skipped,
        hist_restart=hr[:nh].copy(), hist_r=hrr[:nh].copy(), hist_mu=hmu[:nh].copy(),
        hist_theta=hth[:nh].copy(),
        T=T[: r * r].reshape(r, r, order="F").copy() if r else None,
        U=U[: n * r].reshape(r, n).T.copy() if (U is not None and r) else None,
        ortho_max=rep.ortho_max, tmatch_max=rep.tmatch_max, rank_max=rep.rank_max,
        wall_s=rep.wall_s)


class RefSession:
    """A reference deflated solve advanced one call at a time (oracle/_ref
    refd_session_*): run(max_restarts=1, fixed_iterations=True) is the next
    restart cycle of one solve, x and the Deflator carried over."""

    def __init__(self, ne: int, lam: float = 6.8, threads: int = 0, r_max: int = 20,
                 assembly_threads: int | None = None):
        L = lib()
        h = L.refd_system_create(ne, lam, None,
                                 threads if assembly_threads is None else assembly_threads)
        if not h:
            raise RuntimeError(_err())
        try:
            self.n = L.refd_system_n(h)
            self.nnz = L.refd_system_nnz(h)
            self.h = L.refd_session_create(h, ne, threads, r_max)
        finally:
            L.refd_system_free(h)
        if not self.h:
            raise RuntimeError(_err())

    def run(self, m=50, max_restarts=1, rel_tol=1e-10, fixed_iterations=True):
        rep = RefdReport()
        if lib().refd_session_run(self.h, m, max_restarts, rel_tol, int(fixed_iterations),
                                  C.byref(rep)):
            raise RuntimeError(_err())
        return rep

    def reset(self):
        lib().refd_session_reset(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().refd_session_free(self.h)
            self.h = None


class RefDeflator:
    """Direct handle on the reference Deflator (push_vector / truncate / apply)."""

    def __init__(self, r_max=20, drop=1):
        self.h = lib().refd_deflator_create(r_max, drop)
        if not self.h:
            raise ValueError(_err())

    def __del__(self):
        if getattr(self, "h", None):
            lib().refd_deflator_free(self.h)
            self.h = None

    def push(self, A: Csr, cand) -> bool:
        return bool(lib().refd_deflator_push(self.h, A.n, A.nnz, A.row_ptr, A.col_idx,
                                             A.values, np.ascontiguousarray(cand, np.float64)))

    def truncate(self):
        lib().refd_deflator_truncate(self.h)

    def observe(self, v):
        lib().refd_deflator_observe(self.h, v)

    def reset(self):
        lib().refd_deflator_reset(self.h)

    def apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        w = np.empty_like(v)
        lib().refd_deflator_apply(self.h, v.size, v, w)
        return w

    def state(self, n):
        r, mu, sk = C.c_uint32(), C.c_double(), C.c_uint32()
        lib().refd_deflator_state(self.h, C.byref(r), C.byref(mu), C.byref(sk), None, None, n)
        rr = r.value
        T = np.zeros(max(1, rr * rr))
        U = np.zeros(max(1, rr * n))
        lib().refd_deflator_state(self.h, C.byref(r), C.byref(mu), C.byref(sk), T.ctypes.data,
                                  U.ctypes.data, n)
        return dict(rank=rr, mu=mu.value, skipped=sk.value,
                    T=T[: rr * rr].reshape(rr, rr, order="F"),
                    U=U[: rr * n].reshape(rr, n).T if rr else np.zeros((n, 0)))


def newton(ne, lam=6.8, *, max_iters=30, update_tol=1e-8, m=50, max_restarts=100,
           rel_tol=1e-10, use_deflation=True, continuation=False, continuation_steps=4,
           threads=0):
    n = (2 * ne + 1) ** 3
    u = np.zeros(n)
    cap = max_iters * max(1, continuation_steps)
    recs = (RefdNewtonRec * cap)()
    nrec, conv, fres, wall = C.c_uint32(), C.c_int32(), C.c_double(), C.c_double()
    rc = lib().refd_newton(ne, lam, max_iters, update_tol, m, max_restarts, rel_tol,
                           int(use_deflation), int(continuation), continuation_steps, threads,
                           u, recs, cap, C.byref(nrec), C.byref(conv), C.byref(fres),
                           C.byref(wall))
    if rc:
        raise RuntimeError(_err())
    its = [dict(iter=r.iter, lam=r.lam, update_inf=r.update_inf,
                residual_norm=r.residual_norm, gmres_restarts=r.gmres_restarts,
                gmres_inner=r.gmres_inner) for r in recs[: nrec.value]]
    return dict(u=u, iters=its, converged=bool(conv.value), final_residual=fres.value,
                wall_s=wall.value)


def diag_csr(d) -> Csr:
    d = np.asarray(d, np.float64)
    n = d.size
    return Csr(n, np.arange(n + 1, dtype=np.uint32), np.arange(n, dtype=np.uint32), d.copy())
