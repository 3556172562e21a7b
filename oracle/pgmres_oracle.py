"""CPU restatement of the reference's deflated GMRES(m) — TEST INFRASTRUCTURE ONLY.

This is the checker, never the product: only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg may import it.  The product path
(paper_1906_04051_b200) never calls into oracle/ and fails loudly if its CUDA
library is missing.

Each function restates one reference routine (file:line into
/root/reference/proj) in numpy/scipy:

  spmv ............... src/sparse.cpp:9-19 (ascending-column row sums)
  Workspace .......... src/gmres.cpp:9-115 (begin_cycle, arnoldi_step with
                       conditional second MGS sweep, Givens update, back-sub,
                       correction)
  gmres_restarted .... src/gmres.cpp:132-218
  Deflator ........... src/deflation.cpp:85-279 (apply, observe_ritz,
                       push_vector, truncate, refresh_lu, update_from_restart,
                       hessenberg_block, smallest/largest Ritz iterations)
  deflated_gmres ..... src/deflation.cpp:281-291

`orth="cgs2"` switches arnoldi_step to the unconditional two-pass classical
Gram-Schmidt the device path runs (SURVEY.md §8(c) shows it keeps parity), so
tests can separate "algorithm variant" from "rounding" differences.
`orth="dcgs2"` is a numerical prototype of delayed CGS2 (a
candidate device algorithm): the SpMV runs on the lagged once-orthogonalised
vector and the reorthogonalisation + Arnoldi correction happen one step
later; tests/test_oracle.py measures its parity before any device code.

Parity of this restatement is PINNED against the reference itself: the
golden fixtures in tests/golden/ are produced by oracle/_ref (the reference's
own sources compiled verbatim, see oracle/Makefile and
tests/golden/make_golden.py), and tests/test_oracle.py checks this module
against them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


class GmresError(RuntimeError):
    """Mirrors the std::runtime_error messages of src/gmres.cpp."""


def csr_matrix(n, row_ptr, col_idx, values):
    return sp.csr_matrix((np.asarray(values, np.float64), np.asarray(col_idx, np.int64),
                          np.asarray(row_ptr, np.int64)), shape=(n, n))


def spmv(A: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    """y = A x, each row accumulated in ascending column order (sparse.cpp:9-19).

    scipy's csr_matvec is the same sequential loop, so this is bitwise equal
    to the reference for sorted CSR."""
    return A @ x


@dataclass
class GmresConfig:  # include/dgmres/gmres.hpp:17-23
    m: int = 50
    max_restarts: int = 100
    rel_tol: float = 1e-8
    fixed_iterations: bool = False
    breakdown_scale: float = 1e-14


@dataclass
class DeflationConfig:  # include/dgmres/deflation.hpp:15-22
    r_max: int = 20
    drop: int = 1
    accept_tol: float = 1e-8
    inv_power_maxit: int = 500
    inv_power_tol: float = 1e-10
    power_maxit: int = 200


@dataclass
class GmresReport:  # include/dgmres/gmres.hpp:31-44
    beta0: float = 0.0
    inner: list = field(default_factory=list)  # (restart, inner, monitored)
    explicit_residual: list = field(default_factory=list)
    restarts: int = 0
    total_inner: int = 0
    converged: bool = False
    breakdown: bool = False
    final_relative: float = 0.0

    @property
    def monitored(self):
        return np.array([r[2] for r in self.inner])


class Workspace:
    """GmresWorkspace (gmres.hpp:49-92, gmres.cpp:9-115)."""

    def __init__(self, n, m, orth="mgs"):
        if m == 0:
            raise ValueError("GmresWorkspace: m must be positive")  # gmres.cpp:10
        self.n, self.m, self.orth = n, m, orth
        self.V = np.zeros((m + 1, n))
        self.h_rot = np.zeros((m + 1, m), order="F")
        self.h_orig = np.zeros((m + 1, m), order="F")
        self.g = np.zeros(m + 1)
        self.cs = np.zeros(m)
        self.sn = np.zeros(m)

    def begin_cycle(self, r, beta):  # gmres.cpp:21-26
        self.V[0] = r
        if beta > 0.0:
            self.V[0] *= 1.0 / beta
        self.g[:] = 0.0
        self.g[0] = beta

    def arnoldi_step(self, opA, opM, k):  # gmres.cpp:28-65
        w = opA(opM(self.V[k])) if opM is not None else opA(self.V[k])
        w = np.array(w, copy=True)
        if self.orth == "cgs2":
            h1 = self.V[: k + 1] @ w
            w -= h1 @ self.V[: k + 1]
            h2 = self.V[: k + 1] @ w
            w -= h2 @ self.V[: k + 1]
            self.h_rot[: k + 1, k] = h1 + h2
            self.h_orig[: k + 1, k] = h1 + h2
            hnext = math.sqrt(float(w @ w))
        else:
            for i in range(k + 1):  # modified Gram-Schmidt sweep
                h = float(self.V[i] @ w)
                self.h_rot[i, k] = h
                self.h_orig[i, k] = h
                w -= h * self.V[i]
            hnext = math.sqrt(float(w @ w))
            mass = hnext * hnext + float(np.sum(self.h_orig[: k + 1, k] ** 2))
            if hnext > 0.0 and hnext * hnext < 0.5 * mass:  # conditional 2nd sweep
                for i in range(k + 1):
                    c = float(self.V[i] @ w)
                    self.h_rot[i, k] += c
                    self.h_orig[i, k] += c
                    w -= c * self.V[i]
                hnext = math.sqrt(float(w @ w))
        self.h_rot[k + 1, k] = hnext
        self.h_orig[k + 1, k] = hnext
        if hnext > 0.0:
            self.V[k + 1] = w * (1.0 / hnext)
        return hnext

    def apply_rotations_and_update(self, k):  # gmres.cpp:67-90
        H = self.h_rot
        for i in range(k):
            hi, hj = H[i, k], H[i + 1, k]
            H[i, k] = self.cs[i] * hi + self.sn[i] * hj
            H[i + 1, k] = -self.sn[i] * hi + self.cs[i] * hj
        a, b = H[k, k], H[k + 1, k]
        r = math.hypot(a, b)
        if r == 0.0:
            self.cs[k], self.sn[k] = 1.0, 0.0
        else:
            self.cs[k], self.sn[k] = a / r, b / r
        H[k, k] = r
        H[k + 1, k] = 0.0
        self.g[k + 1] = -self.sn[k] * self.g[k]
        self.g[k] = self.cs[k] * self.g[k]
        return abs(self.g[k + 1])

    def solve_least_squares(self, k):  # gmres.cpp:92-107
        y = self.g[:k].copy()
        for i in range(k - 1, -1, -1):
            d = self.h_rot[i, i]
            if d == 0.0:
                raise GmresError("gmres: singular projection in least squares")
            s = y[i] - float(self.h_rot[i, i + 1:k] @ y[i + 1:k])
            y[i] = s / d
        return y

    def correction(self, y):  # gmres.cpp:109-115
        return y @ self.V[: y.size] if y.size else np.zeros(self.n)

    def hess(self, i, j):
        return self.h_orig[i, j]


def _dcgs2_cycle(ws, opA, opM, cfg, rep, restart, beta_cycle):
    """One restart cycle of delayed CGS2 (one global reduction per step).

    Step k runs the operator on the lagged vector u_k (orthogonalised once
    against q_0..q_{k-1}) and, from ONE batch of dot products
    [Q^T u_k, u_k.u_k, Q^T w, u_k.w], finishes u_k's second pass (column k-1 of
    H gets + a, h_{k,k-1} = beta) and forms the first pass of the next vector
    through the Arnoldi relation A M^-1 Q = Q H.  Column k-1's Givens update and
    termination tests therefore happen at step k; the cycle end needs one
    closing reduction (no operator application)."""
    m = ws.m
    op = (lambda v: opA(opM(v))) if opM is not None else opA
    Q = ws.V
    steps, lucky = 0, False
    # step 0: q_0 is final
    w = np.array(op(Q[0]), copy=True)
    h1 = np.array([float(Q[0] @ w)])
    u = w - h1[0] * Q[0]
    ws.h_orig[0, 0] = h1[0]
    for k in range(1, m + 1):
        a = Q[:k] @ u
        alpha = float(u @ u)
        if k < m:
            w = np.array(op(u), copy=True)
            b = Q[:k] @ w
            gamma = float(u @ w)
        beta = math.sqrt(max(alpha - float(a @ a), 0.0))
        if not math.isfinite(beta):
            raise GmresError(f"gmres: non-finite Arnoldi coefficient at restart {restart}, "
                             f"step {k - 1}")
        # column k-1 complete: second-pass coefficients and the subdiagonal
        ws.h_orig[:k, k - 1] += a
        ws.h_orig[k, k - 1] = beta
        ws.h_rot[: k + 1, k - 1] = ws.h_orig[: k + 1, k - 1]
        mon = ws.apply_rotations_and_update(k - 1)
        rep.inner.append((restart, k - 1, mon))
        steps = k
        if beta < cfg.breakdown_scale * beta_cycle:
            lucky = True
            break
        if not cfg.fixed_iterations and mon <= cfg.rel_tol * rep.beta0:
            break
        if k == m:
            break
        q = (u - a @ Q[:k]) / beta
        Q[k] = q
        # A M^-1 q_k = (w - Q_{k+1} H[:k+1, :k] a) / beta
        Ha = ws.h_orig[: k + 1, :k] @ a
        qw = (gamma - float(a @ b)) / beta
        h1 = np.empty(k + 1)
        h1[:k] = (b - Ha[:k]) / beta
        h1[k] = (qw - Ha[k]) / beta
        wk = (w - Ha @ Q[: k + 1]) / beta
        u = wk - h1 @ Q[: k + 1]
        ws.h_orig[: k + 1, k] = h1
    return steps, lucky


def gmres_restarted(opA, opM, b, x, cfg: GmresConfig, hook=None, orth="mgs"):
    """Right-preconditioned restarted GMRES (gmres.cpp:132-218).  x is updated."""
    n = b.size
    rep = GmresReport()
    ws = Workspace(n, cfg.m, orth)

    def refresh():
        r = b - opA(x)
        return r, math.sqrt(float(r @ r))

    r, beta = refresh()
    rep.beta0 = beta
    if not math.isfinite(beta):
        raise GmresError("gmres: initial residual is not finite")
    if beta == 0.0:
        rep.converged = True
        return rep
    for restart in range(cfg.max_restarts):
        ws.begin_cycle(r, beta)
        steps, lucky = 0, False
        if orth == "dcgs2":
            steps, lucky = _dcgs2_cycle(ws, opA, opM, cfg, rep, restart, beta)
        for k in range(cfg.m if orth != "dcgs2" else 0):
            h = ws.arnoldi_step(opA, opM, k)
            if not math.isfinite(h):
                raise GmresError(f"gmres: non-finite Arnoldi coefficient at restart "
                                 f"{restart}, step {k}")
            mon = ws.apply_rotations_and_update(k)
            rep.inner.append((restart, k, mon))
            steps = k + 1
            if h < cfg.breakdown_scale * beta:
                lucky = True
                break
            if not cfg.fixed_iterations and mon <= cfg.rel_tol * rep.beta0:
                break
        y = ws.solve_least_squares(steps)
        z = ws.correction(y)
        x += opM(z) if opM is not None else z
        if hook is not None:
            hook(ws, steps, restart)
        r, beta = refresh()
        rep.explicit_residual.append(beta)
        rep.restarts = restart + 1
        rep.total_inner += steps
        if not math.isfinite(beta):
            raise GmresError(f"gmres: non-finite residual after restart {restart}")
        if lucky:
            rep.breakdown = rep.converged = True
            break
        if not cfg.fixed_iterations and beta <= cfg.rel_tol * rep.beta0:
            rep.converged = True
            break
        if beta == 0.0:
            rep.converged = True
            break
    rep.final_relative = beta / rep.beta0 if rep.beta0 > 0.0 else 0.0
    if not rep.converged and not cfg.fixed_iterations:
        rep.converged = beta <= cfg.rel_tol * rep.beta0
    return rep


# ---------------------------------------------------------------------------
# Deflation preconditioner (deflation.cpp)

def hessenberg_block(ws: Workspace, k):  # deflation.cpp:15-22
    h = np.zeros((k, k))
    for j in range(k):
        top = min(k - 1, j + 1)
        h[: top + 1, j] = ws.h_orig[: top + 1, j]
    return h


def smallest_ritz_pair(h, maxit, tol):  # deflation.cpp:31-54 (inverse power)
    k = h.shape[0]
    scale = float(np.linalg.norm(h))
    if not (scale > 0.0) or not math.isfinite(scale):
        return False, 0.0, None
    lu = sla.lu_factor(h, check_finite=False)
    z = np.full(k, 1.0 / math.sqrt(k))
    val, vec = 0.0, None
    for _ in range(maxit):
        nxt = sla.lu_solve(lu, z, check_finite=False)
        nz = float(np.linalg.norm(nxt))
        if not math.isfinite(nz) or nz == 0.0:
            return False, val, vec
        z = nxt / nz
        hz = h @ z
        theta = float(z @ hz)
        resid = float(np.linalg.norm(hz - theta * z))
        val, vec = theta, z
        if resid <= tol * scale:
            return True, val, vec
    return False, val, vec


def largest_ritz_value(h, maxit, tol):  # deflation.cpp:57-82 (power iteration)
    k = h.shape[0]
    scale = float(np.linalg.norm(h))
    if not (scale > 0.0) or not math.isfinite(scale):
        return False, 0.0
    z = np.full(k, 1.0 / math.sqrt(k))
    val, have = 0.0, False
    for _ in range(maxit):
        nxt = h @ z
        nz = float(np.linalg.norm(nxt))
        if not math.isfinite(nz) or nz == 0.0:
            return False, val
        z = nxt / nz
        hz = h @ z
        theta = float(z @ hz)
        resid = float(np.linalg.norm(hz - theta * z))
        val, have = theta, True
        if resid <= tol * scale:
            return True, val
    return have, val  # a non-converged iterate still estimates |mu| (:78-80)


class Deflator:
    """M^{-1} = I + U(|mu| T^{-1} - I)U^T (deflation.hpp:35-89)."""

    def __init__(self, cfg: DeflationConfig | None = None):
        self.cfg = cfg or DeflationConfig()
        if self.cfg.r_max == 0:
            raise ValueError("deflation: r_max must be positive")
        if self.cfg.drop == 0:
            raise ValueError("deflation: drop must be positive")
        self.U = None
        self.AU = None
        self.T = None
        self.r = 0
        self.mu = 0.0
        self.skipped = 0
        self.history = []
        self._lu = None

    def reset(self):  # deflation.cpp:91-96
        self.r, self.mu, self.skipped, self.history = 0, 0.0, 0, []

    def apply(self, v):  # deflation.cpp:104-117
        w = np.array(v, copy=True)
        if self.r == 0:
            return w
        Ur = self.U[:, : self.r]
        t = Ur.T @ v
        s = sla.lu_solve(self._lu, t, check_finite=False)
        coeff = abs(self.mu) * s - t
        return w + Ur @ coeff

    def observe_ritz(self, value):  # deflation.cpp:119-121
        if math.isfinite(value) and abs(value) > abs(self.mu):
            self.mu = value

    def push_vector(self, cand, opA):  # deflation.cpp:123-184
        n = cand.size
        if self.U is None or self.U.shape[0] != n:
            self.U = np.zeros((n, self.cfg.r_max + 1), order="F")
            self.AU = np.zeros((n, self.cfg.r_max + 1), order="F")
            self.T = np.zeros((self.cfg.r_max + 1, self.cfg.r_max + 1), order="F")
            self.r = 0
        if self.r >= self.U.shape[1]:
            self.skipped += 1
            return False
        u = np.array(cand, np.float64, copy=True)
        norm_in = math.sqrt(float(u @ u))
        if not (norm_in > 0.0) or not math.isfinite(norm_in):
            self.skipped += 1
            return False
        if self.r > 0:
            Ur = self.U[:, : self.r]
            for _ in range(2):
                u -= Ur @ (Ur.T @ u)
        norm_left = math.sqrt(float(u @ u))
        if not (norm_left >= self.cfg.accept_tol * norm_in):
            self.skipped += 1
            return False
        u *= 1.0 / norm_left
        j = self.r
        self.U[:, j] = u
        self.AU[:, j] = opA(u)
        if j > 0:
            self.T[:j, j] = self.U[:, :j].T @ self.AU[:, j]
            self.T[j, :j] = self.U[:, j] @ self.AU[:, :j]
        self.T[j, j] = float(self.U[:, j] @ self.AU[:, j])
        self.r += 1
        while self.r > self.cfg.r_max:
            before = self.r
            self.truncate()
            if self.r == before:
                break
        self._refresh_lu()
        return True

    def truncate(self):  # deflation.cpp:186-225
        dropped = 0
        while dropped < self.cfg.drop and self.r > 1:
            r = self.r
            tb = self.T[:r, :r].copy()
            vals, vecs = np.linalg.eig(tb)
            dom = int(np.argmax(np.abs(vals)))
            v = vecs[:, dom].real.copy()
            if np.linalg.norm(v) <= 1e-12:
                v = vecs[:, dom].imag.copy()
            vn = float(np.linalg.norm(v))
            if not (vn > 0.0) or not math.isfinite(vn):
                return
            v /= vn
            hv = v.copy()
            sigma = 1.0 if v[r - 1] >= 0.0 else -1.0
            hv[r - 1] += sigma
            denom = float(hv @ hv)
            p = np.eye(r)
            if denom > 0.0:
                p -= (2.0 / denom) * np.outer(hv, hv)
            q = p[:, : r - 1]
            self.U[:, : r - 1] = self.U[:, :r] @ q
            self.AU[:, : r - 1] = self.AU[:, :r] @ q
            self.T[: r - 1, : r - 1] = q.T @ tb @ q
            self.r = r - 1
            dropped += 1
        self._refresh_lu()

    def _refresh_lu(self):  # deflation.cpp:227-230
        if self.r:
            self._lu = sla.lu_factor(self.T[: self.r, : self.r], check_finite=False)

    def update_from_restart(self, ws: Workspace, steps, restart, opA):  # deflation.cpp:232-264
        k = steps
        theta = float("nan")
        added = False
        if k > 0:
            h = hessenberg_block(ws, k)
            ok, big = largest_ritz_value(h, self.cfg.power_maxit, self.cfg.inv_power_tol)
            if ok:
                self.observe_ritz(big)
            ok, val, vec = smallest_ritz_pair(h, self.cfg.inv_power_maxit,
                                              self.cfg.inv_power_tol)
            if ok:
                theta = val
                u = vec @ ws.V[:k]
                added = self.push_vector(u, opA)
            else:
                self.skipped += 1
        else:
            self.skipped += 1
        self.history.append((restart, self.r, self.mu, theta))
        return added

    def T_block(self):
        return self.T[: self.r, : self.r].copy() if self.r else np.zeros((0, 0))


def deflated_gmres(A, b, x, cfg: GmresConfig, d: Deflator, orth="mgs"):
    """deflation.cpp:281-291: opA = spmv, opM = d.apply, hook = harvest."""
    opA = lambda v: spmv(A, v)  # noqa: E731
    return gmres_restarted(opA, d.apply, b, x, cfg,
                           hook=lambda ws, s, rs: d.update_from_restart(ws, s, rs, opA),
                           orth=orth)
