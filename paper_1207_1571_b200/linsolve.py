"""Jacobi-preconditioned CG and BiCGStab on the device (reference: linsolve.py).

Each solve is one persistent cooperative kernel in libfvb (fvb_op_cg /
fvb_op_bicgstab): same normalised residual ||b - Ax|| / max(||b||, 1e-30),
same convergence check on entry and right after each residual update,
same breakdown tests and messages, initial guess left untouched, solution
returned as a new array.  Dot products are deterministic tree reductions
(they differ from OpenBLAS ddot only by rounding).
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import context_for
from .errors import SolverError

STAGES = ("smvp", "daxpy", "dot", "reduction", "precond", "other")
RESIDUAL_FLOOR = 1e-30
BREAKDOWN_EPS = 1e-300

__all__ = ["STAGES", "SolverError", "SolveConfig", "SolveReport", "cg", "bicgstab",
           "bicgstab_batched", "residual_norm", "jacobi_apply"]


@dataclass
class SolveConfig:
    tolerance: float = 1e-7
    abs_tolerance: float = 0.0
    max_iters: int = 1000
    record_stages: bool = False

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")


@dataclass
class SolveReport:
    iterations: int
    initial_residual: float
    final_residual: float
    converged: bool
    wall_time: float = 0.0
    stage_times: dict = field(default_factory=dict)


def stage_times_of(r, record):
    """StageTimer buckets (linsolve.py:18-79) from the persistent kernel's
    device timers: the SpMV passes carry the fused p-update/preconditioner,
    the vector passes carry z = r/D and the dot partials, the grid/team
    reductions are "reduction"; setup and launch are the "other" remainder."""
    if not record:
        return {}
    d = dict.fromkeys(STAGES, 0.0)
    d["smvp"] = float(r.t_smvp)
    d["daxpy"] = float(r.t_daxpy)
    d["reduction"] = float(r.t_reduction)
    d["other"] = max(float(r.wall_time) - d["smvp"] - d["daxpy"] - d["reduction"], 0.0)
    return d


def _report(r, cfg):
    return SolveReport(iterations=int(r.iterations), initial_residual=float(r.initial_residual),
                       final_residual=float(r.final_residual), converged=bool(r.converged),
                       wall_time=float(r.wall_time), stage_times=stage_times_of(r, cfg.record_stages))


def _solve(fn, A, b, x0, cfg, ncomp=1):
    p = A.pattern
    ctx = context_for(None, None, p)
    V = _lib.f64(A.V)
    crs = _lib.f64(A.crs_val)
    bb = _lib.f64(b)
    xx0 = _lib.f64(x0)
    x = np.empty_like(bb)
    P = _lib.ptr
    reps = (_lib.SolveReportC * ncomp)()
    args = [ctx.h]
    if ncomp != 1 or fn is _lib.lib.fvb_op_bicgstab_batched:
        args.append(ncomp)
    rc = fn(*args, P(V), P(crs), P(bb), P(xx0), P(x), float(cfg.tolerance),
            float(cfg.abs_tolerance), int(cfg.max_iters), reps)
    _lib.check(rc, SolverError)
    return x, [_report(reps[i], cfg) for i in range(ncomp)]


def cg(A, b, x0, cfg: SolveConfig):
    """Jacobi-PCG (linsolve.py:102-172); A must be symmetric in values."""
    x, reps = _solve(_lib.lib.fvb_op_cg, A, b, x0, cfg)
    return x, reps[0]


def bicgstab(A, b, x0, cfg: SolveConfig):
    """Jacobi-PBiCGStab with shadow-residual restart (linsolve.py:175-282)."""
    x, reps = _solve(_lib.lib.fvb_op_bicgstab, A, b, x0, cfg)
    return x, reps[0]


def bicgstab_batched(A, B, X0, cfg: SolveConfig):
    """Three right-hand sides (columns of B, shape (n, 3)) against one matrix,
    sharing every matrix read; each column keeps its own scalars and stop
    rule, so the result equals three independent bicgstab calls."""
    Bs = np.ascontiguousarray(np.asarray(B, dtype=float).T)
    Xs = np.ascontiguousarray(np.asarray(X0, dtype=float).T)
    x, reps = _solve(_lib.lib.fvb_op_bicgstab_batched, A, Bs.reshape(-1), Xs.reshape(-1), cfg,
                     ncomp=Bs.shape[0])
    return x.reshape(Bs.shape).T.copy(), reps


def jacobi_apply(diag, r):
    """z = r / diag, the Jacobi preconditioner as a standalone helper
    (linsolve.py:82-87; the device solvers fuse it into their passes).
    SolverError names the first zero diagonal row, as the solvers do."""
    diag = np.asarray(diag, dtype=float)
    bad = np.flatnonzero(diag == 0.0)
    if bad.size:
        raise SolverError(f"singular preconditioner: zero diagonal at row {int(bad[0])}")
    return np.asarray(r, dtype=float) / diag


def residual_norm(A, x, b):
    """||b - A x|| / max(||b||, 1e-30) with the device SpMV."""
    from .sparse import smvp

    return float(np.linalg.norm(b - smvp(A, x)) / max(np.linalg.norm(b), RESIDUAL_FLOOR))
