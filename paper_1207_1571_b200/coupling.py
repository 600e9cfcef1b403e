"""PISO time steps and SIMPLE sweeps, device-resident (reference: coupling.py).

``init_state`` uploads the mesh, geometry-derived face tables, pattern and
boundary tables to one libfvb context; from then on u, p and the face
flux live in HBM and one C-ABI call (fvb_piso_step / fvb_simple_sweep)
advances a whole step: momentum assembly, three batched BiCGStab solves,
n_correctors x (HbyA, pressure assembly, PCG, flux and velocity
correction), with no per-iteration host round trip.

The RunState keeps the reference's bookkeeping (outer, t, cum_iters,
residual_log, wall, ops, stage_times) and exposes u.values, p.values and
flux as host views that are downloaded lazily; a view handed to the user
(or assigned by the user) is treated as authoritative and uploaded again
before the next device step, so in-place host edits behave as in the
reference.
"""

import ctypes as C
import time
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from .device import DeviceContext, bc_table
from .errors import CouplingError
from .fvm import (
    Field,
    SchemeConfig,
    bc_from_tuple,
    is_value_bc,
    make_scalar,
    make_vector,
)
from .linsolve import SolveConfig, SolveReport, stage_times_of
from .mesh import compute_geometry
from .sparse import build_pattern

__all__ = ["CouplingError", "CouplingConfig", "RunState", "init_state", "simple_outer_iteration",
           "piso_time_step", "continuity_error", "kinetic_energy", "run_case",
           "RESIDUAL_COLUMNS"]

RESIDUAL_COLUMNS = ("solver", "field", "outer_iter", "inner_iters", "initial_res", "final_res")


@dataclass
class CouplingConfig:
    """Algorithm knobs (coupling.py:68-129)."""

    algorithm: str = "simple"
    nu: float = 1e-6
    alpha_u: float = 0.7
    alpha_p: float = 0.3
    n_correctors: int = 2
    n_nonorth_correctors: int = 0
    dt: float = 1e-3
    end_time: float = 1.0
    outer_tol: float = 1e-5
    max_outer: int = 2000
    scheme: SchemeConfig = dc_field(default_factory=SchemeConfig)
    momentum: SolveConfig = dc_field(default_factory=lambda: SolveConfig(tolerance=1e-7))
    pressure: SolveConfig = dc_field(default_factory=lambda: SolveConfig(tolerance=1e-7))
    pressure_ref_cell: int = 0
    pressure_ref_value: float = 0.0

    def __post_init__(self):
        if self.algorithm not in ("simple", "piso"):
            raise CouplingError(f"unknown algorithm {self.algorithm!r}")
        for name in ("alpha_u", "alpha_p"):
            a = getattr(self, name)
            if not 0.0 < a <= 1.0:
                raise CouplingError(f"{name} must lie in (0, 1]")
        if self.n_correctors < 1:
            raise CouplingError("n_correctors must be >= 1")
        if self.n_nonorth_correctors < 0:
            raise CouplingError("n_nonorth_correctors must be >= 0")
        if self.dt <= 0.0:
            raise CouplingError("dt must be positive")

    @classmethod
    def from_case_config(cls, cc, record_stages=False):
        scheme = SchemeConfig(convection=cc.convection, nonorth_correction=cc.nonorth_correction,
                              limiter=cc.limiter)
        return cls(
            algorithm=cc.algorithm, nu=cc.nu, alpha_u=cc.alpha_u, alpha_p=cc.alpha_p,
            n_correctors=cc.n_correctors, n_nonorth_correctors=cc.n_nonorth_correctors,
            dt=cc.dt, end_time=cc.end_time, outer_tol=cc.outer_tol, max_outer=cc.max_outer,
            scheme=scheme,
            momentum=SolveConfig(tolerance=cc.bicgstab_tol, max_iters=cc.max_iters,
                                 record_stages=record_stages),
            pressure=SolveConfig(tolerance=cc.cg_tol, max_iters=cc.max_iters,
                                 record_stages=record_stages),
            pressure_ref_cell=cc.pressure_ref_cell, pressure_ref_value=cc.pressure_ref_value)


class _DeviceState:
    """u, p, flux and their boundary arrays resident on the device."""

    def __init__(self, ctx, n, nf, nb):
        self.ctx = ctx
        self.n, self.nf, self.nb = n, nf, nb
        self.host = {}          # name -> host array (valid copy or user-owned view)
        self.host_dirty = set()  # names whose host copy may be newer than the device

    def _download(self):
        n, nf, nb = self.n, self.nf, self.nb
        u = np.empty(3 * n)
        p = np.empty(n)
        fl = np.empty(nf)
        ub = np.empty(3 * nb)
        pb = np.empty(nb)
        P = _lib.ptr
        _lib.check(_lib.lib.fvb_get_state(self.ctx.h, P(u), P(p), P(fl), P(ub), P(pb)))
        self.host = {"u": np.ascontiguousarray(u.reshape(3, n).T), "p": p, "flux": fl,
                     "ub": np.ascontiguousarray(ub.reshape(3, nb).T), "pb": pb}

    def get(self, name):
        if name not in self.host:
            self._download()
        self.host_dirty.add(name)  # the caller may edit it in place
        return self.host[name]

    def set(self, name, value):
        if name not in self.host:
            self._download()
        shape = self.host[name].shape
        arr = np.array(value, dtype=float)
        if arr.shape != shape:
            arr = np.broadcast_to(arr, shape).copy()
        self.host[name] = arr
        self.host_dirty.add(name)

    def push(self):
        """Upload host views that may have been modified."""
        if not self.host_dirty:
            return
        P = _lib.ptr
        args = {}
        for name in self.host_dirty:
            a = self.host[name]
            if name in ("u", "ub"):
                a = np.ascontiguousarray(np.asarray(a, dtype=float).T)
            args[name] = _lib.f64(a)
        _lib.check(_lib.lib.fvb_set_state(
            self.ctx.h, P(args.get("u")), P(args.get("p")), P(args.get("flux")),
            P(args.get("ub")), P(args.get("pb"))))
        self.host_dirty.clear()

    def invalidate(self):
        self.host = {}
        self.host_dirty.clear()


class DeviceField(Field):
    """Field whose values/boundary live in a _DeviceState."""

    def __init__(self, name, mesh, bcs, dev, vkey, bkey):
        self._dev, self._vkey, self._bkey = dev, vkey, bkey
        self.name, self.mesh, self.bcs, self.face_flux = name, mesh, dict(bcs), None

    @property
    def values(self):
        return self._dev.get(self._vkey)

    @values.setter
    def values(self, v):
        self._dev.set(self._vkey, v)

    @property
    def boundary(self):
        return self._dev.get(self._bkey)

    @boundary.setter
    def boundary(self, v):
        self._dev.set(self._bkey, v)

    @property
    def rank(self):
        return "vector" if self._vkey == "u" else "scalar"


@dataclass
class RunState:
    """Outer-loop state plus bookkeeping (coupling.py:132-175)."""

    mesh: object
    geom: object
    pattern: object
    u: object
    p: object
    t: float = 0.0
    outer: int = 0
    pin_pressure: bool = True
    converged: bool = False
    cum_iters: dict = dc_field(default_factory=lambda: {"cg": 0, "bicgstab": 0})
    residual_log: list = dc_field(default_factory=list)
    stage_times: dict = dc_field(default_factory=dict)
    wall: dict = dc_field(default_factory=dict)
    ops: dict = dc_field(default_factory=dict)
    _res_scale: dict = dc_field(default_factory=dict)
    _dev: object = None
    _ctx: object = None

    @property
    def flux(self):
        return self._dev.get("flux")

    @flux.setter
    def flux(self, v):
        self._dev.set("flux", v)

    def log_solve(self, solver, name, report):
        self.cum_iters[solver] += report.iterations
        self.residual_log.append((solver, name, self.outer, report.iterations,
                                  report.initial_residual, report.final_residual))
        for stage, sec in report.stage_times.items():
            bucket = self.stage_times.setdefault(solver, {})
            bucket[stage] = bucket.get(stage, 0.0) + sec

    def add_wall(self, section, seconds):
        self.wall[section] = self.wall.get(section, 0.0) + seconds

    def add_op(self, name, seconds):
        rec = self.ops.setdefault(name, [0.0, 0])
        rec[0] += seconds
        rec[1] += 1

    def normalized(self, slot, res):
        seen = max(self._res_scale.get(slot, 0.0), res)
        self._res_scale[slot] = seen
        return res / max(seen, 1e-30)


def init_state(case, cfg, device=None) -> RunState:
    """Geometry, pattern, fields, BCs at t = 0 and the plain initial flux,
    all resident on one device context (coupling.py:182-213)."""
    mesh = case.mesh
    geom = compute_geometry(mesh)
    pattern = build_pattern(mesh)
    missing = [p.name for p in mesh.patches if p.name not in case.config.boundary]
    if missing:
        raise CouplingError(f"no boundary conditions for patches {missing}")
    u_bcs = {name: bc_from_tuple(bs.u) for name, bs in case.config.boundary.items()}
    p_bcs = {name: bc_from_tuple(bs.p) for name, bs in case.config.boundary.items()}
    # host-side templates validate patch coverage exactly like the reference
    make_vector("u", mesh, u_bcs)
    make_scalar("p", mesh, p_bcs)
    pin = not any(is_value_bc(bc) for bc in p_bcs.values())
    if pin and not 0 <= cfg.pressure_ref_cell < mesh.n_cells:
        raise CouplingError(
            f"pressure reference cell {cfg.pressure_ref_cell} outside 0..{mesh.n_cells - 1}")
    ctx = DeviceContext(device)
    ctx.upload_mesh(mesh, geom)
    ctx.upload_pattern(pattern, faces=True)
    dev = _DeviceState(ctx, mesh.n_cells, mesh.n_faces, mesh.n_boundary)
    u = DeviceField("u", mesh, u_bcs, dev, "u", "ub")
    p = DeviceField("p", mesh, p_bcs, dev, "p", "pb")
    state = RunState(mesh=mesh, geom=geom, pattern=pattern, u=u, p=p, pin_pressure=pin,
                     _dev=dev, _ctx=ctx)
    state._u_bcs = bc_table(u, geom, 0.0)
    kinds, patch, fixed, speeds = state._u_bcs
    ctx.set_bcs(0, kinds, patch, fixed, len(mesh.patches))
    pk, pp, pf, _ = bc_table(p, geom, 0.0)
    ctx.set_bcs(1, pk, pp, pf, len(mesh.patches))
    # apply_bcs(u), apply_bcs(p) at t = 0 and flux = S.u_f (coupling.py:193-201)
    _apply_device_bcs(state, 0.0)
    _lib.check(_lib.lib.fvb_plain_flux(ctx.h), CouplingError)
    dev.invalidate()
    return state


def _speeds(state, t):
    """Per-patch inflow speeds of timed / mass-flow u conditions at time t."""
    _, _, _, speeds = bc_table(state.u, state.geom, t)
    return speeds


def _apply_device_bcs(state, t):
    state._dev.push()
    sp = _lib.f64(_speeds(state, t))
    _lib.check(_lib.lib.fvb_state_apply_bcs(state._ctx.h, _lib.ptr(sp)))
    state._dev.invalidate()


def _step_cfg(state, cfg):
    s = _lib.StepCfgC()
    s.algorithm = 1 if cfg.algorithm == "piso" else 0
    s.scheme = 0 if cfg.scheme.convection == "upwind" else 1
    s.nonorth_correction = int(bool(cfg.scheme.nonorth_correction))
    s.n_correctors = cfg.n_correctors
    s.n_nonorth_correctors = cfg.n_nonorth_correctors
    s.pin_pressure = int(bool(state.pin_pressure))
    s.pressure_ref_cell = cfg.pressure_ref_cell
    s.mom_max_iters = cfg.momentum.max_iters
    s.p_max_iters = cfg.pressure.max_iters
    s.record_stages = int(bool(cfg.pressure.record_stages))
    s.nu = cfg.nu
    s.alpha_u = cfg.alpha_u
    s.alpha_p = cfg.alpha_p
    s.dt = cfg.dt
    s.t = state.t
    s.limiter = cfg.scheme.limiter
    s.mom_tol = cfg.momentum.tolerance
    s.mom_abs_tol = cfg.momentum.abs_tolerance
    s.p_tol = cfg.pressure.tolerance
    s.p_abs_tol = cfg.pressure.abs_tolerance
    s.pressure_ref_value = cfg.pressure_ref_value
    return s


_FIELD_NAMES = ("ux", "uy", "uz", "p")
_OP_NAMES = ("ddt", "convection", "laplacian", "gradient", "divergence")  # fvb_step_report order


def _run_device_step(state, cfg, piso):
    state._dev.push()
    scfg = _step_cfg(state, cfg)
    rep = _lib.StepReportC()
    sp = _lib.f64(_speeds(state, state.t))
    fn = _lib.lib.fvb_piso_step if piso else _lib.lib.fvb_simple_sweep
    t0 = time.perf_counter()
    rc = fn(state._ctx.h, C.byref(scfg), _lib.ptr(sp), C.byref(rep))
    state._dev.invalidate()
    state._last_solves = []
    for k in range(rep.n_solves):
        r = rep.rep[k]
        solver = "cg" if rep.solver[k] == 0 else "bicgstab"
        # (solver, iterations, device seconds of the persistent solver kernel)
        state._last_solves.append((solver, int(r.iterations), float(r.wall_time)))
        sc = cfg.pressure if solver == "cg" else cfg.momentum
        # the 3 batched momentum solves share one kernel: its stage times are
        # booked once (on ux)
        shared = solver == "bicgstab" and rep.field[k] != 0
        st = {} if shared else stage_times_of(r, sc.record_stages)
        state.log_solve(solver, _FIELD_NAMES[rep.field[k]],
                        SolveReport(int(r.iterations), float(r.initial_residual),
                                    float(r.final_residual), bool(r.converged),
                                    float(r.wall_time), st))
    if rc != 0:
        msg = _lib.last_error().replace("{outer}", str(state.outer))
        if rc in (_lib.E_COUPLING,):
            raise CouplingError(msg)
        raise _lib._ERR.get(rc, RuntimeError)(msg)
    state.add_wall("momentum_assembly", rep.t_momentum_assembly)
    state.add_wall("momentum_solve", rep.t_momentum_solve)
    state.add_wall("pressure_assembly", rep.t_pressure_assembly)
    state.add_wall("pressure_solve", rep.t_pressure_solve)
    state.add_wall("correction", rep.t_correction)
    for i, name in enumerate(_OP_NAMES):
        if rep.op_calls[i]:
            rec = state.ops.setdefault(name, [0.0, 0])
            rec[0] += float(rep.op_seconds[i])
            rec[1] += int(rep.op_calls[i])
    state._last_step_s = time.perf_counter() - t0
    return float(rep.mom_res), float(rep.p_res)


def simple_outer_iteration(state, cfg):
    """One SIMPLE sweep; normalised (momentum, pressure) residuals (coupling.py:347-353)."""
    state.outer += 1
    mom_res, p_res = _run_device_step(state, cfg, piso=False)
    return state.normalized("u", mom_res), state.normalized("p", p_res)


def piso_time_step(state, cfg):
    """Advance one dt: predictor + n_correctors corrections (coupling.py:356-370)."""
    state.outer += 1
    state.t = state.outer * cfg.dt
    return _run_device_step(state, cfg, piso=True)


def continuity_error(state) -> float:
    """max |div(flux)| (coupling.py:373-375)."""
    state._dev.push()
    out = C.c_double()
    _lib.check(_lib.lib.fvb_continuity_error(state._ctx.h, C.byref(out)))
    return float(out.value)


def kinetic_energy(state) -> float:
    u = state.u.values
    return float(0.5 * (state.geom.cell_volume * (u ** 2).sum(axis=1)).sum())


def run_case(case, cfg=None, writer=None, verbose=False, record_stages=False) -> RunState:
    """Drive a case to its stopping point (coupling.py:382-423)."""
    if cfg is None:
        cfg = CouplingConfig.from_case_config(case.config, record_stages=record_stages)
    state = init_state(case, cfg)
    every = case.config.write_interval
    t_start = time.perf_counter()
    if cfg.algorithm == "simple":
        for _ in range(cfg.max_outer):
            ru, rp = simple_outer_iteration(state, cfg)
            if verbose:
                print(f"iter {state.outer}: u {ru:.3e} p {rp:.3e} "
                      f"(cg {state.cum_iters['cg']}, bicgstab {state.cum_iters['bicgstab']})")
            if every and state.outer % every == 0 and writer is not None:
                writer(state, f"{state.outer:06d}")
            if max(ru, rp) < cfg.outer_tol:
                state.converged = True
                break
    else:
        n_steps = int(round(cfg.end_time / cfg.dt))
        for _ in range(n_steps):
            ru, rp = piso_time_step(state, cfg)
            if verbose:
                print(f"step {state.outer} t={state.t:.6g}: u {ru:.3e} p {rp:.3e} "
                      f"(cg {state.cum_iters['cg']}, bicgstab {state.cum_iters['bicgstab']})")
            if every and state.outer % every == 0 and writer is not None:
                writer(state, f"{state.outer:06d}")
        state.converged = True
    state.add_wall("total", time.perf_counter() - t_start)
    if writer is not None:
        writer(state, "final")
    if verbose and not state.converged:
        print(f"not converged after {state.outer} iterations")
    return state


def _plain_flux(u, geom):
    """S . u_f with 0 on empty faces (coupling.py:206-213), on the device."""
    from .device import context_for, set_field_bcs
    from .fvm import _soa

    ctx = context_for(u.mesh, geom, None)
    set_field_bcs(ctx, u, geom)
    vals = _soa(u.values, 3)
    bnd = _soa(u.boundary, 3)
    out = np.empty(u.mesh.n_faces)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_face_flux(ctx.h, P(vals), P(bnd), P(out)))
    return out
